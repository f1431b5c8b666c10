// radix.cuh — device-wide primitives: stable LSD radix sort of
// (uint64 key, int32 value) pairs and exclusive prefix sums.  Host drivers
// launch on the context stream; all buffers are device memory.
#pragma once

#include "ctx.h"

namespace scls {

// Stable sort of (keys, vals) by key bits [begin_bit, end_bit).  Ping-pongs
// between (keys, vals) and (keys_alt, vals_alt); *swapped tells the caller
// which pair holds the result.
scls_status radix_sort_pairs(scls_ctx* ctx, int64_t n, uint64_t* keys, int32_t* vals,
                             uint64_t* keys_alt, int32_t* vals_alt, int begin_bit,
                             int end_bit, bool* swapped);

// out[i] = sum(in[0..i)), total written to *d_total (device) if non-null.
scls_status scan_exclusive(scls_ctx* ctx, int64_t n, const int32_t* in, int32_t* out,
                           int32_t* d_total);

// Sort permutation of a pool by (eff, arrival, id) -- the order of the stable
// LSD path on (bias32(eff), ordered_bits(arrival), bias64(id)), input position
// last -- through eff buckets: a counting scatter by eff (one histogram, one
// scan, one scatter), then one CTA per bucket sorting (arrival, id, position)
// in registers and shared memory.  The plan comes from the device: the eff
// range d_eff_range[0..1] (biased int32, the key-stats kernel's min / max),
// so no host round trip precedes the sort.  When the range has more than
// kBucketMaxBins values, the average bucket is too large, or one bucket is
// larger than kBucketCap, *d_overflow (device int) is set and perm holds a
// valid but unsorted permutation; the caller then uses the LSD sort.
constexpr int kBucketMaxBins = 1 << 16;
constexpr int kBucketCap = 2048;
scls_status bucket_sort_perm(scls_ctx* ctx, int64_t n, const int32_t* eff, const double* arr,
                             const int64_t* id, const unsigned long long* d_eff_range, int32_t* perm,
                             int32_t* d_overflow);

// Number of significant bits of v (0 for v == 0).
inline int bit_width(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

}  // namespace scls
