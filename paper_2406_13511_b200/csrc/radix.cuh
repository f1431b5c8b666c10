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

// Number of significant bits of v (0 for v == 0).
inline int bit_width(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }

}  // namespace scls
