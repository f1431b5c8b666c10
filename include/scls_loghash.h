/* scls_loghash.h — the event-log digests reported per trace by scls_simulate.
 *
 * Shared verbatim by the CUDA simulator, the C oracle (oracle/scls_oracle.c)
 * and the wrapper around the compiled reference (oracle/ref_capi.cpp), so a
 * digest mismatch always means a behavioural difference, never a hashing one.
 *
 *   byte-wise FNV-1a-64 over little-endian 8-byte words:
 *     h_complete_ids  request id of every `complete` record, in log order
 *     h_dispatch      (batch, worker, n, l_in) of every `dispatch` record
 *     h_complete_t    IEEE bits of the `t` of every `complete` record
 *   word-wise FNV-1a-64 (h = (h ^ w) * prime) over every EventRecord field
 *   (event_log.h:52-69) and member (event_log.h:41-47):
 *     h_log
 */
#ifndef SCLS_LOGHASH_H_
#define SCLS_LOGHASH_H_

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define SCLS_HD __host__ __device__ __forceinline__
#else
#define SCLS_HD static inline
#endif

#define SCLS_FNV_OFFSET 1469598103934665603ULL
#define SCLS_FNV_PRIME 1099511628211ULL

SCLS_HD uint64_t scls_fnv_bytes(uint64_t h, uint64_t w) {
  for (int i = 0; i < 8; ++i) {
    h ^= (w >> (8 * i)) & 0xffu;
    h *= SCLS_FNV_PRIME;
  }
  return h;
}

SCLS_HD uint64_t scls_fnv_word(uint64_t h, uint64_t w) {
  return (h ^ w) * SCLS_FNV_PRIME;
}

SCLS_HD uint64_t scls_dbits(double x) {
  uint64_t u;
#if defined(__CUDA_ARCH__)
  u = (uint64_t)__double_as_longlong(x);
#else
  memcpy(&u, &x, sizeof u);
#endif
  return u;
}

/* Fold one EventRecord header (everything but the member list). */
SCLS_HD uint64_t scls_hash_record(uint64_t h, int32_t kind, double t, int64_t request,
                                  int32_t worker, int64_t batch, int32_t n,
                                  int32_t l_in, int32_t planned_l_out,
                                  int32_t served_l_out, double est_serve_s,
                                  int32_t input_len, int32_t gen_len,
                                  double response_s, int32_t slices,
                                  double next_interval_s, int32_t member_count) {
  h = scls_fnv_word(h, (uint64_t)(int64_t)kind);
  h = scls_fnv_word(h, scls_dbits(t));
  h = scls_fnv_word(h, (uint64_t)request);
  h = scls_fnv_word(h, (uint64_t)(int64_t)worker);
  h = scls_fnv_word(h, (uint64_t)batch);
  h = scls_fnv_word(h, (uint64_t)(int64_t)n);
  h = scls_fnv_word(h, (uint64_t)(int64_t)l_in);
  h = scls_fnv_word(h, (uint64_t)(int64_t)planned_l_out);
  h = scls_fnv_word(h, (uint64_t)(int64_t)served_l_out);
  h = scls_fnv_word(h, scls_dbits(est_serve_s));
  h = scls_fnv_word(h, (uint64_t)(int64_t)input_len);
  h = scls_fnv_word(h, (uint64_t)(int64_t)gen_len);
  h = scls_fnv_word(h, scls_dbits(response_s));
  h = scls_fnv_word(h, (uint64_t)(int64_t)slices);
  h = scls_fnv_word(h, scls_dbits(next_interval_s));
  h = scls_fnv_word(h, (uint64_t)(int64_t)member_count);
  return h;
}

SCLS_HD uint64_t scls_hash_member(uint64_t h, int64_t request, int32_t eff, int32_t pad,
                                  int32_t gen, int32_t invalid) {
  h = scls_fnv_word(h, (uint64_t)request);
  h = scls_fnv_word(h, (uint64_t)(int64_t)eff);
  h = scls_fnv_word(h, (uint64_t)(int64_t)pad);
  h = scls_fnv_word(h, (uint64_t)(int64_t)gen);
  h = scls_fnv_word(h, (uint64_t)(int64_t)invalid);
  return h;
}

#endif /* SCLS_LOGHASH_H_ */
