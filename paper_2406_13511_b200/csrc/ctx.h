// ctx.h — the per-(thread, device, stream) context behind scls_ctx: error
// state, a grow-only device scratch arena, pinned staging memory and the
// CUDA events that time each phase of a call.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "scls_capi.h"

struct scls_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t err_request = -1;
  int64_t launches = 0;
  float timings[8] = {0};
  cudaEvent_t ev[16] = {};
  int sm_count = 148;
  unsigned long long* dp_prof = nullptr;  // device counters when profiling is on
  bool sim_digests = true;                // scls_simulate computes the log digests
  int dp_cluster = 1;                     // CTAs per monotone-DP cluster (1, 2 or 4)
  int dp_last_cluster = 1;                // what the last monotone DP launch used
  int dp_mode = 0;                        // 0 auto, 1 force the chain kernel (tests)
  bool dp_last_mono = false;              // the last DP ran the monotone decision kernel
  bool sim_concurrent = true;             // scls_simulate runs its per-policy launches concurrently
  bool ils_split = true;                  // metrics-only ILS / SLS: simulation kernel (32 / W jobs per warp) + merge kernel
  bool ils_lockstep = false;              // metrics-only ILS: the lock-step kernel instead of independent lanes
  cudaStream_t side[3] = {};              // forked streams for those launches (created on first use)
  bool force_large_path = false;          // batch_requests: the multi-kernel path even for small pools (tests)
  bool force_lsd_sort = false;            // batch_requests: the LSD radix sort instead of the eff-bucket sort
  void* comm = nullptr;                   // ncclComm_t of scls_comm_init (multi.cu)
  int world = 1, rank = 0;

  // Named grow-only device buffers (scratch reused across calls).
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  std::vector<Buf> bufs;
  // Pinned host staging for small readbacks.
  void* pinned = nullptr;
  size_t pinned_cap = 0;
  // Pinned host staging for small entry-point arguments and results (one
  // host<->device copy each way instead of one pageable copy per array).
  void* stage = nullptr;
  size_t stage_cap = 0;

  void* buf(int slot, size_t bytes);
  void* host_pinned(size_t bytes);
  void* host_stage(size_t bytes);
};

namespace scls {

// Scratch slots (ctx->buf).  0..29 belong to the entry points, the rest to
// shared primitives, so nested calls never alias each other's buffers.
enum ScratchSlot : int {
  kSlotRadixCounts = 30,
  kSlotRadixOffs = 31,
  kSlotBucket = 32,   // 32..35: eff-bucket sort
  kSlotScan = 40,     // 40..55: two per recursion level
  kSlotStage = 60,    // 60..79: host<->device staging of entry-point arguments
  kSlotSim = 80,      // 80..109: simulator
  kSlotGen = 110,     // 110..119: device trace generation
  kSlotMulti = 120,   // 120..123: sharded sweep (local grid, gather buffers)
  kNumSlots = 124,
};

// Status plumbing shared by the C-ABI entry points.
scls_status set_error(scls_ctx* ctx, scls_status st, const std::string& msg);
scls_status cuda_error(scls_ctx* ctx, cudaError_t e, const char* where);

#define SCLS_CUDA(call)                                             \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::scls::cuda_error(ctx, _e, #call); \
  } while (0)

#define SCLS_LAUNCHED()                                                         \
  do {                                                                          \
    ++ctx->launches;                                                            \
    cudaError_t _e = cudaPeekAtLastError();                                     \
    if (_e != cudaSuccess) return ::scls::cuda_error(ctx, _e, "kernel launch"); \
  } while (0)

void comm_release(scls_ctx* ctx);  // multi.cu

inline int div_up(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace scls
