// multi.cu — the sweep sharded over GPUs: the reference runs
// sweep values one after another (experiment.cpp:62-85); here the trace
// dimension is split into contiguous shards, each shard is generated and
// simulated on its own device by the single-device sweep (scls_run_sweep),
// and the fixed-size result records are all-gathered with ONE ncclAllGather
// (NVLink / NVSwitch) -- the only collective of the path.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": in a PyTorch process
// this resolves to the NCCL torch already mapped), so the library has no
// link-time NCCL dependency and single-GPU users never touch it.
//
// Per shard the gather moves one padded block:
//   [n_cfgs][n_max] scls_trace_result  ++  [n_cfgs][n_max][hist_bins] int64
// where n_max = ceil(n_traces / N) (shard sizes differ by at most one).
// After the gather, block r holds shard r's jobs (c, t - lo_r); a reorder of
// n_shards * n_cfgs contiguous runs yields the scls_run_sweep order
// j = c * n_traces + t.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ctx.h"

namespace scls {
namespace {

// ---- NCCL, resolved at run time ---------------------------------------------------------
struct Nccl {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
#define SCLS_NCCL_SYM(field, name)                                   \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #name));    \
  if (!n.field) {                                                    \
    n.why = "libnccl.so.2 lacks " #name;                             \
    return;                                                          \
  }
    SCLS_NCCL_SYM(get_unique_id, ncclGetUniqueId)
    SCLS_NCCL_SYM(comm_init_rank, ncclCommInitRank)
    SCLS_NCCL_SYM(comm_init_all, ncclCommInitAll)
    SCLS_NCCL_SYM(comm_destroy, ncclCommDestroy)
    SCLS_NCCL_SYM(comm_count, ncclCommCount)
    SCLS_NCCL_SYM(all_gather, ncclAllGather)
    SCLS_NCCL_SYM(group_start, ncclGroupStart)
    SCLS_NCCL_SYM(group_end, ncclGroupEnd)
    SCLS_NCCL_SYM(error_string, ncclGetErrorString)
#undef SCLS_NCCL_SYM
    n.ok = true;
  });
  return n;
}

std::string nccl_msg(ncclResult_t r, const char* where) {
  return std::string("NCCL error ") + (nccl().error_string ? nccl().error_string(r) : "?") + " at " + where;
}

// One shard's padded block (records, then histograms) in a byte buffer.
struct Block {
  size_t rec_bytes, hist_bytes, bytes;
  Block(int32_t n_cfgs, int64_t n_max, int32_t hist_bins)
      : rec_bytes(sizeof(scls_trace_result) * (size_t)n_cfgs * n_max),
        hist_bytes(sizeof(int64_t) * (size_t)n_cfgs * n_max * hist_bins),
        bytes(((rec_bytes + hist_bytes + 255) / 256) * 256) {}
};

// Runs one shard [lo, hi) of the sweep on ctx's device and packs its jobs
// into the padded send block (records at c * n_max, histograms likewise).
// grid: every config on every trace (scls_run_sweep); else run i pairs specs[i]
// with cfgs[i] (scls_run_experiments) and the block holds one row per run.
scls_status run_shard(scls_ctx* ctx, bool grid, int64_t lo, int64_t hi, int64_t n_max,
                      const scls_workload_spec* specs, int32_t n_cfgs, const scls_sched_cfg* cfgs,
                      const scls_latency* lat, const scls_memory* memm, int32_t hist_bins, char* send, const Block& B,
                      float* shard_ms) {
  const int64_t nl = hi - lo;
  if (!grid) n_cfgs = 1;
  *shard_ms = 0.f;
  if (nl == 0) return SCLS_OK;
  const size_t rec = sizeof(scls_trace_result), hb = sizeof(int64_t) * (size_t)hist_bins;
  auto* d_res = (scls_trace_result*)ctx->buf(kSlotMulti + 0, rec * (size_t)n_cfgs * nl);
  auto* d_hist = hist_bins > 0 ? (int64_t*)ctx->buf(kSlotMulti + 1, hb * (size_t)n_cfgs * nl) : nullptr;
  if (!d_res || (hist_bins > 0 && !d_hist)) return set_error(ctx, SCLS_ERR_CUDA, "shard allocation failed");
  scls_status st = grid ? scls_run_sweep(ctx, (int32_t)nl, specs + lo, n_cfgs, cfgs, lat, memm, d_res, hist_bins,
                                         d_hist, nullptr, SCLS_MEM_DEVICE)
                        : scls_run_experiments(ctx, (int32_t)nl, specs + lo, cfgs + lo, lat, memm, d_res, hist_bins,
                                               d_hist, nullptr, SCLS_MEM_DEVICE);
  if (st) return st;
  *shard_ms = ctx->timings[0];
  // local job c * nl + tl -> block row c * n_max + tl
  SCLS_CUDA(cudaMemcpy2DAsync(send, rec * n_max, d_res, rec * nl, rec * nl, n_cfgs, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  if (hist_bins > 0)
    SCLS_CUDA(cudaMemcpy2DAsync(send + B.rec_bytes, hb * n_max, d_hist, hb * nl, hb * nl, n_cfgs,
                                cudaMemcpyDeviceToDevice, ctx->stream));
  return SCLS_OK;
}

// Gathered blocks [n_shards][Block] -> the grid in job order, on `stream`.
scls_status reorder(scls_ctx* ctx, cudaStream_t stream, const char* gathered, const Block& B, int32_t n_shards,
                    int64_t n_traces, int64_t n_max, int32_t n_cfgs, int32_t hist_bins, scls_trace_result* results,
                    int64_t* slice_hist, cudaMemcpyKind kind) {
  const size_t rec = sizeof(scls_trace_result), hb = sizeof(int64_t) * (size_t)hist_bins;
  for (int32_t r = 0; r < n_shards; ++r) {
    int64_t lo, hi;
    scls_shard_range(n_traces, r, n_shards, &lo, &hi);
    if (hi == lo) continue;
    const char* blk = gathered + B.bytes * r;
    // block rows c * n_max + [0, hi - lo) -> results[c * n_traces + lo ...]
    SCLS_CUDA(cudaMemcpy2DAsync((char*)results + rec * lo, rec * n_traces, blk, rec * n_max, rec * (hi - lo), n_cfgs,
                                kind, stream));
    if (hist_bins > 0)
      SCLS_CUDA(cudaMemcpy2DAsync((char*)slice_hist + hb * lo, hb * n_traces, blk + B.rec_bytes, hb * n_max,
                                  hb * (hi - lo), n_cfgs, kind, stream));
  }
  return SCLS_OK;
}

bool args_ok(int32_t n_traces, const scls_workload_spec* specs, int32_t n_cfgs, const scls_sched_cfg* cfgs,
             const scls_latency* lat, const scls_memory* memm, const scls_trace_result* results, int32_t hist_bins,
             const int64_t* slice_hist) {
  return n_traces >= 0 && (n_traces == 0 || specs) && n_cfgs >= 1 && cfgs && lat && memm && results &&
         hist_bins >= 0 && (hist_bins == 0 || slice_hist) && (int64_t)n_traces * n_cfgs <= INT32_MAX;
}

}  // namespace

void comm_release(scls_ctx* ctx) {
  if (ctx->comm && nccl().ok) nccl().comm_destroy((ncclComm_t)ctx->comm);
  ctx->comm = nullptr;
  ctx->world = 1;
  ctx->rank = 0;
}

}  // namespace scls

using namespace scls;

extern "C" void scls_shard_range(int64_t total, int32_t shard, int32_t n_shards, int64_t* lo, int64_t* hi) {
  if (n_shards < 1 || shard < 0 || shard >= n_shards || total < 0) {
    *lo = *hi = 0;
    return;
  }
  *lo = total * shard / n_shards;
  *hi = total * (shard + 1) / n_shards;
}

extern "C" int32_t scls_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

extern "C" scls_status scls_comm_unique_id(uint8_t out[128]) {
  if (!out) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null output");
  if (!nccl().ok) return set_error(nullptr, SCLS_ERR_CUDA, nccl().why);
  ncclUniqueId id;
  const ncclResult_t r = nccl().get_unique_id(&id);
  if (r != ncclSuccess) return set_error(nullptr, SCLS_ERR_CUDA, nccl_msg(r, "ncclGetUniqueId"));
  std::memcpy(out, id.internal, sizeof id.internal);
  return SCLS_OK;
}

extern "C" scls_status scls_comm_init(scls_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128]) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  if (world < 1 || rank < 0 || rank >= world || !id) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad rank");
  if (!nccl().ok) return set_error(ctx, SCLS_ERR_CUDA, nccl().why);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  comm_release(ctx);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof uid.internal);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, world, uid, rank);
  if (r != ncclSuccess) return set_error(ctx, SCLS_ERR_CUDA, nccl_msg(r, "ncclCommInitRank"));
  ctx->comm = c;
  ctx->world = world;
  ctx->rank = rank;
  return SCLS_OK;
}

extern "C" int32_t scls_comm_size(const scls_ctx* ctx) {
  if (!ctx || !ctx->comm || !nccl().ok) return 1;
  int n = 0;
  return nccl().comm_count((ncclComm_t)ctx->comm, &n) == ncclSuccess ? n : -1;
}

extern "C" scls_status scls_run_sweep_sharded(scls_ctx* ctx, int32_t n_traces, const scls_workload_spec* specs,
                                              int32_t n_cfgs, const scls_sched_cfg* cfgs, const scls_latency* lat,
                                              const scls_memory* memm, scls_trace_result* results,
                                              int32_t hist_bins, int64_t* slice_hist, int32_t mem) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  if (!args_ok(n_traces, specs, n_cfgs, cfgs, lat, memm, results, hist_bins, slice_hist))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  const int32_t world = ctx->comm ? ctx->world : 1;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t n_max = (n_traces + world - 1) / world;
  int64_t lo, hi;
  scls_shard_range(n_traces, ctx->rank, world, &lo, &hi);
  const Block B(n_cfgs, n_max, hist_bins);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  char* send = (char*)ctx->buf(kSlotMulti + 2, B.bytes);
  char* recv = (char*)ctx->buf(kSlotMulti + 3, B.bytes * world);
  if (!send || !recv) return set_error(ctx, SCLS_ERR_CUDA, "gather allocation failed");
  float shard_ms = 0.f;
  scls_status st = run_shard(ctx, true, lo, hi, n_max, specs, n_cfgs, cfgs, lat, memm, hist_bins, send, B, &shard_ms);
  if (st) return st;
  const int64_t launches = ctx->launches;
  SCLS_CUDA(cudaEventRecord(ctx->ev[4], ctx->stream));
  if (world > 1) {
    const ncclResult_t r = nccl().all_gather(send, recv, B.bytes, ncclInt8, (ncclComm_t)ctx->comm, ctx->stream);
    if (r != ncclSuccess) return set_error(ctx, SCLS_ERR_CUDA, nccl_msg(r, "ncclAllGather"));
  } else {
    SCLS_CUDA(cudaMemcpyAsync(recv, send, B.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  st = reorder(ctx, ctx->stream, recv, B, world, n_traces, n_max, n_cfgs, hist_bins, results, slice_hist,
               mem == SCLS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  if (st) return st;
  SCLS_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  ctx->timings[6] = shard_ms;
  cudaEventElapsedTime(&ctx->timings[5], ctx->ev[4], ctx->ev[5]);
  ctx->timings[0] = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ctx->launches = launches;
  return SCLS_OK;
}

// ---- one process, many GPUs -----------------------------------------------------------------

struct scls_multi {
  std::vector<int32_t> dev;
  std::vector<scls_ctx*> ctx;
  std::vector<ncclComm_t> comm;  // empty: peer-copy gather (a device listed twice)
  std::string err;
};

namespace {
scls_status multi_error(scls_multi* m, scls_status st, const std::string& msg) {
  m->err = msg;
  return st;
}
}  // namespace

extern "C" scls_status scls_multi_create(int32_t n_dev, const int32_t* devices, scls_multi** out) {
  if (!out || n_dev < 1 || !devices) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  *out = nullptr;
  auto* m = new scls_multi();
  m->dev.assign(devices, devices + n_dev);
  for (int32_t i = 0; i < n_dev; ++i) {
    scls_ctx* c = nullptr;
    const scls_status st = scls_ctx_create(devices[i], nullptr, &c);
    if (st) {
      scls_multi_destroy(m);
      return st;
    }
    m->ctx.push_back(c);
  }
  std::vector<int32_t> sorted(m->dev);
  std::sort(sorted.begin(), sorted.end());
  const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
  if (distinct && n_dev > 1) {
    if (!nccl().ok) {
      scls_multi_destroy(m);
      return set_error(nullptr, SCLS_ERR_CUDA, nccl().why);
    }
    m->comm.resize(n_dev);
    const ncclResult_t r = nccl().comm_init_all(m->comm.data(), n_dev, m->dev.data());
    if (r != ncclSuccess) {
      m->comm.clear();
      scls_multi_destroy(m);
      return set_error(nullptr, SCLS_ERR_CUDA, nccl_msg(r, "ncclCommInitAll"));
    }
  } else if (n_dev > 1) {
    // shards sharing a device: enable peer access where it exists (copies work either way)
    for (int32_t a = 0; a < n_dev; ++a)
      for (int32_t b = 0; b < n_dev; ++b)
        if (m->dev[a] != m->dev[b]) {
          int can = 0;
          cudaDeviceCanAccessPeer(&can, m->dev[a], m->dev[b]);
          if (can) {
            cudaSetDevice(m->dev[a]);
            cudaDeviceEnablePeerAccess(m->dev[b], 0);
            cudaGetLastError();
          }
        }
  }
  *out = m;
  return SCLS_OK;
}

extern "C" void scls_multi_destroy(scls_multi* m) {
  if (!m) return;
  for (size_t i = 0; i < m->comm.size(); ++i)
    if (m->comm[i]) {
      cudaSetDevice(m->dev[i]);
      nccl().comm_destroy(m->comm[i]);
    }
  for (scls_ctx* c : m->ctx) scls_ctx_destroy(c);
  delete m;
}

extern "C" size_t scls_multi_last_error(const scls_multi* m, char* buf, size_t cap) {
  const std::string& s = m ? m->err : std::string();
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

extern "C" scls_status scls_multi_set_option(scls_multi* m, int32_t option, int64_t value) {
  if (!m) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null multi context");
  for (scls_ctx* c : m->ctx) {
    const scls_status st = scls_set_option(c, option, value);
    if (st) return multi_error(m, st, c->err);
  }
  return SCLS_OK;
}

extern "C" int32_t scls_multi_uses_nccl(const scls_multi* m) { return m && !m->comm.empty() ? 1 : 0; }

namespace {
scls_status multi_run(scls_multi* m, bool grid, int32_t n_traces, const scls_workload_spec* specs, int32_t n_cfgs,
                      const scls_sched_cfg* cfgs, const scls_latency* lat, const scls_memory* memm,
                      scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist, float* out_ms) {
  if (!m) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null multi context");
  m->err.clear();
  if (!args_ok(n_traces, specs, n_cfgs, cfgs, lat, memm, results, hist_bins, slice_hist) ||
      (!grid && n_cfgs != n_traces))
    return multi_error(m, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  const int32_t rows = grid ? n_cfgs : 1;  // block rows per shard
  const auto t0 = std::chrono::steady_clock::now();
  const int32_t N = (int32_t)m->ctx.size();
  const int64_t n_max = (n_traces + N - 1) / N;
  const Block B(rows, n_max, hist_bins);
  std::vector<char*> send(N), recv(N);
  std::vector<float> shard_ms(N, 0.f);
  std::vector<scls_status> st(N, SCLS_OK);
  // one host thread per shard: generate + simulate + pack
  std::vector<std::thread> th;
  for (int32_t i = 0; i < N; ++i)
    th.emplace_back([&, i] {
      scls_ctx* c = m->ctx[i];
      cudaSetDevice(c->device);
      send[i] = (char*)c->buf(kSlotMulti + 2, B.bytes);
      recv[i] = (char*)c->buf(kSlotMulti + 3, B.bytes * N);
      if (!send[i] || !recv[i]) {
        st[i] = set_error(c, SCLS_ERR_CUDA, "gather allocation failed");
        return;
      }
      int64_t lo, hi;
      scls_shard_range(n_traces, i, N, &lo, &hi);
      st[i] = run_shard(c, grid, lo, hi, n_max, specs, n_cfgs, cfgs, lat, memm, hist_bins, send[i], B,
                        &shard_ms[i]);
      if (!st[i] && cudaStreamSynchronize(c->stream) != cudaSuccess) st[i] = set_error(c, SCLS_ERR_CUDA, "shard sync");
    });
  for (auto& t : th) t.join();
  for (int32_t i = 0; i < N; ++i)
    if (st[i]) return multi_error(m, st[i], "shard " + std::to_string(i) + ": " + m->ctx[i]->err);
  // the gather: every device receives every block
  scls_ctx* c0 = m->ctx[0];
  cudaSetDevice(c0->device);
  cudaEventRecord(c0->ev[4], c0->stream);
  if (!m->comm.empty()) {
    nccl().group_start();
    for (int32_t i = 0; i < N; ++i) {
      cudaSetDevice(m->ctx[i]->device);
      const ncclResult_t r = nccl().all_gather(send[i], recv[i], B.bytes, ncclInt8, m->comm[i], m->ctx[i]->stream);
      if (r != ncclSuccess) {
        nccl().group_end();
        return multi_error(m, SCLS_ERR_CUDA, nccl_msg(r, "ncclAllGather"));
      }
    }
    const ncclResult_t r = nccl().group_end();
    if (r != ncclSuccess) return multi_error(m, SCLS_ERR_CUDA, nccl_msg(r, "ncclGroupEnd"));
  } else {
    for (int32_t i = 0; i < N; ++i)
      for (int32_t r = 0; r < N; ++r) {
        cudaSetDevice(m->ctx[i]->device);
        if (cudaMemcpyPeerAsync(recv[i] + B.bytes * r, m->ctx[i]->device, send[r], m->ctx[r]->device, B.bytes,
                                m->ctx[i]->stream) != cudaSuccess)
          return multi_error(m, SCLS_ERR_CUDA, "peer copy failed");
      }
  }
  for (int32_t i = 0; i < N; ++i) {
    cudaSetDevice(m->ctx[i]->device);
    if (cudaStreamSynchronize(m->ctx[i]->stream) != cudaSuccess) return multi_error(m, SCLS_ERR_CUDA, "gather sync");
  }
  // device 0's copy of the grid -> the caller's host buffers, job order
  cudaSetDevice(c0->device);
  scls_status s0 = reorder(c0, c0->stream, recv[0], B, N, n_traces, n_max, rows, hist_bins, results, slice_hist,
                           cudaMemcpyDeviceToHost);
  if (s0) return multi_error(m, s0, c0->err);
  cudaEventRecord(c0->ev[5], c0->stream);
  if (cudaStreamSynchronize(c0->stream) != cudaSuccess) return multi_error(m, SCLS_ERR_CUDA, "result copy");
  if (out_ms) {
    for (int32_t i = 0; i < N; ++i) out_ms[i] = shard_ms[i];
    cudaEventElapsedTime(&out_ms[N], c0->ev[4], c0->ev[5]);
    out_ms[N + 1] = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return SCLS_OK;
}
}  // namespace

extern "C" scls_status scls_multi_run_sweep(scls_multi* m, int32_t n_traces, const scls_workload_spec* specs,
                                            int32_t n_cfgs, const scls_sched_cfg* cfgs, const scls_latency* lat,
                                            const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                            int64_t* slice_hist, float* out_ms) {
  return multi_run(m, true, n_traces, specs, n_cfgs, cfgs, lat, memm, results, hist_bins, slice_hist, out_ms);
}

extern "C" scls_status scls_multi_run_experiments(scls_multi* m, int32_t n_runs, const scls_workload_spec* specs,
                                                  const scls_sched_cfg* cfgs, const scls_latency* lat,
                                                  const scls_memory* memm, scls_trace_result* results,
                                                  int32_t hist_bins, int64_t* slice_hist, float* out_ms) {
  return multi_run(m, false, n_runs, specs, n_runs, cfgs, lat, memm, results, hist_bins, slice_hist, out_ms);
}
