// capi.cu — the C-ABI entry points of include/scls_capi.h: context
// management, argument checking, host<->device staging, phase timing, and
// dispatch to the device implementations.  There is no CPU compute path: if
// the device is unusable every compute entry point returns SCLS_ERR_CUDA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "batcher.cuh"
#include "ctx.h"
#include "scls_common.cuh"
#include "sim.cuh"

static thread_local std::string g_tls_err;
static thread_local int64_t g_tls_request = -1;

void* scls_ctx::buf(int slot, size_t bytes) {
  if ((int)bufs.size() <= slot) bufs.resize(slot + 1);
  Buf& b = bufs[slot];
  if (bytes == 0) bytes = 1;
  if (b.cap >= bytes) return b.p;
  if (b.p) {
    cudaStreamSynchronize(stream);
    cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
  }
  size_t cap = std::max(bytes, (size_t)256);
  cap = cap + cap / 4;
  if (cudaMalloc(&b.p, cap) != cudaSuccess) {
    b.p = nullptr;
    return nullptr;
  }
  b.cap = cap;
  return b.p;
}

void* scls_ctx::host_pinned(size_t bytes) {
  if (pinned_cap >= bytes) return pinned;
  if (pinned) {
    cudaStreamSynchronize(stream);
    cudaFreeHost(pinned);
  }
  pinned_cap = std::max(bytes, (size_t)4096);
  if (cudaMallocHost(&pinned, pinned_cap) != cudaSuccess) {
    pinned = nullptr;
    pinned_cap = 0;
  }
  return pinned;
}

void* scls_ctx::host_stage(size_t bytes) {
  if (stage_cap >= bytes) return stage;
  if (stage) {
    cudaStreamSynchronize(stream);
    cudaFreeHost(stage);
  }
  stage_cap = std::max(bytes, (size_t)65536);
  if (cudaMallocHost(&stage, stage_cap) != cudaSuccess) {
    stage = nullptr;
    stage_cap = 0;
  }
  return stage;
}

namespace scls {

scls_status set_error(scls_ctx* ctx, scls_status st, const std::string& msg) {
  if (ctx) ctx->err = msg;
  else g_tls_err = msg;
  return st;
}

scls_status cuda_error(scls_ctx* ctx, cudaError_t e, const char* where) {
  return set_error(ctx, SCLS_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + where);
}

namespace {

// Stage a caller array onto the device (or pass device pointers through).
template <typename T>
scls_status stage_in(scls_ctx* ctx, int slot, const T* p, int64_t count, int32_t mem, const T** out) {
  if (mem == SCLS_MEM_DEVICE || count == 0) {
    *out = p;
    return SCLS_OK;
  }
  T* d = (T*)ctx->buf(kSlotStage + slot, sizeof(T) * (size_t)count);
  if (!d) return set_error(ctx, SCLS_ERR_CUDA, "staging allocation failed");
  SCLS_CUDA(cudaMemcpyAsync(d, p, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, ctx->stream));
  *out = d;
  return SCLS_OK;
}

template <typename T>
T* stage_out_buf(scls_ctx* ctx, int slot, T* p, int64_t count, int32_t mem) {
  if (mem == SCLS_MEM_DEVICE || p == nullptr) return p;
  return (T*)ctx->buf(kSlotStage + slot, sizeof(T) * (size_t)std::max<int64_t>(count, 1));
}

template <typename T>
scls_status copy_out(scls_ctx* ctx, T* host, const T* dev, int64_t count, int32_t mem) {
  if (mem == SCLS_MEM_DEVICE || host == nullptr || count == 0) return SCLS_OK;
  SCLS_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * (size_t)count, cudaMemcpyDeviceToHost, ctx->stream));
  return SCLS_OK;
}

scls_status begin_call(scls_ctx* ctx) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  ctx->err.clear();
  ctx->err_request = -1;
  ctx->launches = 0;
  std::fill(ctx->timings, ctx->timings + 8, 0.f);
  SCLS_CUDA(cudaSetDevice(ctx->device));
  return SCLS_OK;
}

void collect_timings(scls_ctx* ctx, int last_event) {
  cudaEventSynchronize(ctx->ev[last_event]);
  for (int i = 1; i <= last_event; ++i) cudaEventElapsedTime(&ctx->timings[i], ctx->ev[i - 1], ctx->ev[i]);
  cudaEventElapsedTime(&ctx->timings[0], ctx->ev[0], ctx->ev[last_event]);
}

bool check_memory_arg(scls_ctx* ctx, const scls_memory* m) {
  if (!m) return false;
  if (m->kind == SCLS_MEM_RULE_TABLE && (m->n_rules < 1 || m->n_rules > SCLS_MAX_RULES)) return false;
  if (m->kind != SCLS_MEM_RULE_TABLE && m->kind != SCLS_MEM_ANALYTIC) return false;
  (void)ctx;
  return true;
}

// ---- batched estimator kernels -------------------------------------------------

__global__ void bst_kernel(int64_t count, const int32_t* __restrict__ n, const int32_t* __restrict__ l_in,
                           const int32_t* __restrict__ l_out, Lat lat, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = batch_serve_time(lat, n[i], l_in[i], l_out[i]);
}

__global__ void oom_kernel(int64_t count, const int32_t* __restrict__ n, const int32_t* __restrict__ l_in,
                           int32_t slice, Mem mem, uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = would_oom(mem, n[i], l_in[i], slice) ? 1 : 0;
}

__global__ void mbs_kernel(int64_t count, const int32_t* __restrict__ l_in, int32_t slice, Mem mem,
                           int32_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = max_batch_size(mem, l_in[i], slice);
}

__global__ void iota_ids_kernel(int64_t nb, int64_t first, int64_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) ids[i] = first + i;
}

}  // namespace
}  // namespace scls

using namespace scls;

extern "C" {

int32_t scls_abi_version(void) { return SCLS_ABI_VERSION; }

scls_status scls_ctx_create(int32_t device, void* stream, scls_ctx** out) {
  if (!out) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null output pointer");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_error(nullptr, SCLS_ERR_CUDA,
                     std::string("no CUDA device available (") + cudaGetErrorString(e) +
                         "); the scheduling core has no CPU fallback");
  if (device < 0 || device >= count) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "bad device index");
  if (cudaSetDevice(device) != cudaSuccess) return set_error(nullptr, SCLS_ERR_CUDA, "cudaSetDevice failed");
  scls_ctx* ctx = new scls_ctx();
  ctx->device = device;
  if (stream) {
    ctx->stream = (cudaStream_t)stream;
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return set_error(nullptr, SCLS_ERR_CUDA, "stream creation failed");
    }
    ctx->own_stream = true;
  }
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  *out = ctx;
  return SCLS_OK;
}

void scls_ctx_destroy(scls_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  scls::comm_release(ctx);
  for (auto& b : ctx->bufs)
    if (b.p) cudaFree(b.p);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->stage) cudaFreeHost(ctx->stage);
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto& st : ctx->side)
    if (st) cudaStreamDestroy(st);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

size_t scls_last_error(const scls_ctx* ctx, char* buf, size_t cap) {
  const std::string& s = ctx ? ctx->err : g_tls_err;
  if (buf && cap) {
    const size_t k = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), k);
    buf[k] = '\0';
  }
  return s.size();
}

int64_t scls_last_request_id(const scls_ctx* ctx) { return ctx ? ctx->err_request : g_tls_request; }

void scls_last_timings(const scls_ctx* ctx, float out_ms[8]) {
  for (int i = 0; i < 8; ++i) out_ms[i] = ctx ? ctx->timings[i] : 0.f;
}

int64_t scls_last_launch_count(const scls_ctx* ctx) { return ctx ? ctx->launches : 0; }

scls_status scls_set_option(scls_ctx* ctx, int32_t option, int64_t value) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  if (option == SCLS_OPT_SIM_DIGESTS) {
    ctx->sim_digests = value != 0;
    return SCLS_OK;
  }
  if (option == SCLS_OPT_DP_KERNEL) {
    ctx->dp_mode = (int)value;
    return SCLS_OK;
  }
  if (option == SCLS_OPT_SIM_CONCURRENT) {
    ctx->sim_concurrent = value != 0;
    return SCLS_OK;
  }
  if (option == SCLS_OPT_DP_CLUSTER) {
    if (value != 1 && value != 2 && value != 4) return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "DP cluster size must be 1, 2 or 4");
    ctx->dp_cluster = (int)value;
    return SCLS_OK;
  }
  if (option == SCLS_OPT_ILS_KERNEL) {
    ctx->ils_lockstep = value == 1;
    ctx->ils_split = value != 2;
    return SCLS_OK;
  }
  if (option == SCLS_OPT_BATCH_PATH) {
    ctx->force_large_path = value != 0;
    ctx->force_lsd_sort = value == 2;
    return SCLS_OK;
  }
  return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "unknown option");
}

scls_status scls_debug_dp_profile(scls_ctx* ctx, int32_t enable, uint64_t out[8]) {
  if (!ctx) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null context");
  SCLS_CUDA(cudaSetDevice(ctx->device));
  if (enable && !ctx->dp_prof) {
    SCLS_CUDA(cudaMalloc(&ctx->dp_prof, 8 * sizeof(unsigned long long)));
    SCLS_CUDA(cudaMemset(ctx->dp_prof, 0, 8 * sizeof(unsigned long long)));
  }
  if (out) {
    for (int i = 0; i < 8; ++i) out[i] = 0;
    if (ctx->dp_prof) {
      SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
      SCLS_CUDA(cudaMemcpy(out, ctx->dp_prof, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
      SCLS_CUDA(cudaMemset(ctx->dp_prof, 0, 8 * sizeof(unsigned long long)));
    }
  }
  if (!enable && ctx->dp_prof) {
    cudaFree(ctx->dp_prof);
    ctx->dp_prof = nullptr;
  }
  return SCLS_OK;
}

// ---- validation: cost_model.cpp:70-87, memory_model.cpp:92-120, sched_policies.cpp:45-57

scls_status scls_validate_latency(const scls_latency* m) {
  if (!m) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null latency model");
  const double c[8] = {m->p1, m->p2, m->p3, m->p4, m->d1, m->d2, m->d3, m->d4};
  for (double v : c)
    if (!std::isfinite(v)) return set_error(nullptr, SCLS_ERR_DEGENERATE_MODEL, "latency model has a non-finite coefficient");
  if (m->n_cap < 1 || m->l_cap < 1)
    return set_error(nullptr, SCLS_ERR_DEGENERATE_MODEL, "latency model operating range caps must be >= 1");
  auto negative = [&](double c1, double c2, double c3, double c4) {
    for (int n : {1, (int)m->n_cap})
      for (int l : {1, (int)m->l_cap}) {
        volatile double v = c1 * double(n) * double(l);
        v = v + c2 * n;
        v = v + c3 * l;
        v = v + c4;
        if (!(v >= 0.0)) return true;
      }
    return false;
  };
  if (negative(m->p1, m->p2, m->p3, m->p4))
    return set_error(nullptr, SCLS_ERR_DEGENERATE_MODEL, "latency model predicts negative prefill time within operating range");
  if (negative(m->d1, m->d2, m->d3, m->d4))
    return set_error(nullptr, SCLS_ERR_DEGENERATE_MODEL, "latency model predicts negative decode-step time within operating range");
  return SCLS_OK;
}

scls_status scls_validate_memory(const scls_memory* m) {
  if (!m) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null memory model");
  if (m->kind == SCLS_MEM_ANALYTIC) {
    for (double v : {m->m_cap, m->m_model, m->m_engine, m->delta, m->zeta})
      if (!std::isfinite(v)) return set_error(nullptr, SCLS_ERR_ERROR, "memory model has a non-finite field");
    if (!(m->m_cap > m->m_model + m->m_engine)) return set_error(nullptr, SCLS_ERR_ERROR, "memory model needs m_cap > m_model + m_engine");
    if (!(m->delta > 0.0)) return set_error(nullptr, SCLS_ERR_ERROR, "memory model needs delta > 0");
    if (!(m->zeta > 0.0 && m->zeta <= 1.0)) return set_error(nullptr, SCLS_ERR_ERROR, "memory model needs zeta in (0, 1]");
    return SCLS_OK;
  }
  if (m->kind != SCLS_MEM_RULE_TABLE) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "unknown memory model kind");
  if (m->n_rules < 1) return set_error(nullptr, SCLS_ERR_ERROR, "rule-table memory model needs >= 1 row");
  if (m->n_rules > SCLS_MAX_RULES) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "too many rule-table rows");
  for (int i = 0; i < m->n_rules; ++i) {
    if (m->rule_max_n[i] < 1) return set_error(nullptr, SCLS_ERR_ERROR, "rule-table max batch sizes must be >= 1");
    if (i > 0) {
      if (m->rule_threshold[i] >= m->rule_threshold[i - 1])
        return set_error(nullptr, SCLS_ERR_ERROR, "rule-table thresholds must be strictly decreasing");
      if (m->rule_max_n[i] < m->rule_max_n[i - 1])
        return set_error(nullptr, SCLS_ERR_ERROR, "rule-table max batch sizes must not decrease as thresholds do");
    }
  }
  return SCLS_OK;
}

scls_status scls_validate_sched(const scls_sched_cfg* c) {
  if (!c) return set_error(nullptr, SCLS_ERR_INVALID_ARGUMENT, "null scheduler config");
  if (!(c->lambda > 0.0 && c->lambda < 1.0)) return set_error(nullptr, SCLS_ERR_ERROR, "lambda must lie in (0, 1)");
  if (!(c->gamma > 0.0)) return set_error(nullptr, SCLS_ERR_ERROR, "gamma must be > 0");
  if (c->slice_len < 1) return set_error(nullptr, SCLS_ERR_ERROR, "slice_len must be >= 1");
  if (c->max_gen_limit < c->slice_len) return set_error(nullptr, SCLS_ERR_ERROR, "slice_len must not exceed max_gen_limit");
  if (c->fixed_batch_size < 1) return set_error(nullptr, SCLS_ERR_ERROR, "fixed_batch_size must be >= 1");
  if (c->max_concurrent < 1) return set_error(nullptr, SCLS_ERR_ERROR, "max_concurrent must be >= 1");
  if (c->worker_count < 1) return set_error(nullptr, SCLS_ERR_ERROR, "worker_count must be >= 1");
  if (c->policy < SCLS_POLICY_SCLS || c->policy > SCLS_POLICY_ILS)
    return set_error(nullptr, SCLS_ERR_ERROR, "unknown policy (expected scls, sls, or ils)");
  return SCLS_OK;
}

// ---- estimators ---------------------------------------------------------------------

scls_status scls_batch_serve_time(scls_ctx* ctx, int64_t count, const int32_t* n, const int32_t* l_in,
                                  const int32_t* l_out, const scls_latency* lat, double* out, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  if (count < 0 || !lat || (count && (!n || !l_in || !l_out || !out)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return SCLS_OK;
  const int32_t *dn, *dl, *dk;
  if ((st = stage_in(ctx, 0, n, count, mem, &dn)) || (st = stage_in(ctx, 1, l_in, count, mem, &dl)) ||
      (st = stage_in(ctx, 2, l_out, count, mem, &dk)))
    return st;
  double* dout = stage_out_buf(ctx, 3, out, count, mem);
  if (!dout) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  bst_kernel<<<std::min(div_up(count, 256), ctx->sm_count * 16), 256, 0, ctx->stream>>>(count, dn, dl, dk, make_lat(*lat), dout);
  SCLS_LAUNCHED();
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  if ((st = copy_out(ctx, out, dout, count, mem))) return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  collect_timings(ctx, 1);
  return SCLS_OK;
}

scls_status scls_would_oom(scls_ctx* ctx, int64_t count, const int32_t* n, const int32_t* l_in, int32_t slice_len,
                           const scls_memory* memm, uint8_t* out, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  if (count < 0 || !check_memory_arg(ctx, memm) || (count && (!n || !l_in || !out)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return SCLS_OK;
  const int32_t *dn, *dl;
  if ((st = stage_in(ctx, 0, n, count, mem, &dn)) || (st = stage_in(ctx, 1, l_in, count, mem, &dl))) return st;
  uint8_t* dout = stage_out_buf(ctx, 3, out, count, mem);
  if (!dout) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  oom_kernel<<<std::min(div_up(count, 256), ctx->sm_count * 16), 256, 0, ctx->stream>>>(count, dn, dl, slice_len, make_mem(*memm), dout);
  SCLS_LAUNCHED();
  if ((st = copy_out(ctx, out, dout, count, mem))) return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return SCLS_OK;
}

scls_status scls_max_batch_size(scls_ctx* ctx, int64_t count, const int32_t* l_in, int32_t slice_len,
                                const scls_memory* memm, int32_t* out, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  if (count < 0 || !check_memory_arg(ctx, memm) || (count && (!l_in || !out)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (count == 0) return SCLS_OK;
  const int32_t* dl;
  if ((st = stage_in(ctx, 1, l_in, count, mem, &dl))) return st;
  int32_t* dout = stage_out_buf(ctx, 3, out, count, mem);
  if (!dout) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  mbs_kernel<<<std::min(div_up(count, 256), ctx->sm_count * 16), 256, 0, ctx->stream>>>(count, dl, slice_len, make_mem(*memm), dout);
  SCLS_LAUNCHED();
  if ((st = copy_out(ctx, out, dout, count, mem))) return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return SCLS_OK;
}

// ---- batcher / offloader / fused tick -----------------------------------------------

// Host-memory calls on pools up to kPackMax requests stage their three input
// arrays through one pinned buffer (one H2D copy) and read their five result
// arrays back as one region (one D2H copy, scattered on the host after the
// sync): at these sizes each pageable copy costs more than the kernels.
constexpr int64_t kPackMax = 1 << 16;
struct BatchPack {
  bool on = false;
  char* h_out = nullptr;  // pinned: the result region after the D2H copy
  char* d_out = nullptr;  // device: order | seg_begin | l_in | est | member_id
  size_t off[5] = {}, bytes = 0;
};

static size_t pack_align(size_t x) { return (x + 15) & ~(size_t)15; }

static scls_status batch_impl(scls_ctx* ctx, int64_t n, const int32_t* eff_len, const double* arrival,
                              const int64_t* id, int32_t slice_len, const scls_latency* lat,
                              const scls_memory* memm, int64_t first_batch_id, scls_batches* out,
                              int32_t mem, BatchOutputs* dev_out_keep, BatchPack* pk) {
  scls_status st;
  if (n < 0 || !lat || !check_memory_arg(ctx, memm) || !out || (n && (!eff_len || !arrival || !id)) ||
      (n && (!out->seg_begin || !out->l_in || !out->est)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  out->n_batches = 0;
  if (n == 0) {
    if (mem == SCLS_MEM_HOST) out->seg_begin[0] = 0;
    else SCLS_CUDA(cudaMemsetAsync(out->seg_begin, 0, sizeof(int32_t), ctx->stream));
    return SCLS_OK;
  }
  const int32_t* d_eff;
  const double* d_arr;
  const int64_t* d_id;
  BatchOutputs d{};
  pk->on = mem == SCLS_MEM_HOST && n <= kPackMax;
  if (pk->on) {
    const size_t be = pack_align(4 * (size_t)n), ba = pack_align(8 * (size_t)n), bi = pack_align(8 * (size_t)n);
    const size_t in_bytes = be + ba + bi;
    pk->off[0] = 0;                                          // order
    pk->off[1] = pk->off[0] + pack_align(4 * (size_t)n);     // seg_begin (n + 1)
    pk->off[2] = pk->off[1] + pack_align(4 * (size_t)(n + 1));  // l_in
    pk->off[3] = pk->off[2] + pack_align(4 * (size_t)n);     // est
    pk->off[4] = pk->off[3] + pack_align(8 * (size_t)n);     // member_id
    pk->bytes = pk->off[4] + pack_align(8 * (size_t)n);
    char* h = (char*)ctx->host_stage(in_bytes + pk->bytes);
    char* din = (char*)ctx->buf(kSlotStage + 8, in_bytes);
    pk->d_out = (char*)ctx->buf(kSlotStage + 9, pk->bytes);
    if (!h || !din || !pk->d_out) return set_error(ctx, SCLS_ERR_CUDA, "staging allocation failed");
    std::memcpy(h, eff_len, 4 * (size_t)n);
    std::memcpy(h + be, arrival, 8 * (size_t)n);
    std::memcpy(h + be + ba, id, 8 * (size_t)n);
    SCLS_CUDA(cudaMemcpyAsync(din, h, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
    pk->h_out = h + in_bytes;
    d_eff = (const int32_t*)din;
    d_arr = (const double*)(din + be);
    d_id = (const int64_t*)(din + be + ba);
    d.order = out->order ? (int32_t*)(pk->d_out + pk->off[0]) : nullptr;
    d.seg_begin = (int32_t*)(pk->d_out + pk->off[1]);
    d.l_in = (int32_t*)(pk->d_out + pk->off[2]);
    d.est = (double*)(pk->d_out + pk->off[3]);
    d.member_id = out->member_id ? (int64_t*)(pk->d_out + pk->off[4]) : nullptr;
  } else {
    if ((st = stage_in(ctx, 0, eff_len, n, mem, &d_eff)) || (st = stage_in(ctx, 1, arrival, n, mem, &d_arr)) ||
        (st = stage_in(ctx, 2, id, n, mem, &d_id)))
      return st;
    d.order = stage_out_buf(ctx, 3, out->order, n, mem);
    d.seg_begin = stage_out_buf(ctx, 4, out->seg_begin, n + 1, mem);
    d.l_in = stage_out_buf(ctx, 5, out->l_in, n, mem);
    d.est = stage_out_buf(ctx, 6, out->est, n, mem);
    d.member_id = stage_out_buf(ctx, 7, out->member_id, n, mem);
  }
  if (!d.seg_begin || !d.l_in || !d.est) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  BatchInputs in{n, d_eff, d_arr, d_id, slice_len, lat, memm};
  int64_t nb = 0;
  if ((st = batch_requests_device(ctx, in, d, &nb, nullptr))) return st;
  out->n_batches = nb;
  (void)first_batch_id;  // batch b has id first_batch_id + b (documented in scls_capi.h)
  if (dev_out_keep) *dev_out_keep = d;
  return SCLS_OK;
}

static scls_status batch_copy_out(scls_ctx* ctx, int64_t n, const BatchOutputs& d, scls_batches* out, int32_t mem,
                                  const BatchPack& pk) {
  scls_status st;
  const int64_t nb = out->n_batches;
  if (pk.on) {  // the used prefix of the result region (member_id is last)
    const size_t used = out->member_id ? pk.bytes : pk.off[4];
    SCLS_CUDA(cudaMemcpyAsync(pk.h_out, pk.d_out, used, cudaMemcpyDeviceToHost, ctx->stream));
    return SCLS_OK;
  }
  if ((st = copy_out(ctx, out->order, d.order, n, mem)) || (st = copy_out(ctx, out->seg_begin, d.seg_begin, nb + 1, mem)) ||
      (st = copy_out(ctx, out->l_in, d.l_in, nb, mem)) || (st = copy_out(ctx, out->est, d.est, nb, mem)) ||
      (st = copy_out(ctx, out->member_id, d.member_id, n, mem)))
    return st;
  return SCLS_OK;
}

// After the stream sync: scatter the packed result region into the caller's arrays.
static void batch_finish(int64_t n, scls_batches* out, const BatchPack& pk) {
  if (!pk.on || n == 0) return;
  const int64_t nb = out->n_batches;
  if (out->order) std::memcpy(out->order, pk.h_out + pk.off[0], 4 * (size_t)n);
  std::memcpy(out->seg_begin, pk.h_out + pk.off[1], 4 * (size_t)(nb + 1));
  std::memcpy(out->l_in, pk.h_out + pk.off[2], 4 * (size_t)nb);
  std::memcpy(out->est, pk.h_out + pk.off[3], 8 * (size_t)nb);
  if (out->member_id) std::memcpy(out->member_id, pk.h_out + pk.off[4], 8 * (size_t)n);
}

scls_status scls_batch_requests(scls_ctx* ctx, int64_t n, const int32_t* eff_len, const double* arrival,
                                const int64_t* id, int32_t slice_len, const scls_latency* lat,
                                const scls_memory* memm, int64_t first_batch_id, scls_batches* out, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  BatchOutputs d{};
  BatchPack pk;
  if ((st = batch_impl(ctx, n, eff_len, arrival, id, slice_len, lat, memm, first_batch_id, out, mem, &d, &pk))) return st;
  if (n == 0) return SCLS_OK;
  if ((st = batch_copy_out(ctx, n, d, out, mem, pk))) return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  batch_finish(n, out, pk);
  collect_timings(ctx, 4);
  ctx->timings[7] = ctx->dp_last_mono ? 1.f : 0.f;
  return SCLS_OK;
}

scls_status scls_offload(scls_ctx* ctx, int64_t n_batches, const int64_t* batch_id, const double* est,
                         int32_t n_workers, const int32_t* worker_id, double* load_inout,
                         int64_t* out_batch_id, int32_t* out_worker, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  if (n_batches < 0 || n_workers < 0 || (n_batches && (!batch_id || !est || !out_batch_id || !out_worker)) ||
      (n_workers && (!worker_id || !load_inout)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  if (n_batches == 0) return SCLS_OK;  // offloader.cpp:26
  if (n_workers == 0) return set_error(ctx, SCLS_ERR_NO_WORKERS, "cannot offload batches: no workers configured");
  const int64_t* d_bid;
  const double* d_est;
  const int32_t* d_wid;
  if ((st = stage_in(ctx, 0, batch_id, n_batches, mem, &d_bid)) || (st = stage_in(ctx, 1, est, n_batches, mem, &d_est)) ||
      (st = stage_in(ctx, 2, worker_id, n_workers, mem, &d_wid)))
    return st;
  double* d_load;
  if (mem == SCLS_MEM_DEVICE) {
    d_load = load_inout;
  } else {
    d_load = (double*)ctx->buf(kSlotStage + 3, sizeof(double) * n_workers);
    if (!d_load) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    SCLS_CUDA(cudaMemcpyAsync(d_load, load_inout, sizeof(double) * n_workers, cudaMemcpyHostToDevice, ctx->stream));
  }
  int64_t* d_ob = stage_out_buf(ctx, 4, out_batch_id, n_batches, mem);
  int32_t* d_ow = stage_out_buf(ctx, 5, out_worker, n_batches, mem);
  if (!d_ob || !d_ow) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
  SCLS_CUDA(cudaEventRecord(ctx->ev[0], ctx->stream));
  if ((st = offload_device(ctx, n_batches, d_bid, d_est, n_workers, d_wid, d_load, d_ob, d_ow))) return st;
  SCLS_CUDA(cudaEventRecord(ctx->ev[1], ctx->stream));
  if ((st = copy_out(ctx, out_batch_id, d_ob, n_batches, mem)) || (st = copy_out(ctx, out_worker, d_ow, n_batches, mem)) ||
      (st = copy_out(ctx, load_inout, (const double*)d_load, n_workers, mem)))
    return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  collect_timings(ctx, 1);
  ctx->timings[5] = ctx->timings[1];
  ctx->timings[1] = 0.f;
  return SCLS_OK;
}

scls_status scls_schedule(scls_ctx* ctx, int64_t n, const int32_t* eff_len, const double* arrival,
                          const int64_t* id, int32_t slice_len, const scls_latency* lat,
                          const scls_memory* memm, int64_t first_batch_id, int32_t n_workers,
                          const int32_t* worker_id, double* load_inout, scls_batches* out,
                          int64_t* out_batch_id, int32_t* out_worker, int32_t mem) {
  scls_status st = begin_call(ctx);
  if (st) return st;
  if (n_workers < 0 || (n_workers && (!worker_id || !load_inout)) || (n && (!out_batch_id || !out_worker)))
    return set_error(ctx, SCLS_ERR_INVALID_ARGUMENT, "bad arguments");
  BatchOutputs d{};
  BatchPack pk;
  if ((st = batch_impl(ctx, n, eff_len, arrival, id, slice_len, lat, memm, first_batch_id, out, mem, &d, &pk))) return st;
  const int64_t nb = out->n_batches;
  if (nb > 0 && n_workers == 0) return set_error(ctx, SCLS_ERR_NO_WORKERS, "cannot offload batches: no workers configured");
  if (nb > 0) {
    int64_t* d_bid = (int64_t*)ctx->buf(kSlotStage + 10, sizeof(int64_t) * nb);
    if (!d_bid) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    iota_ids_kernel<<<div_up(nb, 256), 256, 0, ctx->stream>>>(nb, first_batch_id, d_bid);
    SCLS_LAUNCHED();
    const int32_t* d_wid;
    if ((st = stage_in(ctx, 11, worker_id, n_workers, mem, &d_wid))) return st;
    double* d_load;
    if (mem == SCLS_MEM_DEVICE) {
      d_load = load_inout;
    } else {
      d_load = (double*)ctx->buf(kSlotStage + 12, sizeof(double) * n_workers);
      if (!d_load) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
      SCLS_CUDA(cudaMemcpyAsync(d_load, load_inout, sizeof(double) * n_workers, cudaMemcpyHostToDevice, ctx->stream));
    }
    int64_t* d_ob = stage_out_buf(ctx, 13, out_batch_id, nb, mem);
    int32_t* d_ow = stage_out_buf(ctx, 14, out_worker, nb, mem);
    if (!d_ob || !d_ow) return set_error(ctx, SCLS_ERR_CUDA, "allocation failed");
    if ((st = offload_device(ctx, nb, d_bid, d.est, n_workers, d_wid, d_load, d_ob, d_ow))) return st;
    SCLS_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
    if ((st = copy_out(ctx, out_batch_id, d_ob, nb, mem)) || (st = copy_out(ctx, out_worker, d_ow, nb, mem)) ||
        (st = copy_out(ctx, load_inout, (const double*)d_load, n_workers, mem)))
      return st;
  } else if (n > 0) {
    SCLS_CUDA(cudaEventRecord(ctx->ev[5], ctx->stream));
  }
  if (n > 0 && (st = batch_copy_out(ctx, n, d, out, mem, pk))) return st;
  SCLS_CUDA(cudaStreamSynchronize(ctx->stream));
  batch_finish(n, out, pk);
  if (n > 0) collect_timings(ctx, 5);
  ctx->timings[7] = ctx->dp_last_mono ? 1.f : 0.f;
  return SCLS_OK;
}

}  // extern "C"
