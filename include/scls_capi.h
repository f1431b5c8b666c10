/* scls_capi.h — C-ABI boundary of the B200-native SCLS scheduling core.
 *
 * Plain C types only (no torch, no C++), so any FFI (ctypes, cgo, JNI) or the
 * C++ drop-in layer (paper_2406_13511_b200/dropin/, which re-creates the
 * reference's own headers on top of it) can bind it.  Every entry point
 * replaces one public function of the reference library `slicesim`
 * (/root/reference/proj/core/include/slicesim/*.h); the replaced interface is
 * cited on each declaration as reference file:line.
 *
 * Conventions
 *   - A context (scls_ctx) binds one CUDA device and one stream.  Calls are
 *     stream-ordered and synchronous with respect to the host: when a call
 *     returns, its outputs are valid.  One context per host thread.
 *   - `mem` selects where the caller's array arguments live: SCLS_MEM_HOST
 *     (pageable or pinned host memory; the library copies in/out inside the
 *     call) or SCLS_MEM_DEVICE (device pointers on the context's device).
 *   - Errors map 1:1 onto the reference exception classes (errors.h:26-87).
 *     scls_last_error() returns the message, scls_last_request_id() the
 *     offending request of an InfeasibleRequestError (errors.h:51-56).
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     entry point fails with SCLS_ERR_CUDA.
 */
#ifndef SCLS_CAPI_H_
#define SCLS_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCLS_ABI_VERSION 1
#define SCLS_MAX_RULES 32

/* errors.h:26-87 — one code per exception class. */
typedef enum scls_status {
  SCLS_OK = 0,
  SCLS_ERR_ERROR = 1,                /* slicesim::Error (validation)          */
  SCLS_ERR_INSUFFICIENT_SAMPLES = 2, /* InsufficientSamplesError              */
  SCLS_ERR_DEGENERATE_MODEL = 3,     /* DegenerateModelError                  */
  SCLS_ERR_WRONG_KIND = 4,           /* WrongKindError                        */
  SCLS_ERR_INFEASIBLE_REQUEST = 5,   /* InfeasibleRequestError{request_id}    */
  SCLS_ERR_NO_WORKERS = 6,           /* NoWorkersError                        */
  SCLS_ERR_PARSE = 7,                /* ParseError                            */
  SCLS_ERR_LIMIT_VIOLATION = 8,      /* LimitViolationError                   */
  SCLS_ERR_EMPTY_LOG = 9,            /* EmptyLogError                         */
  SCLS_ERR_NON_TERMINATION = 10,     /* NonTerminationError                   */
  SCLS_ERR_INVALID_ARGUMENT = 11,    /* C-ABI misuse (null pointer, bad size) */
  SCLS_ERR_CUDA = 12,                /* no device / launch failure            */
  SCLS_ERR_CAPACITY = 13             /* caller buffer (event log) too small   */
} scls_status;

enum { SCLS_MEM_HOST = 0, SCLS_MEM_DEVICE = 1 };

/* cost_model.h:29-39 LatencyModel. */
typedef struct scls_latency {
  double p1, p2, p3, p4; /* prefill: p1*n*l + p2*n + p3*l + p4 */
  double d1, d2, d3, d4; /* decode step: d1*n*l + d2*n + d3*l + d4 */
  double rmse_prefill, rmse_decode;
  int32_t n_cap, l_cap;
} scls_latency;

enum { SCLS_MEM_ANALYTIC = 0, SCLS_MEM_RULE_TABLE = 1 };

/* memory_model.h:20-53 MemoryModel (rule rows inline, <= SCLS_MAX_RULES). */
typedef struct scls_memory {
  int32_t kind;    /* SCLS_MEM_ANALYTIC | SCLS_MEM_RULE_TABLE */
  int32_t n_rules;
  double m_cap, m_model, m_engine, delta, zeta;
  int32_t rule_threshold[SCLS_MAX_RULES]; /* strictly decreasing */
  int32_t rule_max_n[SCLS_MAX_RULES];
} scls_memory;

enum { SCLS_POLICY_SCLS = 0, SCLS_POLICY_SLS = 1, SCLS_POLICY_ILS = 2 };

/* sched_policies.h:39-48 SchedulerConfig (+ the Simulator horizon,
 * sim_engine.h:61-62). */
typedef struct scls_sched_cfg {
  int32_t policy;
  int32_t slice_len;
  int32_t max_gen_limit;
  int32_t fixed_batch_size;
  int32_t max_concurrent;
  int32_t worker_count;  // >= 1; the device simulator takes up to 1024
  double lambda;
  double gamma;
  double horizon_s;
} scls_sched_cfg;

enum { SCLS_DIST_UNIFORM = 0, SCLS_DIST_LOGNORMAL = 1, SCLS_DIST_HISTOGRAM = 2 };
#define SCLS_MAX_BUCKETS 30

/* workload.h:32-50 LengthDist (histogram buckets inline). */
typedef struct scls_length_dist {
  int32_t kind;
  int32_t lo, hi;  /* uniform */
  double mu, sigma; /* log-normal */
  int32_t cap;
  int32_t n_buckets; /* histogram: n_buckets weights, n_buckets+1 edges */
  int32_t edges[SCLS_MAX_BUCKETS + 1];
  double weights[SCLS_MAX_BUCKETS];
} scls_length_dist;

/* workload.h:54-62 WorkloadSpec. */
typedef struct scls_workload_spec {
  double rate;
  double duration_s;
  scls_length_dist input_len_dist;
  scls_length_dist gen_len_dist;
  int32_t max_input_limit;
  int32_t max_gen_limit;
  uint64_t seed;
} scls_workload_spec;

typedef struct scls_ctx scls_ctx;

/* ---- context ------------------------------------------------------------ */
int32_t scls_abi_version(void);
/* stream: a cudaStream_t (NULL = a private non-blocking stream). */
scls_status scls_ctx_create(int32_t device, void* stream, scls_ctx** out);
void scls_ctx_destroy(scls_ctx* ctx);
/* Message of the last failed call on this context (thread-local when ctx is
 * NULL); returns the full message length. */
size_t scls_last_error(const scls_ctx* ctx, char* buf, size_t cap);
int64_t scls_last_request_id(const scls_ctx* ctx);
/* Device time (ms, CUDA events on the context stream) of the phases of the
 * last call: [0]=total, [1]=sort, [2]=estimate/window tables, [3]=DP chain,
 * [4]=backtrack+emit, [5]=offload, [6]=simulate, [7]=device trace generation
 * (scls_run_sweep / scls_generate_batch) or, after a batcher call, 1.0 when
 * the monotone DP kernel ran. */
void scls_last_timings(const scls_ctx* ctx, float out_ms[8]);
/* Number of CUDA kernel launches issued by the last call. */
int64_t scls_last_launch_count(const scls_ctx* ctx);
/* Context options.  SCLS_OPT_SIM_DIGESTS (default 1): scls_simulate fills
 * the h_* log digests of scls_trace_result; 0 skips them (the metrics are
 * computed either way, and the digests are zero). */
enum { SCLS_OPT_SIM_DIGESTS = 1, SCLS_OPT_DP_KERNEL = 2, SCLS_OPT_SIM_CONCURRENT = 3, SCLS_OPT_ILS_KERNEL = 4,
       SCLS_OPT_BATCH_PATH = 5, SCLS_OPT_DP_CLUSTER = 6 };
/* SCLS_OPT_DP_KERNEL: 0 (default) picks the monotone decision kernel when the
 * model allows it and some window exceeds 32 rows, else the serial-chain
 * kernel; 1 forces the chain kernel; 2 forces the decision kernel when the
 * model allows it.  SCLS_OPT_SIM_CONCURRENT (default 1): the simulator's
 * per-policy launches run concurrently on forked streams (0: in sequence on
 * the context stream; results are identical).  Each launch takes its jobs
 * longest first, so the policies' tails overlap: 65.8 vs 70.1 ms on the C5
 * sweep.  SCLS_OPT_ILS_KERNEL
 * (default 0): metrics-only ILS and SLS run every instance / worker in its own
 * lane and merge the completions (csrc/sim_indep.cuh; each as a simulation
 * kernel packing 32 / W jobs per warp plus a merge kernel with a warp per
 * job); 1 forces the lock-step kernels that process the global event order
 * directly; 2 runs each policy in one kernel (ILS: packs of two jobs whose
 * merges follow in series; SLS: one job per warp) (results identical).
 * SCLS_OPT_BATCH_PATH (default 0): batch_requests / schedule take the fused
 * four-launch small-pool path for n <= 4096 and the multi-kernel path above;
 * 1 forces the multi-kernel path at every size; 2 does that and sorts with
 * the 8-bit LSD radix sort instead of the eff-bucket sort (results
 * identical).
 * SCLS_OPT_DP_CLUSTER (default 1): the monotone DP kernel runs as a
 * thread-block cluster of this many CTAs (1, 2 or 4): the older far
 * candidates go to the peer CTAs, exchanged over distributed shared memory
 * (results identical).  Measured slower than one CTA on the C3 pool (2: 58,
 * 4: 70 vs 51 ms: the per-tile DSMEM handshake costs more than the far scan
 * it moves), so 1 is the default. */
scls_status scls_set_option(scls_ctx* ctx, int32_t option, int64_t value);
/* Diagnostics: enable/disable clock64 phase counters in the DP chain kernel
 * and read-and-reset them (cycles: main chain, main barrier wait, helper
 * staging, helper far candidates, helper wait, helper-warp count). */
scls_status scls_debug_dp_profile(scls_ctx* ctx, int32_t enable, uint64_t out[8]);

/* ---- validation (host only; mirrors the reference validators) ----------- */
scls_status scls_validate_latency(const scls_latency* m);   /* cost_model.cpp:70-87    */
/* cost_model.h:45-50 ProfileSample (phase 0 = prefill, 1 = decode). */
typedef struct scls_profile_sample {
  int32_t phase;
  int32_t batch_size;
  int32_t length;
  int32_t pad_;
  double latency_s;
} scls_profile_sample;
/* cost_model.cpp:96-160 fit (cost_model.h:80): least squares of the prefill
 * and decode surfaces c1*n*l + c2*n + c3*l + c4 by column-pivoting Householder
 * QR, rmse per phase, then validate.  Host computation (a 4-parameter
 * problem).  SCLS_ERR_INSUFFICIENT_SAMPLES with the reference's messages
 * (fewer than 4 samples / 2 sizes / 2 lengths in a phase, or rank < 4);
 * SCLS_ERR_DEGENERATE_MODEL when the fitted model fails validate. */
scls_status scls_fit_latency(const scls_profile_sample* samples, int64_t n, int32_t n_cap, int32_t l_cap,
                             scls_latency* out);
scls_status scls_validate_memory(const scls_memory* m);     /* memory_model.cpp:92-120 */
scls_status scls_validate_sched(const scls_sched_cfg* cfg); /* sched_policies.cpp:45-57 */

/* ---- estimators: batched device evaluation ------------------------------
 * Replaces cost_model.h:54-66 batch_serve_time and memory_model.h:62-66
 * would_oom / max_batch_size, evaluated for `count` candidates at once with
 * the reference's exact fp64 operation order. */
scls_status scls_batch_serve_time(scls_ctx* ctx, int64_t count, const int32_t* n,
                                  const int32_t* l_in, const int32_t* l_out,
                                  const scls_latency* lat, double* out, int32_t mem);
scls_status scls_would_oom(scls_ctx* ctx, int64_t count, const int32_t* n,
                           const int32_t* l_in, int32_t slice_len,
                           const scls_memory* memm, uint8_t* out, int32_t mem);
scls_status scls_max_batch_size(scls_ctx* ctx, int64_t count, const int32_t* l_in,
                                int32_t slice_len, const scls_memory* memm,
                                int32_t* out, int32_t mem);

/* ---- batcher: batcher.h:40-43 batch_requests ------------------------------
 * Inputs (length n): effective input length, arrival time, id.
 * Outputs (caller-allocated; capacities n, n+1, n, n, n, n):
 *   order[p]      input index of the p-th request in (eff, arrival, id) order
 *   seg_begin[b]  first sorted position of batch b; seg_begin[n_batches] = n
 *   l_in[b], est[b]  batch input length and est_serve_time
 *   member_id[p]  id of the p-th member in batch order (= id[order[p]]); may be NULL
 * Batch b has id first_batch_id + b and planned_l_out = slice_len. */
typedef struct scls_batches {
  int64_t n_batches;
  int32_t* order;
  int32_t* seg_begin;
  int32_t* l_in;
  double* est;
  int64_t* member_id;
} scls_batches;

scls_status scls_batch_requests(scls_ctx* ctx, int64_t n, const int32_t* eff_len,
                                const double* arrival, const int64_t* id,
                                int32_t slice_len, const scls_latency* lat,
                                const scls_memory* memm, int64_t first_batch_id,
                                scls_batches* out, int32_t mem);

/* ---- offloader: offloader.h:39-44 offload ----------------------------------
 * Batches in creation order (ids, estimates); workers (ids, loads, mutated in
 * place).  Outputs the (batch_id, worker_id) assignment sequence. */
scls_status scls_offload(scls_ctx* ctx, int64_t n_batches, const int64_t* batch_id,
                         const double* est, int32_t n_workers, const int32_t* worker_id,
                         double* load_inout, int64_t* out_batch_id, int32_t* out_worker,
                         int32_t mem);

/* Fused batch_requests + offload (the SCLS tick, sched_policies.cpp:93-112).
 * out_batch_id/out_worker have capacity n. */
scls_status scls_schedule(scls_ctx* ctx, int64_t n, const int32_t* eff_len,
                          const double* arrival, const int64_t* id, int32_t slice_len,
                          const scls_latency* lat, const scls_memory* memm,
                          int64_t first_batch_id, int32_t n_workers,
                          const int32_t* worker_id, double* load_inout,
                          scls_batches* out, int64_t* out_batch_id, int32_t* out_worker,
                          int32_t mem);

/* ---- simulator: sim_engine.h:61-67 Simulator::run + metrics.h:41 compute ---
 * Runs `n_traces` independent simulations.  Trace t owns requests
 * [req_offset[t], req_offset[t+1]) of the concatenated arrays, given in
 * arrival order with ids 0..n_t-1 (sim_engine.cpp:102-114), and config
 * cfg[cfg_index[t]] (cfg_index may be NULL: cfg[0] for all).
 *
 * Per-trace results: the MetricsReport fields (metrics.h:26-36), the status
 * (NonTermination / Infeasible / EmptyLog map to codes, never traps), and
 * FNV-1a-64 hashes of the completion order, the dispatch sequence and the
 * completion times, plus a word-wise hash of the whole
 * event log.  slice_hist[t*hist_bins + s] counts requests completed after s
 * slices (fraction = count / completed, metrics.cpp:109-111). */
typedef struct scls_trace_result {
  int32_t status;
  int32_t worker_count;
  int64_t error_request_id;
  int64_t n_requests;
  int64_t completed;
  double throughput;
  double avg_response_s;
  double p95_response_s;
  double ct_std_s;
  double avg_pad_tokens;
  double avg_invalid_tokens;
  double avg_batch_size;
  double early_return_ratio;
  int64_t total_pad;
  int64_t total_invalid;
  int64_t batch_count;
  int64_t batch_members;
  int64_t early_returns;
  int64_t n_events;     /* EventRecords the reference log would hold */
  int64_t n_dispatches;
  int64_t n_ticks;
  uint64_t h_complete_ids;
  uint64_t h_dispatch;
  uint64_t h_complete_t;
  uint64_t h_log;
  double sim_clock;     /* clock at the last processed event */
} scls_trace_result;

/* Optional full event log (EventRecord, event_log.h:52-69; members
 * event_log.h:41-47) for traces whose index is < n_logged.  Trace t writes
 * records [rec_offset[t], rec_offset[t]+rec_count[t]) and members likewise;
 * capacity per trace = rec_cap / mem_cap.  Device pointers when mem =
 * SCLS_MEM_DEVICE. */
typedef struct scls_event_record {
  double t;
  double est_serve_s;
  double response_s;
  double next_interval_s;
  int64_t request;
  int64_t batch;
  int32_t kind; /* event_log.h:27-34 order: arrival, tick, dispatch, batch_start, batch_end, complete */
  int32_t worker;
  int32_t n;
  int32_t l_in;
  int32_t planned_l_out;
  int32_t served_l_out;
  int32_t input_len;
  int32_t gen_len;
  int32_t slices;
  int32_t member_count;
  int64_t member_offset; /* into the member array, relative to the trace */
} scls_event_record;

typedef struct scls_member {
  int64_t request;
  int32_t effective_input;
  int32_t pad;
  int32_t gen;
  int32_t invalid;
} scls_member;

typedef struct scls_event_log {
  int32_t n_logged;
  int64_t rec_cap;     /* records per trace */
  int64_t mem_cap;     /* members per trace */
  scls_event_record* records; /* n_logged * rec_cap */
  scls_member* members;       /* n_logged * mem_cap */
  int64_t* rec_count;         /* n_logged */
  int64_t* mem_count;         /* n_logged */
} scls_event_log;

scls_status scls_simulate(scls_ctx* ctx, int32_t n_traces, const int64_t* req_offset,
                          const double* arrival, const int32_t* input_len,
                          const int32_t* gen_len, int32_t n_cfgs,
                          const scls_sched_cfg* cfgs, const int32_t* cfg_index,
                          const scls_latency* lat, const scls_memory* memm,
                          scls_trace_result* results, int32_t hist_bins,
                          int64_t* slice_hist, scls_event_log* log, int32_t mem);

/* The sweep grid (experiment.h:60 sweep; experiment.cpp runs every policy /
 * slice / worker configuration on the same generated trace): every config in
 * `cfgs` on every trace, each trace's requests staged once.  Job j =
 * c * n_traces + t simulates trace t under cfgs[c]; results / slice_hist /
 * log are indexed by job (n_cfgs * n_traces entries).  Same statuses and
 * per-job results as scls_simulate with the traces repeated per config. */
scls_status scls_simulate_grid(scls_ctx* ctx, int32_t n_traces, const int64_t* req_offset,
                               const double* arrival, const int32_t* input_len,
                               const int32_t* gen_len, int32_t n_cfgs,
                               const scls_sched_cfg* cfgs, const scls_latency* lat,
                               const scls_memory* memm, scls_trace_result* results,
                               int32_t hist_bins, int64_t* slice_hist, scls_event_log* log,
                               int32_t mem);

/* The sweep entry point with generation on the device: experiment.h:37,52-53
 * run_experiment / sweep (experiment.cpp:39-85 = generate -> Simulator::run ->
 * compute per run).  Trace t is generated from specs[t] on the device
 * (workload.cpp:163-181, bit-exact: mt19937_64, top-53-bit uniforms, glibc
 * 2.39's log for the gaps; uniform and histogram lengths — log-normal specs
 * fail with SCLS_ERR_ERROR), then every config runs on every trace exactly as
 * scls_simulate_grid (job j = c * n_traces + t).  specs / cfgs are host
 * structs; `mem` places results / slice_hist / log.  Timings: [7] = generation. */
scls_status scls_run_sweep(scls_ctx* ctx, int32_t n_traces, const scls_workload_spec* specs,
                           int32_t n_cfgs, const scls_sched_cfg* cfgs, const scls_latency* lat,
                           const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                           int64_t* slice_hist, scls_event_log* log, int32_t mem);

/* experiment.h:37 run_experiment for n_runs independent runs (the body of the
 * reference's sweep loop, experiment.cpp:67-83): run i generates specs[i] on
 * the device and simulates it under cfgs[i].  Same generator, statuses and
 * per-run results as scls_run_sweep (results indexed by run). */
scls_status scls_run_experiments(scls_ctx* ctx, int32_t n_runs, const scls_workload_spec* specs,
                                 const scls_sched_cfg* cfgs, const scls_latency* lat,
                                 const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                 int64_t* slice_hist, scls_event_log* log, int32_t mem);

/* workload.h:78 generate for n_specs traces at once, on the device (same
 * sampler and restrictions as scls_run_sweep).  Trace t's requests are
 * [req_offset[t], req_offset[t+1]) of the concatenated outputs (ids = arrival
 * ranks); req_offset has n_specs + 1 entries.  SCLS_ERR_CAPACITY (req_offset
 * still filled) when the total exceeds `cap`.  `mem` places the outputs. */
scls_status scls_generate_batch(scls_ctx* ctx, int32_t n_specs, const scls_workload_spec* specs,
                                int64_t cap, int64_t* req_offset, double* arrival,
                                int32_t* input_len, int32_t* gen_len, int32_t mem);

/* ---- multi-GPU sweep: SURVEY §8(e), the reference's sequential sweep loop
 * (experiment.cpp:62-85) sharded over devices ---------------------------------
 * The trace dimension is the only one that shards: trace t belongs to shard
 * floor(t * N / n_traces) (contiguous ranges, scls_shard_range).  Each shard is
 * generated and simulated on its own device exactly as scls_run_sweep, and
 * the fixed-size per-job result records (+ histograms) are then all-gathered
 * with one ncclAllGather over NVLink -- the only collective -- so every device
 * ends with the full grid in the scls_run_sweep job order (j = c * n_traces + t).
 *
 * Two launch shapes:
 *  - one process per GPU (torchrun): every rank creates its context, joins a
 *    communicator with scls_comm_init (the 128-byte id comes from
 *    scls_comm_unique_id on rank 0, broadcast by the caller), then calls
 *    scls_run_sweep_sharded with the GLOBAL spec list;
 *  - one process, many GPUs: scls_multi_create binds N devices (one context
 *    and one host thread each, one NCCL clique via ncclCommInitAll) and
 *    scls_multi_run_sweep runs the sharded sweep across them.  A device may
 *    appear more than once (shards sharing a GPU); the gather then uses peer
 *    copies instead of NCCL, which cannot put two ranks on one device.
 * NCCL is loaded at run time (libnccl.so.2); without it these calls fail with
 * SCLS_ERR_CUDA, except a 1-shard run, which needs no collective. */
void scls_shard_range(int64_t total, int32_t shard, int32_t n_shards, int64_t* lo, int64_t* hi);
scls_status scls_comm_unique_id(uint8_t out[128]);
scls_status scls_comm_init(scls_ctx* ctx, int32_t world, int32_t rank, const uint8_t id[128]);
/* Ranks of the context's communicator as NCCL reports them (1 without one). */
int32_t scls_comm_size(const scls_ctx* ctx);
/* results / slice_hist: n_cfgs * n_traces entries (the whole grid) in `mem`
 * (device memory = this rank's device).  Timings: [6] = this rank's shard
 * (generate + simulate), [5] = the gather + reorder, [0] = total. */
scls_status scls_run_sweep_sharded(scls_ctx* ctx, int32_t n_traces, const scls_workload_spec* specs,
                                   int32_t n_cfgs, const scls_sched_cfg* cfgs, const scls_latency* lat,
                                   const scls_memory* memm, scls_trace_result* results, int32_t hist_bins,
                                   int64_t* slice_hist, int32_t mem);

/* Number of visible CUDA devices (0 without a usable driver). */
int32_t scls_device_count(void);

typedef struct scls_multi scls_multi;
scls_status scls_multi_create(int32_t n_dev, const int32_t* devices, scls_multi** out);
void scls_multi_destroy(scls_multi* m);
size_t scls_multi_last_error(const scls_multi* m, char* buf, size_t cap);
/* scls_set_option on every device context of the group. */
scls_status scls_multi_set_option(scls_multi* m, int32_t option, int64_t value);
/* 1 when the gather runs over NCCL (distinct devices), 0 for peer copies. */
int32_t scls_multi_uses_nccl(const scls_multi* m);
/* results / slice_hist in host memory.  out_ms (optional, n_dev + 2 floats):
 * per-device shard time (device events), then the gather and the wall time. */
scls_status scls_multi_run_sweep(scls_multi* m, int32_t n_traces, const scls_workload_spec* specs, int32_t n_cfgs,
                                 const scls_sched_cfg* cfgs, const scls_latency* lat, const scls_memory* memm,
                                 scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                                 float* out_ms);

/* scls_run_experiments across the devices: run i (specs[i] under cfgs[i])
 * belongs to shard floor(i * N / n_runs); results / slice_hist by run, host memory. */
scls_status scls_multi_run_experiments(scls_multi* m, int32_t n_runs, const scls_workload_spec* specs,
                                       const scls_sched_cfg* cfgs, const scls_latency* lat, const scls_memory* memm,
                                       scls_trace_result* results, int32_t hist_bins, int64_t* slice_hist,
                                       float* out_ms);

/* Diagnostics: the device port of glibc's log (csrc/glibc_log.cuh) on n
 * inputs, for the bit-exactness check against the host libm. */
scls_status scls_debug_log(scls_ctx* ctx, int64_t n, const double* x, double* y, int32_t mem);
/* The same for fn = 0 log, 1 exp, 2 cos (csrc/glibc_expcos.cuh: the FMA
 * builds of glibc's exp and cos behind the log-normal lengths,
 * workload.cpp:112-118,136-141; cos for |x| < 105414350, exp exact for
 * |x| < 512 and +inf / +0 beyond). */
scls_status scls_debug_libm(scls_ctx* ctx, int32_t fn, int64_t n, const double* x, double* y, int32_t mem);

/* ---- workload: workload.h:78 generate ------------------------------------
 * Host-side Poisson trace generation (mt19937_64 + glibc log, the reference's
 * exact sampler; workload.cpp:100-181).  Writes up to `cap` requests and sets
 * *n to the full count; SCLS_ERR_CAPACITY when cap < *n. */
scls_status scls_generate(const scls_workload_spec* spec, int64_t cap, int64_t* n,
                          double* arrival, int32_t* input_len, int32_t* gen_len);

/* The reference microbenchmark's synthetic pool (bench_batcher.cpp:27-42):
 * mt19937_64(seed); request i: id i, arrival U*100, input 1+floor(U*1024),
 * generation 1+floor(U*1024).  Host-side input preparation. */
scls_status scls_make_pool(int64_t n, uint64_t seed, int32_t* input_len, double* arrival,
                           int64_t* id, int32_t* gen_len);

#ifdef __cplusplus
}
#endif

#endif /* SCLS_CAPI_H_ */
