"""ctypes mirror of include/scls_capi.h (the C-ABI boundary) plus the
reference's builtin models and presets as C structs.

The struct layouts must match scls_capi.h field for field; tests check that
the library exports every declared symbol.  The builtin constants restate
/root/reference/proj/core/src/run_config.cpp:216-241 (latency + memory models)
and workload.cpp:276-291 (length presets); the scheduler defaults restate
sched_policies.h:39-48 and run_config.h:41.
"""
from __future__ import annotations

import ctypes as C
import os

SCLS_ABI_VERSION = 1
SCLS_MAX_RULES = 32
SCLS_MAX_BUCKETS = 30

MEM_HOST, MEM_DEVICE = 0, 1
ANALYTIC, RULE_TABLE = 0, 1
POLICY_SCLS, POLICY_SLS, POLICY_ILS = 0, 1, 2
POLICIES = {"scls": POLICY_SCLS, "sls": POLICY_SLS, "ils": POLICY_ILS}
DIST_UNIFORM, DIST_LOGNORMAL, DIST_HISTOGRAM = 0, 1, 2

# errors.h:26-87 class names, indexed by scls_status.
STATUS_NAMES = {
    0: "OK",
    1: "Error",
    2: "InsufficientSamplesError",
    3: "DegenerateModelError",
    4: "WrongKindError",
    5: "InfeasibleRequestError",
    6: "NoWorkersError",
    7: "ParseError",
    8: "LimitViolationError",
    9: "EmptyLogError",
    10: "NonTerminationError",
    11: "InvalidArgument",
    12: "CudaError",
    13: "CapacityError",
}
OK = 0
ERR_INFEASIBLE_REQUEST = 5
ERR_NO_WORKERS = 6
ERR_EMPTY_LOG = 9
ERR_NON_TERMINATION = 10
ERR_INVALID_ARGUMENT = 11
ERR_CUDA = 12
ERR_CAPACITY = 13

# event_log.h:27-34
EVENT_KINDS = ["arrival", "tick", "dispatch", "batch_start", "batch_end", "complete"]


class Latency(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("p1", "p2", "p3", "p4", "d1", "d2", "d3", "d4",
                 "rmse_prefill", "rmse_decode")] + [
        ("n_cap", C.c_int32), ("l_cap", C.c_int32)]


class ProfileSample(C.Structure):
    """cost_model.h:45-50 (phase 0 prefill, 1 decode)."""
    _fields_ = [("phase", C.c_int32), ("batch_size", C.c_int32), ("length", C.c_int32), ("pad_", C.c_int32),
                ("latency_s", C.c_double)]


class Memory(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_rules", C.c_int32),
                ("m_cap", C.c_double), ("m_model", C.c_double),
                ("m_engine", C.c_double), ("delta", C.c_double),
                ("zeta", C.c_double),
                ("rule_threshold", C.c_int32 * SCLS_MAX_RULES),
                ("rule_max_n", C.c_int32 * SCLS_MAX_RULES)]


class SchedCfg(C.Structure):
    _fields_ = [("policy", C.c_int32), ("slice_len", C.c_int32),
                ("max_gen_limit", C.c_int32), ("fixed_batch_size", C.c_int32),
                ("max_concurrent", C.c_int32), ("worker_count", C.c_int32),
                ("lambda_", C.c_double), ("gamma", C.c_double),
                ("horizon_s", C.c_double)]


class LengthDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("lo", C.c_int32), ("hi", C.c_int32),
                ("mu", C.c_double), ("sigma", C.c_double), ("cap", C.c_int32),
                ("n_buckets", C.c_int32),
                ("edges", C.c_int32 * (SCLS_MAX_BUCKETS + 1)),
                ("weights", C.c_double * SCLS_MAX_BUCKETS)]


class WorkloadSpec(C.Structure):
    _fields_ = [("rate", C.c_double), ("duration_s", C.c_double),
                ("input_len_dist", LengthDist), ("gen_len_dist", LengthDist),
                ("max_input_limit", C.c_int32), ("max_gen_limit", C.c_int32),
                ("seed", C.c_uint64)]


class Batches(C.Structure):
    _fields_ = [("n_batches", C.c_int64), ("order", C.POINTER(C.c_int32)),
                ("seg_begin", C.POINTER(C.c_int32)), ("l_in", C.POINTER(C.c_int32)),
                ("est", C.POINTER(C.c_double)), ("member_id", C.POINTER(C.c_int64))]


class TraceResult(C.Structure):
    _fields_ = [("status", C.c_int32), ("worker_count", C.c_int32),
                ("error_request_id", C.c_int64), ("n_requests", C.c_int64),
                ("completed", C.c_int64)] + [
        (n, C.c_double) for n in
        ("throughput", "avg_response_s", "p95_response_s", "ct_std_s",
         "avg_pad_tokens", "avg_invalid_tokens", "avg_batch_size",
         "early_return_ratio")] + [
        (n, C.c_int64) for n in
        ("total_pad", "total_invalid", "batch_count", "batch_members",
         "early_returns", "n_events", "n_dispatches", "n_ticks")] + [
        (n, C.c_uint64) for n in
        ("h_complete_ids", "h_dispatch", "h_complete_t", "h_log")] + [
        ("sim_clock", C.c_double)]


class EventRecord(C.Structure):
    _fields_ = [("t", C.c_double), ("est_serve_s", C.c_double),
                ("response_s", C.c_double), ("next_interval_s", C.c_double),
                ("request", C.c_int64), ("batch", C.c_int64)] + [
        (n, C.c_int32) for n in
        ("kind", "worker", "n", "l_in", "planned_l_out", "served_l_out",
         "input_len", "gen_len", "slices", "member_count")] + [
        ("member_offset", C.c_int64)]


class Member(C.Structure):
    _fields_ = [("request", C.c_int64), ("effective_input", C.c_int32),
                ("pad", C.c_int32), ("gen", C.c_int32), ("invalid", C.c_int32)]


class EventLog(C.Structure):
    _fields_ = [("n_logged", C.c_int32), ("rec_cap", C.c_int64),
                ("mem_cap", C.c_int64), ("records", C.POINTER(EventRecord)),
                ("members", C.POINTER(Member)), ("rec_count", C.POINTER(C.c_int64)),
                ("mem_count", C.POINTER(C.c_int64))]


# ---- builtin models (run_config.cpp:216-241) --------------------------------

def latency_model(p1=0.0, p2=0.0, p3=0.0, p4=0.0, d1=0.0, d2=0.0, d3=0.0, d4=0.0,
                  n_cap=64, l_cap=4096) -> Latency:
    return Latency(p1, p2, p3, p4, d1, d2, d3, d4, 0.0, 0.0, n_cap, l_cap)


def builtin_latency_model() -> Latency:
    return latency_model(2e-6, 1e-3, 5e-5, 0.02, 1e-7, 2e-4, 3e-6, 0.02)


def rule_table(rows) -> Memory:
    m = Memory()
    m.kind = RULE_TABLE
    m.n_rules = len(rows)
    if len(rows) > SCLS_MAX_RULES:
        raise ValueError("too many rule rows")
    for i, (thr, mx) in enumerate(rows):
        m.rule_threshold[i] = thr
        m.rule_max_n[i] = mx
    return m


def analytic(m_cap, m_model, m_engine, delta, zeta=1.0) -> Memory:
    m = Memory()
    m.kind = ANALYTIC
    m.m_cap, m.m_model, m.m_engine, m.delta, m.zeta = m_cap, m_model, m_engine, delta, zeta
    return m


def builtin_memory_model() -> Memory:
    return rule_table([(1024, 12), (512, 22), (0, 28)])


def builtin_analytic_memory_model() -> Memory:
    return analytic(80e9, 26e9, 4e9, 786432.0, 0.9)


def sched_cfg(policy="scls", slice_len=128, max_gen_limit=1024, lambda_=0.5, gamma=3.0,
              fixed_batch_size=12, max_concurrent=12, worker_count=8,
              horizon_s=1e7) -> SchedCfg:
    p = POLICIES[policy] if isinstance(policy, str) else int(policy)
    return SchedCfg(p, slice_len, max_gen_limit, fixed_batch_size, max_concurrent,
                    worker_count, lambda_, gamma, horizon_s)


# ---- workload presets (workload.cpp:276-291) ---------------------------------

def uniform_dist(lo, hi) -> LengthDist:
    d = LengthDist()
    d.kind, d.lo, d.hi = DIST_UNIFORM, lo, hi
    return d


def lognormal_dist(mu, sigma, cap) -> LengthDist:
    d = LengthDist()
    d.kind, d.mu, d.sigma, d.cap = DIST_LOGNORMAL, mu, sigma, cap
    return d


def histogram_dist(edges, weights) -> LengthDist:
    d = LengthDist()
    d.kind = DIST_HISTOGRAM
    d.n_buckets = len(weights)
    for i, e in enumerate(edges):
        d.edges[i] = e
    for i, w in enumerate(weights):
        d.weights[i] = w
    return d


def codefuse_like_input_dist() -> LengthDist:
    return histogram_dist([1, 128, 256, 512, 1024], [0.30, 0.25, 0.25, 0.20])


def codefuse_like_gen_dist() -> LengthDist:
    return histogram_dist([1, 64, 128, 256, 511, 1024], [0.10, 0.15, 0.30, 0.30, 0.15])


def long_gen_dist() -> LengthDist:
    return histogram_dist([1, 512, 513, 1024], [0.40, 0.0, 0.60])


def workload_spec(rate=20.0, duration_s=600.0, input_dist=None, gen_dist=None,
                  max_input_limit=1024, max_gen_limit=1024, seed=42) -> WorkloadSpec:
    """Defaults of default_run_config() (run_config.cpp:109-114): codefuse-like."""
    return WorkloadSpec(rate, duration_s,
                        input_dist if input_dist is not None else codefuse_like_input_dist(),
                        gen_dist if gen_dist is not None else codefuse_like_gen_dist(),
                        max_input_limit, max_gen_limit, seed)


def repo_root() -> str:
    return os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
