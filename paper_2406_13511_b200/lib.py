"""ctypes binding of libscls_b200.so (the C-ABI in include/scls_capi.h).

This is the Python face of the CUDA scheduling core.  There is no CPU
fallback: if the shared library is missing the import of `load()` raises, and
if no CUDA device is usable `Context()` raises SclsError(CudaError).

Method names and argument meanings mirror the reference API
(/root/reference/proj/core/include/slicesim/*.h):
  batch_requests   batcher.h:40-43       offload        offloader.h:39-40
  schedule         sched_policies.cpp:93-112 (batch_requests + offload)
  simulate         sim_engine.h:61-67 + metrics.h:41 for many traces
  generate         workload.h:78         batch_serve_time/would_oom/max_batch_size
                                          cost_model.h:54-66, memory_model.h:62-66
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import capi

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libscls_b200.so")
# Diagnostics only (profiling builds): another build of the same library.
LIB_PATH = os.environ.get("SCLS_B200_LIB", LIB_PATH)

# Every symbol include/scls_capi.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "scls_abi_version", "scls_ctx_create", "scls_ctx_destroy", "scls_last_error",
    "scls_last_request_id", "scls_last_timings", "scls_last_launch_count",
    "scls_validate_latency", "scls_validate_memory", "scls_validate_sched",
    "scls_batch_serve_time", "scls_would_oom", "scls_max_batch_size",
    "scls_batch_requests", "scls_offload", "scls_schedule", "scls_simulate",
    "scls_simulate_grid", "scls_generate", "scls_make_pool", "scls_debug_dp_profile", "scls_set_option",
    "scls_run_sweep", "scls_run_experiments", "scls_generate_batch", "scls_debug_log", "scls_debug_libm",
    "scls_shard_range", "scls_comm_unique_id", "scls_comm_init", "scls_comm_size", "scls_run_sweep_sharded",
    "scls_multi_create", "scls_multi_destroy", "scls_multi_last_error", "scls_multi_uses_nccl",
    "scls_multi_run_sweep", "scls_multi_run_experiments", "scls_device_count",
    "scls_multi_set_option", "scls_fit_latency",
]


class SclsError(RuntimeError):
    """Carries the scls_status code; `name` is the reference exception class."""

    def __init__(self, status, msg, request_id=-1):
        self.status = status
        self.name = capi.STATUS_NAMES.get(status, str(status))
        self.request_id = request_id
        super().__init__(f"{self.name}: {msg}")


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built (run __graft_entry__.build()); "
                          "the scheduling core has no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    P = C.POINTER
    i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
    L, M, S = P(capi.Latency), P(capi.Memory), P(capi.SchedCfg)
    sigs = {
        "scls_abi_version": (i32, []),
        "scls_ctx_create": (i32, [i32, vp, P(vp)]),
        "scls_ctx_destroy": (None, [vp]),
        "scls_last_error": (C.c_size_t, [vp, C.c_char_p, C.c_size_t]),
        "scls_last_request_id": (i64, [vp]),
        "scls_last_timings": (None, [vp, P(C.c_float)]),
        "scls_last_launch_count": (i64, [vp]),
        "scls_validate_latency": (i32, [L]),
        "scls_validate_memory": (i32, [M]),
        "scls_validate_sched": (i32, [S]),
        "scls_batch_serve_time": (i32, [vp, i64, vp, vp, vp, L, vp, i32]),
        "scls_would_oom": (i32, [vp, i64, vp, vp, i32, M, vp, i32]),
        "scls_max_batch_size": (i32, [vp, i64, vp, i32, M, vp, i32]),
        "scls_batch_requests": (i32, [vp, i64, vp, vp, vp, i32, L, M, i64, P(capi.Batches), i32]),
        "scls_offload": (i32, [vp, i64, vp, vp, i32, vp, vp, vp, vp, i32]),
        "scls_schedule": (i32, [vp, i64, vp, vp, vp, i32, L, M, i64, i32, vp, vp,
                                P(capi.Batches), vp, vp, i32]),
        "scls_simulate": (i32, [vp, i32, vp, vp, vp, vp, i32, S, vp, L, M,
                                P(capi.TraceResult), i32, vp, P(capi.EventLog), i32]),
        "scls_simulate_grid": (i32, [vp, i32, vp, vp, vp, vp, i32, S, L, M,
                                     P(capi.TraceResult), i32, vp, P(capi.EventLog), i32]),
        "scls_generate": (i32, [P(capi.WorkloadSpec), i64, P(i64), vp, vp, vp]),
        "scls_fit_latency": (i32, [vp, i64, i32, i32, P(capi.Latency)]),
        "scls_make_pool": (i32, [i64, C.c_uint64, vp, vp, vp, vp]),
        "scls_debug_dp_profile": (i32, [vp, i32, vp]),
        "scls_set_option": (i32, [vp, i32, i64]),
        "scls_run_sweep": (i32, [vp, i32, P(capi.WorkloadSpec), i32, S, L, M,
                                 P(capi.TraceResult), i32, vp, P(capi.EventLog), i32]),
        "scls_run_experiments": (i32, [vp, i32, P(capi.WorkloadSpec), S, L, M,
                                       P(capi.TraceResult), i32, vp, P(capi.EventLog), i32]),
        "scls_generate_batch": (i32, [vp, i32, P(capi.WorkloadSpec), i64, vp, vp, vp, vp, i32]),
        "scls_debug_log": (i32, [vp, i64, vp, vp, i32]),
        "scls_debug_libm": (i32, [vp, i32, i64, vp, vp, i32]),
        "scls_shard_range": (None, [i64, i32, i32, P(i64), P(i64)]),
        "scls_comm_unique_id": (i32, [vp]),
        "scls_comm_init": (i32, [vp, i32, i32, vp]),
        "scls_comm_size": (i32, [vp]),
        "scls_run_sweep_sharded": (i32, [vp, i32, P(capi.WorkloadSpec), i32, S, L, M,
                                         P(capi.TraceResult), i32, vp, i32]),
        "scls_multi_create": (i32, [i32, vp, P(vp)]),
        "scls_multi_destroy": (None, [vp]),
        "scls_multi_last_error": (C.c_size_t, [vp, C.c_char_p, C.c_size_t]),
        "scls_multi_uses_nccl": (i32, [vp]),
        "scls_multi_run_sweep": (i32, [vp, i32, P(capi.WorkloadSpec), i32, S, L, M,
                                       P(capi.TraceResult), i32, vp, vp]),
        "scls_multi_run_experiments": (i32, [vp, i32, P(capi.WorkloadSpec), S, L, M,
                                             P(capi.TraceResult), i32, vp, vp]),
        "scls_device_count": (i32, []),
        "scls_multi_set_option": (i32, [vp, i32, i64]),
    }
    for name, (res, args) in sigs.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.scls_abi_version() != capi.SCLS_ABI_VERSION:
        raise ImportError("libscls_b200.so ABI version mismatch")
    _lib = lib
    return lib


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _dev_ptr(t):
    """torch CUDA tensor -> device pointer (mem=SCLS_MEM_DEVICE calls)."""
    return C.c_void_p(t.data_ptr())


class Context:
    """One scls_ctx: a CUDA device + stream (NULL: a private stream)."""

    def __init__(self, device=0, stream=None):
        self.lib = load()
        h = C.c_void_p()
        st = self.lib.scls_ctx_create(device, stream, C.byref(h))
        if st:
            raise self._error(st, None)
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.scls_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- diagnostics ------------------------------------------------------------
    def _error(self, st, h):
        lib = self.lib if hasattr(self, "lib") else load()
        buf = C.create_string_buffer(4096)
        lib.scls_last_error(h, buf, 4096)
        return SclsError(st, buf.value.decode(errors="replace"), lib.scls_last_request_id(h))

    def _check(self, st):
        if st:
            raise self._error(st, self.h)

    def timings(self):
        """Device ms of the last call: total, sort, estimate, dp, backtrack+emit,
        offload, simulate, generate."""
        out = (C.c_float * 8)()
        self.lib.scls_last_timings(self.h, out)
        d = dict(zip(["total", "sort", "estimate", "dp", "backtrack", "offload", "simulate", "generate"],
                     list(out)))
        d["dp_mono"] = d["generate"]  # slot 7 of a batcher call: 1.0 when the monotone DP kernel ran
        return d

    def set_digests(self, on):
        """SCLS_OPT_SIM_DIGESTS: compute the per-trace log digests (default on)."""
        self._check(self.lib.scls_set_option(self.h, 1, 1 if on else 0))

    def set_concurrent(self, on):
        """SCLS_OPT_SIM_CONCURRENT: run the per-policy simulator launches concurrently (default on)."""
        self._check(self.lib.scls_set_option(self.h, 3, 1 if on else 0))

    def set_ils_lockstep(self, on):
        """SCLS_OPT_ILS_KERNEL: 1 = the lock-step metrics-only ILS kernel, 0 = independent instance lanes."""
        self._check(self.lib.scls_set_option(self.h, 4, 1 if on else 0))

    def set_ils_kernel(self, mode):
        """SCLS_OPT_ILS_KERNEL: 0 independent lanes, simulation and merge kernels split (default);
        1 lock-step; 2 independent lanes in one kernel (packs of two jobs, merges in series)."""
        self._check(self.lib.scls_set_option(self.h, 4, int(mode)))

    def set_batch_path(self, large):
        """SCLS_OPT_BATCH_PATH: 1 forces the multi-kernel batch_requests path for small pools too;
        2 also replaces the eff-bucket sort by the LSD radix sort."""
        self._check(self.lib.scls_set_option(self.h, 5, int(large) if not isinstance(large, bool) else int(large)))

    def set_dp_cluster(self, ctas):
        """SCLS_OPT_DP_CLUSTER: CTAs per monotone-DP cluster (1, 2 or 4; default 1)."""
        self._check(self.lib.scls_set_option(self.h, 6, int(ctas)))

    def set_dp_kernel(self, mode):
        """SCLS_OPT_DP_KERNEL: 0 auto (monotone decision kernel when allowed), 1 chain."""
        self._check(self.lib.scls_set_option(self.h, 2, int(mode)))

    def dp_profile(self, enable=True):
        """Read-and-reset the DP kernel's clock64 phase counters."""
        out = np.zeros(8, np.uint64)
        self._check(self.lib.scls_debug_dp_profile(self.h, 1 if enable else 0, _ptr(out)))
        return out

    def launches(self):
        return self.lib.scls_last_launch_count(self.h)

    # -- estimators (batched) -----------------------------------------------------
    def batch_serve_time(self, n, l_in, l_out, lat):
        n = np.ascontiguousarray(n, np.int32)
        l_in = np.ascontiguousarray(l_in, np.int32)
        l_out = np.ascontiguousarray(l_out, np.int32)
        out = np.zeros(len(n), np.float64)
        self._check(self.lib.scls_batch_serve_time(self.h, len(n), _ptr(n), _ptr(l_in), _ptr(l_out),
                                                   C.byref(lat), _ptr(out), capi.MEM_HOST))
        return out

    def would_oom(self, n, l_in, slice_len, mem):
        n = np.ascontiguousarray(n, np.int32)
        l_in = np.ascontiguousarray(l_in, np.int32)
        out = np.zeros(len(n), np.uint8)
        self._check(self.lib.scls_would_oom(self.h, len(n), _ptr(n), _ptr(l_in), slice_len,
                                            C.byref(mem), _ptr(out), capi.MEM_HOST))
        return out.astype(bool)

    def max_batch_size(self, l_in, slice_len, mem):
        l_in = np.ascontiguousarray(l_in, np.int32)
        out = np.zeros(len(l_in), np.int32)
        self._check(self.lib.scls_max_batch_size(self.h, len(l_in), _ptr(l_in), slice_len,
                                                 C.byref(mem), _ptr(out), capi.MEM_HOST))
        return out

    # -- batcher / offloader ----------------------------------------------------------
    def batch_requests(self, eff, arrival, ids, slice_len, lat, mem, first_batch_id=0):
        """batcher.h:40-43 -> dict(order, seg_begin, l_in, est, batch_id, member_id)."""
        eff = np.ascontiguousarray(eff, np.int32)
        arrival = np.ascontiguousarray(arrival, np.float64)
        ids = np.ascontiguousarray(ids, np.int64)
        n = len(eff)
        order = np.zeros(max(n, 1), np.int32)
        seg = np.zeros(n + 1, np.int32)
        l_in = np.zeros(max(n, 1), np.int32)
        est = np.zeros(max(n, 1), np.float64)
        mid = np.zeros(max(n, 1), np.int64)
        out = capi.Batches(0, order.ctypes.data_as(C.POINTER(C.c_int32)),
                           seg.ctypes.data_as(C.POINTER(C.c_int32)),
                           l_in.ctypes.data_as(C.POINTER(C.c_int32)),
                           est.ctypes.data_as(C.POINTER(C.c_double)),
                           mid.ctypes.data_as(C.POINTER(C.c_int64)))
        self._check(self.lib.scls_batch_requests(self.h, n, _ptr(eff), _ptr(arrival), _ptr(ids),
                                                 slice_len, C.byref(lat), C.byref(mem),
                                                 first_batch_id, C.byref(out), capi.MEM_HOST))
        k = out.n_batches
        return dict(n_batches=k, order=order[:n], seg_begin=seg[:k + 1], l_in=l_in[:k],
                    est=est[:k], batch_id=np.arange(first_batch_id, first_batch_id + k, dtype=np.int64),
                    member_id=mid[:n])

    def offload(self, batch_id, est, worker_id, loads):
        """offloader.h:39-40 -> (assigned batch ids, workers, new loads)."""
        batch_id = np.ascontiguousarray(batch_id, np.int64)
        est = np.ascontiguousarray(est, np.float64)
        worker_id = np.ascontiguousarray(worker_id, np.int32)
        loads = np.array(loads, np.float64)
        nb = len(est)
        ob = np.zeros(max(nb, 1), np.int64)
        ow = np.zeros(max(nb, 1), np.int32)
        self._check(self.lib.scls_offload(self.h, nb, _ptr(batch_id), _ptr(est), len(worker_id),
                                          _ptr(worker_id), _ptr(loads), _ptr(ob), _ptr(ow),
                                          capi.MEM_HOST))
        return ob[:nb], ow[:nb], loads

    def schedule(self, eff, arrival, ids, slice_len, lat, mem, worker_id, loads, first_batch_id=0):
        """One SCLS tick: batch_requests then offload (sched_policies.cpp:93-112)."""
        eff = np.ascontiguousarray(eff, np.int32)
        arrival = np.ascontiguousarray(arrival, np.float64)
        ids = np.ascontiguousarray(ids, np.int64)
        worker_id = np.ascontiguousarray(worker_id, np.int32)
        loads = np.array(loads, np.float64)
        n = len(eff)
        seg = np.zeros(n + 1, np.int32)
        l_in = np.zeros(max(n, 1), np.int32)
        est = np.zeros(max(n, 1), np.float64)
        mid = np.zeros(max(n, 1), np.int64)
        ob = np.zeros(max(n, 1), np.int64)
        ow = np.zeros(max(n, 1), np.int32)
        out = capi.Batches(0, None, seg.ctypes.data_as(C.POINTER(C.c_int32)),
                           l_in.ctypes.data_as(C.POINTER(C.c_int32)),
                           est.ctypes.data_as(C.POINTER(C.c_double)),
                           mid.ctypes.data_as(C.POINTER(C.c_int64)))
        self._check(self.lib.scls_schedule(self.h, n, _ptr(eff), _ptr(arrival), _ptr(ids), slice_len,
                                           C.byref(lat), C.byref(mem), first_batch_id,
                                           len(worker_id), _ptr(worker_id), _ptr(loads),
                                           C.byref(out), _ptr(ob), _ptr(ow), capi.MEM_HOST))
        k = out.n_batches
        return dict(n_batches=k, seg_begin=seg[:k + 1], l_in=l_in[:k], est=est[:k],
                    member_id=mid[:n], assign_batch=ob[:k], assign_worker=ow[:k], loads=loads)

    def schedule_device(self, n, eff, arrival, ids, slice_len, lat, mem, worker_id, loads, out_bufs,
                        first_batch_id=0):
        """Device-resident tick: every array is a torch CUDA tensor (mem=DEVICE)."""
        seg, l_in, est, mid, ob, ow = out_bufs
        out = capi.Batches(0, None, C.cast(C.c_void_p(seg.data_ptr()), C.POINTER(C.c_int32)),
                           C.cast(C.c_void_p(l_in.data_ptr()), C.POINTER(C.c_int32)),
                           C.cast(C.c_void_p(est.data_ptr()), C.POINTER(C.c_double)),
                           C.cast(C.c_void_p(mid.data_ptr()), C.POINTER(C.c_int64)))
        self._check(self.lib.scls_schedule(self.h, n, _dev_ptr(eff), _dev_ptr(arrival), _dev_ptr(ids),
                                           slice_len, C.byref(lat), C.byref(mem), first_batch_id,
                                           worker_id.numel(), _dev_ptr(worker_id), _dev_ptr(loads),
                                           C.byref(out), _dev_ptr(ob), _dev_ptr(ow), capi.MEM_DEVICE))
        return out.n_batches

    # -- simulator ------------------------------------------------------------------------
    def simulate(self, traces, cfgs, lat, mem, cfg_index=None, hist_bins=64, n_logged=0,
                 rec_cap=0, mem_cap=0):
        """Simulator::run + compute for every trace (list of (arrival, input_len,
        gen_len)).  Returns (results, hist[, log])."""
        offs, arr, inp, gen = _flatten(traces)
        return self.simulate_flat(offs, arr, inp, gen, cfgs, lat, mem, cfg_index, hist_bins,
                                  n_logged, rec_cap, mem_cap)

    def simulate_flat(self, offs, arr, inp, gen, cfgs, lat, mem, cfg_index=None, hist_bins=64,
                      n_logged=0, rec_cap=0, mem_cap=0):
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        ntr = len(offs) - 1
        cfg_arr = (capi.SchedCfg * len(cfgs))(*cfgs)
        idx = None if cfg_index is None else np.ascontiguousarray(cfg_index, np.int32)
        res = (capi.TraceResult * max(ntr, 1))()
        hist = np.zeros(max(ntr * hist_bins, 1), np.int64)
        log = None
        if n_logged:
            recs = (capi.EventRecord * (n_logged * rec_cap))()
            mems = (capi.Member * max(n_logged * mem_cap, 1))()
            rc = np.zeros(n_logged, np.int64)
            mc = np.zeros(n_logged, np.int64)
            st = capi.EventLog(n_logged, rec_cap, mem_cap, recs, mems,
                               rc.ctypes.data_as(C.POINTER(C.c_int64)),
                               mc.ctypes.data_as(C.POINTER(C.c_int64)))
            log = dict(struct=st, records=recs, members=mems, rec_count=rc, mem_count=mc,
                       rec_cap=rec_cap, mem_cap=mem_cap)
        self._check(self.lib.scls_simulate(self.h, ntr, _ptr(np.ascontiguousarray(offs, np.int64)),
                                           _ptr(arr), _ptr(inp), _ptr(gen), len(cfgs), cfg_arr,
                                           _ptr(idx), C.byref(lat), C.byref(mem), res, hist_bins,
                                           _ptr(hist), C.byref(log["struct"]) if log else None,
                                           capi.MEM_HOST))
        hist = hist[:ntr * hist_bins].reshape(ntr, hist_bins)
        if log is not None:
            return res, hist, log
        return res, hist

    def simulate_grid(self, traces, cfgs, lat, mem, hist_bins=64):
        """scls_simulate_grid: every config on every trace, each trace staged
        once.  Returns (results, hist) with results[c][t] and hist[c, t]."""
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        offs, arr, inp, gen = _flatten(traces)
        res, hist = self.simulate_grid_flat(offs, arr, inp, gen, cfgs, lat, mem, hist_bins)
        ntr = len(traces)
        return [[res[c * ntr + t] for t in range(ntr)] for c in range(len(cfgs))], hist

    def simulate_grid_flat(self, offs, arr, inp, gen, cfgs, lat, mem, hist_bins=64):
        ntr, nc = len(offs) - 1, len(cfgs)
        cfg_arr = (capi.SchedCfg * nc)(*cfgs)
        res = (capi.TraceResult * max(ntr * nc, 1))()
        hist = np.zeros(max(ntr * nc * hist_bins, 1), np.int64)
        self._check(self.lib.scls_simulate_grid(self.h, ntr, _ptr(np.ascontiguousarray(offs, np.int64)),
                                                _ptr(arr), _ptr(inp), _ptr(gen), nc, cfg_arr,
                                                C.byref(lat), C.byref(mem), res, hist_bins, _ptr(hist), None,
                                                capi.MEM_HOST))
        # flat job order: res[c * ntr + t]
        return res, hist[:ntr * nc * hist_bins].reshape(nc, ntr, hist_bins)

    # -- device trace generation (workload.h:78) and the sweep (experiment.h:37,52-53) --
    def generate_batch(self, specs):
        """generate() for every spec on the device -> (req_offset, arrival, input_len, gen_len)."""
        specs = list(specs)
        n = len(specs)
        sp = (capi.WorkloadSpec * max(n, 1))(*specs)
        offs = np.zeros(n + 1, np.int64)
        st = self.lib.scls_generate_batch(self.h, n, sp, 0, _ptr(offs), None, None, None, capi.MEM_HOST)
        if st not in (0, capi.ERR_CAPACITY):
            self._check(st)
        tot = int(offs[-1])
        arr = np.zeros(max(tot, 1), np.float64)
        inp = np.zeros(max(tot, 1), np.int32)
        gen = np.zeros(max(tot, 1), np.int32)
        self._check(self.lib.scls_generate_batch(self.h, n, sp, tot, _ptr(offs), _ptr(arr), _ptr(inp), _ptr(gen),
                                                 capi.MEM_HOST))
        return offs, arr[:tot], inp[:tot], gen[:tot]

    def run_sweep(self, specs, cfgs, lat, mem, hist_bins=64, n_logged=0, rec_cap=0, mem_cap=0):
        """scls_run_sweep: generate every trace on the device, then every config
        on every trace.  Returns (results, hist[, log]); results[c * ntr + t]."""
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        specs = list(specs)
        ntr, nc = len(specs), len(cfgs)
        sp = (capi.WorkloadSpec * max(ntr, 1))(*specs)
        cfg_arr = (capi.SchedCfg * nc)(*cfgs)
        res = (capi.TraceResult * max(ntr * nc, 1))()
        hist = np.zeros(max(ntr * nc * hist_bins, 1), np.int64)
        log = None
        if n_logged:
            recs = (capi.EventRecord * (n_logged * rec_cap))()
            mems = (capi.Member * max(n_logged * mem_cap, 1))()
            rc = np.zeros(n_logged, np.int64)
            mc = np.zeros(n_logged, np.int64)
            st = capi.EventLog(n_logged, rec_cap, mem_cap, recs, mems,
                               rc.ctypes.data_as(C.POINTER(C.c_int64)),
                               mc.ctypes.data_as(C.POINTER(C.c_int64)))
            log = dict(struct=st, records=recs, members=mems, rec_count=rc, mem_count=mc,
                       rec_cap=rec_cap, mem_cap=mem_cap)
        self._check(self.lib.scls_run_sweep(self.h, ntr, sp, nc, cfg_arr, C.byref(lat), C.byref(mem), res,
                                            hist_bins, _ptr(hist), C.byref(log["struct"]) if log else None,
                                            capi.MEM_HOST))
        hist = hist[:ntr * nc * hist_bins].reshape(nc, ntr, hist_bins)
        if log is not None:
            return res, hist, log
        return res, hist

    def run_experiments(self, specs, cfgs, lat, mem, hist_bins=64):
        """scls_run_experiments: run i = generate(specs[i]) simulated under cfgs[i]."""
        specs, cfgs = list(specs), list(cfgs)
        n = len(specs)
        assert len(cfgs) == n
        sp = (capi.WorkloadSpec * max(n, 1))(*specs)
        cfg_arr = (capi.SchedCfg * max(n, 1))(*cfgs)
        res = (capi.TraceResult * max(n, 1))()
        hist = np.zeros(max(n * hist_bins, 1), np.int64)
        self._check(self.lib.scls_run_experiments(self.h, n, sp, cfg_arr, C.byref(lat), C.byref(mem), res,
                                                  hist_bins, _ptr(hist), None, capi.MEM_HOST))
        return res, hist[:n * hist_bins].reshape(n, hist_bins)

    # -- the sharded sweep (one process per GPU, NCCL gather in the library) ----------
    def comm_init(self, world, rank, uid):
        """scls_comm_init: join the NCCL communicator `uid` (128 bytes from comm_unique_id())."""
        b = (C.c_uint8 * 128).from_buffer_copy(bytes(uid))
        self._check(self.lib.scls_comm_init(self.h, world, rank, b))

    def comm_size(self):
        return self.lib.scls_comm_size(self.h)

    def run_sweep_sharded(self, specs, cfgs, lat, mem, hist_bins=64):
        """scls_run_sweep_sharded with host outputs: this rank's shard of the
        GLOBAL spec list, gathered so every rank returns the whole grid
        (results[c * ntr + t], hist[c, t])."""
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        if isinstance(specs, C.Array):  # a prebuilt scls_workload_spec array is passed as is
            sp, ntr = specs, len(specs)
        else:
            specs = list(specs)
            ntr = len(specs)
            sp = (capi.WorkloadSpec * max(ntr, 1))(*specs)
        nc = len(cfgs)
        cfg_arr = (capi.SchedCfg * nc)(*cfgs)
        res = (capi.TraceResult * max(ntr * nc, 1))()
        hist = np.zeros(max(ntr * nc * hist_bins, 1), np.int64)
        self._check(self.lib.scls_run_sweep_sharded(self.h, ntr, sp, nc, cfg_arr, C.byref(lat), C.byref(mem), res,
                                                    hist_bins, _ptr(hist), capi.MEM_HOST))
        return res, hist[:ntr * nc * hist_bins].reshape(nc, ntr, hist_bins)

    def debug_log(self, x):
        """The device port of glibc log on x (float64 array)."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        self._check(self.lib.scls_debug_log(self.h, len(x), _ptr(x), _ptr(y), capi.MEM_HOST))
        return y

    def debug_libm(self, fn, x):
        """The device port of glibc log / exp / cos (fn = "log" | "exp" | "cos") on x."""
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros_like(x)
        code = {"log": 0, "exp": 1, "cos": 2}[fn]
        self._check(self.lib.scls_debug_libm(self.h, code, len(x), _ptr(x), _ptr(y), capi.MEM_HOST))
        return y


def shard_range(total, shard, n_shards):
    """scls_shard_range: contiguous [lo, hi) of `shard` (trace t -> floor(t * N / total))."""
    lo, hi = C.c_int64(), C.c_int64()
    load().scls_shard_range(total, shard, n_shards, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def comm_unique_id():
    """scls_comm_unique_id (rank 0): 128 bytes to broadcast to every rank."""
    lib = load()
    b = (C.c_uint8 * 128)()
    st = lib.scls_comm_unique_id(b)
    if st:
        buf = C.create_string_buffer(4096)
        lib.scls_last_error(None, buf, 4096)
        raise SclsError(st, buf.value.decode())
    return bytes(b)


class Multi:
    """scls_multi: one process driving several GPUs (a shard and a host
    thread per entry of `devices`; NCCL gather when the devices are distinct)."""

    def __init__(self, devices):
        self.lib = load()
        devs = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        st = self.lib.scls_multi_create(len(devices), devs, C.byref(h))
        if st:
            buf = C.create_string_buffer(4096)
            self.lib.scls_last_error(None, buf, 4096)
            raise SclsError(st, buf.value.decode())
        self.h = h
        self.n = len(devices)

    def close(self):
        if getattr(self, "h", None):
            self.lib.scls_multi_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_digests(self, on):
        """SCLS_OPT_SIM_DIGESTS on every device context (default on)."""
        st = self.lib.scls_multi_set_option(self.h, 1, 1 if on else 0)
        if st:
            raise SclsError(st, "scls_multi_set_option failed")

    def uses_nccl(self):
        return bool(self.lib.scls_multi_uses_nccl(self.h))

    def run_sweep(self, specs, cfgs, lat, mem, hist_bins=64):
        """Returns (results, hist, ms) with ms = per-shard device ms, gather ms, wall ms."""
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        specs = list(specs)
        ntr, nc = len(specs), len(cfgs)
        sp = (capi.WorkloadSpec * max(ntr, 1))(*specs)
        cfg_arr = (capi.SchedCfg * nc)(*cfgs)
        res = (capi.TraceResult * max(ntr * nc, 1))()
        hist = np.zeros(max(ntr * nc * hist_bins, 1), np.int64)
        ms = np.zeros(self.n + 2, np.float32)
        st = self.lib.scls_multi_run_sweep(self.h, ntr, sp, nc, cfg_arr, C.byref(lat), C.byref(mem), res,
                                           hist_bins, _ptr(hist), _ptr(ms))
        if st:
            buf = C.create_string_buffer(4096)
            self.lib.scls_multi_last_error(self.h, buf, 4096)
            raise SclsError(st, buf.value.decode())
        return res, hist[:ntr * nc * hist_bins].reshape(nc, ntr, hist_bins), ms

    def run_experiments(self, specs, cfgs, lat, mem, hist_bins=64):
        """scls_multi_run_experiments: run i = specs[i] under cfgs[i], runs sharded over the devices."""
        specs, cfgs = list(specs), list(cfgs)
        n = len(specs)
        sp = (capi.WorkloadSpec * max(n, 1))(*specs)
        cfg_arr = (capi.SchedCfg * max(n, 1))(*cfgs)
        res = (capi.TraceResult * max(n, 1))()
        hist = np.zeros(max(n * hist_bins, 1), np.int64)
        ms = np.zeros(self.n + 2, np.float32)
        st = self.lib.scls_multi_run_experiments(self.h, n, sp, cfg_arr, C.byref(lat), C.byref(mem), res,
                                                 hist_bins, _ptr(hist), _ptr(ms))
        if st:
            buf = C.create_string_buffer(4096)
            self.lib.scls_multi_last_error(self.h, buf, 4096)
            raise SclsError(st, buf.value.decode())
        return res, hist[:n * hist_bins].reshape(n, hist_bins), ms


def _flatten(traces):
    """List of (arrival, input_len, gen_len) -> (req_offset, arrival, input_len, gen_len)."""
    offs = np.zeros(len(traces) + 1, np.int64)
    for i, t in enumerate(traces):
        offs[i + 1] = offs[i] + len(t[0])
    tot = max(int(offs[-1]), 1)
    arr = np.zeros(tot, np.float64)
    inp = np.zeros(tot, np.int32)
    gen = np.zeros(tot, np.int32)
    for i, (a, b, g) in enumerate(traces):
        arr[offs[i]:offs[i + 1]] = a
        inp[offs[i]:offs[i + 1]] = b
        gen[offs[i]:offs[i + 1]] = g
    return offs, arr, inp, gen


def generate(spec):
    """workload.h:78 (host) -> (arrival, input_len, gen_len)."""
    lib = load()
    n = C.c_int64(0)
    st = lib.scls_generate(C.byref(spec), 0, C.byref(n), None, None, None)
    if st not in (0, capi.ERR_CAPACITY):
        buf = C.create_string_buffer(4096)
        lib.scls_last_error(None, buf, 4096)
        raise SclsError(st, buf.value.decode())
    k = n.value
    arr = np.zeros(max(k, 1), np.float64)
    inp = np.zeros(max(k, 1), np.int32)
    gen = np.zeros(max(k, 1), np.int32)
    st = lib.scls_generate(C.byref(spec), k, C.byref(n), _ptr(arr), _ptr(inp), _ptr(gen))
    if st:
        raise SclsError(st, "generate failed")
    return arr[:k], inp[:k], gen[:k]


def fit_latency(samples, n_cap=64, l_cap=4096):
    """cost_model.cpp:140-160 fit: samples = [(phase 0|1 or "prefill"|"decode",
    batch_size, length, latency_s)] -> capi.Latency (host computation)."""
    lib = load()
    rows = list(samples)
    arr = (capi.ProfileSample * max(len(rows), 1))()
    for i, (ph, n, l, t) in enumerate(rows):
        arr[i].phase = {"prefill": 0, "decode": 1}.get(ph, ph)
        arr[i].batch_size, arr[i].length, arr[i].latency_s = n, l, t
    out = capi.Latency()
    st = lib.scls_fit_latency(arr, len(rows), n_cap, l_cap, C.byref(out))
    if st:
        buf = C.create_string_buffer(4096)
        lib.scls_last_error(None, buf, 4096)
        raise SclsError(st, buf.value.decode())
    return out


def make_pool(n, seed=7):
    """bench_batcher.cpp:27-42 -> (eff, arrival, ids, gen_len)."""
    lib = load()
    eff = np.zeros(max(n, 1), np.int32)
    arr = np.zeros(max(n, 1), np.float64)
    ids = np.zeros(max(n, 1), np.int64)
    gen = np.zeros(max(n, 1), np.int32)
    st = lib.scls_make_pool(n, seed, _ptr(eff), _ptr(arr), _ptr(ids), _ptr(gen))
    if st:
        raise SclsError(st, "make_pool failed")
    return eff[:n], arr[:n], ids[:n], gen[:n]
