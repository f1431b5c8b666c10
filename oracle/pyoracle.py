"""Python bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module, and only as the checker (never the thing
measured or shipped).

  RefLib     oracle/_ref/libscls_ref.so — the unmodified reference core
             compiled from /root/reference sources (oracle/Makefile `ref`).
  OracleLib  oracle/libscls_oracle.so  — the C restatement, oracle/scls_oracle.c.

Both expose the same methods, so a test can run either checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2406_13511_b200 import capi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libscls_ref.so")
ORACLE_SO = os.path.join(HERE, "libscls_oracle.so")


class CheckerError(RuntimeError):
    def __init__(self, status, msg, request_id=-1):
        super().__init__(f"{capi.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.request_id = request_id


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class _Checker:
    prefix = ""

    def __init__(self, path):
        self.path = path
        self.lib = C.CDLL(path)
        self._bind()

    def _f(self, name):
        return getattr(self.lib, self.prefix + name)

    def _bind(self):
        L, M, S = C.POINTER(capi.Latency), C.POINTER(capi.Memory), C.POINTER(capi.SchedCfg)
        i32, i64, f64 = C.c_int32, C.c_int64, C.c_double
        P = C.POINTER
        sig = {
            "last_error": (C.c_size_t, [C.c_char_p, C.c_size_t]),
            "last_request_id": (i64, []),
            "batch_serve_time": (f64, [L, i32, i32, i32]),
            "prefill_time": (f64, [L, i32, i32]),
            "decode_step_time": (f64, [L, i32, i32]),
            "decode_time": (f64, [L, i32, i32, i32]),
            "would_oom": (i32, [M, i32, i32, i32]),
            "max_batch_size": (i32, [M, i32, i32]),
            "next_interval": (f64, [f64, f64, f64]),
            "validate_latency": (i32, [L]),
            "validate_memory": (i32, [M]),
            "validate_sched": (i32, [S]),
            "batch_requests": (i32, [i64, P(i32), P(f64), P(i64), i32, L, M, i64, P(i64),
                                     P(i32), P(i32), P(f64), P(i64), P(i64)]),
            "offload": (i32, [i64, P(i64), P(f64), i32, P(i32), P(f64), P(i64), P(i32)]),
            "generate": (i32, [P(capi.WorkloadSpec), i64, P(i64), P(f64), P(i32), P(i32)]),
            "simulate": (i32, [i32, P(i64), P(f64), P(i32), P(i32), S, P(i32), L, M,
                               P(capi.TraceResult), i32, P(i64), P(capi.EventLog), i32]),
        }
        for name, (res, args) in sig.items():
            fn = self._f(name)
            fn.restype = res
            fn.argtypes = args

    # -- helpers --------------------------------------------------------------
    def _raise(self, st):
        buf = C.create_string_buffer(4096)
        self._f("last_error")(buf, 4096)
        raise CheckerError(st, buf.value.decode(errors="replace"),
                           self._f("last_request_id")())

    def batch_serve_time(self, lat, n, l_in, l_out):
        return self._f("batch_serve_time")(C.byref(lat), n, l_in, l_out)

    def prefill_time(self, lat, n, l_in):
        return self._f("prefill_time")(C.byref(lat), n, l_in)

    def decode_time(self, lat, n, l_in, l_out):
        return self._f("decode_time")(C.byref(lat), n, l_in, l_out)

    def decode_step_time(self, lat, ctx, n):
        return self._f("decode_step_time")(C.byref(lat), ctx, n)

    def would_oom(self, mem, n, l_in, s):
        return bool(self._f("would_oom")(C.byref(mem), n, l_in, s))

    def max_batch_size(self, mem, l_in, s):
        return self._f("max_batch_size")(C.byref(mem), l_in, s)

    def next_interval(self, lam, gamma, min_load):
        return self._f("next_interval")(lam, gamma, min_load)

    def validate_latency(self, lat):
        return self._f("validate_latency")(C.byref(lat))

    def validate_memory(self, mem):
        return self._f("validate_memory")(C.byref(mem))

    def validate_sched(self, cfg):
        return self._f("validate_sched")(C.byref(cfg))

    def batch_requests(self, eff, arrival, ids, slice_len, lat, mem, first_batch_id=0):
        """batcher.h:40-43 -> dict(seg_begin, l_in, est, batch_id, member_id)."""
        eff = np.ascontiguousarray(eff, np.int32)
        arrival = np.ascontiguousarray(arrival, np.float64)
        ids = np.ascontiguousarray(ids, np.int64)
        n = len(eff)
        nb = C.c_int64(0)
        seg = np.zeros(n + 1, np.int32)
        l_in = np.zeros(max(n, 1), np.int32)
        est = np.zeros(max(n, 1), np.float64)
        bid = np.zeros(max(n, 1), np.int64)
        mid = np.zeros(max(n, 1), np.int64)
        st = self._f("batch_requests")(n, _p(eff, C.c_int32), _p(arrival, C.c_double),
                                       _p(ids, C.c_int64), slice_len, C.byref(lat),
                                       C.byref(mem), first_batch_id, C.byref(nb),
                                       _p(seg, C.c_int32), _p(l_in, C.c_int32),
                                       _p(est, C.c_double), _p(bid, C.c_int64),
                                       _p(mid, C.c_int64))
        if st:
            self._raise(st)
        k = nb.value
        return dict(n_batches=k, seg_begin=seg[:k + 1], l_in=l_in[:k], est=est[:k],
                    batch_id=bid[:k], member_id=mid[:n])

    def offload(self, batch_id, est, worker_id, loads):
        """offloader.h:39-40 -> (assigned batch ids, assigned workers, new loads)."""
        batch_id = np.ascontiguousarray(batch_id, np.int64)
        est = np.ascontiguousarray(est, np.float64)
        worker_id = np.ascontiguousarray(worker_id, np.int32)
        loads = np.array(loads, np.float64)
        nb = len(est)
        ob = np.zeros(max(nb, 1), np.int64)
        ow = np.zeros(max(nb, 1), np.int32)
        st = self._f("offload")(nb, _p(batch_id, C.c_int64), _p(est, C.c_double),
                                len(worker_id), _p(worker_id, C.c_int32),
                                _p(loads, C.c_double), _p(ob, C.c_int64), _p(ow, C.c_int32))
        if st:
            self._raise(st)
        return ob[:nb], ow[:nb], loads

    def generate(self, spec):
        """workload.h:78 -> (arrival, input_len, gen_len)."""
        n = C.c_int64(0)
        z = np.zeros(1, np.float64)
        zi = np.zeros(1, np.int32)
        st = self._f("generate")(C.byref(spec), 0, C.byref(n), _p(z, C.c_double),
                                 _p(zi, C.c_int32), _p(zi, C.c_int32))
        if st not in (0, capi.ERR_CAPACITY):
            self._raise(st)
        k = n.value
        arr = np.zeros(max(k, 1), np.float64)
        inp = np.zeros(max(k, 1), np.int32)
        gen = np.zeros(max(k, 1), np.int32)
        st = self._f("generate")(C.byref(spec), k, C.byref(n), _p(arr, C.c_double),
                                 _p(inp, C.c_int32), _p(gen, C.c_int32))
        if st:
            self._raise(st)
        return arr[:k], inp[:k], gen[:k]

    def simulate(self, traces, cfgs, lat, mem, cfg_index=None, hist_bins=64,
                 n_logged=0, rec_cap=0, mem_cap=0, threads=1):
        """One Simulator::run + compute per trace.  traces: list of
        (arrival, input_len, gen_len).  Returns (results, hist[, log])."""
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
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        cfg_arr = (capi.SchedCfg * len(cfgs))(*cfgs)
        idx = None if cfg_index is None else np.ascontiguousarray(cfg_index, np.int32)
        res = (capi.TraceResult * len(traces))()
        hist = np.zeros(len(traces) * hist_bins, np.int64)
        log = None
        logp = None
        if n_logged:
            log = _alloc_log(n_logged, rec_cap, mem_cap)
            logp = C.byref(log["struct"])
        st = self._f("simulate")(len(traces), _p(offs, C.c_int64), _p(arr, C.c_double),
                                 _p(inp, C.c_int32), _p(gen, C.c_int32), cfg_arr,
                                 None if idx is None else _p(idx, C.c_int32),
                                 C.byref(lat), C.byref(mem), res, hist_bins,
                                 _p(hist, C.c_int64), logp, threads)
        if st:
            self._raise(st)
        hist = hist.reshape(len(traces), hist_bins)
        if log is not None:
            return res, hist, log
        return res, hist


def _alloc_log(n_logged, rec_cap, mem_cap):
    recs = (capi.EventRecord * (n_logged * rec_cap))()
    mems = (capi.Member * max(n_logged * mem_cap, 1))()
    rc = np.zeros(n_logged, np.int64)
    mc = np.zeros(n_logged, np.int64)
    s = capi.EventLog(n_logged, rec_cap, mem_cap, recs, mems,
                      _p(rc, C.c_int64), _p(mc, C.c_int64))
    return dict(struct=s, records=recs, members=mems, rec_count=rc, mem_count=mc,
                rec_cap=rec_cap, mem_cap=mem_cap)


class RefLib(_Checker):
    prefix = "ref_"

    def run_sweep(self, specs, cfgs, lat, mem, hist_bins=16, threads=1):
        """ref_run_sweep: the reference's sweep body for every (config, trace):
        generate once per trace, Simulator::run + compute per config, no
        digests.  Returns (results[c * ntr + t], hist [nc, ntr, bins])."""
        fn = self.lib.ref_run_sweep
        fn.restype = C.c_int32
        fn.argtypes = [C.c_int32, C.POINTER(capi.WorkloadSpec), C.c_int32, C.POINTER(capi.SchedCfg),
                       C.POINTER(capi.Latency), C.POINTER(capi.Memory), C.POINTER(capi.TraceResult), C.c_int32,
                       C.POINTER(C.c_int64), C.c_int32]
        specs = list(specs)
        if isinstance(cfgs, capi.SchedCfg):
            cfgs = [cfgs]
        ntr, nc = len(specs), len(cfgs)
        sp = (capi.WorkloadSpec * max(ntr, 1))(*specs)
        ca = (capi.SchedCfg * nc)(*cfgs)
        res = (capi.TraceResult * max(ntr * nc, 1))()
        hist = np.zeros(max(ntr * nc * hist_bins, 1), np.int64)
        st = fn(ntr, sp, nc, ca, C.byref(lat), C.byref(mem), res, hist_bins, _p(hist, C.c_int64), threads)
        if st:
            self._raise(st)
        return res, hist[:ntr * nc * hist_bins].reshape(nc, ntr, hist_bins)


def _ref_fit(self, samples, n_cap=64, l_cap=4096):
    """ref_fit_latency: the reference's own fit (cost_model.cpp:140-160)."""
    fn = self.lib.ref_fit_latency
    fn.restype = C.c_int32
    rows = list(samples)
    arr = (capi.ProfileSample * max(len(rows), 1))()
    for i, (ph, n, l, t) in enumerate(rows):
        arr[i].phase = {"prefill": 0, "decode": 1}.get(ph, ph)
        arr[i].batch_size, arr[i].length, arr[i].latency_s = n, l, t
    out = capi.Latency()
    st = fn(arr, C.c_int64(len(rows)), n_cap, l_cap, C.byref(out))
    if st:
        self._raise(st)
    return out


RefLib.fit_latency = _ref_fit


class OracleLib(_Checker):
    prefix = "orc_"

    def make_pool(self, n, seed=7):
        """bench_batcher.cpp:27-42 -> (eff, arrival, ids, gen_len)."""
        fn = self.lib.orc_make_pool
        fn.restype = C.c_int32
        eff = np.zeros(max(n, 1), np.int32)
        arr = np.zeros(max(n, 1), np.float64)
        ids = np.zeros(max(n, 1), np.int64)
        gen = np.zeros(max(n, 1), np.int32)
        fn(C.c_int64(n), C.c_uint64(seed), _p(eff, C.c_int32), _p(arr, C.c_double),
           _p(ids, C.c_int64), _p(gen, C.c_int32))
        return eff[:n], arr[:n], ids[:n], gen[:n]


_cache = {}


def ref_lib():
    if "ref" not in _cache:
        if not os.path.exists(REF_SO):
            return None
        _cache["ref"] = RefLib(REF_SO)
    return _cache["ref"]


def oracle_lib():
    if "orc" not in _cache:
        _cache["orc"] = OracleLib(ORACLE_SO)
    return _cache["orc"]
