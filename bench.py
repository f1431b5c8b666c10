"""bench.py — the driver's benchmark.

Headline (BASELINE.json metric, configs[4]): simulated traces/s of the
Monte Carlo sweep — 4096 traces (1024 seeds x arrival rates 10/15/20/25 req/s,
600 s, 8 instances, S = 128, codefuse-like lengths, builtin latency model and
rule-table memory) x the three policies {SCLS, SLS, ILS}: 12,288 simulations
per step.  One step is the reference's sweep() (experiment.cpp:62-85:
generate -> Simulator::run -> compute per run) through the C-ABI
scls_run_sweep_sharded: the rank's contiguous shard of traces is generated on
its GPU from the WorkloadSpecs (bit-exact with generate()), every policy runs
on every trace, and the library all-gathers the fixed-size result records
with one ncclAllGather (the only collective).  Weak scaling: every rank runs
the 4096-trace sweep (its own seeds), so N GPUs simulate 4096 N traces per
step; `value` is the whole job's traces/s.  Device time, CUDA events on the
launching stream, max over ranks.

Parity, outside the timed region: rank 0 runs the unmodified reference
(oracle/_ref, compiled from /root/reference) on ALL 4096 traces x 3 policies
of its shard on the host cores -- that run is also the cpu_baseline -- and
compares every MetricsReport field, the slice histogram and the counters of
all 12,288 jobs with the gathered device grid (at N > 1 also the first 32
traces of every other rank's shard).

The same JSON line carries the scheduling-core number (configs[2]): requests
scheduled/s for batch_requests + offload of the 1M-request pool
(bench_batcher.cpp make_pool(2^20, 7), analytic KV cap, S = 128, 8 workers),
with its phase breakdown and roofline, and C1 / C2 / C4 latency lines.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment relaunches itself under
torch.distributed.run with N ranks (one per GPU, 127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2406_13511_b200 import capi  # noqa: E402  (ctypes structs only)

METRIC = ("requests scheduled/sec (sort+DP batching+offload) and simulated traces/sec "
          "at 1/2/4/8 B200")
RATES = (10.0, 15.0, 20.0, 25.0)
POLICIES = ("scls", "sls", "ils")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--traces", type=int, default=4096)
    p.add_argument("--duration", type=float, default=600.0)
    p.add_argument("--no-c3", action="store_true", help="skip the C1-C4 side lines")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU reference run (parity + cpu_baseline)")
    return p.parse_args()


def trace_spec(i, duration):
    return capi.workload_spec(rate=RATES[i % 4], duration_s=duration, seed=1000 + i // 4)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(name):
    """dram bytes per launch of a kernel from the committed ncu summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(name, {}).get("dram_bytes")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
def ref_checker():
    """(library, kind): the compiled reference (oracle/_ref) when present, else the C port."""
    from oracle.pyoracle import RefLib, REF_SO, OracleLib, ORACLE_SO
    try:
        return RefLib(REF_SO), "reference"
    except OSError:
        return OracleLib(ORACLE_SO), "port"


def ref_sweep(lib, kind, specs, cfgs, lat, mem, hist_bins, cores):
    """The reference's sweep body on the host cores: per trace generate() once,
    then Simulator::run + compute for every policy (ref_run_sweep)."""
    if kind == "reference":
        return lib.run_sweep(specs, cfgs, lat, mem, hist_bins=hist_bins, threads=cores)
    traces = [lib.generate(sp) for sp in specs]  # the C port: same work, composed here
    res, hist = [], []
    for c in cfgs:
        r, h = lib.simulate(traces, c, lat, mem, hist_bins=hist_bins, threads=cores)
        res.extend(r)
        hist.append(h)
    out = (capi.TraceResult * len(res))(*res)
    return out, np.stack(hist)


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    compiled from /root/reference sources) on the host cores, rank 0 only,
    on the SAME workload as our arm: every step is the full 4096-trace x 3
    policy sweep, with the same warm-up and step counts."""
    if rank != 0:
        return
    lib, kind = ref_checker()
    cores = os.cpu_count() or 1
    specs = [trace_spec(i, args.duration) for i in range(args.traces)]
    lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
    cfgs = [capi.sched_cfg(policy=p) for p in POLICIES]

    def step():
        t0 = time.perf_counter()
        ref_sweep(lib, kind, specs, cfgs, lat, mem, 16, cores)
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    sec = sum(times) / len(times)
    value = 3 * args.traces / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "traces/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the reference's own generate(): Poisson arrivals, codefuse-like lengths)",
            "config": {"workload": f"C5 Monte Carlo sweep: {args.traces} traces (seeds x rates 10/15/20/25 req/s), "
                                   f"{args.duration:.0f} s, 8 instances, S=128, max_gen 1024, x {{SCLS,SLS,ILS}} = "
                                   f"{3 * args.traces} simulations per step", "traces": args.traces,
                       "host_threads": cores},
            "cpu_baseline": {"value": value, "unit": "traces/s", "cores": cores, "kind": kind,
                             "sample": f"every step the full per-GPU workload: {args.traces} traces x 3 policies "
                                       "(generate once per trace + Simulator::run + compute per policy, "
                                       "one digest-free counting pass per log); at N > 1 the host runs one "
                                       "GPU's share (the host cores do not grow with N)"},
            "e2e": {"value": value, "unit": "traces/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def bench_c3(ctx, torch, lib, capi, stream, steps, warmup):
    """configs[2]: batch_requests + offload on the 1M pool, device-resident and e2e."""
    n = 1 << 20
    eff, arr, ids, _ = lib.make_pool(n, 7)
    lat, mem = capi.builtin_latency_model(), capi.builtin_analytic_memory_model()
    dev = torch.device("cuda")
    d_eff = torch.from_numpy(eff).to(dev)
    d_arr = torch.from_numpy(arr).to(dev)
    d_ids = torch.from_numpy(ids).to(dev)
    wid = torch.arange(8, dtype=torch.int32, device=dev)
    loads = torch.zeros(8, dtype=torch.float64, device=dev)
    outs = (torch.empty(n + 1, dtype=torch.int32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(n, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.int64, device=dev),
            torch.empty(n, dtype=torch.int64, device=dev), torch.empty(n, dtype=torch.int32, device=dev))
    for _ in range(warmup):
        loads.zero_()
        ctx.schedule_device(n, d_eff, d_arr, d_ids, 128, lat, mem, wid, loads, outs)
    ms, phases, launches = [], [], 0
    for _ in range(steps):
        loads.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        nb = ctx.schedule_device(n, d_eff, d_arr, d_ids, 128, lat, mem, wid, loads, outs)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        phases.append(ctx.timings())
        launches += ctx.launches()
    # e2e: host buffers through the C-ABI (H2D + D2H inside the call)
    e2e = []
    p_eff = torch.from_numpy(eff).pin_memory().numpy()
    p_arr = torch.from_numpy(arr).pin_memory().numpy()
    p_ids = torch.from_numpy(ids).pin_memory().numpy()
    for _ in range(steps):
        t0 = time.perf_counter()
        r = ctx.schedule(p_eff, p_arr, p_ids, 128, lat, mem, np.arange(8, dtype=np.int32), [0.0] * 8)
        e2e.append(time.perf_counter() - t0)
    med = statistics.median(ms)
    ph = {k: round(statistics.median(p[k] for p in phases), 3) for k in ("sort", "estimate", "dp", "backtrack", "offload")}
    # parity vs the committed reference golden (11,820 batches, sum est)
    tot = 0.0
    for e in r["est"]:
        tot += float(e)
    peak, _ = peaks()

    def hbm(bytes_per_req, ms):
        gbs = bytes_per_req * n / (ms / 1e3) / 1e9 if ms else None
        return {"bytes_per_request": bytes_per_req, "ms": ms, "achieved_gbs": gbs,
                "frac": gbs / peak if gbs else None, "peak_gbs": peak}

    # the sort and the estimator are HBM-shaped (24 B/request for
    # the sort; the estimator reads the sorted key and writes a row's L / K:
    # 16 B/request); the DP is the serial chain, reported in ns per row against
    # the measured DADD+DSETP+SEL dependent-step floor (25.9 cycles @ 1965 MHz,
    # tools/ubench_chain.cu) with the committed ncu issue counters.
    dp = issue_line("dp_mono_kernel_1m", "dp_mono_kernel", n, "rows", ph["dp"])
    dp["ns_per_row"] = ph["dp"] * 1e6 / n
    dp["chain_floor_ns_per_row"] = 25.9 / 1.965
    return {"metric": "requests scheduled/s", "config": "C3: make_pool(2^20, 7), analytic KV cap, S=128, 8 workers",
            "value": n / (med / 1e3), "ms_per_call": med, "phases_ms": ph,
            "hbm": {"sort": hbm(24, ph["sort"]), "estimate": hbm(16, ph["estimate"])},
            "issue_efficiency": {"dp": dp},
            "e2e_value": n / statistics.median(e2e), "e2e_ms": statistics.median(e2e) * 1e3,
            "n_batches": int(nb), "sum_est": repr(tot),
            "parity": "ok" if (nb == 11820 and repr(tot) == "70831.31070040006") else "MISMATCH",
            "gpu_launches_per_call": launches // max(steps, 1)}


def bench_scheduler_sweep(ctx, lib):
    """Per-call latency of batch_requests across pool sizes: the reference's
    own microbenchmark sizes (bench_batcher.cpp:44-57: make_pool(n, 7), S =
    128, builtin rule-table memory, n = 16..4096) and 2^14..2^20.  Device time
    (CUDA events, inputs resident), e2e through the C-ABI with host arrays
    (H2D + D2H inside), and the compiled reference on one host core (the
    reference API is one serial call), every result compared."""
    lib_ref, kind = ref_checker()
    lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
    rows = []
    for n in (16, 64, 256, 1024, 4096, 1 << 14, 1 << 16, 1 << 18, 1 << 20):
        eff, arr, ids, _ = lib.make_pool(n, 7)
        reps = 50 if n <= 4096 else (10 if n <= 1 << 16 else 3)
        dev, e2e = [], []
        for _ in range(reps + 2):
            t0 = time.perf_counter()
            r = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
            e2e.append(time.perf_counter() - t0)
            dev.append(ctx.timings()["total"])
        cpu = []
        for _ in range(max(3, reps // 5)):
            t0 = time.perf_counter()
            w = lib_ref.batch_requests(eff, arr, ids, 128, lat, mem)
            cpu.append(time.perf_counter() - t0)
        same = (r["n_batches"] == w["n_batches"] and all(np.array_equal(r[k], w[k])
                                                          for k in ("seg_begin", "l_in", "est", "member_id")))
        dv, ev, cv = statistics.median(dev[2:]) * 1e3, statistics.median(e2e[2:]) * 1e6, statistics.median(cpu) * 1e6
        rows.append({"n": n, "batches": int(r["n_batches"]), "device_us": round(dv, 1), "e2e_us": round(ev, 1),
                     "cpu_us": round(cv, 1), "e2e_speedup": round(cv / ev, 2), "parity": "ok" if same else "MISMATCH",
                     "path": "small (4 launches)" if n <= 4096 else "multi-kernel"})
    return {"metric": "batch_requests latency per call", "memory": "rule table (builtin_memory_model)", "S": 128,
            "cpu": f"{kind}, 1 host core", "rows": rows}


def bench_configs(ctx, lib, capi, steps):
    """BASELINE configs[0], [1], [3] as latency lines next to the headline:
    C1 (1 instance, rate 2, 500 s, SCLS), C2 (8 instances, rate 20, 500 s, SCLS)
    and C4 (one 5000 s / ~100k-request trace x {SCLS, SLS, ILS} x slice
    {32, 64, 128, 256} x max_gen {256, 512, 1024}), each generated and
    simulated on the device through scls_run_experiments; the CPU reference
    (oracle/_ref) runs the same jobs on the host cores; every TraceResult
    field is compared with it."""
    from oracle.pyoracle import RefLib, REF_SO, OracleLib, ORACLE_SO
    try:
        ref, kind = RefLib(REF_SO), "reference"
    except OSError:
        ref, kind = OracleLib(ORACLE_SO), "port"
    lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
    cases = {
        "C1": [(capi.workload_spec(rate=2.0, duration_s=500.0, seed=42), capi.sched_cfg(policy="scls", worker_count=1))],
        "C2": [(capi.workload_spec(rate=20.0, duration_s=500.0, seed=42), capi.sched_cfg(policy="scls"))],
    }
    c4 = []
    for pol in POLICIES:
        for S in (32, 64, 128, 256):
            for G in (256, 512, 1024):
                if S <= G:
                    c4.append((capi.workload_spec(rate=20.0, duration_s=5000.0, seed=42, max_gen_limit=G),
                               capi.sched_cfg(policy=pol, slice_len=S, max_gen_limit=G)))
    cases["C4"] = c4
    cores = os.cpu_count() or 1
    ctx.set_digests(False)  # the reference's run/sweep report metrics only
    out = {}
    for name, jobs in cases.items():
        specs = [j[0] for j in jobs]
        cfgs = [j[1] for j in jobs]
        ms = []
        for _ in range(max(3, steps)):
            res, _h = ctx.run_experiments(specs, cfgs, lat, mem, hist_bins=16)
            ms.append(ctx.timings()["total"])
        traces = [ref.generate(sp) for sp in specs]
        t0 = time.perf_counter()
        want, _wh = ref.simulate(traces, cfgs, lat, mem, cfg_index=list(range(len(jobs))), hist_bins=16,
                                 threads=cores)
        cpu_s = time.perf_counter() - t0
        bad = sum(1 for i in range(len(jobs)) for f, _ in capi.TraceResult._fields_
                  if f not in ("sim_clock", "h_complete_ids", "h_dispatch", "h_complete_t", "h_log")
                  and getattr(res[i], f) != getattr(want[i], f))
        out[name] = {"jobs": len(jobs), "requests_per_trace": int(len(traces[0][0])),
                     "device_ms": round(statistics.median(ms), 3),
                     "cpu_reference_ms": round(cpu_s * 1e3, 1), "cpu_cores": min(cores, len(jobs)),
                     "cpu_kind": kind, "mismatches": bad}
    return out


SIM_NCU = {"scls": ("sim_kernel_scls_4096", "sim_kernel<SCLS>"),
           "ils": ("sim_ils_indep_4096", "sim_ils_indep_kernel<split> (+ sim_ils_merge_kernel)"),
           "sls": ("sim_sls_pack_4096", "sim_sls_pack_kernel (+ sim_sls_merge_kernel)")}
REPORT_FIELDS = [f for f, _ in capi.TraceResult._fields_
                 if f not in ("sim_clock", "h_complete_ids", "h_dispatch", "h_complete_t", "h_log")]
FIELD_WORD = {f: getattr(capi.TraceResult, f).offset // 8 for f, _ in capi.TraceResult._fields_}


def ncu_row(name):
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f).get(name)
    except Exception:
        return None


def issue_line(name, kname, units, unit_name, ms):
    """SM / warp-issue efficiency of a latency-bound kernel (north star):
    units/s measured live, and the ncu counters of the committed capture."""
    row = ncu_row(name) or {}
    return {"kernel": kname, unit_name + "_per_launch": units, "launch_ms": ms,
            unit_name + "_per_s": units / (ms / 1e3) if ms else None,
            "issue_active_pct": row.get("issue_active_pct"), "warps_active_pct": row.get("warps_active_pct"),
            "top_stalls": row.get("stall_share"), "ncu_capture": row.get("report")}


def run_ours(args, rank, world, dist):
    import torch

    from paper_2406_13511_b200 import lib, sweep

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    ctx = lib.Context(local, C.c_void_p(stream.cuda_stream))
    if world > 1:  # the library's own NCCL communicator (the gather runs inside scls_run_sweep_sharded)
        sweep.join_comm(ctx, rank, world, dist)
    nranks = ctx.comm_size()
    assert nranks == world, (nranks, world)
    # weak scaling (the trace dimension is partitioned): every rank
    # runs the C5 sweep of args.traces traces; rank r's traces are the global
    # indices [r * traces, (r + 1) * traces) -- distinct seeds
    T = args.traces * world
    lo, hi = sweep.shard_range(T, rank, world)
    ntr = hi - lo
    lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
    cfgs = [capi.sched_cfg(policy=p) for p in POLICIES]
    nfields = C.sizeof(capi.TraceResult) // 8
    hist_bins = 16
    # the whole grid (every rank holds it after the gather), policy-major: job c * T + t
    d_res = torch.empty(3 * T * nfields, dtype=torch.int64, device=dev)
    d_hist = torch.empty(3 * T * hist_bins, dtype=torch.int64, device=dev)
    ctx.set_digests(False)  # the reference's sweep reports metrics only
    cfg_arr = (capi.SchedCfg * 3)(*cfgs)
    spec_arr = (capi.WorkloadSpec * T)(*[trace_spec(i, args.duration) for i in range(T)])
    res_ptr = C.cast(C.c_void_p(d_res.data_ptr()), C.POINTER(capi.TraceResult))

    def sweep_step():
        # experiment.cpp sweep, sharded: this rank's traces generated on the
        # device (workload.cpp:163-181, bit-exact), every policy on each, the
        # result records all-gathered (ncclAllGather inside the library)
        st = ctx.lib.scls_run_sweep_sharded(ctx.h, T, spec_arr, 3, cfg_arr, C.byref(lat), C.byref(mem), res_ptr,
                                            hist_bins, C.c_void_p(d_hist.data_ptr()), capi.MEM_DEVICE)
        ctx._check(st)

    for _ in range(args.warmup):
        sweep_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = 0
    shard_ms, gather_ms = [], []
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            sweep_step()
            launches += ctx.launches()
            tm = ctx.timings()
            shard_ms.append(tm["simulate"])
            gather_ms.append(tm["offload"])
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    elapsed = e0.elapsed_time(e1) / 1e3
    t_max = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    elapsed = float(t_max.item())
    value = 3 * T * args.steps / elapsed
    grid = d_res.view(3 * T, nfields).cpu().numpy().copy()
    grid_hist = d_hist.view(3, T, hist_bins).cpu().numpy().copy()

    # per-policy launches of this rank's shard alone (outside the timed region):
    # the kernel times and event counts behind the roofline / issue lines
    specs_local = [trace_spec(i, args.duration) for i in range(lo, hi)]
    pol_ms, pol_events, pol_gen = {}, {}, []
    for k, p in enumerate(POLICIES):
        ms = []
        for _ in range(2):
            r, _h = ctx.run_sweep(specs_local, [cfgs[k]], lat, mem, hist_bins=hist_bins)
            tm = ctx.timings()
            ms.append(tm["simulate"])
            pol_gen.append(tm["generate"])
        pol_ms[p] = statistics.median(ms)
        pol_events[p] = int(sum(r[i].n_events for i in range(ntr)))
    nreq = int(grid[:T, FIELD_WORD["n_requests"]].sum())  # requests of the sweep (one row per trace)

    # e2e through the public C-ABI with host buffers: WorkloadSpecs in from the
    # host (H2D inside the call), the gathered grid out to host memory (D2H)
    ctx.run_sweep_sharded(spec_arr, cfgs, lat, mem, hist_bins=hist_bins)  # warm-up of the host path
    e2e_t = []
    for _ in range(max(3, args.steps)):
        t0 = time.perf_counter()
        ctx.run_sweep_sharded(spec_arr, cfgs, lat, mem, hist_bins=hist_bins)
        e2e_t.append(time.perf_counter() - t0)
    t_e2e = torch.tensor([statistics.median(e2e_t)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    h2d = ntr * C.sizeof(capi.WorkloadSpec)
    d2h = 3 * T * (C.sizeof(capi.TraceResult) + 8 * hist_bins)
    statuses = sorted(set(int(x) & 0xffffffff for x in grid[:, 0]))

    if rank != 0:
        return
    hbm, peak_src = peaks()
    dom = max(pol_ms, key=pol_ms.get)  # the dominant launch
    ncu_name, kname = SIM_NCU[dom]
    sim_s = pol_ms[dom] / 1e3
    shard_req = int(grid[lo:hi, FIELD_WORD["n_requests"]].sum())
    bytes_per_launch = shard_req * 16 + ntr * (C.sizeof(capi.TraceResult) + 8 * hist_bins)
    achieved = bytes_per_launch / sim_s / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "traces/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: every step generates its traces on the device from WorkloadSpecs (the reference "
                "sampler: mt19937_64, glibc log gaps, codefuse-like lengths; bit-exact with generate())",
        "config": {"workload": f"C5 Monte Carlo sweep (experiment.cpp sweep: generate + simulate + metrics): "
                               f"{T} traces (seeds x rates 10/15/20/25 req/s), {args.duration:.0f} s, 8 instances, "
                               f"S=128, max_gen 1024, x {{SCLS,SLS,ILS}} = {3 * T} simulations per step",
                   "traces": T, "traces_per_gpu": args.traces, "requests": nreq,
                   "parallelism": f"trace-sharded dp{world}",
                   "l2": "generated traces (%.0f MB per rank) > L2, rewritten every step" % (shard_req * 16 / 1e6)},
        "e2e": {"value": 3 * T / float(t_e2e.item()), "unit": "traces/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "comm": {"backend": "nccl (library-owned communicator, scls_comm_init)" if world > 1 else "none (one rank)",
                 "nranks": nranks, "comm_nranks_ok": nranks == world,
                 "gather_ms_per_step": statistics.median(gather_ms), "shard_ms_per_step": statistics.median(shard_ms)},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": achieved / hbm, "traffic": ncu_traffic(ncu_name),
                     "peak_source": peak_src, "bytes_per_launch": bytes_per_launch,
                     "launch_ms": pol_ms[dom],
                     # the bound that applies: warp-issue slots (ncu smsp__issue_active of the
                     # committed capture of this kernel on the current build)
                     "issue_frac": ((ncu_row(ncu_name) or {}).get("issue_active_pct") or 0.0) / 100.0 or None,
                     "note": "the simulators are event-chain (issue / latency) bound, not HBM bound: "
                             "algorithmic bytes = 16 B/request in + result records out; the issue efficiency "
                             "the north star asks for is in `issue_efficiency`"},
        "issue_efficiency": {p: issue_line(SIM_NCU[p][0], SIM_NCU[p][1], pol_events[p], "events", pol_ms[p])
                             for p in POLICIES},
        "kernel_ms_per_policy": pol_ms,
        "generate_ms_per_shard": statistics.median(pol_gen),
        "statuses": statuses,
        "clocks": clk.summary(),
    }
    if not args.no_c3:
        line["scheduler_c3"] = bench_c3(ctx, torch, lib, capi, stream, max(2, args.steps // 2), 2)
        line["scheduler_sweep"] = bench_scheduler_sweep(ctx, lib)
        line["configs_c1_c2_c4"] = bench_configs(ctx, lib, capi, args.steps)
    if not args.no_cpu:
        # every job of rank 0's shard (the N = 1 workload) and the first 32
        # traces of every other rank's shard
        check = list(range(0, args.traces)) + [t for r in range(1, world)
                                               for t in range(r * args.traces, r * args.traces + 32)]
        cpu, parity = cpu_reference(args, T, check, cfgs, lat, mem, hist_bins, grid, grid_hist)
        line["cpu_baseline"] = cpu
        line["parity"] = parity
        if not args.no_c3:
            line["cpu_baseline"]["scheduler_c3"] = cpu_c3()
    print(json.dumps(line), flush=True)


def cpu_reference(args, T, check, cfgs, lat, mem, hist_bins, grid, grid_hist):
    """The unmodified reference on the traces `check` (all of them at one GPU)
    x 3 policies on this host's cores, then every job compared with the device
    grid (policy-major, T traces): every MetricsReport field, the slice
    histogram and the counters.  The timed part over rank 0's shard is the
    cpu_baseline (the N = 1 workload)."""
    lib, kind = ref_checker()
    cores = os.cpu_count() or 1
    n0 = min(len(check), args.traces)
    specs = [trace_spec(i, args.duration) for i in check]
    t0 = time.perf_counter()
    want0, want_hist0 = ref_sweep(lib, kind, specs[:n0], cfgs, lat, mem, hist_bins, cores)
    sec = time.perf_counter() - t0
    parts = [(want0, want_hist0, n0)]
    if len(specs) > n0:
        w1, h1 = ref_sweep(lib, kind, specs[n0:], cfgs, lat, mem, hist_bins, cores)
        parts.append((w1, h1, len(specs) - n0))
    cpu = {"value": 3 * n0 / sec, "unit": "traces/s", "cores": cores, "kind": kind,
           "sample": f"the full workload: {n0} traces x 3 policies (generate once per trace + Simulator::run + "
                     f"compute per policy, one digest-free counting pass per log), {cores} host threads"}
    nfields = C.sizeof(capi.TraceResult) // 8
    word = sorted(set(FIELD_WORD[f] for f in REPORT_FIELDS))  # status + worker_count share word 0
    bad = set()
    base = 0
    for want, want_hist, m in parts:
        wg = np.frombuffer(C.string_at(C.addressof(want), 3 * m * C.sizeof(capi.TraceResult)),
                           np.int64).reshape(3, m, nfields)
        ts = np.asarray(check[base:base + m])
        for c in range(3):
            rows = grid[c * T + ts]
            bj = np.nonzero((rows[:, word] != wg[c][:, word]).any(axis=1))[0]
            bh = np.nonzero((grid_hist[c, ts] != want_hist.reshape(3, m, -1)[c]).any(axis=1))[0]
            bad |= {int(c * T + ts[j]) for j in set(bj) | set(bh)}
        base += m
    jobs = 3 * len(check)
    parity = {"checked": f"{jobs} jobs ({len(check)} traces x 3 policies{'' if len(check) == T else ' of ' + str(T)}) "
                         f"vs the {kind} on the host: every MetricsReport field bit-exact, slice histogram, "
                         "completed/batch/pad/invalid/event counters",
              "jobs": jobs, "mismatched_jobs": len(bad), "first_mismatches": sorted(bad)[:8]}
    return cpu, parity


def cpu_c3():
    """C3 on one host thread (the reference API is one serial call)."""
    from oracle.pyoracle import OracleLib, ORACLE_SO
    lib, kind = ref_checker()
    eff, arr, ids, _ = (OracleLib(ORACLE_SO)).make_pool(1 << 20, 7)
    t0 = time.perf_counter()
    res = lib.batch_requests(eff, arr, ids, 128, capi.builtin_latency_model(), capi.builtin_analytic_memory_model())
    lib.offload(res["batch_id"], res["est"], np.arange(8, dtype=np.int32), [0.0] * 8)
    sec3 = time.perf_counter() - t0
    return {"value": (1 << 20) / sec3, "unit": "requests scheduled/s", "cores": 1,
            "kind": kind, "sample": "one batch_requests + offload of the 1M pool"}


def relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run
    with N ranks (the driver's own launch shape) and return its exit code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, dist)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
