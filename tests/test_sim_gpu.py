"""GPU parity of the trace-batched simulator (scls_simulate) against the C
oracle, the compiled reference's golden fixtures and SURVEY Appendix B.
Every TraceResult field is compared bit for bit (metrics are fp64 values
computed in the reference's order; digests cover every event record)."""
import itertools

import numpy as np
import pytest

from paper_2406_13511_b200 import capi
from tests.helpers import MEMORIES

pytestmark = pytest.mark.gpu

FIELDS = [f for f, _ in capi.TraceResult._fields_ if f != "sim_clock"]


def assert_results_equal(a, b, msg=""):
    for f in FIELDS:
        assert getattr(a, f) == getattr(b, f), (msg, f, getattr(a, f), getattr(b, f))


def test_golden_runs(ctx, orc, golden):
    lat = capi.builtin_latency_model()
    for run in golden["simulate"]:
        spec = capi.workload_spec(rate=run["rate"], duration_s=run["duration_s"], seed=run["seed"])
        trace = orc.generate(spec)
        cfg = capi.sched_cfg(policy=run["policy"], worker_count=run["workers"],
                             slice_len=run["slice_len"], max_gen_limit=run["max_gen_limit"])
        res, hist = ctx.simulate([trace], cfg, lat, MEMORIES[run["memory"]]())
        for f in FIELDS:
            v = getattr(res[0], f)
            got = float(v).hex() if isinstance(v, float) else int(v)
            assert got == run[f], (run["name"], f)
        assert [int(x) for x in hist[0]] == run["hist"], run["name"]


def test_many_traces_one_launch(ctx, orc):
    """A mixed sweep (3 policies x slices x workers x seeds) in one call."""
    lat = capi.builtin_latency_model()
    mem = MEMORIES["rule"]()
    cfgs, traces, idx = [], [], []
    for pol, s, w in itertools.product(("scls", "sls", "ils"), (32, 128, 256), (1, 3, 8)):
        cfgs.append(capi.sched_cfg(policy=pol, slice_len=s, worker_count=w, max_gen_limit=max(s, 512)))
    for i in range(54):
        spec = capi.workload_spec(rate=float(5 + i % 20), duration_s=40.0, seed=500 + i)
        traces.append(orc.generate(spec))
        idx.append(i % len(cfgs))
    a, ha = ctx.simulate(traces, cfgs, lat, mem, cfg_index=idx)
    b, hb = orc.simulate(traces, cfgs, lat, mem, cfg_index=idx)
    for t in range(len(traces)):
        assert_results_equal(a[t], b[t], t)
    assert np.array_equal(ha, hb)


def test_random_configs_vs_oracle(ctx, orc):
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(42)
    traces, cfgs, mems = [], [], []
    for trial in range(60):
        pol = ("scls", "sls", "ils")[trial % 3]
        spec = capi.workload_spec(rate=float(rng.uniform(2, 40)), duration_s=float(rng.uniform(5, 60)),
                                  seed=1000 + trial,
                                  gen_dist=(capi.codefuse_like_gen_dist(), capi.long_gen_dist(),
                                            capi.uniform_dist(1, 300))[(trial // 3) % 3])
        trace = orc.generate(spec)
        cfg = capi.sched_cfg(policy=pol, worker_count=int(rng.integers(1, 33)),
                             slice_len=int(rng.choice([1, 7, 16, 64, 128, 512])), max_gen_limit=1024,
                             fixed_batch_size=int(rng.integers(1, 40)),
                             max_concurrent=int(rng.integers(1, 60)),
                             lambda_=float(rng.uniform(0.05, 0.95)), gamma=float(rng.uniform(0.5, 6)))
        mname = ("rule", "analytic", "rule")[trial % 3]
        a, ha = ctx.simulate([trace], cfg, lat, MEMORIES[mname]())
        b, hb = orc.simulate([trace], cfg, lat, MEMORIES[mname]())
        assert_results_equal(a[0], b[0], (trial, pol, mname))
        assert np.array_equal(ha, hb), trial


def _log_rows(log, t):
    recs = log["records"]
    mems = log["members"]
    n = int(log["rec_count"][t])
    m = int(log["mem_count"][t])
    base = t * log["rec_cap"]
    mbase = t * log["mem_cap"]
    out = []
    for i in range(n):
        r = recs[base + i]
        row = tuple(getattr(r, f) for f, _ in capi.EventRecord._fields_ if f != "member_offset")
        mm = tuple((mems[mbase + r.member_offset + j].request, mems[mbase + r.member_offset + j].effective_input,
                    mems[mbase + r.member_offset + j].pad, mems[mbase + r.member_offset + j].gen,
                    mems[mbase + r.member_offset + j].invalid) for j in range(r.member_count))
        out.append((row, mm))
    return out, m


def test_full_event_logs(ctx, orc):
    """Record-by-record equality of the event log (event_log.h:52-69)."""
    lat = capi.builtin_latency_model()
    traces = [orc.generate(capi.workload_spec(rate=12.0, duration_s=25.0, seed=77 + i)) for i in range(3)]
    for pol in ("scls", "sls", "ils"):
        cfg = capi.sched_cfg(policy=pol, worker_count=3, slice_len=64)
        a, _, la = ctx.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=3, rec_cap=20000, mem_cap=20000)
        b, _, lb = orc.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=3, rec_cap=20000, mem_cap=20000)
        for t in range(3):
            ra, ma = _log_rows(la, t)
            rb, mb = _log_rows(lb, t)
            assert len(ra) == len(rb) and ma == mb, (pol, t)
            for i, (x, y) in enumerate(zip(ra, rb)):
                assert x == y, (pol, t, i, x, y)


def test_digests_off_keeps_metrics(ctx, orc):
    lat = capi.builtin_latency_model()
    trace = orc.generate(capi.workload_spec(rate=20.0, duration_s=60.0))
    cfg = capi.sched_cfg()
    a, _ = ctx.simulate([trace], cfg, lat, MEMORIES["rule"]())
    ctx.set_digests(False)
    try:
        b, _ = ctx.simulate([trace], cfg, lat, MEMORIES["rule"]())
    finally:
        ctx.set_digests(True)
    for f in FIELDS:
        if not f.startswith("h_"):
            assert getattr(a[0], f) == getattr(b[0], f), f
    assert b[0].h_log == 0


def test_error_statuses(ctx, orc):
    lat = capi.builtin_latency_model()
    trace = orc.generate(capi.workload_spec(rate=20.0, duration_s=10.0))
    # NonTerminationError (sim_engine_test.cpp:176-181)
    cfg = capi.sched_cfg(worker_count=1, horizon_s=0.5)
    for pol in ("scls", "sls", "ils"):
        cfg.policy = capi.POLICIES[pol]
        a, _ = ctx.simulate([trace], cfg, lat, MEMORIES["rule"]())
        b, _ = orc.simulate([trace], cfg, lat, MEMORIES["rule"]())
        assert a[0].status == capi.ERR_NON_TERMINATION == b[0].status
        assert_results_equal(a[0], b[0], pol)
    # empty workload -> EmptyLogError
    empty = (np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32))
    a, _ = ctx.simulate([empty], capi.sched_cfg(), lat, MEMORIES["rule"]())
    assert a[0].status == capi.ERR_EMPTY_LOG
    # arrivals out of order -> Error
    bad = (np.array([1.0, 0.5]), np.array([10, 10], np.int32), np.array([10, 10], np.int32))
    a, _ = ctx.simulate([bad], capi.sched_cfg(), lat, MEMORIES["rule"]())
    assert a[0].status == 1
    # a length < 1 -> INVALID_ARGUMENT for that trace only, every policy and
    # kernel (lock-step, independent-lane), other traces unaffected
    for g0, i0 in ((0, 10), (-3, 10), (10, 0)):
        zero = (np.array([0.0, 0.5, 1.0]), np.array([10, i0, 10], np.int32), np.array([10, g0, 10], np.int32))
        for pol in ("scls", "sls", "ils"):
            for digests in (True, False):
                ctx.set_digests(digests)
                a, _ = ctx.simulate([trace, zero, zero, trace], capi.sched_cfg(policy=pol), lat, MEMORIES["rule"]())
                ctx.set_digests(True)
                assert [r.status for r in a] == [0, capi.ERR_INVALID_ARGUMENT, capi.ERR_INVALID_ARGUMENT, 0], pol
                if digests:
                    b, _ = orc.simulate([trace], capi.sched_cfg(policy=pol), lat, MEMORIES["rule"]())
                    assert_results_equal(a[3], b[0], pol)
    # invalid config -> Error, other traces unaffected
    a, _ = ctx.simulate([trace, trace], [capi.sched_cfg(), capi.sched_cfg(lambda_=2.0)], lat,
                        MEMORIES["rule"](), cfg_index=[0, 1])
    assert a[0].status == 0 and a[1].status == 1
    # infeasible request under SCLS -> InfeasibleRequestError with the id
    tight = capi.analytic(1100.0, 1.0, 1.0, 1.0, 1.0)
    a, _ = ctx.simulate([trace], capi.sched_cfg(), lat, tight)
    b, _ = orc.simulate([trace], capi.sched_cfg(), lat, tight)
    assert a[0].status == capi.ERR_INFEASIBLE_REQUEST == b[0].status
    assert a[0].error_request_id == b[0].error_request_id


def test_known_answers(ctx):
    """sim_engine_test.cpp:62-88, 141-166: one short request; SLS 24 at t=0."""
    lat = capi.builtin_latency_model()
    one = (np.array([0.0]), np.array([100], np.int32), np.array([100], np.int32))
    a, _, log = ctx.simulate([one], capi.sched_cfg(worker_count=1), lat, MEMORIES["rule"](),
                             n_logged=1, rec_cap=64, mem_cap=64)
    from oracle.pyoracle import oracle_lib
    expected = oracle_lib().batch_serve_time(lat, 1, 100, 100)
    assert a[0].completed == 1 and a[0].avg_response_s == expected
    sls = (np.zeros(24), np.full(24, 50, np.int32), np.full(24, 60, np.int32))
    cfg = capi.sched_cfg(policy="sls", worker_count=1, fixed_batch_size=12)
    a, _, log = ctx.simulate([sls], cfg, lat, MEMORIES["rule"](), n_logged=1, rec_cap=256, mem_cap=256)
    recs = [log["records"][i] for i in range(int(log["rec_count"][0]))]
    starts = [r.t for r in recs if r.kind == 3]
    ends = [r.t for r in recs if r.kind == 4]
    assert len(starts) == 2 and starts[0] == 0.0 and starts[1] == ends[0]


def test_c4_scale_trace(ctx, orc):
    """configs[3] scale: one 100k-request trace (5000 s at 20 req/s) under each
    policy, bit-exact against the oracle; plus the slice-length grid on a
    shorter trace."""
    lat = capi.builtin_latency_model()
    big = orc.generate(capi.workload_spec(rate=20.0, duration_s=5000.0, seed=42))
    assert len(big[0]) > 99000
    for pol in ("scls", "sls", "ils"):
        cfg = capi.sched_cfg(policy=pol)
        a, ha = ctx.simulate([big], cfg, lat, MEMORIES["rule"]())
        b, hb = orc.simulate([big], cfg, lat, MEMORIES["rule"]())
        assert_results_equal(a[0], b[0], pol)
        assert np.array_equal(ha, hb)
    small = orc.generate(capi.workload_spec(rate=20.0, duration_s=300.0, seed=7))
    cfgs = [capi.sched_cfg(policy=p, slice_len=s, max_gen_limit=g)
            for p in ("scls", "sls", "ils") for s in (32, 64, 128, 256) for g in (256, 512, 1024) if s <= g]
    a, ha = ctx.simulate([small] * len(cfgs), cfgs, lat, MEMORIES["rule"](), cfg_index=list(range(len(cfgs))))
    b, hb = orc.simulate([small] * len(cfgs), cfgs, lat, MEMORIES["rule"](), cfg_index=list(range(len(cfgs))))
    for i in range(len(cfgs)):
        assert_results_equal(a[i], b[i], i)
    assert np.array_equal(ha, hb)


def test_metrics_only_path_vs_oracle(ctx, orc):
    """Digests off selects the lean metrics-only kernels (the sweep/bench path):
    every report field must still match the oracle bit for bit."""
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(77)
    traces, cfgs = [], []
    for trial in range(48):
        pol = ("ils", "scls", "sls")[trial % 3]
        traces.append(orc.generate(capi.workload_spec(rate=float(rng.uniform(2, 30)),
                                                      duration_s=float(rng.uniform(10, 90)), seed=3000 + trial)))
        cfgs.append(capi.sched_cfg(policy=pol, worker_count=int(rng.integers(1, 33)),
                                   slice_len=int(rng.choice([16, 64, 128])), max_gen_limit=1024,
                                   fixed_batch_size=int(rng.integers(1, 30)),
                                   max_concurrent=int(rng.integers(1, 40)),
                                   horizon_s=1e7 if trial % 7 else 20.0))
    idx = list(range(len(cfgs)))
    ctx.set_digests(False)
    try:
        a, ha = ctx.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    finally:
        ctx.set_digests(True)
    b, hb = orc.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    for t in range(len(traces)):
        for f in FIELDS:
            if not f.startswith("h_"):
                assert getattr(a[t], f) == getattr(b[t], f), (t, cfgs[t].policy, f)
    assert np.array_equal(ha, hb)


def test_metrics_only_edge_times(ctx, orc):
    """The lean ILS kernel keys event times by raw IEEE bits only when every
    time is provably positive; zero / negative arrivals, models whose step
    time may be zero, and exact time ties (duplicate arrivals, integer-valued
    models) must take the general key path or the tie-break and still match."""
    base = orc.generate(capi.workload_spec(rate=12.0, duration_s=40.0, seed=4242))
    arr, inp, gen = (np.asarray(x) for x in base)
    dup = np.repeat(arr[: len(arr) // 2], 2)
    n2 = len(dup)
    variants = {
        "zero_start": (arr - arr[0], inp, gen),
        "negative": (arr - 5.0, inp, gen),
        "duplicates": (dup, inp[:n2], gen[:n2]),
        "plain": (arr, inp, gen),
    }
    lats = {
        "builtin": capi.builtin_latency_model(),
        "no_const": capi.latency_model(p1=2e-6, p3=5e-5, d1=1e-7, d3=3e-6),
        "integer": capi.latency_model(p4=1.0, d4=1.0),
        "neg_coeff": capi.latency_model(p4=0.02, d3=3e-6, d4=0.02, d2=-1e-5),
    }
    for lname, lat in lats.items():
        traces, cfgs = [], []
        for vname, tr in variants.items():
            for pol in ("ils", "scls", "sls"):
                traces.append(tuple(np.ascontiguousarray(x) for x in tr))
                cfgs.append(capi.sched_cfg(policy=pol, worker_count=4, max_concurrent=6, fixed_batch_size=6))
        idx = list(range(len(cfgs)))
        ctx.set_digests(False)
        try:
            a, ha = ctx.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
        finally:
            ctx.set_digests(True)
        b, hb = orc.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
        for t in range(len(traces)):
            for f in FIELDS:
                if not f.startswith("h_"):
                    assert getattr(a[t], f) == getattr(b[t], f), (lname, t, cfgs[t].policy, f)
        assert np.array_equal(ha, hb), lname


@pytest.mark.parametrize("digests", [False, True])
@pytest.mark.parametrize("concurrent", [True, False])
def test_simulate_grid_matches_per_trace_runs(ctx, orc, digests, concurrent):
    """scls_simulate_grid (each trace staged once, every config on every
    trace, per-policy launches on forked streams) must equal the oracle run
    on the repeated traces, job by job."""
    lat = capi.builtin_latency_model()
    traces = [orc.generate(capi.workload_spec(rate=r, duration_s=45.0, seed=900 + i))
              for i, r in enumerate((6.0, 11.0, 17.0, 23.0, 29.0))]
    cfgs = [capi.sched_cfg(policy=p, worker_count=w, slice_len=sl)
            for p, w, sl in (("scls", 4, 64), ("sls", 3, 128), ("ils", 5, 128), ("scls", 8, 128), ("ils", 2, 64))]
    ctx.set_digests(digests)
    ctx.set_concurrent(concurrent)
    try:
        got, gh = ctx.simulate_grid(traces, cfgs, lat, MEMORIES["rule"](), hist_bins=16)
    finally:
        ctx.set_digests(True)
        ctx.set_concurrent(True)
    rep = [t for _ in cfgs for t in traces]
    idx = [c for c in range(len(cfgs)) for _ in traces]
    want, wh = orc.simulate(rep, cfgs, lat, MEMORIES["rule"](), cfg_index=idx, hist_bins=16)
    for c in range(len(cfgs)):
        for t in range(len(traces)):
            a, b = got[c][t], want[c * len(traces) + t]
            for f in FIELDS:
                if digests or not f.startswith("h_"):
                    assert getattr(a, f) == getattr(b, f), (c, t, f)
    assert np.array_equal(gh.reshape(-1, 16), np.asarray(wh).reshape(-1, 16))


@pytest.mark.parametrize("lockstep", [False, True])
def test_ils_kernels_agree_and_tie_fallback(ctx, orc, lockstep):
    """Metrics-only ILS and SLS: the independent-lane kernels (default) and the
    lock-step kernels both match the oracle, including traces whose instances
    evolve identically (exact cross-instance time ties: the independent
    kernels hand those jobs to the lock-step kernels), simultaneous arrivals
    and NonTermination horizons."""
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(11)
    traces, cfgs = [], []
    for trial in range(80):
        pol = ("ils", "sls")[trial % 2]
        tr = orc.generate(capi.workload_spec(rate=float(rng.uniform(2, 40)),
                                             duration_s=float(rng.uniform(10, 120)), seed=8100 + trial))
        if trial % 7 == 3:  # bursts of simultaneous arrivals
            tr = (np.floor(np.asarray(tr[0]) * 2.0) / 2.0, tr[1], tr[2])
        traces.append(tr)
        cfgs.append(capi.sched_cfg(policy=pol, worker_count=int(rng.integers(1, 33)),
                                   max_gen_limit=int(rng.choice([64, 512, 1024])),
                                   max_concurrent=int(rng.integers(1, 20)),
                                   fixed_batch_size=int(rng.integers(1, 40)),
                                   horizon_s=1e7 if trial % 5 else float(rng.uniform(5, 60))))
    # identical instances: every instance gets the same requests at the same times
    for pol in ("ils", "sls"):
        for w in (2, 4, 8):
            k = 6
            arr = np.repeat(np.arange(1, k + 1, dtype=np.float64), w)
            inp = np.repeat(np.arange(100, 100 + 10 * k, 10, dtype=np.int32), w)
            gen = np.repeat(np.arange(5, 5 + 3 * k, 3, dtype=np.int32), w)
            traces.append((arr, inp, gen))
            cfgs.append(capi.sched_cfg(policy=pol, worker_count=w, max_concurrent=3, fixed_batch_size=2))
    idx = list(range(len(cfgs)))
    ctx.set_digests(False)
    ctx.set_ils_lockstep(lockstep)
    try:
        a, ha = ctx.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    finally:
        ctx.set_digests(True)
        ctx.set_ils_lockstep(False)
    b, hb = orc.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    for t in range(len(traces)):
        for f in FIELDS:
            if not f.startswith("h_"):
                assert getattr(a[t], f) == getattr(b[t], f), (t, f, getattr(a[t], f), getattr(b[t], f))
    assert np.array_equal(ha, hb)


@pytest.mark.slow
def test_randomized_metrics_only_sweep_vs_reference(ctx, orc):
    """A larger randomized parity sweep of the metrics-only kernels (the
    bench path): 360 traces generated on the device under random configs of
    all three policies -- workers 1..32, slices 16..512, max-gen 64..1024,
    batch caps, concurrency caps, short horizons, both memory models --
    against the compiled reference, every report field and histogram."""
    from oracle import pyoracle
    ref = pyoracle.ref_lib() or orc
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(2026)
    for mem in (MEMORIES["rule"](), MEMORIES["analytic"]()):
        specs, cfgs = [], []
        for trial in range(180):
            G = int(rng.choice([64, 256, 512, 1024]))
            S = int(rng.choice([s for s in (16, 32, 64, 128, 256, 512) if s <= G]))
            specs.append(capi.workload_spec(rate=float(rng.uniform(0.5, 40)), duration_s=float(rng.uniform(5, 150)),
                                            seed=int(rng.integers(0, 2 ** 40)), max_gen_limit=G))
            cfgs.append(capi.sched_cfg(policy=("scls", "sls", "ils")[trial % 3], worker_count=int(rng.integers(1, 33)),
                                       slice_len=S, max_gen_limit=G, fixed_batch_size=int(rng.integers(1, 48)),
                                       max_concurrent=int(rng.integers(1, 24)),
                                       horizon_s=1e7 if trial % 9 else float(rng.uniform(5, 80))))
        ctx.set_digests(False)
        try:
            a, ha = ctx.run_experiments(specs, cfgs, lat, mem, hist_bins=64)
        finally:
            ctx.set_digests(True)
        traces = [ref.generate(s) for s in specs]
        b, hb = ref.simulate(traces, cfgs, lat, mem, cfg_index=list(range(len(cfgs))), hist_bins=64, threads=8)
        for t in range(len(specs)):
            for f in FIELDS:
                if not f.startswith("h_"):
                    assert getattr(a[t], f) == getattr(b[t], f), (t, cfgs[t].policy, f)
        assert np.array_equal(ha, np.asarray(hb).reshape(ha.shape))


@pytest.mark.parametrize("digests", [True, False])
def test_wide_worker_counts_vs_oracle(ctx, orc, digests):
    """More than 32 workers / instances (the reference allows any count,
    sched_policies.cpp:56): the wide lock-step variant (ceil(W/32) worker
    slots per lane in the trace's arena, any W) against the oracle, mixed with narrow configs in one launch, with
    and without digests (without: the metrics-only launch path)."""
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(33)
    cfgs, traces, idx = [], [], []
    for i, w in enumerate((33, 40, 64, 100, 257, 1024, 1025, 3000, 8)):
        for pol in ("scls", "sls", "ils"):
            cfgs.append(capi.sched_cfg(policy=pol, worker_count=w, slice_len=int(rng.choice([16, 64, 128])),
                                       max_gen_limit=512, fixed_batch_size=int(rng.integers(1, 12)),
                                       max_concurrent=int(rng.integers(1, 16))))
    for j in range(len(cfgs)):
        spec = capi.workload_spec(rate=float(rng.uniform(20, 400)), duration_s=float(rng.uniform(4, 20)),
                                  seed=3300 + j)
        traces.append(orc.generate(spec))
        idx.append(j)
    ctx.set_digests(digests)
    try:
        a, ha = ctx.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    finally:
        ctx.set_digests(True)
    b, hb = orc.simulate(traces, cfgs, lat, MEMORIES["rule"](), cfg_index=idx)
    for t in range(len(traces)):
        for f in FIELDS:
            if digests or not f.startswith("h_"):
                assert getattr(a[t], f) == getattr(b[t], f), (t, cfgs[t].worker_count, cfgs[t].policy, f)
    assert np.array_equal(ha, hb)


def test_wide_worker_event_logs(ctx, orc):
    lat = capi.builtin_latency_model()
    traces = [orc.generate(capi.workload_spec(rate=150.0, duration_s=6.0, seed=91 + i)) for i in range(2)]
    for pol in ("scls", "sls", "ils"):
        cfg = capi.sched_cfg(policy=pol, worker_count=70, slice_len=64, max_concurrent=4, fixed_batch_size=4)
        a, _, la = ctx.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=2, rec_cap=40000, mem_cap=40000)
        b, _, lb = orc.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=2, rec_cap=40000, mem_cap=40000)
        for t in range(2):
            assert_results_equal(a[t], b[t], (pol, t))
            ra, ma = _log_rows(la, t)
            rb, mb = _log_rows(lb, t)
            assert len(ra) == len(rb) and ma == mb, (pol, t)
            assert ra == rb, pol
            assert max(r[0][7] for r in ra) >= 33  # workers above 32 were used (record field `worker`)


def test_worker_counts_beyond_1024(ctx, orc):
    """Any worker_count >= 1 (sched_policies.cpp:56): 1,500 / 5,000 workers,
    every policy, event logs record by record and the report."""
    lat = capi.builtin_latency_model()
    traces = [orc.generate(capi.workload_spec(rate=2000.0, duration_s=3.0, seed=97 + i)) for i in range(2)]
    for w in (1500, 5000):
        for pol in ("scls", "sls", "ils"):
            cfg = capi.sched_cfg(policy=pol, worker_count=w, slice_len=64, max_concurrent=3, fixed_batch_size=3)
            a, _, la = ctx.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=2, rec_cap=200000,
                                    mem_cap=200000)
            b, _, lb = orc.simulate(traces, cfg, lat, MEMORIES["rule"](), n_logged=2, rec_cap=200000,
                                    mem_cap=200000)
            for t in range(2):
                assert_results_equal(a[t], b[t], (w, pol, t))
                ra, ma = _log_rows(la, t)
                rb, mb = _log_rows(lb, t)
                assert ra == rb and ma == mb, (w, pol, t)
                if pol != "scls":  # round-robin assignment reaches every worker
                    assert max(r[0][7] for r in ra) >= 1024, (w, pol)


@pytest.mark.parametrize("pol", ["ils", "sls"])
def test_packed_jobs_mixed_outcomes(ctx, orc, pol):
    """Several jobs of one config share a warp (ILS packs: up to 32 / W jobs):
    normal jobs, jobs with exact cross-instance ties (handed to the lock-step
    kernel from inside a pack), jobs that fail validation (unsorted arrivals)
    and NonTermination horizons, all in the same packs, against the oracle."""
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(5)
    traces = []
    for i in range(40):
        kind = i % 8
        if kind == 5:  # identical instances: exact time ties
            k, w = 5, 4
            traces.append((np.repeat(np.arange(1, k + 1, dtype=np.float64), w),
                           np.repeat(np.arange(100, 100 + 10 * k, 10, dtype=np.int32), w),
                           np.repeat(np.arange(5, 5 + 3 * k, 3, dtype=np.int32), w)))
        elif kind == 6:  # unsorted arrivals: Error from the simulator's constructor checks
            tr = orc.generate(capi.workload_spec(rate=10.0, duration_s=20.0, seed=700 + i))
            arr = np.asarray(tr[0]).copy()
            arr[[3, 4]] = arr[[4, 3]] if arr[3] != arr[4] else (arr[3] + 1.0, arr[4])
            traces.append((arr, tr[1], tr[2]))
        else:
            traces.append(orc.generate(capi.workload_spec(rate=float(rng.uniform(5, 30)),
                                                          duration_s=float(rng.uniform(20, 90)), seed=700 + i)))
    cfgs = [capi.sched_cfg(policy=pol, worker_count=4, max_concurrent=3, fixed_batch_size=3),
            capi.sched_cfg(policy=pol, worker_count=4, max_concurrent=3, fixed_batch_size=3, horizon_s=15.0)]
    ctx.set_digests(False)
    try:
        a, ha = ctx.simulate_grid(traces, cfgs, lat, MEMORIES["rule"](), hist_bins=16)
    finally:
        ctx.set_digests(True)
    statuses = set()
    for c, cfg in enumerate(cfgs):
        b, hb = orc.simulate(traces, cfg, lat, MEMORIES["rule"](), hist_bins=16)
        for t in range(len(traces)):
            statuses.add(b[t].status)
            for f in FIELDS:
                if not f.startswith("h_"):
                    assert getattr(a[c][t], f) == getattr(b[t], f), (c, t, f, getattr(a[c][t], f), getattr(b[t], f))
        assert np.array_equal(ha[c], hb), c
    assert len(statuses) >= 3, statuses  # ok, error and non-termination all occurred


@pytest.mark.gpu
@pytest.mark.slow
def test_sweep_600s_regime_vs_reference(ctx, ref):
    """The headline's regime (bench.py / BASELINE configs[4]): 600 s traces at
    rates 10-25 req/s, 8 instances, S = 128, generated on the device, under
    SCLS / SLS / ILS with the metrics-only kernels the sweep uses (independent
    ILS / SLS lanes, two-job ILS packs), against the reference's own sweep
    body (generate + Simulator::run + compute) on the host: every job, every
    report field, the slice histogram and the counters.  Fresh seeds (not the
    bench's), plus 4- and 16-instance configs."""
    import os
    T = 384
    specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=70000 + i)
             for i in range(T)]
    lat, mem = capi.builtin_latency_model(), MEMORIES["rule"]()
    cfgs = [capi.sched_cfg(policy=p, worker_count=w) for w in (8, 4, 16) for p in ("scls", "sls", "ils")]
    ctx.set_digests(False)
    try:
        got, got_h = ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
    finally:
        ctx.set_digests(True)
    want, want_h = ref.run_sweep(specs, cfgs, lat, mem, hist_bins=16, threads=os.cpu_count() or 1)
    skip = ("sim_clock", "h_complete_ids", "h_dispatch", "h_complete_t", "h_log")
    bad = [(j, f) for j in range(len(cfgs) * T) for f, _ in capi.TraceResult._fields_
           if f not in skip and getattr(got[j], f) != getattr(want[j], f)]
    assert not bad, bad[:10]
    assert np.array_equal(got_h, want_h)
    assert all(got[j].status == 0 for j in range(len(cfgs) * T))
