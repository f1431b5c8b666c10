"""GPU parity of the scheduling core (batch_requests, offload, schedule,
batched estimators) against the C oracle and the golden fixtures.
Bit-exact: batch boundaries, members, l_in, est bits, assignments, loads."""
import numpy as np
import pytest

from paper_2406_13511_b200 import capi
from paper_2406_13511_b200.lib import SclsError
from tests.helpers import (MEMORIES, padding_heavy_model, planned_total, random_instances,
                           reference_model, sha)

pytestmark = pytest.mark.gpu


def assert_same_batches(a, b, ctx_msg=""):
    assert a["n_batches"] == b["n_batches"], ctx_msg
    for k in ("seg_begin", "l_in", "est", "member_id"):
        assert np.array_equal(a[k], b[k]), (ctx_msg, k)


def test_golden_pools(ctx, orc, golden):
    """bench_batcher.cpp pools up to 2^20 (configs[2]) vs the reference's
    fingerprints; the 1M analytic pool is SURVEY's C3 (11,820 batches)."""
    lat = capi.builtin_latency_model()
    for case in golden["batcher"]:
        eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
        res = ctx.batch_requests(eff, arr, ids, case["slice_len"], lat, MEMORIES[case["memory"]]())
        msg = (case["n"], case["slice_len"], case["memory"])
        assert res["n_batches"] == case["n_batches"], msg
        assert float(planned_total(res["est"])).hex() == case["sum_est"], msg
        assert sha(res["seg_begin"].astype(np.int32)) == case["seg"], msg
        assert sha(res["l_in"].astype(np.int32)) == case["l_in"], msg
        assert sha(res["est"].astype(np.float64)) == case["est"], msg
        assert sha(res["member_id"].astype(np.int64)) == case["member"], msg


def test_random_instances_vs_oracle(ctx, orc):
    """batcher_test.cpp:126-166 instances (600), incl. arrival ties."""
    lat = reference_model()
    for i, (eff, arr, ids, s, mem) in enumerate(random_instances(trials=600)):
        a = ctx.batch_requests(eff, arr, ids, s, lat, mem, 3)
        b = orc.batch_requests(eff, arr, ids, s, lat, mem, 3)
        assert_same_batches(a, b, i)
        # order[] is the sorted permutation
        assert np.array_equal(ids[a["order"]], a["member_id"])


def test_medium_pools_all_models(ctx, orc):
    rng = np.random.default_rng(11)
    for n in (31, 32, 33, 63, 64, 65, 1000, 4097, 20000):
        eff = rng.integers(1, 2048, n).astype(np.int32)
        arr = rng.random(n) * 50
        ids = rng.permutation(n).astype(np.int64) - n // 2  # negative ids too
        for mname in ("rule", "analytic", "tight"):
            for s in (1, 16, 128):
                lat = capi.builtin_latency_model()
                a = ctx.batch_requests(eff, arr, ids, s, lat, MEMORIES[mname]())
                b = orc.batch_requests(eff, arr, ids, s, lat, MEMORIES[mname]())
                assert_same_batches(a, b, (n, mname, s))


def test_huge_windows_use_global_path(ctx, orc):
    """Analytic model with S=1: K(L) reaches ~28k, beyond the smem ring."""
    rng = np.random.default_rng(5)
    n = 40000
    eff = np.sort(rng.integers(1, 64, n)).astype(np.int32)
    arr = rng.random(n)
    ids = np.arange(n, dtype=np.int64)
    mem = capi.builtin_analytic_memory_model()
    lat = capi.builtin_latency_model()
    a = ctx.batch_requests(eff, arr, ids, 1, lat, mem)
    b = orc.batch_requests(eff, arr, ids, 1, lat, mem)
    assert_same_batches(a, b)


def test_ties_and_degenerate_keys(ctx, orc):
    rule = MEMORIES["rule"]()
    flat = capi.latency_model(p2=1.0)  # every partition costs the same: pure tie-breaking
    for n in (2, 33, 100, 3000):
        eff = np.full(n, 100, np.int32)
        arr = np.zeros(n)
        ids = np.arange(n, dtype=np.int64)[::-1].copy()
        assert_same_batches(ctx.batch_requests(eff, arr, ids, 128, flat, rule),
                            orc.batch_requests(eff, arr, ids, 128, flat, rule), n)
    # -0.0 vs +0.0 arrivals compare equal (ties fall to id)
    eff = np.array([5, 5, 5, 5], np.int32)
    arr = np.array([0.0, -0.0, 0.0, -0.0])
    ids = np.array([3, 2, 1, 0], np.int64)
    assert_same_batches(ctx.batch_requests(eff, arr, ids, 128, reference_model(), rule),
                        orc.batch_requests(eff, arr, ids, 128, reference_model(), rule))


def test_known_answers(ctx):
    rule = MEMORIES["rule"]()
    r = ctx.batch_requests([100, 100], [0.0, 0.0], [0, 1], 128, capi.latency_model(p2=1.0), rule)
    assert r["n_batches"] == 2
    r = ctx.batch_requests([10] * 8 + [1024], [0.0] * 9, list(range(9)), 128,
                           padding_heavy_model(), rule)
    assert r["n_batches"] == 2 and r["member_id"][-1] == 8 and r["l_in"].tolist() == [10, 1024]
    r = ctx.batch_requests([600, 600, 10, 10], [2.0, 1.0, 3.0, 0.5], [3, 1, 2, 0], 128,
                           padding_heavy_model(), rule)
    assert r["member_id"].tolist() == [0, 2, 1, 3] and r["seg_begin"].tolist() == [0, 2, 4]
    r = ctx.batch_requests([10, 310, 610, 910, 1210, 1510], [0.0] * 6, list(range(6)), 128,
                           reference_model(), rule, first_batch_id=42)
    assert r["batch_id"][0] == 42
    r = ctx.batch_requests([], [], [], 128, reference_model(), rule)
    assert r["n_batches"] == 0


def test_infeasible_singleton(ctx, orc):
    mem = capi.analytic(105.0, 3.0, 2.0, 1.0, 1.0)
    with pytest.raises(SclsError) as e:
        ctx.batch_requests([200], [0.0], [7], 10, reference_model(), mem)
    assert e.value.status == capi.ERR_INFEASIBLE_REQUEST and e.value.request_id == 7
    # the first offender in sorted order (batcher.cpp:40-46)
    with pytest.raises(SclsError) as e:
        ctx.batch_requests([50, 300, 200, 90], [0.0, 1.0, 2.0, 3.0], [10, 11, 12, 13], 10,
                           reference_model(), mem)
    assert e.value.request_id == 12


def test_offload_fixtures(ctx, orc, golden):
    ob, ow, nl = ctx.offload([0, 1, 2, 3], [6.0, 10.0, 2.0, 6.0], [0, 1], [0.0, 0.0])
    assert list(zip(ob.tolist(), ow.tolist())) == [(1, 0), (0, 1), (3, 1), (2, 0)]
    assert nl.tolist() == [12.0, 12.0]
    ob, ow, nl = ctx.offload([5], [4.0], [0, 1, 2], [5.0, 3.0, 9.0])
    assert ow.tolist() == [1] and nl.tolist() == [5.0, 7.0, 9.0]
    ob, ow, _ = ctx.offload([0, 1], [1.0, 1.0], [0, 1, 2], [2.0, 2.0, 2.0])
    assert ow.tolist() == [0, 1]
    ob, ow, _ = ctx.offload([10, 11, 12], [3.0, 3.0, 3.0], [0], [0.0])
    assert ob.tolist() == [10, 11, 12]
    with pytest.raises(SclsError) as e:
        ctx.offload([0], [1.0], [], [])
    assert e.value.status == capi.ERR_NO_WORKERS
    lat = capi.builtin_latency_model()
    for case in golden["offload"]:
        eff, arr, ids, _ = orc.make_pool(case["n"], 7)
        res = orc.batch_requests(eff, arr, ids, 128, lat, MEMORIES[case["memory"]]())
        loads = [float.fromhex(x) for x in case["loads"]]
        ob, ow, nl = ctx.offload(res["batch_id"], res["est"], np.arange(8, dtype=np.int32), loads)
        assert sha(ob) == case["batch"] and sha(ow) == case["worker"]
        assert [float(x).hex() for x in nl] == case["final_loads"]


def test_offload_random_vs_oracle(ctx, orc):
    rng = np.random.default_rng(12345)
    for trial in range(200):
        nw = int(rng.integers(1, 40))
        nb = int(rng.integers(0, 300))
        loads = rng.random(nw) * 10
        if trial % 4 == 0:
            loads = np.round(loads)  # load ties
        if trial % 5 == 1:
            loads = np.round(loads) - 5.0  # negative loads, -0.0 beside +0.0
            loads[::2] = np.where(loads[::2] == 0.0, -0.0, loads[::2])
        est = 0.01 + rng.random(nb) * 5
        if trial % 3 == 0:
            est = np.round(est, 1)  # estimate ties
        wid = rng.permutation(nw).astype(np.int32)
        bid = np.arange(nb, dtype=np.int64) + 100
        a = ctx.offload(bid, est, wid, loads)
        b = orc.offload(bid, est, wid, loads)
        for x, y in zip(a, b):
            assert np.array_equal(x, y), trial


def test_schedule_equals_batch_then_offload(ctx, orc):
    eff, arr, ids, _ = orc.make_pool(50000, 3)
    lat = capi.builtin_latency_model()
    mem = MEMORIES["analytic"]()
    loads = [0.5 * w for w in range(8)]
    s = ctx.schedule(eff, arr, ids, 128, lat, mem, np.arange(8, dtype=np.int32), loads, 7)
    b = orc.batch_requests(eff, arr, ids, 128, lat, mem, 7)
    ob, ow, nl = orc.offload(b["batch_id"], b["est"], np.arange(8, dtype=np.int32), loads)
    assert_same_batches(s, b)
    assert np.array_equal(s["assign_batch"], ob) and np.array_equal(s["assign_worker"], ow)
    assert np.array_equal(s["loads"], nl)


def test_batched_estimators(ctx, orc):
    rng = np.random.default_rng(2)
    lat = capi.builtin_latency_model()
    n = rng.integers(1, 500, 5000).astype(np.int32)
    l_in = rng.integers(1, 4096, 5000).astype(np.int32)
    l_out = rng.integers(-2, 1024, 5000).astype(np.int32)
    got = ctx.batch_serve_time(n, l_in, l_out, lat)
    want = np.array([orc.batch_serve_time(lat, int(a), int(b), int(c)) for a, b, c in zip(n, l_in, l_out)])
    assert np.array_equal(got, want)
    for mname in ("rule", "analytic", "tight"):
        mem = MEMORIES[mname]()
        got = ctx.would_oom(n[:2000], l_in[:2000], 128, mem)
        want = np.array([orc.would_oom(mem, int(a), int(b), 128) for a, b in zip(n[:2000], l_in[:2000])])
        assert np.array_equal(got, want), mname
        got = ctx.max_batch_size(l_in[:2000], 32, mem)
        want = np.array([orc.max_batch_size(mem, int(b), 32) for b in l_in[:2000]])
        assert np.array_equal(got, want), mname


@pytest.fixture
def chain_ctx(ctx):
    ctx.set_dp_kernel(1)
    yield ctx
    ctx.set_dp_kernel(0)


def test_kernel_choice(ctx, orc):
    eff, arr, ids, _ = orc.make_pool(4096, 7)
    ctx.batch_requests(eff, arr, ids, 128, capi.builtin_latency_model(), MEMORIES["analytic"]())
    assert ctx.timings()["dp_mono"] == 1.0  # builtin analytic model: monotone, windows > 32
    neg = capi.latency_model(2e-6, 1e-3, 5e-5, 0.02, 1e-7, 2e-4, 3e-6, -0.0)  # sign bit set
    ctx.batch_requests(eff, arr, ids, 128, neg, MEMORIES["analytic"]())
    assert ctx.timings()["dp_mono"] == 0.0


def test_chain_kernel_golden_pools(chain_ctx, orc, golden):
    """The serial-chain kernel (non-monotone models' path) on the same goldens."""
    lat = capi.builtin_latency_model()
    for case in golden["batcher"]:
        if case["n"] > 65536:
            continue
        eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
        res = chain_ctx.batch_requests(eff, arr, ids, case["slice_len"], lat, MEMORIES[case["memory"]]())
        assert res["n_batches"] == case["n_batches"]
        assert sha(res["seg_begin"].astype(np.int32)) == case["seg"]
        assert sha(res["est"].astype(np.float64)) == case["est"]


def test_non_monotone_models_vs_oracle(ctx, orc):
    """Models outside the monotone conditions take the chain kernel; still exact."""
    rng = np.random.default_rng(9)
    lats = [capi.latency_model(2e-6, 1e-3, 5e-5, 0.02, 1e-7, 2e-4, 3e-6, -0.0),
            capi.latency_model(-1e-7, 1e-3, 5e-5, 0.5, 1e-7, 2e-4, 3e-6, 0.02)]
    for lat in lats:
        for n in (100, 5000):
            eff = rng.integers(1, 1500, n).astype(np.int32)
            arr = rng.random(n)
            ids = np.arange(n, dtype=np.int64)
            for mname in ("rule", "analytic"):
                assert_same_batches(ctx.batch_requests(eff, arr, ids, 64, lat, MEMORIES[mname]()),
                                    orc.batch_requests(eff, arr, ids, 64, lat, MEMORIES[mname]()), (n, mname))


def test_decision_kernel_forced_small_windows(ctx, orc, golden):
    """The monotone decision kernel on rule-table pools (windows <= 28) too."""
    ctx.set_dp_kernel(2)
    try:
        lat = capi.builtin_latency_model()
        for case in golden["batcher"]:
            if case["n"] > 65536 or case["memory"] != "rule":
                continue
            eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
            res = ctx.batch_requests(eff, arr, ids, case["slice_len"], lat, MEMORIES["rule"]())
            assert ctx.timings()["dp_mono"] == 1.0
            assert sha(res["seg_begin"].astype(np.int32)) == case["seg"]
            assert sha(res["est"].astype(np.float64)) == case["est"]
    finally:
        ctx.set_dp_kernel(0)


@pytest.mark.gpu
def test_golden_large_pools(ctx, orc):
    """Pools of 2^22 and 2^24 requests (the north star's ">= 1M-request
    pools"): batches and the 8-worker offload vs the reference's fingerprints
    (tests/golden/golden_large.json, make_golden.py --large)."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_large.json")
    lat = capi.builtin_latency_model()
    for case in json.load(open(path))["pools"]:
        eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
        assert sha(eff) + sha(arr) == case["pool"]
        r = ctx.schedule(eff, arr, ids, case["slice_len"], lat, MEMORIES[case["memory"]](),
                         np.arange(8, dtype=np.int32), [0.0] * 8)
        msg = (case["n"], case["memory"])
        assert r["n_batches"] == case["n_batches"], msg
        assert float(planned_total(r["est"])).hex() == case["sum_est"], msg
        assert sha(r["seg_begin"].astype(np.int32)) == case["seg"], msg
        assert sha(r["l_in"].astype(np.int32)) == case["l_in"], msg
        assert sha(r["est"].astype(np.float64)) == case["est"], msg
        assert sha(r["member_id"].astype(np.int64)) == case["member"], msg
        assert sha(r["assign_batch"]) == case["assign_batch"], msg
        assert sha(r["assign_worker"]) == case["assign_worker"], msg
        assert [float(x).hex() for x in r["loads"]] == case["final_loads"], msg


@pytest.mark.gpu
def test_small_pool_path_matches_large_path(ctx, orc):
    """The fused small-pool path (csrc/small.cu, n <= 4096) against the
    multi-kernel path and the C oracle: every size class, all memory models,
    arrival ties, negative ids, an infeasible request."""
    rng = np.random.default_rng(5)
    lat = capi.builtin_latency_model()
    sizes = (1, 2, 3, 31, 32, 33, 100, 460, 1000, 1500, 2048, 4031, 4032, 4033, 4095, 4096)
    for n in sizes:
        eff = rng.integers(1, 2048, n).astype(np.int32)
        arr = np.round(rng.random(n) * 20, 1)  # ties
        ids = rng.permutation(n).astype(np.int64) - n // 3
        for mname in ("rule", "analytic", "tight"):
            mem = MEMORIES[mname]()
            try:
                want = orc.batch_requests(eff, arr, ids, 128, lat, mem)
            except Exception as e:  # infeasible under the tight model
                with pytest.raises(lib_error()) as ei:
                    ctx.batch_requests(eff, arr, ids, 128, lat, mem)
                assert ei.value.request_id == e.request_id, (n, mname)
                continue
            small = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
            ctx.set_batch_path(True)
            try:
                large = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
            finally:
                ctx.set_batch_path(False)
            assert_same_batches(small, want, (n, mname, "small"))
            assert_same_batches(large, want, (n, mname, "large"))
            assert np.array_equal(small["order"], large["order"])
    # the bitonic (n <= 1024) and LSD (above) sorts on full-key ties: few eff
    # values, arrivals that tie (+-0.0 included) and duplicate ids
    mem = MEMORIES["rule"]()
    for n in (2, 16, 500, 1023, 1024, 1025, 3000):
        eff = rng.integers(1, 6, n).astype(np.int32)
        arr = np.round(rng.random(n) * 3, 0)
        arr[::5] = -0.0
        ids = rng.integers(-3, 4, n).astype(np.int64)
        want = orc.batch_requests(eff, arr, ids, 128, lat, mem)
        small = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
        assert_same_batches(small, want, (n, "ties"))
        assert np.array_equal(ids[small["order"]], small["member_id"])


def lib_error():
    from paper_2406_13511_b200.lib import SclsError
    return SclsError


@pytest.mark.parametrize("ctas", [1, 2, 4])
def test_dp_cluster_sizes_bit_exact(ctx, orc, golden, ctas):
    """The monotone DP as one CTA or a 2 / 4-CTA cluster (far candidates over
    DSMEM): the reference's fingerprints on the 2^20 goldens and the oracle on
    pools whose windows exceed a tile (the analytic and tight KV caps)."""
    lat = capi.builtin_latency_model()
    ctx.set_dp_cluster(ctas)
    try:
        for case in golden["batcher"]:
            if case["memory"] == "rule" or case["n"] < 8192:
                continue
            eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
            res = ctx.batch_requests(eff, arr, ids, case["slice_len"], lat, MEMORIES[case["memory"]]())
            msg = (ctas, case["n"], case["slice_len"], case["memory"])
            assert res["n_batches"] == case["n_batches"], msg
            assert sha(res["seg_begin"].astype(np.int32)) == case["seg"], msg
            assert sha(res["est"].astype(np.float64)) == case["est"], msg
        rng = np.random.default_rng(5 + ctas)
        for n in (4097, 9000, 33333):
            eff = rng.integers(1, 3000, n).astype(np.int32)
            arr = rng.random(n) * 50
            ids = rng.permutation(n).astype(np.int64)
            for mname in ("analytic", "tight"):
                a = ctx.batch_requests(eff, arr, ids, 128, lat, MEMORIES[mname]())
                b = orc.batch_requests(eff, arr, ids, 128, lat, MEMORIES[mname]())
                assert_same_batches(a, b, (ctas, n, mname))
    finally:
        ctx.set_dp_cluster(1)


def test_bucket_sort_matches_lsd_sort(ctx, orc):
    """The eff-bucket sort (default for eff ranges <= 2^16) and the LSD radix
    sort (SCLS_OPT_BATCH_PATH 2) give the same batches as the oracle:
    uniform and skewed eff, a bucket above the shared-memory cap (the
    overflow fallback), eff ranges beyond 2^16 (LSD directly), equal and
    +-0.0 arrivals, duplicate and negative ids, buckets whose arrival images
    tie in runs short enough for the in-place fix-up and too long for it."""
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(17)
    cases = []
    n = 50000
    cases.append((rng.integers(1, 1025, n), rng.random(n) * 100, rng.permutation(n)))           # C3-like
    e = rng.integers(1, 1025, n)
    e[: n // 5] = 77                                                                              # 10k in one bucket
    cases.append((e, rng.random(n) * 100, rng.permutation(n)))
    cases.append((rng.integers(1, 200000, n), rng.random(n) * 100, rng.permutation(n)))       # range > 2^16
    a = np.round(rng.random(n) * 10, 1)
    a[::7] = 0.0
    a[1::7] = -0.0
    cases.append((rng.integers(1, 300, n), a, rng.integers(-50, 50, n)))                      # ties, dup ids
    cases.append((rng.integers(1, 100, n), np.full(n, 5.0), rng.permutation(n)))              # one arrival: long runs
    a = np.floor(rng.random(n) * 24) * 0.5
    a[: n // 2] = rng.random(n // 2) * 1e-300                                                  # subnormal spread
    cases.append((rng.integers(1, 60, n), a, rng.permutation(n)))                              # runs of ~35 and short
    for i, (eff, arr, ids) in enumerate(cases):
        eff = eff.astype(np.int32)
        arr = np.asarray(arr, np.float64)
        ids = np.asarray(ids, np.int64)
        want = orc.batch_requests(eff, arr, ids, 128, lat, MEMORIES["rule"]())
        for path in (0, 2):
            ctx.set_batch_path(path)
            try:
                got = ctx.batch_requests(eff, arr, ids, 128, lat, MEMORIES["rule"]())
            finally:
                ctx.set_batch_path(0)
            assert_same_batches(got, want, (i, path))
            assert np.array_equal(ids[got["order"]], got["member_id"])


def test_host_staging_boundary(ctx, orc):
    """Host-memory calls up to 2^16 requests stage through one pinned buffer
    (capi.cu BatchPack), larger ones array by array: both sides of the
    boundary against the oracle, batch_requests and schedule."""
    lat = capi.builtin_latency_model()
    mem = MEMORIES["analytic"]()
    for n in (65535, 65536, 65537):
        eff, arr, ids, _ = orc.make_pool(n, 11)
        want = orc.batch_requests(eff, arr, ids, 128, lat, mem)
        got = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
        assert_same_batches(got, want, n)
        assert np.array_equal(ids[got["order"]], got["member_id"])
        loads = [0.25 * w for w in range(8)]
        s = ctx.schedule(eff, arr, ids, 128, lat, mem, np.arange(8, dtype=np.int32), loads)
        ob, ow, nl = orc.offload(want["batch_id"], want["est"], np.arange(8, dtype=np.int32), loads)
        assert_same_batches(s, want, (n, "schedule"))
        assert np.array_equal(s["assign_batch"], ob) and np.array_equal(s["assign_worker"], ow)
        assert np.array_equal(s["loads"], nl)
