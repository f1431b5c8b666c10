"""Pin the checker: the C restatement (oracle/scls_oracle.c) against the
committed golden fixtures (generated from the unmodified reference by
tests/golden/make_golden.py) and, where the reference build exists, against
the reference itself on fresh random inputs.  CPU only."""
import itertools

import numpy as np
import pytest

from paper_2406_13511_b200 import capi
from tests.helpers import (MEMORIES, padding_heavy_model, planned_total, random_instances,
                           reference_model, sha)


def _batch_fingerprint(res):
    return dict(n_batches=int(res["n_batches"]), sum_est=float(planned_total(res["est"])).hex(),
                seg=sha(res["seg_begin"].astype(np.int32)), l_in=sha(res["l_in"].astype(np.int32)),
                est=sha(res["est"].astype(np.float64)), member=sha(res["member_id"].astype(np.int64)))


def test_oracle_batcher_matches_golden(orc, golden):
    lat = capi.builtin_latency_model()
    for case in golden["batcher"]:
        eff, arr, ids, _ = orc.make_pool(case["n"], case["seed"])
        res = orc.batch_requests(eff, arr, ids, case["slice_len"], lat, MEMORIES[case["memory"]]())
        fp = _batch_fingerprint(res)
        for k, v in fp.items():
            assert v == case[k], (case["n"], case["slice_len"], case["memory"], k)


def test_survey_c3_goldens(golden):
    """the 1M-pool totals."""
    c3 = {(c["memory"], c["slice_len"]): c for c in golden["batcher"] if c["n"] == 1 << 20}
    assert c3[("analytic", 128)]["n_batches"] == 11820
    assert c3[("analytic", 128)]["sum_est_dec"] == "70831.31070040006"
    assert c3[("rule", 128)]["n_batches"] == 48802
    assert c3[("rule", 128)]["sum_est_dec"] == "176179.4680023956"


def test_oracle_simulate_matches_golden(orc, golden):
    lat = capi.builtin_latency_model()
    for run in golden["simulate"]:
        spec = capi.workload_spec(rate=run["rate"], duration_s=run["duration_s"], seed=run["seed"])
        trace = orc.generate(spec)
        cfg = capi.sched_cfg(policy=run["policy"], worker_count=run["workers"],
                             slice_len=run["slice_len"], max_gen_limit=run["max_gen_limit"])
        res, hist = orc.simulate([trace], cfg, lat, MEMORIES[run["memory"]]())
        for name, _ in capi.TraceResult._fields_:
            v = getattr(res[0], name)
            want = run[name]
            got = float(v).hex() if isinstance(v, float) else int(v)
            assert got == want, (run["name"], name)
        assert [int(x) for x in hist[0]] == run["hist"], run["name"]


def test_appendix_b_digests(golden):
    """SURVEY Appendix B hashes, restated from the survey text."""
    want = {"C1": ("d67eadb1564cf8ae", "ba7b871703f6feed", "ebfd446318ea1381"),
            "C2": ("f159746c84c8b282", "30c6c2156bfcb5c1", "927be780954435c4"),
            "defaults-scls": ("0af787c41608bfc9", "4a354d341c5bbf88", "a0165b0b5da14e03"),
            "defaults-sls": ("f2e9442cb5b918e9", "4c2a96a756eee1f5", "fd23fa361170a781"),
            "defaults-ils": ("b13ae330bfe0cca9", "91779f7cc9faf291", "57c9640f531eafe2")}
    runs = {r["name"]: r for r in golden["simulate"]}
    for name, (hc, hd, ht) in want.items():
        r = runs[name]
        assert "%016x" % r["h_complete_ids"] == hc
        assert "%016x" % r["h_dispatch"] == hd
        assert "%016x" % r["h_complete_t"] == ht


def test_oracle_generate_matches_golden(orc, golden):
    for g in golden["generate"]:
        a, i, gl = orc.generate(capi.workload_spec(rate=g["rate"], duration_s=g["duration_s"],
                                                   seed=g["seed"]))
        assert len(a) == g["n"]
        assert sha(a) == g["arrival"] and sha(i) == g["input_len"] and sha(gl) == g["gen_len"]


def test_oracle_offload_matches_golden(orc, golden):
    lat = capi.builtin_latency_model()
    for case in golden["offload"]:
        eff, arr, ids, _ = orc.make_pool(case["n"], 7)
        res = orc.batch_requests(eff, arr, ids, 128, lat, MEMORIES[case["memory"]]())
        loads = [float.fromhex(x) for x in case["loads"]]
        ob, ow, nl = orc.offload(res["batch_id"], res["est"], np.arange(8, dtype=np.int32), loads)
        assert sha(ob) == case["batch"] and sha(ow) == case["worker"]
        assert [float(x).hex() for x in nl] == case["final_loads"]


def test_oracle_estimators_match_golden(orc, golden):
    lat = capi.builtin_latency_model()
    it = iter(golden["estimators"]["batch_serve_time"])
    for n in (1, 2, 12, 28, 64, 443):
        for L in (1, 100, 511, 1024, 2047):
            for lo in (0, 1, 32, 128, 1024):
                assert float(orc.batch_serve_time(lat, n, L, lo)).hex() == next(it)
    for mname, vals in golden["estimators"]["max_batch_size"].items():
        got = [orc.max_batch_size(MEMORIES[mname](), L, s)
               for L in (1, 2, 50, 100, 511, 512, 1000, 1024, 2000, 4000) for s in (1, 32, 128)]
        assert got == vals, mname


def test_offload_hand_fixture(orc):
    """offloader_test.cpp:48-63: {10,6,6,2} onto two idle workers."""
    ob, ow, nl = orc.offload([0, 1, 2, 3], [6.0, 10.0, 2.0, 6.0], [0, 1], [0.0, 0.0])
    assert list(zip(ob.tolist(), ow.tolist())) == [(1, 0), (0, 1), (3, 1), (2, 0)]
    assert nl.tolist() == [12.0, 12.0]


def test_memory_alg2_exhaustive(orc, ref):
    """memory_model_test.cpp:72-86: would_oom / max_batch_size over the table."""
    for mem in (MEMORIES["rule"](), MEMORIES["analytic"](), MEMORIES["tight"]()):
        for L in range(1, 2049, 7):
            for s in (1, 32, 128):
                assert orc.max_batch_size(mem, L, s) == ref.max_batch_size(mem, L, s)
                for n in (1, 2, 11, 12, 13, 27, 28, 29, 48, 49, 50, 64, 442, 443, 444):
                    assert orc.would_oom(mem, n, L, s) == ref.would_oom(mem, n, L, s)


def test_oracle_vs_ref_random_batches(orc, ref):
    """batcher_test.cpp:126-166 style random instances, both checkers."""
    lat = reference_model()
    for eff, arr, ids, s, mem in random_instances(trials=300):
        a = orc.batch_requests(eff, arr, ids, s, lat, mem, 5)
        b = ref.batch_requests(eff, arr, ids, s, lat, mem, 5)
        for k in ("seg_begin", "l_in", "est", "batch_id", "member_id"):
            assert np.array_equal(a[k], b[k]), k


def test_brute_force_optimality(orc):
    """batcher_test.cpp:92-118: the DP total equals the exhaustive minimum,
    bit for bit (same arithmetic, same accumulation order)."""
    lat = reference_model()
    for eff, arr, ids, s, mem in random_instances(trials=120, seed=7, max_n=8):
        res = orc.batch_requests(eff, arr, ids, s, lat, mem)
        order = sorted(range(len(eff)), key=lambda i: (int(eff[i]), float(arr[i]), int(ids[i])))
        L = [int(eff[i]) for i in order]
        n = len(L)
        best = float("inf")
        for mask in range(1 << (n - 1)):
            total, start, ok = 0.0, 0, True
            for i in range(n):
                if i == n - 1 or (mask >> i) & 1:
                    cnt = i - start + 1
                    if orc.would_oom(mem, cnt, L[i], s):
                        ok = False
                        break
                    total += orc.batch_serve_time(lat, cnt, L[i], s)
                    start = i + 1
            if ok and total < best:
                best = total
        assert planned_total(res["est"]) == best


def test_batcher_known_answers(orc):
    """batcher_test.cpp:168-275 fixtures."""
    rule = MEMORIES["rule"]()
    # TiesPreferTheSmallerTrailingBatch: flat model, two requests -> two singletons
    flat = capi.latency_model(p2=1.0)
    r = orc.batch_requests([100, 100], [0.0, 0.0], [0, 1], 128, flat, rule)
    assert r["n_batches"] == 2
    # IsolatesLongOutlierWhenPaddingDominates
    r = orc.batch_requests([10] * 8 + [1024], [0.0] * 9, list(range(9)), 128,
                           padding_heavy_model(), rule)
    assert r["n_batches"] == 2 and r["member_id"][-1] == 8 and r["l_in"].tolist() == [10, 1024]
    # SegmentsFollowSortedEffectiveInputOrder
    r = orc.batch_requests([600, 600, 10, 10], [2.0, 1.0, 3.0, 0.5], [3, 1, 2, 0], 128,
                           padding_heavy_model(), rule)
    assert r["member_id"].tolist() == [0, 2, 1, 3] and r["seg_begin"].tolist() == [0, 2, 4]
    # ThrowsWhenASingletonCannotFit
    from oracle.pyoracle import CheckerError
    with pytest.raises(CheckerError) as e:
        orc.batch_requests([200], [0.0], [7], 10, reference_model(), capi.analytic(105.0, 3.0, 2.0, 1.0, 1.0))
    assert e.value.status == capi.ERR_INFEASIBLE_REQUEST and e.value.request_id == 7


def test_oracle_vs_ref_random_sims(orc, ref):
    lat = capi.builtin_latency_model()
    rng = np.random.default_rng(3)
    for trial, (pol, mname) in enumerate(itertools.product(("scls", "sls", "ils"),
                                                           ("rule", "analytic", "tight"))):
        spec = capi.workload_spec(rate=float(rng.uniform(5, 30)), duration_s=30.0, seed=100 + trial)
        trace = ref.generate(spec)
        cfg = capi.sched_cfg(policy=pol, worker_count=int(rng.integers(1, 9)),
                             slice_len=int(rng.choice([16, 64, 128])), max_gen_limit=512,
                             fixed_batch_size=int(rng.integers(1, 16)),
                             max_concurrent=int(rng.integers(1, 16)))
        a, ha = orc.simulate([trace], cfg, lat, MEMORIES[mname]())
        b, hb = ref.simulate([trace], cfg, lat, MEMORIES[mname]())
        for name, _ in capi.TraceResult._fields_:
            assert getattr(a[0], name) == getattr(b[0], name), (pol, mname, name)
        assert np.array_equal(ha, hb)


def test_error_paths_match_ref(orc, ref):
    lat = capi.builtin_latency_model()
    # horizon shorter than the run -> NonTerminationError (sim_engine_test.cpp:176-181)
    trace = ref.generate(capi.workload_spec(rate=20.0, duration_s=10.0))
    cfg = capi.sched_cfg(worker_count=1, horizon_s=0.5)
    for chk in (orc, ref):
        res, _ = chk.simulate([trace], cfg, lat, MEMORIES["rule"]())
        assert res[0].status == capi.ERR_NON_TERMINATION
    # empty workload -> EmptyLogError from compute (metrics.cpp:31)
    for chk in (orc, ref):
        res, _ = chk.simulate([(np.zeros(0), np.zeros(0, np.int32), np.zeros(0, np.int32))],
                              capi.sched_cfg(), lat, MEMORIES["rule"]())
        assert res[0].status == capi.ERR_EMPTY_LOG
    # arrivals out of order -> Error (sim_engine.cpp:110-114)
    for chk in (orc, ref):
        res, _ = chk.simulate([(np.array([1.0, 0.5]), np.array([10, 10], np.int32),
                                np.array([10, 10], np.int32))], capi.sched_cfg(), lat,
                              MEMORIES["rule"]())
        assert res[0].status == 1
    # invalid config -> Error
    for chk in (orc, ref):
        res, _ = chk.simulate([trace], capi.sched_cfg(worker_count=0), lat, MEMORIES["rule"]())
        assert res[0].status == 1
