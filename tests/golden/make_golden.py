"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py          # golden.json
    python tests/golden/make_golden.py --large                        # golden_large.json

Every number here comes from oracle/_ref/libscls_ref.so, i.e. the reference
core compiled from /root/reference/proj/core/src (oracle/Makefile).  The
fixtures pin the C oracle and the CUDA path on machines without the
reference (the GPU box).  Arrays are fingerprinted with sha256 over their
little-endian bytes; scalars are stored exactly (floats as hex).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import RefLib, REF_SO, OracleLib, ORACLE_SO  # noqa: E402
from paper_2406_13511_b200 import capi  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def fx(x):
    return float(x).hex()


MEMORIES = {
    "rule": capi.builtin_memory_model,
    "analytic": capi.builtin_analytic_memory_model,
    "tight": lambda: capi.analytic(5005.0, 3.0, 2.0, 1.0, 1.0),
}


def batcher_cases():
    cases = []
    for n in (1, 2, 7, 16, 100, 1024, 5000, 65536, 1 << 20):
        for slice_len in (32, 128):
            for mname in ("rule", "analytic", "tight"):
                if mname == "tight" and n > 5000:
                    continue
                if n == 1 << 20 and slice_len == 32:
                    continue
                cases.append((n, 7, slice_len, mname))
    return cases


def batch_record(res):
    seg = res["seg_begin"].astype(np.int32)
    total = 0.0
    for e in res["est"]:
        total += float(e)  # planned_total (batcher_test.cpp:120-124), batch order
    return dict(n_batches=int(res["n_batches"]), sum_est=fx(total), sum_est_dec=repr(total),
                seg=sha(seg), l_in=sha(res["l_in"].astype(np.int32)),
                est=sha(res["est"].astype(np.float64)),
                member=sha(res["member_id"].astype(np.int64)))


def sim_record(r, hist):
    d = {}
    for name, _ in capi.TraceResult._fields_:
        v = getattr(r, name)
        d[name] = fx(v) if isinstance(v, float) else int(v)
    d["hist"] = [int(x) for x in hist]
    return d


def main():
    ref = RefLib(REF_SO)
    orc = OracleLib(ORACLE_SO)
    lat = capi.builtin_latency_model()
    out = {"source": "oracle/_ref/libscls_ref.so built from /root/reference/proj/core/src",
           "batcher": [], "offload": [], "simulate": [], "generate": [], "estimators": {}}

    # batcher on the reference microbenchmark pools (bench_batcher.cpp:27-42)
    for n, seed, slice_len, mname in batcher_cases():
        eff, arr, ids, _ = orc.make_pool(n, seed)
        res = ref.batch_requests(eff, arr, ids, slice_len, lat, MEMORIES[mname]())
        rec = dict(n=n, seed=seed, slice_len=slice_len, memory=mname, pool=sha(eff) + sha(arr))
        rec.update(batch_record(res))
        out["batcher"].append(rec)
        print("batcher", n, slice_len, mname, rec["n_batches"], rec["sum_est_dec"], flush=True)

    # offload: the batches of a few pools onto 8 workers at load 0, and with
    # staggered initial loads
    for n, mname in ((1024, "rule"), (65536, "analytic"), (1 << 20, "rule")):
        eff, arr, ids, _ = orc.make_pool(n, 7)
        res = ref.batch_requests(eff, arr, ids, 128, lat, MEMORIES[mname]())
        for loads in ([0.0] * 8, [float(w) * 0.5 for w in range(8)]):
            ob, ow, nl = ref.offload(res["batch_id"], res["est"], np.arange(8, dtype=np.int32), loads)
            out["offload"].append(dict(n=n, memory=mname, loads=[fx(x) for x in loads],
                                       batch=sha(ob), worker=sha(ow),
                                       final_loads=[fx(x) for x in nl]))

    # generate (workload.cpp:163-181)
    for rate, dur, seed in ((20.0, 600.0, 42), (2.0, 500.0, 42), (25.0, 600.0, 1003)):
        spec = capi.workload_spec(rate=rate, duration_s=dur, seed=seed)
        a, i, g = ref.generate(spec)
        out["generate"].append(dict(rate=rate, duration_s=dur, seed=seed, n=len(a),
                                    arrival=sha(a), input_len=sha(i), gen_len=sha(g)))

    # simulate: SURVEY Appendix B runs plus sweeps over policies / slices
    runs = [("C1", "scls", 2.0, 500.0, 1, 128, 1024, 42, "rule"),
            ("C2", "scls", 20.0, 500.0, 8, 128, 1024, 42, "rule"),
            ("defaults-scls", "scls", 20.0, 600.0, 8, 128, 1024, 42, "rule"),
            ("defaults-sls", "sls", 20.0, 600.0, 8, 128, 1024, 42, "rule"),
            ("defaults-ils", "ils", 20.0, 600.0, 8, 128, 1024, 42, "rule")]
    for pol in ("scls", "sls", "ils"):
        for s, mg in ((32, 256), (64, 512), (256, 1024)):
            runs.append((f"{pol}-s{s}-mg{mg}", pol, 15.0, 120.0, 4, s, mg, 1001, "rule"))
        runs.append((f"{pol}-analytic", pol, 20.0, 120.0, 8, 128, 1024, 1002, "analytic"))
    for name, pol, rate, dur, w, s, mg, seed, mname in runs:
        spec = capi.workload_spec(rate=rate, duration_s=dur, seed=seed, max_gen_limit=1024)
        trace = ref.generate(spec)
        cfg = capi.sched_cfg(policy=pol, worker_count=w, slice_len=s, max_gen_limit=mg)
        res, hist = ref.simulate([trace], cfg, lat, MEMORIES[mname]())
        rec = dict(name=name, policy=pol, rate=rate, duration_s=dur, workers=w, slice_len=s,
                   max_gen_limit=mg, seed=seed, memory=mname)
        rec.update(sim_record(res[0], hist[0]))
        out["simulate"].append(rec)
        print("simulate", name, res[0].status, res[0].completed, flush=True)

    # estimator grids
    grid = []
    for n in (1, 2, 12, 28, 64, 443):
        for L in (1, 100, 511, 1024, 2047):
            for lo in (0, 1, 32, 128, 1024):
                grid.append(fx(ref.batch_serve_time(lat, n, L, lo)))
    out["estimators"]["batch_serve_time"] = grid
    mbs = {}
    for mname in MEMORIES:
        mbs[mname] = [ref.max_batch_size(MEMORIES[mname](), L, s)
                      for L in (1, 2, 50, 100, 511, 512, 1000, 1024, 2000, 4000) for s in (1, 32, 128)]
    out["estimators"]["max_batch_size"] = mbs

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


def main_large():
    """C3-style pools beyond 2^20 (bench_batcher.cpp make_pool, seed 7, S = 128):
    n = 2^22 and 2^24 under the analytic KV cap and the rule table, batches
    fingerprinted, then offloaded onto 8 workers at load 0."""
    ref = RefLib(REF_SO)
    orc = OracleLib(ORACLE_SO)
    lat = capi.builtin_latency_model()
    out = {"source": "oracle/_ref/libscls_ref.so built from /root/reference/proj/core/src",
           "pools": []}
    for n in (1 << 22, 1 << 24):
        eff, arr, ids, _ = orc.make_pool(n, 7)
        for mname in ("analytic", "rule"):
            res = ref.batch_requests(eff, arr, ids, 128, lat, MEMORIES[mname]())
            rec = dict(n=n, seed=7, slice_len=128, memory=mname, pool=sha(eff) + sha(arr))
            rec.update(batch_record(res))
            ob, ow, nl = ref.offload(res["batch_id"], res["est"], np.arange(8, dtype=np.int32), [0.0] * 8)
            rec.update(assign_batch=sha(ob), assign_worker=sha(ow), final_loads=[fx(x) for x in nl])
            out["pools"].append(rec)
            print("large", n, mname, rec["n_batches"], rec["sum_est_dec"], flush=True)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_large.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    if "--large" in sys.argv:
        main_large()
    else:
        main()
