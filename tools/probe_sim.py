"""C5-style sweep probe: N traces (600 s, rates 10..25, 8 workers) x policy."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
from oracle.pyoracle import oracle_lib
ntr = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = lib.Context(0)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
traces = [lib.generate(capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4)) for i in range(ntr)]
nreq = sum(len(t[0]) for t in traces)
for pol in ("scls", "sls", "ils"):
    cfg = capi.sched_cfg(policy=pol)
    for dig in (True, False):
        ctx.set_digests(dig)
        t0 = time.time(); res, hist = ctx.simulate(traces, cfg, lat, mem); wall = time.time() - t0
        st = set(r.status for r in res)
        print(pol, "digests" if dig else "metrics", "traces %d reqs %d status %s wall %.1f ms sim %.1f ms -> %.1f traces/s" % (
            ntr, nreq, st, wall * 1e3, ctx.timings()["simulate"], ntr / (ctx.timings()["simulate"] / 1e3)), flush=True)
    ctx.set_digests(True)
    res, hist = ctx.simulate(traces[:8], cfg, lat, mem)
    k = min(ntr, 8)
    ref = oracle_lib().simulate(traces[:k], cfg, lat, mem)[0]
    bad = sum(1 for i in range(k) for f, _ in capi.TraceResult._fields_ if f != "sim_clock" and getattr(res[i], f) != getattr(ref[i], f))
    print(pol, "oracle mismatches on first %d traces: %d" % (k, bad))
