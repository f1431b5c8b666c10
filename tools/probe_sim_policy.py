"""Per-policy simulate time at sweep scale (device-resident inputs)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
import bench
ntr = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
pols = sys.argv[2].split(",") if len(sys.argv) > 2 else ["scls", "sls", "ils"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
ctx = lib.Context(0)
ctx.set_digests(False)
traces = bench.gen_traces(list(range(ntr)), 600.0, lib.generate)
offs, arr, inp, gen = bench.flatten(traces)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
for pol in pols:
    for r in range(reps):
        res, hist = ctx.simulate_flat(offs, arr, inp, gen, capi.sched_cfg(policy=pol), lat, mem, hist_bins=16)
        print(pol, ntr, "sim %.1f ms total %.1f ms -> %.0f traces/s" % (ctx.timings()["simulate"], ctx.timings()["total"], ntr / ctx.timings()["simulate"] * 1e3), set(x.status for x in res), flush=True)
