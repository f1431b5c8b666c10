"""scls_simulate_grid on the C5 sweep: concurrent vs sequential policy launches."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2406_13511_b200 import capi, lib
import bench
ntr = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = lib.Context(0)
ctx.set_digests(False)
traces = bench.gen_traces(list(range(ntr)), 600.0, lib.generate)
offs, arr, inp, gen = bench.flatten(traces)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
for conc in (True, False, True, False):
    ctx.set_concurrent(conc)
    ctx.simulate_grid_flat(offs, arr, inp, gen, cfgs, lat, mem, hist_bins=16)
    print("concurrent" if conc else "sequential", "sim %.1f ms" % ctx.timings()["simulate"], flush=True)
