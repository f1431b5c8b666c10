"""ILS / SLS sweep timing at a given worker count (default 1)."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
import bench
W = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ntr = 4096
ctx = lib.Context(0)
ctx.set_digests(False)
traces = bench.gen_traces(list(range(ntr)), 600.0, lib.generate)
offs, arr, inp, gen = bench.flatten(traces)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
for pol in ("ils", "sls"):
    for r in range(2):
        res, hist = ctx.simulate_flat(offs, arr, inp, gen, capi.sched_cfg(policy=pol, worker_count=W), lat, mem, hist_bins=16)
    print(pol, "W", W, "sim %.1f ms" % ctx.timings()["simulate"], "avg_resp_sum %.17g" % sum(x.avg_response_s for x in res),
          set(x.status for x in res), flush=True)
