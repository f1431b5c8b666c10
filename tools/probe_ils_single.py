"""One rate-25 trace per SM (148 traces): the ILS kernel's per-trace latency."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
pol = sys.argv[1] if len(sys.argv) > 1 else "ils"
ntr = int(sys.argv[2]) if len(sys.argv) > 2 else 148
ctx = lib.Context(0)
ctx.set_digests(False)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
traces = [lib.generate(capi.workload_spec(rate=25.0, duration_s=600.0, seed=1000 + i)) for i in range(ntr)]
ctx.simulate(traces, capi.sched_cfg(policy=pol), lat, mem, hist_bins=16)
print(pol, ntr, "sim %.1f ms" % ctx.timings()["simulate"])
