"""Per-phase clock64 breakdown of the SCLS simulator kernel (build with
make -C paper_2406_13511_b200/csrc EXTRA=-DSCLS_SIM_PROF)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
ntr = int(sys.argv[1]) if len(sys.argv) > 1 else 148
rates = [float(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["25"])]
ctx = lib.Context(0)
ctx.set_digests(False)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
traces = [lib.generate(capi.workload_spec(rate=rates[i % len(rates)], duration_s=600.0, seed=1000 + i)) for i in range(ntr)]
res, hist = ctx.simulate(traces, capi.sched_cfg(policy="scls"), lat, mem, hist_bins=16)
print("sim %.1f ms" % ctx.timings()["simulate"])
p = hist[:, 4:16].astype(np.float64).mean(axis=0)
names = ["argmin", "arrivals", "tick: keys", "tick: sort", "tick: rows", "tick: DP", "tick: backtrack+emit",
         "tick: offload", "misc", "tick: interval", "batch done", "-"]
tot = p.sum()
for n, v in zip(names, p):
    print("%-22s %12.0f cycles/trace  %5.1f%%" % (n, v, 100 * v / tot))
print("total %.0f cycles/trace = %.1f ms at 1.965 GHz" % (tot, tot / 1.965e6))
