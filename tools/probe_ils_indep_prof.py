"""Per-phase clock64 breakdown of the independent-lane ILS kernel.  Build:
  make -C paper_2406_13511_b200/csrc EXTRA=-DSCLS_ILS_PROF OUT=$PWD/build/prof/libscls_b200.so OBJDIR=$PWD/build/prof/obj
then run with SCLS_B200_LIB=build/prof/libscls_b200.so."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
ntr = int(sys.argv[1]) if len(sys.argv) > 1 else 148
rate = float(sys.argv[2]) if len(sys.argv) > 2 else 25.0
ctx = lib.Context(0)
ctx.set_digests(False)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
specs = [capi.workload_spec(rate=rate, duration_s=600.0, seed=1000 + i) for i in range(ntr)]
for _ in range(2):
    res, hist = ctx.run_sweep(specs, [capi.sched_cfg(policy="ils")], lat, mem, hist_bins=16)
print("sim %.2f ms" % ctx.timings()["simulate"])
h = hist[0][:, 4:8].astype(np.float64)
for name, col in zip(["phase1 (instances)", "merge", "finish_report"], range(3)):
    print("%-20s mean %10.0f  max %10.0f cycles" % (name, h[:, col].mean(), h[:, col].max()))
print("completions/trace mean %.0f" % h[:, 3].mean())
c = hist[0][:, 8:15].astype(np.float64).mean(axis=0)
print("lane 0: fast steps %.0f, slow boundaries %.0f, arrivals %.0f, outer iterations %.0f" % tuple(c[:4]))
print("lane 0 cycles: fast %.0f (%.0f/step)  arrival %.0f (%.0f each)  slow %.0f (%.0f each)" %
      (c[4], c[4] / max(c[0], 1), c[5], c[5] / max(c[2], 1), c[6], c[6] / max(c[1], 1)))
x = hist[0][:, 15].astype(np.int64)
print("warp fast-loop trips %.0f, warp outer iterations %.0f" % ((x >> 32).mean(), (x & 0xffffffff).mean()))
