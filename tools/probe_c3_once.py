"""One C3 schedule call (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2406_13511_b200 import capi, lib
ctx = lib.Context(0)
eff, arr, ids, _ = lib.make_pool(1 << 20, 7)
r = ctx.schedule(eff, arr, ids, 128, capi.builtin_latency_model(), capi.builtin_analytic_memory_model(),
                 np.arange(8, dtype=np.int32), [0.0] * 8)
print(r["n_batches"], ctx.timings())
