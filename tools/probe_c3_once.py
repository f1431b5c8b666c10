"""C3 schedule calls (an ncu target): prints the phase split of the last of
`reps` calls (default 1; warm numbers need reps >= 3)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2406_13511_b200 import capi, lib
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = lib.Context(0)
eff, arr, ids, _ = lib.make_pool(1 << 20, 7)
for _ in range(reps):
    r = ctx.schedule(eff, arr, ids, 128, capi.builtin_latency_model(), capi.builtin_analytic_memory_model(),
                     np.arange(8, dtype=np.int32), [0.0] * 8)
print(r["n_batches"], {k: round(v, 3) for k, v in ctx.timings().items()})
