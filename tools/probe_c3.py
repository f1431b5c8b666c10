"""Quick C3 probe: 1M-pool batch_requests + offload timings (device phases)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib

ctx = lib.Context(0)
eff, arr, ids, _ = lib.make_pool(1 << 20, 7)
lat = capi.builtin_latency_model()
for name, mem in (("analytic", capi.builtin_analytic_memory_model()), ("rule", capi.builtin_memory_model())):
    for rep in range(3):
        t = time.time()
        r = ctx.schedule(eff, arr, ids, 128, lat, mem, np.arange(8, dtype=np.int32), [0.0] * 8)
        wall = time.time() - t
        tot = 0.0
        for e in r["est"]:
            tot += float(e)
        print(name, r["n_batches"], repr(tot), "wall %.2f ms" % (wall * 1e3),
              {k: round(v, 3) for k, v in ctx.timings().items()}, "launches", ctx.launches(), flush=True)
