import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2406_13511_b200 import capi, lib
ctx = lib.Context(0)
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
for n in (16, 1024, 4096):
    eff, arr, ids, _ = lib.make_pool(n, 7)
    ts = []; dv = []
    for _ in range(30):
        t0 = time.perf_counter(); r = ctx.batch_requests(eff, arr, ids, 128, lat, mem); ts.append(time.perf_counter() - t0)
        dv.append(ctx.timings()["total"])
    print(n, "e2e_us", round(np.median(ts) * 1e6, 1), "dev_us", round(np.median(dv) * 1e3, 1), ctx.timings())
