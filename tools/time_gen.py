"""Quick timing of device generation and the generate+simulate sweep (C5 shape)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2406_13511_b200 import capi, lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4) for i in range(T)]
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for _ in range(3):
        offs, arr, inp, gen = ctx.generate_batch(specs)
        print("generate_batch", ctx.timings()["generate"], "ms", offs[-1], "requests")
    for _ in range(3):
        t0 = time.perf_counter()
        ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
        t = ctx.timings()
        print("run_sweep wall %.2f ms" % ((time.perf_counter() - t0) * 1e3), {k: round(v, 3) for k, v in t.items()})
