"""Split of one C5 sweep call (device events): generation, simulator setup
(caps, cost tables, arena), the simulator launches, and the rest."""
import sys
import time
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
T = 4096
specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4) for i in range(T)]
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for _ in range(4):
        t0 = time.perf_counter()
        ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
        wall = (time.perf_counter() - t0) * 1e3
        d = ctx.timings()
        print("wall %.1f total %.1f generate %.1f setup %.1f simulate %.1f" %
              (wall, d["total"], d["generate"], d["estimate"], d["simulate"]), flush=True)
