import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
T = 4096
specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4) for i in range(T)]
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for conc in (False, True):
        ctx.set_concurrent(conc)
        ts = []
        for _ in range(4):
            ctx.run_sweep(specs, cfgs, lat, mem, hist_bins=16)
            ts.append(ctx.timings()["total"])
        print("concurrent", conc, "total ms", [round(x, 1) for x in ts])
