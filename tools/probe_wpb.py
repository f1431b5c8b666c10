import sys, time
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for n in (1, 12, 36):
        specs = [capi.workload_spec(rate=25.0, duration_s=600.0, seed=1000 + i) for i in range(n)]
        cf = [capi.sched_cfg(policy="scls")] * n
        ts = []
        for _ in range(3):
            ctx.run_experiments(specs, cf, lat, mem, hist_bins=16)
            ts.append(ctx.timings()["simulate"])
        print(n, "jobs scls", round(min(ts), 2), "ms", flush=True)
