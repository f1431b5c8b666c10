"""Per-policy device time of the C5 sweep shape (4096 traces, rates
10/15/20/25, generated on the device): python tools/probe_policy_sweep.py [traces]"""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
specs = [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=600.0, seed=1000 + i // 4) for i in range(T)]
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    out = {}
    for p in ("scls", "ils", "sls"):
        ts = []
        for _ in range(3):
            ctx.run_sweep(specs, [capi.sched_cfg(policy=p)], lat, mem, hist_bins=16)
            ts.append(ctx.timings()["simulate"])
        out[p] = round(min(ts), 2)
    print(out, "sum", round(sum(out.values()), 2))
