"""C4 grid in one scls_run_experiments call: phase timings."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
specs, cfgs = [], []
for pol in ("scls", "sls", "ils"):
    for S in (32, 64, 128, 256):
        for G in (256, 512, 1024):
            if S <= G:
                specs.append(capi.workload_spec(rate=20.0, duration_s=5000.0, seed=42, max_gen_limit=G))
                cfgs.append(capi.sched_cfg(policy=pol, slice_len=S, max_gen_limit=G))
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for conc in (True, False):
        ctx.set_concurrent(conc)
        for _ in range(2):
            ctx.run_experiments(specs, cfgs, lat, mem, hist_bins=16)
            print("concurrent", conc, {k: round(v, 2) for k, v in ctx.timings().items()}, flush=True)
