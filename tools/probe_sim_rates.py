"""Per-rate simulate time: is a policy kernel latency-bound per trace
(time ~ flat in trace count) or throughput-bound (time ~ trace count)?
Traces are generated on the device (scls_run_sweep)."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
pols = sys.argv[1:] or ["ils", "scls", "sls"]
ctx = lib.Context(0)
ctx.set_digests(False)
lat = capi.builtin_latency_model(); mem = capi.builtin_memory_model()
for pol in pols:
    for rate in (10.0, 15.0, 20.0, 25.0):
        for ntr in (1, 148, 1024, 4096):
            specs = [capi.workload_spec(rate=rate, duration_s=600.0, seed=1000 + i) for i in range(ntr)]
            ts = []
            for _ in range(2):
                ctx.run_sweep(specs, [capi.sched_cfg(policy=pol)], lat, mem, hist_bins=16)
                ts.append(ctx.timings()["simulate"])
            print(pol, "rate", rate, "traces", ntr, "sim %.2f ms" % min(ts), flush=True)
