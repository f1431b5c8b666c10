"""C4 (one 5000 s trace, ~100k requests) per job: device ms of each policy x
slice x max_gen configuration run alone, next to the CPU reference."""
import sys, time
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
from oracle.pyoracle import RefLib, REF_SO
ref = RefLib(REF_SO)
lat, mem = capi.builtin_latency_model(), capi.builtin_memory_model()
with lib.Context(0) as ctx:
    ctx.set_digests(False)
    for pol in ("scls", "sls", "ils"):
        for S in (32, 64, 128, 256):
            for G in (256, 512, 1024):
                if S > G:
                    continue
                sp = capi.workload_spec(rate=20.0, duration_s=5000.0, seed=42, max_gen_limit=G)
                cf = capi.sched_cfg(policy=pol, slice_len=S, max_gen_limit=G)
                ts = []
                for _ in range(2):
                    ctx.run_experiments([sp], [cf], lat, mem, hist_bins=16)
                    ts.append(ctx.timings()["simulate"])
                tr = ref.generate(sp)
                t0 = time.perf_counter()
                ref.simulate([tr], cf, lat, mem)
                cpu = (time.perf_counter() - t0) * 1e3
                print(f"{pol:4s} S={S:3d} G={G:4d}  device {min(ts):8.2f} ms   cpu {cpu:8.1f} ms", flush=True)
