"""Device-time probes used while tuning kernels (diagnostics, not tests):

  python tools/probe.py sweep [traces]     per-policy kernel ms of the C5 sweep shape
  python tools/probe.py scls-dp [traces]   SCLS kernel ms per tick-DP mode (auto / chain)
  python tools/probe.py one <policy> [traces] one device-generated sweep of one policy (ncu target)
  python tools/probe.py c4                 every C4 job alone, device ms next to the reference (1 thread)
  python tools/probe.py step [traces]      the 3-policy C5 step (simulate phase), 5 reps
  python tools/probe.py scls-prof [traces] [rates]
                                           per-phase clock64 split of the SCLS kernel
                                           (needs SCLS_B200_LIB = a -DSCLS_SIM_PROF build)
"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib  # noqa: E402

LAT, MEM = capi.builtin_latency_model(), capi.builtin_memory_model()


def specs(T, rates=(10.0, 15.0, 20.0, 25.0)):
    return [capi.workload_spec(rate=rates[i % len(rates)], duration_s=600.0, seed=1000 + i // len(rates))
            for i in range(T)]


def kernel_ms(ctx, sp, cfg, reps=3):
    ts = []
    for _ in range(reps):
        ctx.run_sweep(sp, [cfg], LAT, MEM, hist_bins=16)
        ts.append(ctx.timings()["simulate"])
    return round(min(ts), 2)


def main():
    cmd = sys.argv[1] if len(sys.argv) > 1 else "sweep"
    T = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 4096
    with lib.Context(0) as ctx:
        ctx.set_digests(False)
        if cmd == "sweep":
            out = {p: kernel_ms(ctx, specs(T), capi.sched_cfg(policy=p)) for p in ("scls", "ils", "sls")}
            print(out, "sum", round(sum(out.values()), 2))
        elif cmd == "step":  # the 3-policy C5 step (simulate only, device-generated traces), 5 reps
            sp = specs(T)
            cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
            ts = []
            for _ in range(5):
                ctx.run_sweep(sp, cfgs, LAT, MEM, hist_bins=16)
                ts.append(ctx.timings()["simulate"])
            print("step simulate ms", [round(t, 2) for t in ts], "median %.2f" % sorted(ts)[2])
        elif cmd == "pairs":  # which policy bounds the concurrent step: every subset's simulate ms
            sp = specs(T)
            for pols in (("scls", "sls", "ils"), ("scls", "sls"), ("scls", "ils"), ("sls", "ils"), ("scls",), ("ils",)):
                cfgs = [capi.sched_cfg(policy=p) for p in pols]
                ts = []
                for _ in range(3):
                    ctx.run_sweep(sp, cfgs, LAT, MEM, hist_bins=16)
                    ts.append(ctx.timings()["simulate"])
                print(pols, "%.2f" % min(ts))
        elif cmd == "scls-dp":
            for mode in (0, 1):
                ctx.set_dp_kernel(mode)
                print("dp mode", mode, "sweep", kernel_ms(ctx, specs(T), capi.sched_cfg()),
                      "one rate-25 trace", kernel_ms(ctx, specs(1, (25.0,)), capi.sched_cfg()))
        elif cmd == "ils":  # SCLS_OPT_ILS_KERNEL 0 (split) vs 2 (one kernel): ILS / SLS alone and the step
            sp = specs(T)
            cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
            for mode in (0, 2, 0, 2):
                ctx.set_ils_kernel(mode)
                r_ils = kernel_ms(ctx, sp, capi.sched_cfg(policy="ils"))
                r_sls = kernel_ms(ctx, sp, capi.sched_cfg(policy="sls"))
                ts = []
                for _ in range(2):
                    ctx.run_sweep(sp, cfgs, LAT, MEM, hist_bins=16)
                    ts.append(ctx.timings()["simulate"])
                print("mode", mode, "ils alone", r_ils, "sls alone", r_sls, "step", [round(t, 2) for t in ts])
            ctx.set_ils_kernel(0)
        elif cmd == "c4":  # every C4 job alone: device ms (and the compiled reference, 1 thread)
            from oracle.pyoracle import ref_lib
            ref = ref_lib()
            import time
            for pol in ("scls", "sls", "ils"):
                for S in (32, 64, 128, 256):
                    for G in (256, 512, 1024):
                        if S > G:
                            continue
                        sp = capi.workload_spec(rate=20.0, duration_s=5000.0, seed=42, max_gen_limit=G)
                        cfg = capi.sched_cfg(policy=pol, slice_len=S, max_gen_limit=G)
                        ts = []
                        for _ in range(2):
                            ctx.run_experiments([sp], [cfg], LAT, MEM, hist_bins=16)
                            ts.append(ctx.timings()["total"])
                        cpu = None
                        if ref is not None:
                            tr = [ref.generate(sp)]
                            t0 = time.perf_counter()
                            ref.simulate(tr, [cfg], LAT, MEM, cfg_index=[0], hist_bins=16)
                            cpu = (time.perf_counter() - t0) * 1e3
                        print(pol, S, G, "device ms %.1f" % min(ts), "cpu ms %.1f" % cpu if cpu else "")
        elif cmd == "one":
            T = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
            ctx.run_sweep(specs(T), [capi.sched_cfg(policy=sys.argv[2])], LAT, MEM, hist_bins=16)
            print(sys.argv[2], "%.2f ms" % ctx.timings()["simulate"])
        elif cmd == "scls-prof":
            rates = [float(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["25"])]
            res, hist = ctx.run_sweep(specs(T, rates), [capi.sched_cfg()], LAT, MEM, hist_bins=16)
            print("sim %.1f ms" % ctx.timings()["simulate"])
            p = hist[0, :, 4:16].astype(np.float64).mean(axis=0)
            names = ["argmin", "arrivals", "tick: keys", "tick: sort", "tick: rows", "tick: DP",
                     "tick: backtrack+emit", "tick: offload", "misc", "tick: interval", "batch done",
                     "tick: DP setup+far"]
            tot = p.sum()
            for n, v in zip(names, p):
                print("%-22s %12.0f cycles/trace  %5.1f%%" % (n, v, 100 * v / tot))
            print("total %.0f cycles/trace = %.1f ms at 1.965 GHz" % (tot, tot / 1.965e6))


if __name__ == "__main__":
    main()
