"""DP kernel phase profile (clock64 counters) on the C3 pools."""
import sys

sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib  # noqa: E402

ctx = lib.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
eff, arr, ids, _ = lib.make_pool(n, 7)
lat = capi.builtin_latency_model()
for name, mem in (("analytic", capi.builtin_analytic_memory_model()), ("rule", capi.builtin_memory_model())):
    ctx.batch_requests(eff, arr, ids, 128, lat, mem)
    ctx.dp_profile(True)
    r = ctx.batch_requests(eff, arr, ids, 128, lat, mem)
    p = ctx.dp_profile(True)
    tiles = (n + 31) // 32
    nh = max(int(p[5]), 1)
    print(name, r["n_batches"], "dp ms %.2f" % ctx.timings()["dp"],
          "per tile cycles: main %.0f (mid %.0f, rounds/tile %.2f) wait %.0f | helper stage %.0f far %.0f wait %.0f" % (
              p[0] / tiles, p[6] / tiles, p[7] / tiles, p[1] / tiles, p[2] / tiles / nh, p[3] / tiles / nh,
              p[4] / tiles / nh))
ctx.dp_profile(False)
eff, arr, ids, _ = lib.make_pool(n, 7)
for ctas in (1, 2, 4):
    ctx.set_dp_cluster(ctas)
    ts = []
    for _ in range(3):
        r = ctx.batch_requests(eff, arr, ids, 128, lat, capi.builtin_analytic_memory_model())
        ts.append(ctx.timings()["dp"])
    print("analytic dp cluster", ctas, "ms", [round(x, 2) for x in ts], r["n_batches"])
ctx.set_dp_cluster(1)
r = ctx.batch_requests(eff, arr, ids, 128, lat, capi.builtin_memory_model())
print("unprofiled rule dp ms %.2f" % ctx.timings()["dp"])
