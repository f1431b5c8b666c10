"""C3 DP tile-barrier diagnostics (needs a -DSCLS_DP_PROF_ARRIVE -DSCLS_DP_PIPE=0 build):
per tile, how long after the main warp the last warp arrives, who, and the
barrier's release latency."""
import sys

sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib  # noqa: E402

ctx = lib.Context(0)
n = 1 << 20
eff, arr, ids, _ = lib.make_pool(n, 7)
lat, mem = capi.builtin_latency_model(), capi.builtin_analytic_memory_model()
ctx.batch_requests(eff, arr, ids, 128, lat, mem)
ctx.dp_profile(True)
ctx.batch_requests(eff, arr, ids, 128, lat, mem)
p = ctx.dp_profile(True)
tiles = (n + 31) // 32
print("helper-last tiles whose helper scans a top segment: %.1f%%" % (100 * p[6] / max(p[5], 1)))
print("dp ms %.2f main work %.0f, last arrival after main %.0f, release %.0f cycles/tile; last = stager %.1f%% helper %.1f%%"
      % (ctx.timings()["dp"], p[0] / tiles, p[2] / tiles, p[3] / tiles, 100 * p[4] / tiles, 100 * p[5] / tiles))
