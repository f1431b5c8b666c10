"""Single batch_requests call (for ncu): 64k analytic pool."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
ctx = lib.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
eff, arr, ids, _ = lib.make_pool(n, 7)
r = ctx.batch_requests(eff, arr, ids, 128, capi.builtin_latency_model(), capi.builtin_analytic_memory_model())
print(r["n_batches"], ctx.timings())
