"""C3 rule-table batch_requests (dp_chain_kernel), an ncu target."""
import sys
sys.path.insert(0, ".")
from paper_2406_13511_b200 import capi, lib
ctx = lib.Context(0)
eff, arr, ids, _ = lib.make_pool(1 << 20, 7)
r = ctx.batch_requests(eff, arr, ids, 128, capi.builtin_latency_model(), capi.builtin_memory_model())
print(r["n_batches"], {k: round(v, 3) for k, v in ctx.timings().items()})
