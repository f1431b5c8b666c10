"""Small helpers shared by the tests (fingerprints, random instances)."""
import hashlib

import numpy as np

from paper_2406_13511_b200 import capi


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


MEMORIES = {
    "rule": capi.builtin_memory_model,
    "analytic": capi.builtin_analytic_memory_model,
    "tight": lambda: capi.analytic(5005.0, 3.0, 2.0, 1.0, 1.0),
}


def reference_model():
    """batcher_test.cpp:33-44 reference_model()."""
    return capi.latency_model(2e-6, 1e-3, 5e-5, 0.02, 1e-7, 2e-4, 3e-6, 0.01)


def padding_heavy_model():
    """batcher_test.cpp:48-59."""
    return capi.latency_model(1e-4, 1e-6, 1e-6, 1e-6, 1e-5, 1e-8, 1e-8, 1e-8)


def planned_total(est):
    t = 0.0
    for e in est:
        t += float(e)
    return t


def random_instances(trials=600, seed=20260815, max_n=10):
    """batcher_test.cpp:126-166 style instances: (eff, arrival, ids, slice, mem)."""
    rng = np.random.default_rng(seed)
    tight = MEMORIES["tight"]()
    rule = MEMORIES["rule"]()
    for trial in range(trials):
        n = 1 + int(rng.integers(0, max_n))
        inp = 1 + rng.integers(0, 1399, n)
        gen = np.where(rng.random(n) < 0.3, rng.integers(0, 256, n), 0)
        arr = np.round(rng.random(n) * 10.0, 1)  # rounding creates arrival ties
        ids = rng.permutation(n).astype(np.int64)
        s = 128 if trial % 2 == 0 else 32
        mem = tight if trial % 3 == 0 else rule
        yield (inp + gen).astype(np.int32), arr, ids, s, mem
