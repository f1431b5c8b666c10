"""The multi-GPU sweep through the C-ABI (csrc/multi.cu) on the
one GPU of the test box: every shard layout must return the single-device
scls_run_sweep grid word for word.

  - scls_multi with devices [0]: one shard, the NCCL-free path;
  - scls_multi with devices [0, 0] / [0, 0, 0]: world 2 / 3 through the
    C-ABI (uneven contiguous shards, padded blocks, peer-copy gather and the
    job-order reorder -- the same code path NCCL feeds on distinct GPUs);
  - scls_run_sweep_sharded on a context with and without a 1-rank NCCL
    communicator (scls_comm_init): the ncclAllGather itself runs."""
import ctypes as C

import numpy as np
import pytest

from paper_2406_13511_b200 import capi, lib

pytestmark = pytest.mark.gpu


def _specs(n):
    return [capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=40.0, seed=500 + i // 4)
            for i in range(n)]


def _words(res, n):
    return np.frombuffer(C.string_at(C.addressof(res), n * C.sizeof(capi.TraceResult)), np.int64)


@pytest.fixture(scope="module")
def want(ctx):
    specs = _specs(11)
    cfgs = [capi.sched_cfg(policy=p) for p in ("scls", "sls", "ils")]
    ctx.set_digests(False)
    res, hist = ctx.run_sweep(specs, cfgs, capi.builtin_latency_model(), capi.builtin_memory_model(), hist_bins=16)
    ctx.set_digests(True)
    return specs, cfgs, _words(res, 33), hist


@pytest.mark.parametrize("devices", [[0], [0, 0], [0, 0, 0]])
def test_multi_matches_single_device(want, devices):
    specs, cfgs, w_res, w_hist = want
    with lib.Multi(devices) as m:
        assert m.uses_nccl() is False  # one device listed (possibly repeatedly)
        m.set_digests(False)  # as `want`: the sweep reports metrics only
        res, hist, ms = m.run_sweep(specs, cfgs, capi.builtin_latency_model(), capi.builtin_memory_model(),
                                    hist_bins=16)
    assert np.array_equal(_words(res, 33), w_res)
    assert np.array_equal(hist, w_hist)
    assert (ms[:len(devices)] > 0).all() and ms[-1] > 0


def test_sharded_world1_without_and_with_nccl(want):
    specs, cfgs, w_res, w_hist = want
    with lib.Context(0) as c:
        c.set_digests(False)
        res, hist = c.run_sweep_sharded(specs, cfgs, capi.builtin_latency_model(), capi.builtin_memory_model(),
                                        hist_bins=16)
        assert np.array_equal(_words(res, 33), w_res) and np.array_equal(hist, w_hist)
        c.comm_init(1, 0, lib.comm_unique_id())
        assert c.comm_size() == 1
        res, hist = c.run_sweep_sharded(specs, cfgs, capi.builtin_latency_model(), capi.builtin_memory_model(),
                                        hist_bins=16)
        assert np.array_equal(_words(res, 33), w_res) and np.array_equal(hist, w_hist)
        assert c.timings()["simulate"] > 0
