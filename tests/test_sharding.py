"""The N>1 path of the sweep on CPU: world size 2 over gloo.  Each rank
simulates its contiguous shard (the C oracle stands in for the GPU here, as
the checker) and the records are all-gathered; the result must equal the
single-process run of the whole sweep, in global trace order."""
import os
import socket

import numpy as np
import pytest

from paper_2406_13511_b200 import capi, sweep


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _traces(total):
    from oracle.pyoracle import oracle_lib
    orc = oracle_lib()
    return [orc.generate(capi.workload_spec(rate=(10.0, 15.0, 20.0, 25.0)[i % 4], duration_s=30.0,
                                            seed=1000 + i // 4)) for i in range(total)]


def _worker(rank, world, port, total, out_path):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.pyoracle import oracle_lib
    lo, hi = sweep.shard_range(total, rank, world)
    traces = _traces(total)[lo:hi]
    res, _ = oracle_lib().simulate(traces, capi.sched_cfg(policy="scls"), capi.builtin_latency_model(),
                                   capi.builtin_memory_model())
    local = torch.from_numpy(sweep.records_to_array(res, hi - lo))
    full = sweep.gather_records(local, total, world, dist)
    if rank == 0:
        np.save(out_path, full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover():
    for total in (1, 7, 4096):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                lo, hi = sweep.shard_range(total, r, world)
                got.extend(range(lo, hi))
            assert got == list(range(total))


def test_gather_world2_gloo(tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    from oracle.pyoracle import oracle_lib
    total = 7  # uneven shards (3 + 4)
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(2, _free_port(), total, out), nprocs=2, join=True,
                       start_method="spawn")
    full = np.load(out)
    res, _ = oracle_lib().simulate(_traces(total), capi.sched_cfg(policy="scls"),
                                   capi.builtin_latency_model(), capi.builtin_memory_model())
    want = sweep.records_to_array(res, total)
    assert np.array_equal(full, want)
    back = sweep.array_to_records(full)
    assert back[3].completed == res[3].completed and back[6].throughput == res[6].throughput


def test_library_shard_range_matches():
    """scls_shard_range (the C++ sharded sweep's partition) == sweep.shard_range."""
    from paper_2406_13511_b200 import lib
    for total in (0, 1, 7, 12288, 4096):
        for world in (1, 2, 3, 8):
            for r in range(world):
                assert lib.shard_range(total, r, world) == sweep.shard_range(total, r, world)


def _comm_worker(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = sweep.join_comm(None, rank, world, dist)  # no GPU here: id exchange only
    with open(f"{out_path}.{rank}", "wb") as f:
        f.write(uid)
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_id_broadcast_world2_gloo(tmp_path):
    """The rank-0 NCCL id reaches every rank intact (scls_comm_unique_id works
    without a GPU; scls_comm_init itself is covered by tests/test_multi_gpu.py)."""
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    out = str(tmp_path / "uid")
    mp.start_processes(_comm_worker, args=(2, _free_port(), out), nprocs=2, join=True, start_method="spawn")
    a, b = open(out + ".0", "rb").read(), open(out + ".1", "rb").read()
    assert len(a) == 128 and a == b
