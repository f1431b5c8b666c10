"""Multi-GPU plumbing of the trace sweep.

The trace dimension of a sweep (reference `sweep`, experiment.cpp:62-85, and
the C5 Monte Carlo grid) is the only dimension that shards: trace t goes to
rank floor(t * N / T) (contiguous ranges).  Each rank generates and
simulates its shard on its own GPU, and the fixed-size per-trace result
records are then all-gathered — the only collective.

On the GPU path both steps live in the library: scls_run_sweep_sharded
(csrc/multi.cu) runs the rank's shard and issues the ncclAllGather itself,
on a communicator the ranks join with scls_comm_init; `join_comm` below
broadcasts the NCCL id over the caller's process group.  `gather_records`
is the torch.distributed restatement of the same gather (gloo in the CPU
tests).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi

RECORD_WORDS = C.sizeof(capi.TraceResult) // 8


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) of the traces owned by `rank`."""
    return rank * total // world, (rank + 1) * total // world


def join_comm(ctx, rank: int, world: int, dist):
    """Rank 0 draws the NCCL unique id (scls_comm_unique_id), every rank
    receives it over `dist` and joins the library's communicator with
    scls_comm_init.  Returns the id (for tests); ctx may be None (CPU tests)."""
    from . import lib
    box = [lib.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    if ctx is not None:
        ctx.comm_init(world, rank, box[0])
    return box[0]


def records_to_array(results, count) -> np.ndarray:
    """TraceResult ctypes array -> int64 [count, RECORD_WORDS] (raw words)."""
    buf = (C.c_int64 * (count * RECORD_WORDS)).from_buffer_copy(
        C.string_at(C.addressof(results), count * C.sizeof(capi.TraceResult)))
    return np.frombuffer(buf, dtype=np.int64).reshape(count, RECORD_WORDS).copy()


def array_to_records(arr: np.ndarray):
    arr = np.ascontiguousarray(arr, np.int64)
    n = arr.shape[0]
    out = (capi.TraceResult * max(n, 1))()
    C.memmove(out, arr.ctypes.data, arr.nbytes)
    return out


def gather_records(local, total: int, world: int, dist, device=None):
    """All-gather per-trace records (torch int64 [n_local, W]) into
    [total, W] in global trace order on every rank."""
    import torch
    n_max = (total + world - 1) // world
    width = local.shape[1]
    pad = torch.zeros((n_max, width), dtype=torch.int64, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    rows = []
    for r in range(world):
        lo, hi = shard_range(total, r, world)
        rows.append(parts[r][:hi - lo])
    return torch.cat(rows, dim=0)
