"""Multi-GPU plumbing of the trace sweep.

The trace dimension of a sweep (reference `sweep`, experiment.cpp:62-85, and
the C5 Monte Carlo grid) is the only dimension that shards: trace t goes to
rank floor(t * N / T) (contiguous ranges).  Each rank simulates its shard on
its own GPU with scls_simulate; the fixed-size per-trace result records are
then all-gathered — the only collective, NCCL over NVLink on the GPU path,
gloo in the CPU tests.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi

RECORD_WORDS = C.sizeof(capi.TraceResult) // 8


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) of the traces owned by `rank`."""
    return rank * total // world, (rank + 1) * total // world


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
