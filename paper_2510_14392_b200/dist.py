"""Multi-GPU sharding of independent instances.

Sweep configurations (C2, C3, C4) are collections of independent run_node
instances, so they shard across GPUs with no data-path collective: rank r of
R owns the instances i with i % R == r (interleaved, which balances the
divergent step counts of neighbouring grid points).  Only results travel:
`gather_results` collects per-instance results on rank 0 for aggregation and
parity checks, over whatever backend torch.distributed was initialised with
(NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from .batch import Batch


def shard_indices(n: int, rank: int, world: int) -> list[int]:
    """Interleaved partition of range(n)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return list(range(rank, n, world))


def shard_batch(batch: Batch, rank: int, world: int) -> tuple[Batch, np.ndarray]:
    """(this rank's sub-batch, global indices of its instances)."""
    idx = shard_indices(batch.n_instances, rank, world)
    return batch.subset(idx), np.asarray(idx, np.int64)


def gather_results(local: np.ndarray, idx: np.ndarray, n_total: int, dist, device=None):
    """All ranks' structured per-instance rows, in global instance order, on
    every rank (all_gather of raw bytes; works for NCCL and gloo)."""
    import torch
    world = dist.get_world_size()
    itemsize = local.dtype.itemsize
    cap = (n_total + world - 1) // world
    buf = np.zeros(cap * itemsize + 8, np.uint8)
    buf[:8] = np.frombuffer(np.int64(len(idx)).tobytes(), np.uint8)
    raw = np.ascontiguousarray(local).view(np.uint8)
    buf[8:8 + raw.size] = raw
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    out = np.zeros(n_total, local.dtype)
    for r, p in enumerate(parts):
        b = p.cpu().numpy()
        k = int(np.frombuffer(b[:8].tobytes(), np.int64)[0])
        rows = np.frombuffer(b[8:8 + k * itemsize].tobytes(), local.dtype)
        out[np.asarray(shard_indices(n_total, r, world), np.int64)[:k]] = rows
    return out
