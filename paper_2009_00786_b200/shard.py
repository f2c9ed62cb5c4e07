"""Multi-GPU sharding of the hot path: one process per GPU.

The dataset is split into contiguous series ranges; rank r
builds its shard with position_offset = its first global row, answers every
query on its shard, and one all-gather of the 16-byte (distance, position)
records per query combines the shards: the lexicographic minimum is the
exact global answer with ties resolved to the lowest position, the same
rule scan_nn uses across its thread ranges (src/scan.cpp:54-59). With the
NCCL backend the records travel over NVLink; the tests run the same code
over gloo on CPU.
"""
from __future__ import annotations

import numpy as np


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) of the `rank`-th of `world` shards."""
    return count * rank // world, count * (rank + 1) // world


def merge_records(records) -> np.ndarray:
    """records: sequence of [nq, 2] float64 arrays (distance, position), one
    per shard in rank order -> per-query lexicographic minimum."""
    best = np.array(records[0], dtype=np.float64, copy=True)
    for r in records[1:]:
        r = np.asarray(r, dtype=np.float64)
        better = (r[:, 0] < best[:, 0]) | ((r[:, 0] == best[:, 0]) & (r[:, 1] < best[:, 1]))
        best[better] = r[better]
    return best


def allgather_merge(records: np.ndarray, device=None, group=None) -> np.ndarray:
    """All-gather every rank's [nq, 2] records and merge them (all ranks get
    the result). `device`: where the collective runs (a CUDA device for
    NCCL, None/'cpu' for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(records, dtype=np.float64))
    if device is not None and str(device) != "cpu":
        t = t.to(device)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t, group=group)
    return merge_records([g.cpu().numpy() for g in gathered])
