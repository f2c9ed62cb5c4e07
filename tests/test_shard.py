"""The N>1 path on CPU: world_size-2 gloo, each rank answers on its
contiguous shard (the oracle stands in for the per-GPU search, as the
checker), and the library's all-gather merge must reproduce the global
exhaustive answer — including ties that straddle the shard boundary."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2009_00786_b200.shard import merge_records, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rows, queries, out):
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2009_00786_b200.shard import allgather_merge

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    b, e = shard_range(len(rows), rank, world)
    local = np.array([orc.scan_nn(rows[b:e], q, 1) for q in queries], dtype=np.float64)
    local[:, 1] += b  # position_offset
    merged = allgather_merge(local)
    out[rank] = merged.tolist()
    dist.destroy_process_group()


def test_shard_range_covers():
    for count in (1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            parts = [shard_range(count, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == count
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def test_merge_is_lexicographic():
    a = np.array([[1.0, 5], [2.0, 9], [3.0, 1]])
    b = np.array([[1.0, 3], [1.5, 20], [3.0, 2]])
    m = merge_records([a, b])
    assert m.tolist() == [[1.0, 3], [1.5, 20], [3.0, 1]]


def test_gloo_two_ranks_equal_global_scan(oracle):
    rows = oracle.generate(3000, 64, 77)
    queries = oracle.generate(6, 64, 78)
    # a tie across the boundary: the same row in both shards
    rows[2500] = rows[400]
    queries = np.concatenate([queries, rows[400:401]])
    world, port = 2, _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, rows, queries, out), nprocs=world, join=True)
        res = [np.array(out[r]) for r in range(world)]
    want = np.array([oracle.scan_nn(rows, q, 1) for q in queries], dtype=np.float64)
    for r in range(world):
        assert np.array_equal(res[r], want)
    assert res[0][-1].tolist() == [0.0, 400.0]
