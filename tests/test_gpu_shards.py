"""GPU parity of the library's sharded path on one B200.

* local shards: tsg_open(k, {0, ..., 0}) splits the index into k contiguous
  shards on the same device, which exchange their seed best-so-far distances
  per batch (host barriers + device snapshots) and merge their result records
  with the device merge kernel - the exchange code of the multi-GPU path with a
  device-memory transport;
* NCCL: a one-device context joined to a one-rank NCCL communicator runs the
  NCCL transport's code (seed-BSF ncclAllReduce captured in the query graph,
  result ncclAllGather + merge kernel);
* position_offset: a shard built with its first global row reports global
  positions;
* gloo world 2: two processes, each building its shard with the library on
  cuda:0, merged with shard.allgather_merge.
Every answer is checked against the oracle's exhaustive scan over the whole
dataset (scan_nn: lowest position on ties, src/scan.cpp:54-59)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2009_00786_b200 as tg  # noqa: E402


def scan_all(oracle, rows, queries):
    return [oracle.scan_nn(rows, q, 0) for q in queries]


def assert_answers(res, want):
    for k, (r, (d, p)) in enumerate(zip(res, want)):
        assert (r.position, r.distance) == (p, d), (k, r.position, r.distance, p, d)


def dataset_with_boundary_tie(oracle, count, n, seed, shards):
    """Random walks with rows duplicated across every shard boundary (the lower
    copy must win), plus queries equal to those rows and to rows of the last shard."""
    rows = oracle.generate(count, n, seed)
    queries = list(oracle.generate(12, n, seed + 1))
    for s in range(1, shards):
        b = count * s // shards
        rows[b + 3] = rows[b - 5]  # same series on both sides of the boundary
        queries.append(rows[b - 5].copy())
        queries.append(rows[b + 7].copy())
    queries.append(rows[count - 1].copy())
    return rows, np.array(queries, np.float32)


@pytest.mark.parametrize("shards,count,leaf", [(2, 6000, 64), (3, 9001, 32), (4, 20000, 200)])
def test_local_shards_equal_global_scan(oracle, shards, count, leaf):
    rows, queries = dataset_with_boundary_tie(oracle, count, 64, 900 + shards, shards)
    ctx = tg.Context((0,) * shards)
    assert ctx.comm_info() == (1, shards, 0)
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=leaf), context=ctx)
    assert index.build_stats().series == count
    want = scan_all(oracle, rows, queries)
    assert_answers(tg.exact_search_batch(index, queries), want)
    # the boundary duplicates resolve to the lower copy
    for s in range(1, shards):
        b = count * s // shards
        r = tg.exact_search(index, rows[b - 5])
        assert (r.position, r.distance) == (b - 5, 0.0)
    index.free()
    ctx.close()


def test_local_shards_many_batches(oracle):
    """More queries than one batch (several exchange rounds per call, and calls
    back to back)."""
    rows = oracle.generate(12000, 64, 31)
    queries = oracle.generate(300, 64, 32)
    want = scan_all(oracle, rows, queries)
    ctx = tg.Context((0, 0))
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=100), context=ctx)
    for _ in range(2):
        assert_answers(tg.exact_search_batch(index, queries), want)
    index.free()
    ctx.close()


def test_local_shards_overflow_reruns(oracle, monkeypatch):
    """Tiny candidate slots: overflowing queries rerun per shard (no exchange),
    and the merge reads the rerun answers."""
    monkeypatch.setenv("TSG_SLOT_CAP", "200")
    rows = oracle.generate(8000, 64, 41)
    queries = oracle.generate(40, 64, 42)
    ctx = tg.Context((0, 0))
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=50), context=ctx)
    assert_answers(tg.exact_search_batch(index, queries), scan_all(oracle, rows, queries))
    index.free()
    ctx.close()


def test_local_shards_dtw_and_approximate(oracle):
    rows = oracle.generate(5000, 64, 51)
    queries = oracle.generate(6, 64, 52)
    ctx = tg.Context((0, 0))
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=64), context=ctx)
    for k, q in enumerate(queries):
        r = tg.exact_search(index, q, tg.Measure.dtw(5))
        d, p = oracle.scan_nn_dtw(rows, q, 5)
        assert (r.position, r.distance) == (p, d), k
        a = tg.approximate_search(index, q)
        assert a.distance >= oracle.scan_nn(rows, q, 0)[0]
    index.free()
    ctx.close()


def test_mixed_devices_rejected():
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two devices")
    with pytest.raises(tg.InvalidArgument, match="all distinct"):
        tg.Context((0, 0, 1))


def test_position_offset_reports_global_positions(oracle):
    rows = oracle.generate(3000, 64, 61)
    queries = oracle.generate(5, 64, 62)
    off = 1_000_000_000
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=64), position_offset=off)
    for r, (d, p) in zip(tg.exact_search_batch(index, queries), scan_all(oracle, rows, queries)):
        assert (r.position, r.distance) == (p + off, d)
    with pytest.raises(tg.InvalidArgument, match="2\\^32-1"):
        tg.build_index(rows, tg.IndexConfig(n=64), position_offset=(1 << 32) - 10)


def test_nccl_one_rank_communicator(oracle):
    """The NCCL transport on one rank: the seed-BSF allreduce is captured into
    the query graph and replayed, results go through the all-gather + merge."""
    rows, queries = dataset_with_boundary_tie(oracle, 7000, 64, 71, 2)
    ctx = tg.Context((0,))
    ctx.comm_init(1, 0, tg.comm_unique_id())
    assert ctx.comm_info() == (2, 1, 0)
    index = tg.build_index(rows, tg.IndexConfig(n=64, leaf_capacity=64), context=ctx, position_offset=0)
    want = scan_all(oracle, rows, queries)
    for _ in range(3):  # capture, then replays
        assert_answers(tg.exact_search_batch(index, queries), want)
    import torch

    dq = torch.from_numpy(queries).cuda()
    assert_answers(tg.exact_search_batch(index, dq), want)
    index.free()
    ctx.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, rows, queries, out):
    import torch.distributed as dist

    import paper_2009_00786_b200 as tgw
    from paper_2009_00786_b200.shard import allgather_merge, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, e = shard_range(len(rows), rank, world)
    index = tgw.build_index(rows[b:e], tgw.IndexConfig(n=rows.shape[1], leaf_capacity=64), position_offset=b)
    res = tgw.exact_search_batch_records(index, queries)
    local = np.stack([res["distance"], res["position"].astype(np.float64)], axis=1)
    out[rank] = allgather_merge(local).tolist()
    index.free()
    dist.destroy_process_group()


def test_gloo_two_ranks_library_shards(oracle):
    """Two processes on cuda:0, each building and searching its shard with the
    library, merged over gloo: equal to the global exhaustive scan."""
    import torch.multiprocessing as mp

    rows, queries = dataset_with_boundary_tie(oracle, 5000, 64, 81, 2)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as mgr:
        out = mgr.dict()
        mp.start_processes(_gloo_worker, args=(world, port, rows, queries, out), nprocs=world, join=True,
                           start_method="spawn")
        res = [np.array(out[r]) for r in range(world)]
    want = np.array(scan_all(oracle, rows, queries), dtype=np.float64)
    for r in range(world):
        assert np.array_equal(res[r], want)
