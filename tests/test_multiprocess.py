"""CPU (gloo, world_size 2): the multi-GPU plumbing — contiguous row shards,
the all-gather of output rows, max-over-ranks timing, and bench.py's own
per-rank row split (rank_rows: c5 strong-scaled over shards of the global
batch) — with the CPU oracle standing in for the per-rank device call (test
infrastructure only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_08455_b200.shard import gather_rows, max_over_ranks, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, L, d, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O

        rng = np.random.default_rng(99)
        X = np.cumsum(rng.standard_normal((B, L, d)) * 0.1, axis=1)  # same global batch on every rank
        lo, hi = shard_rows(B, world, rank)
        local = torch.from_numpy(O.signature(X[lo:hi], N))
        full = gather_rows(local, B)
        slowest = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put((full.numpy(), slowest))
    finally:
        dist.destroy_process_group()


def _bench_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import oracle as O

        B_global, row0, rows, scaling = bench.rank_rows("c5", world, rank)
        rng = np.random.default_rng(5)
        X = np.cumsum(rng.standard_normal((B_global, 3, 2)) * 0.3, axis=1)  # c5's batch, tiny paths
        local = torch.from_numpy(O.signature(X[row0:row0 + rows], 2))
        full = gather_rows(local, B_global)
        weak = bench.rank_rows("c2", world, rank)
        if rank == 0:
            q.put((full.numpy(), scaling, rows, weak))
    finally:
        dist.destroy_process_group()


def test_two_rank_bench_c5_shards():
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, scaling, rows, weak = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    X = np.cumsum(rng.standard_normal((8192, 3, 2)) * 0.3, axis=1)
    assert scaling == "strong" and rows == 4096
    assert np.array_equal(full, O.signature(X, 2))  # the sharded global batch == the single-GPU batch
    assert weak == (256, 0, 128, "weak")  # c2: every rank folds its own 128 rows


@pytest.mark.parametrize("B", [7, 8])
def test_two_rank_shard_gather(B):
    from oracle import oracle as O

    world, L, d, N = 2, 12, 3, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B, L, d, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    full, slowest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(99)
    X = np.cumsum(rng.standard_normal((B, L, d)) * 0.1, axis=1)
    assert np.array_equal(full, O.signature(X, N))  # rows bitwise independent of the split
    assert slowest == float(world)


def test_shard_rows_cover_disjoint():
    for B in (1, 5, 128, 8192, 1001):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_rows(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            for (a, b), (c, e) in zip(spans, spans[1:]):
                assert b == c and a <= b
    with pytest.raises(ValueError):
        shard_rows(4, 2, 2)
