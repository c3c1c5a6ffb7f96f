"""CPU (gloo, world_size 2): the multi-GPU plumbing — contiguous row shards,
the all-gather of output rows, max-over-ranks timing — with the CPU oracle
standing in for the per-rank device call (test infrastructure only)."""
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
