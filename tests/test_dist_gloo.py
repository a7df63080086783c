"""Multi-process (world_size 2, gloo, CPU) coverage of the multi-GPU
split-and-merge host logic: shard ownership and the all-gather of the local
dictionaries / weights that precedes the merge (distributed.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, L, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1403_4781_b200.distributed import exchange_locals, shard_block
    lo, hi = shard_block(L, world, rank)
    K1, m = 3, 4
    # local dictionaries / weights encode their global shard id
    D = torch.stack([torch.full((K1, m), float(t), dtype=torch.float64) for t in range(lo, hi)]) \
        if hi > lo else torch.empty((0, K1, m), dtype=torch.float64)
    w = torch.arange(lo, hi, dtype=torch.float64) + 0.5
    Dall, wall = exchange_locals(D, w, L)
    out[rank] = (Dall[:, 0, 0].tolist(), wall.tolist(), (lo, hi))
    dist.destroy_process_group()


@pytest.mark.parametrize("L", [5, 2, 1, 16])
def test_exchange_locals_two_ranks(L):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), L, out), nprocs=world, join=True)
    blocks = sorted(out[r][2] for r in range(world))
    assert blocks[0][0] == 0 and blocks[-1][1] == L
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    for r in range(world):
        ids, ws, _ = out[r]
        assert ids == [float(t) for t in range(L)]          # shard order, identical on ranks
        assert ws == [t + 0.5 for t in range(L)]


def test_shard_block_partition():
    from paper_1403_4781_b200.distributed import shard_block
    for L in range(1, 40):
        for W in range(1, 9):
            spans = [shard_block(L, W, r) for r in range(W)]
            assert spans[0][0] == 0 and spans[-1][1] == L
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
