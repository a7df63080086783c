"""Multi-GPU split-and-merge: one process per GPU, NCCL over NVLink/NVSwitch.

The split phase partitions naturally: rank r trains the
contiguous block of shards [r*L/W, (r+1)*L/W) with no data-path
communication. The single exchange step is an all-gather of the local
dictionaries D_t (K1 x m f64) and their weights w_t = ||X_t||_F
(trainer.py:248-256); every rank then runs the (small, deterministic) merge
itself, so all ranks return the identical dictionary.

``exchange_locals`` is device-agnostic (NCCL on CUDA tensors, gloo on CPU
tensors), which is what the CPU multi-process tests exercise.
"""

from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist

from . import _engine as E
from .exceptions import InvalidInputError
from .trainer import (SplitMergeResult, merge_data, _derive_seeds, _sync, coding_mode, init_dictionaries,
                      train_device)


def shard_block(L: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of shard ids owned by ``rank`` (sizes differ by <= 1)."""
    base, extra = divmod(L, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def exchange_locals(D_local: torch.Tensor, w_local: torch.Tensor, L: int, group=None):
    """All-gather (L_r, K1, m) local dictionaries and (L_r,) weights into the
    global (L, K1, m) / (L,) arrays in shard order. Blocks are padded to the
    largest block so a single all_gather suffices."""
    world = dist.get_world_size(group)
    blocks = [shard_block(L, world, r) for r in range(world)]
    width = max(hi - lo for lo, hi in blocks)
    K1, m = D_local.shape[1], D_local.shape[2]
    padD = torch.zeros((width, K1, m), dtype=D_local.dtype, device=D_local.device)
    padw = torch.zeros((width,), dtype=w_local.dtype, device=w_local.device)
    padD[:D_local.shape[0]] = D_local
    padw[:w_local.shape[0]] = w_local
    gD = [torch.empty_like(padD) for _ in range(world)]
    gw = [torch.empty_like(padw) for _ in range(world)]
    dist.all_gather(gD, padD, group=group)
    dist.all_gather(gw, padw, group=group)
    D = torch.cat([gD[r][:hi - lo] for r, (lo, hi) in enumerate(blocks)], dim=0)
    w = torch.cat([gw[r][:hi - lo] for r, (lo, hi) in enumerate(blocks)], dim=0)
    return D, w


def split_merge_ranks(Ydev: torch.Tensor, L: int, K1: int, local_cap: int, local_eps: float,
                      local_iters: int, K: int, s2: int, merge_iters: int, seed: int,
                      init="first-columns", prec: str = "fp32", group=None,
                      t_start: float | None = None) -> SplitMergeResult:
    """Distributed split_merge_device: every rank holds the full Y (N, m) on
    its GPU and trains its block of shards; returns the merged dictionary
    (identical on all ranks)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if t_start is None:
        _sync()
        t_start = time.perf_counter()
    N, m = Ydev.shape
    if not 1 <= L <= N:
        raise InvalidInputError("require 1 <= L <= N")
    # split_indices' blocks are consecutive slices of one PCG64 permutation,
    # formed natively and bit-identically on the device (every rank the same)
    base, extra = divmod(N, L)
    all_sizes = [base + (1 if t < extra else 0) for t in range(L)]
    offs = np.concatenate([[0], np.cumsum(all_sizes)]).astype(np.int64)
    lo, hi = shard_block(L, world, rank)
    sizes = all_sizes[lo:hi]
    if min(all_sizes) < K1:
        raise InvalidInputError("first-columns init needs N >= K")
    seeds = _derive_seeds(seed, L + 1)
    if sizes:
        perm = E.split_permutation(N, seed)[int(offs[lo]):int(offs[hi])]
        Ys = E.gather_rows(Ydev, perm, prec)
        off, _ = E.shard_offsets(sizes)
        S = E.ShardSet(Ys, off, sizes, prec)
    _sync()
    t_split = time.perf_counter()
    if sizes:
        D0 = init_dictionaries(S, K1, "first-columns", seeds[lo:hi])
        Dl, codes, _ = train_device(S, D0, local_cap, local_eps, local_iters)
        w = E.code_energy(S, codes)
    else:
        Dl = E.empty((0, K1, m), torch.float64)
        w = E.empty((0,), torch.float64)
    Dall, wall = exchange_locals(Dl, w, L, group)
    w_h = E.d2h(wall)
    t_local = time.perf_counter()
    keep = np.flatnonzero(w_h > 0.0)
    if keep.size == 0:
        raise InvalidInputError("all local code matrices are zero")
    kt = torch.from_numpy(keep).to(E.device())
    Dk, wk = Dall.index_select(0, kt).contiguous(), wall.index_select(0, kt).contiguous()
    cap2, _ = coding_mode(m, K, s2, None, None)
    Sm, D0m = merge_data(Dk, wk, K1, K, init, seeds[L], prec)
    Dm, _, _ = train_device(Sm, D0m, cap2, 0.0, merge_iters)
    _sync()
    t_end = time.perf_counter()
    codings = (local_iters + 1) * N + (merge_iters + 1) * Sm.N
    return SplitMergeResult(E.d2h(Dm[0]).T.copy(), Dm, Dall, w_h, t_split - t_start,
                            t_local - t_split, t_end - t_local, t_end - t_start, codings)
