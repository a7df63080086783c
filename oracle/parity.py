"""CPU PARITY CHECKER — test infrastructure only, never part of the product path.

Compares the GPU's OMP codes with the oracle's (``oracle.omp_raw``, the
bit-exact restatement of ``_kernels.omp_batch_range``, ``_kernels.py:161-173``)
on the same inputs and logs near-ties (BASELINE ``north_star``: "OMP supports
must be identical on >= 99.9% of signals, with near-ties logged").

For every signal whose support differs, the first divergent greedy step k is
located in SELECTION order (both sides record atoms in the order they were
picked, ``_kernels.py:123-127``). With the common prefix S = idx[:k] the
reference's residual r = y - D_S x_S (least squares on S, FP64) gives the
correlations c = D^T r of step k (``_kernels.py:81-96``); the logged gap is

    gap = (|c[a]| - |c[b]|) / |c[a]|,   a = oracle's pick, b = GPU's pick,

i.e. how close the two candidates were in exact arithmetic. A divergence at
the stopping rule instead (same prefix, different count) logs the relative
margin of ||r|| against eps (``_kernels.py:153``) or the pivot against the
singular guard. Only ``tests/``, ``tools/`` and ``bench.py`` import this.
"""

from __future__ import annotations

import numpy as np


def _step_corr(y: np.ndarray, D: np.ndarray, S) -> np.ndarray:
    if len(S) == 0:
        return D.T @ y
    DS = D[:, list(S)]
    x, *_ = np.linalg.lstsq(DS, y, rcond=None)
    return D.T @ (y - DS @ x)


def first_divergence(y, D, ridx, rcnt, gidx, gcnt, eps: float = 0.0):
    """Where and how closely the two greedy traces of one signal diverge."""
    n = min(int(rcnt), int(gcnt))
    k = 0
    while k < n and int(ridx[k]) == int(gidx[k]):
        k += 1
    if k < n:
        c = np.abs(_step_corr(y, D, ridx[:k]))
        a, b = int(ridx[k]), int(gidx[k])
        top = float(c[a])
        return dict(kind="selection", step=k, oracle_atom=a, gpu_atom=b,
                    corr_oracle=top, corr_gpu=float(c[b]),
                    gap=float((top - c[b]) / top) if top > 0 else 0.0)
    # same prefix, different stopping point
    c = _step_corr(y, D, ridx[:n])
    S = list(ridx[:n])
    if S:
        DS = D[:, S]
        x, *_ = np.linalg.lstsq(DS, y, rcond=None)
        rn = float(np.linalg.norm(y - DS @ x))
    else:
        rn = float(np.linalg.norm(y))
    margin = abs(rn - eps) / eps if eps > 0 else float("nan")
    return dict(kind="stop", step=n, oracle_count=int(rcnt), gpu_count=int(gcnt), rnorm=rn,
                eps_margin=margin, next_corr=float(np.abs(c).max()) if c.size else 0.0)


def compare_codes(Y, D, gidx, gval, gcnt, ref, eps: float = 0.0, max_log: int = 50) -> dict:
    """GPU codes (selection-order idx/val rows, counts) vs the oracle's
    ``omp_raw`` result ``ref = (idx, val, counts, status, rnorm)`` for the
    columns of Y (m x n, FP64 values of what the GPU coded) and D (m x K,
    the FP64 values of the GPU's dictionary).

    Returns: n, same_support (fraction), same_order, rel_fro (codes, all
    signals), rel_fro_same_support (signals with identical supports only),
    n_divergent, near_ties (first divergent step per divergent signal, up to
    ``max_log``), max_selection_gap.
    """
    Y = np.asarray(Y, dtype=np.float64)
    D = np.asarray(D, dtype=np.float64)
    ridx, rval, rcnt = ref[0], ref[1], ref[2]
    n = Y.shape[1]
    cap = max(ridx.shape[1], gidx.shape[1])
    same = np.zeros(n, dtype=bool)
    same_order = np.zeros(n, dtype=bool)
    num = np.zeros(n)
    den = np.zeros(n)
    for i in range(n):
        rc, gc = int(rcnt[i]), int(gcnt[i])
        ri, gi = ridx[i, :rc].astype(np.int64), gidx[i, :gc].astype(np.int64)
        rv, gv = rval[i, :rc], gval[i, :gc].astype(np.float64)
        same_order[i] = rc == gc and np.array_equal(ri, gi)
        same[i] = rc == gc and np.array_equal(np.sort(ri), np.sort(gi))
        a = dict(zip(ri.tolist(), rv.tolist()))
        b = dict(zip(gi.tolist(), gv.tolist()))
        num[i] = sum((a.get(j, 0.0) - b.get(j, 0.0)) ** 2 for j in set(a) | set(b))
        den[i] = float(np.dot(rv, rv))
    div = np.flatnonzero(~same)
    ties = []
    for i in div[:max_log]:
        t = first_divergence(Y[:, i], D, ridx[i], rcnt[i], gidx[i], gcnt[i], eps)
        t["signal"] = int(i)
        ties.append(t)
    sel = [t["gap"] for t in ties if t["kind"] == "selection"]
    tot = den.sum()
    return dict(n=int(n), cap=int(cap), same_support=float(same.mean()) if n else 1.0,
                same_order=float(same_order.mean()) if n else 1.0,
                rel_fro=float(np.sqrt(num.sum() / tot)) if tot > 0 else 0.0,
                rel_fro_same_support=float(np.sqrt(num[same].sum() / den[same].sum()))
                if same.any() and den[same].sum() > 0 else 0.0,
                n_divergent=int(div.size), near_ties=ties,
                max_selection_gap=float(max(sel)) if sel else None)


def gpu_codes_host(codes, rows=None):
    """(idx, val, counts) of an engine DeviceCodes as numpy (optionally a row subset)."""
    idx = codes.idx.cpu().numpy()
    val = codes.val.cpu().numpy()
    cnt = codes.counts.cpu().numpy()
    if rows is not None:
        idx, val, cnt = idx[rows], val[rows], cnt[rows]
    return idx, val, cnt
