"""Fused error-bounded coding (sdb_code_step1 + sdb_omp_deferred) vs the
two-kernel path (sdb_correlate + sdb_omp): the codes must be bitwise the
same. The fused GEMM epilogue runs omp_single's first iteration
(_kernels.py:61-154) per signal row and defers the rest to the list-driven
OMP kernel, so every branch of that first step is exercised here: ||y|| <=
eps (including zero signals), one-atom stops, signals within the explicit-
residual band around eps, multi-atom signals, ||y||^2 past the FP32 range,
cap = 1, ragged shards whose
ends straddle 32-row quadrants and 128-row tiles, K < 256 and K not a
multiple of 32.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _data(m, K, sizes, seed, huge=True):
    rng = np.random.default_rng(seed)
    P, N = len(sizes), sum(sizes)
    D = rng.standard_normal((P, K, m))
    D /= np.linalg.norm(D, axis=2, keepdims=True)
    off = np.concatenate([[0], np.cumsum(sizes)])
    Y = np.empty((N, m))
    kind = rng.integers(0, 5, N)
    if huge:
        kind[rng.random(N) < 0.01] = 5
    for p in range(P):
        for i in range(off[p], off[p + 1]):
            k = kind[i]
            if k == 0:      # pure noise, mostly below eps
                Y[i] = rng.standard_normal(m) * 0.8
            elif k == 1:    # one atom plus noise
                Y[i] = 20 * rng.standard_normal() * D[p, rng.integers(K)] + rng.standard_normal(m) * 0.5
            elif k == 2:    # several atoms
                s = rng.integers(2, 6)
                sup = rng.choice(K, s, replace=False)
                Y[i] = (rng.standard_normal(s) * 10) @ D[p, sup] + rng.standard_normal(m) * 0.3
            elif k == 3:    # exact atom (one step, residual ~0)
                Y[i] = 7.0 * D[p, rng.integers(K)]
            elif k == 4:    # zero signal
                Y[i] = 0.0
            else:           # ||y||^2 overflows FP32: deferred by the fused epilogue
                Y[i] = 3e19 * D[p, rng.integers(K)] + 1e18 * rng.standard_normal(m)
    return Y, D, off


def _code(Y, D, sizes, cap, eps, fused):
    from paper_1403_4781_b200 import _engine as E
    Yd = torch.from_numpy(Y.astype(np.float32)).cuda()
    D64 = torch.from_numpy(D).cuda()
    off, mx = E.shard_offsets(sizes)
    ysq = E.signal_sq(Yd)
    old = E.OMP_TC
    E.OMP_TC = False   # the two-kernel reference path (sdb_correlate + sdb_omp)
    try:
        codes = E.code(Yd, off, mx, E.working_dict(D64, "fp32"), E.gram(D64, "fp32"), cap, eps, "fp32",
                       True, ysq=ysq, want_rnorm=not fused)
        torch.cuda.synchronize()
    finally:
        E.OMP_TC = old
    return (codes.idx.cpu().numpy(), codes.val.cpu().numpy(), codes.counts.cpu().numpy(),
            codes.status.cpu().numpy())


@pytest.mark.parametrize("m,K,sizes,cap", [
    (64, 256, [1000, 777, 1, 130], 16),
    (64, 256, [4096], 1),
    (64, 100, [300, 257, 31], 8),
    (16, 24, [50, 70], 4),
    (144, 256, [513, 129], 20),
    (32, 200, [2000], 32),
])
def test_fused_step1_bitwise(m, K, sizes, cap):
    Y, D, _ = _data(m, K, sizes, seed=m * 7 + K + cap)
    eps = float(np.sqrt(m) * 0.9)
    a = _code(Y, D, sizes, cap, eps, fused=True)
    b = _code(Y, D, sizes, cap, eps, fused=False)
    for x, y, name in zip(a, b, ("idx", "val", "counts", "status")):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), name
    # every branch of the first step occurred
    counts = a[2]
    assert (counts == 0).any() and (counts == 1).any()
    if cap > 1:
        assert (counts >= 2).any()


def test_fused_band_signals():
    """Signals whose one-atom residual lands within the explicit-residual band
    (|r^2 - eps^2| <= 1e-4 ||y||^2) are deferred and decided as sdb_omp does."""
    rng = np.random.default_rng(11)
    m, K, N = 64, 256, 3000
    D = rng.standard_normal((1, K, m))
    D /= np.linalg.norm(D, axis=2, keepdims=True)
    eps = 5.0
    Y = np.empty((N, m))
    for i in range(N):
        a = D[0, rng.integers(K)]
        r = rng.standard_normal(m)
        r -= (r @ a) * a                   # orthogonal to the atom
        r *= eps * (1 + rng.uniform(-2e-5, 2e-5)) / np.linalg.norm(r)
        Y[i] = 30 * a + r
    a = _code(Y, D, [N], 8, eps, fused=True)
    b = _code(Y, D, [N], 8, eps, fused=False)
    for x, y, name in zip(a, b, ("idx", "val", "counts", "status")):
        assert np.array_equal(x.view(np.uint8), y.view(np.uint8)), name


def test_fused_vs_oracle_supports():
    """Cross-check with the CPU oracle (FP64 restatement of _kernels.py) on
    the FP32-rounded inputs: identical supports on >= 99.9% of signals."""
    from oracle import oracle as O
    Y, D, off = _data(64, 256, [1500, 1500], seed=5, huge=False)   # FP32 range only
    sizes = [1500, 1500]
    eps = float(np.sqrt(64) * 0.9)
    idx, val, counts, status = _code(Y, D, sizes, 16, eps, fused=True)
    Y32 = Y.astype(np.float32).astype(np.float64)
    D32 = D.astype(np.float32).astype(np.float64)
    same = 0
    for p in range(2):
        oi, ov, oc, ost, _ = O.omp_raw(Y32[off[p]:off[p + 1]].T, D32[p].T, 16, eps)
        for r in range(off[p + 1] - off[p]):
            i = off[p] + r
            same += int(counts[i] == oc[r] and np.array_equal(np.sort(idx[i, :counts[i]]), np.sort(oi[r, :oc[r]])))
    assert same >= 0.999 * len(Y), same


def test_fused_training_bitwise_equals_unfused():
    """A whole error-bounded FP32 split-and-merge training (15 local
    iterations, graph-replayed) gives bitwise the same dictionary with the
    fused coding path as with sdb_correlate + sdb_omp."""
    import benchdata
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device
    Y = benchdata.make_training_data("c2", 7, N=60000)
    Ydev, _ = E.ingest_signals(Y.T, "fp32")
    out = []
    for fuse in (True, False):
        E.FUSE_STEP1 = fuse
        try:
            r = split_merge_device(Ydev, 4, 256, 16, 184.0, 6, 256, 4, 4, 11, prec="fp32")
        finally:
            E.FUSE_STEP1 = True
        out.append(r.D)
    assert np.array_equal(out[0].view(np.uint8), out[1].view(np.uint8))
