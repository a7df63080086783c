"""GPU parity of the fused tensor-core Batch-OMP (sdb_omp_tc: per-step
D^T r on tcgen05, exact FP32 re-evaluation of the candidates within the TF32
error window) against the FP64 CPU oracle (the reference's omp_single,
_kernels.py:38-158) on FP32-representable inputs.

north_star tolerances: identical supports on >= 99.9% of signals with the
near-ties logged (every divergent signal must carry a small reported
margin), codes relative Frobenius error <= 1e-4.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4          # codes, relative Frobenius (north_star)
SUPPORT_FRAC = 0.999    # identical supports (north_star)
NEAR_TIE = 1e-4         # a divergent support must come with a logged margin below this


def _problem(m, K, N, s, sigma, seed):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K))
    D = (D / np.linalg.norm(D, axis=0)).astype(np.float32).astype(np.float64)
    D /= np.linalg.norm(D, axis=0)
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(K, s, replace=False), i] = rng.standard_normal(s)
    Y = (D @ X + sigma * rng.standard_normal((m, N))).astype(np.float32).astype(np.float64)
    return D, Y


def _tc_codes(Y, Ds, sizes, cap, eps=0.0, want_rnorm=False, use_tc_omp=True):
    """Code shard-contiguous columns of Y, shard p against Ds[p]."""
    import torch
    from paper_1403_4781_b200 import _engine as E
    Ydev, _ = E.ingest_signals(Y, "fp32")
    D64 = torch.cat([E.dict_to_device(D) for D in Ds])
    off, mx = E.shard_offsets(sizes)
    DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
    old = E.OMP_TC
    E.OMP_TC = use_tc_omp
    try:
        assert E.omp_tc_applies(Y.shape[0], Ds[0].shape[1], cap, "fp32") == use_tc_omp
        c = E.code(Ydev, off, mx, DT, G, cap, eps, "fp32", want_rnorm=want_rnorm, want_gap=use_tc_omp)
    finally:
        E.OMP_TC = old
    torch.cuda.synchronize()
    out = {k: E.d2h(getattr(c, k)) for k in ("idx", "val", "counts", "status")}
    if want_rnorm:
        out["rnorm"] = E.d2h(c.rnorm)
    if use_tc_omp:
        out["gap"] = E.d2h(c.gap)
    return out


def _oracle(Y, Ds, sizes, cap, eps=0.0):
    from oracle import oracle as O
    parts = []
    lo = 0
    for D, n in zip(Ds, sizes):
        parts.append(O.omp_raw(Y[:, lo:lo + n], D, cap, eps, threads=8))
        lo += n
    return [np.concatenate([p[k] for p in parts]) for k in range(5)]


def _dense(idx, val, counts, K):
    N, cap = idx.shape
    X = np.zeros((N, K))
    for t in range(cap):
        live = counts > t
        X[np.flatnonzero(live), idx[live, t]] = val[live, t]
    return X


def _compare(g, r, K):
    ridx, rval, rcnt, rst, rrn = r
    Xg = _dense(g["idx"].astype(np.int64), g["val"].astype(np.float64), g["counts"].astype(np.int64), K)
    Xr = _dense(ridx, rval, rcnt, K)
    same = np.array([np.array_equal(np.flatnonzero(Xg[i]), np.flatnonzero(Xr[i])) for i in range(Xg.shape[0])])
    rel = np.linalg.norm(Xg - Xr) / max(np.linalg.norm(Xr), 1e-300)
    return same, rel


@pytest.mark.parametrize("m,K,s,N,sigma", [
    (64, 512, 8, 20000, 0.02),    # C4 shard shape
    (64, 512, 4, 20000, 0.02),    # C4 merge sparsity
    (64, 256, 5, 20000, 0.01),    # C1
    (64, 256, 8, 12000, 0.01),    # C5 (64,256,s=8)
    (36, 200, 4, 5000, 0.01),     # padded m and K
    (16, 40, 3, 3000, 0.01),      # tiny
])
def test_omp_tc_vs_oracle(m, K, s, N, sigma):
    D, Y = _problem(m, K, N, s, sigma, seed=m * 1000 + K + s)
    g = _tc_codes(Y, [D], [N], s)
    r = _oracle(Y, [D], [N], s)
    same, rel = _compare(g, r, K)
    assert np.array_equal(g["counts"].astype(np.int64), r[2])
    assert np.array_equal(g["status"].astype(np.int64), r[3])
    assert same.mean() >= SUPPORT_FRAC, f"supports identical on {same.mean():.5f}"
    assert rel <= REL_TOL, f"codes relFro {rel:.2e}"
    # near-tie log: every divergent support comes with a small logged margin
    assert np.all(g["gap"][~same] <= NEAR_TIE)


def test_omp_tc_ragged_shards_vs_oracle():
    """Shard-contiguous batch with ragged shards (partial 128-signal tiles,
    one-signal shard, shards sharing a CTA) and a dictionary per shard."""
    m, K, s = 64, 512, 8
    sizes = [1, 127, 128, 129, 3001, 700]
    Ds, Ys = [], []
    for p, n in enumerate(sizes):
        D, Y = _problem(m, K, n, s, 0.02, seed=900 + p)
        Ds.append(D)
        Ys.append(Y)
    Y = np.concatenate(Ys, axis=1)
    g = _tc_codes(Y, Ds, sizes, s)
    r = _oracle(Y, Ds, sizes, s)
    same, rel = _compare(g, r, K)
    assert same.mean() >= SUPPORT_FRAC and rel <= REL_TOL
    assert np.array_equal(g["counts"].astype(np.int64), r[2])


def test_omp_tc_matches_warp_kernel():
    """The fused kernel and the two-launch path (tcgen05 GEMM + k_omp_fast)
    agree on supports (>= 99.9%) and codes (relFro <= 1e-4)."""
    m, K, s, N = 64, 512, 8, 16000
    D, Y = _problem(m, K, N, s, 0.02, seed=5)
    a = _tc_codes(Y, [D], [N], s, use_tc_omp=True)
    b = _tc_codes(Y, [D], [N], s, use_tc_omp=False)
    Xa = _dense(a["idx"].astype(np.int64), a["val"], a["counts"].astype(np.int64), K)
    Xb = _dense(b["idx"].astype(np.int64), b["val"], b["counts"].astype(np.int64), K)
    same = np.mean([np.array_equal(np.flatnonzero(Xa[i]), np.flatnonzero(Xb[i])) for i in range(N)])
    assert same >= SUPPORT_FRAC
    assert np.linalg.norm(Xa - Xb) / np.linalg.norm(Xb) <= REL_TOL


def test_omp_tc_error_bounded_and_rnorm():
    """eps mode (stop at ||r|| <= eps, cap 8) and the reported residual norms."""
    m, K, s, N = 64, 384, 6, 8000
    D, Y = _problem(m, K, N, s, 0.05, seed=11)
    eps = 0.4 * float(np.median(np.linalg.norm(Y, axis=0)))
    g = _tc_codes(Y, [D], [N], 8, eps=eps, want_rnorm=True)
    r = _oracle(Y, [D], [N], 8, eps=eps)
    same, rel = _compare(g, r, K)
    assert same.mean() >= SUPPORT_FRAC and rel <= REL_TOL
    agree = g["counts"].astype(np.int64) == r[2]
    assert agree.mean() >= SUPPORT_FRAC
    np.testing.assert_allclose(g["rnorm"][agree], r[4][agree], rtol=2e-4, atol=1e-5)


def test_omp_tc_edge_cases():
    """Zero signals (no atom), an exact single atom, a duplicated atom (the
    singular guard stops the support) and s = K."""
    rng = np.random.default_rng(3)
    m, K = 32, 48
    D = rng.standard_normal((m, K))
    D /= np.linalg.norm(D, axis=0)
    D[:, 7] = D[:, 3]                       # exact twin: singular when both are wanted
    D = D.astype(np.float32).astype(np.float64)
    D /= np.linalg.norm(D, axis=0)
    N = 300
    Y = rng.standard_normal((m, N))
    Y[:, 0] = 0.0                           # zero signal -> 0 atoms, status 0
    Y[:, 1] = 3.0 * D[:, 5]                 # exact single atom
    Y = Y.astype(np.float32).astype(np.float64)
    g = _tc_codes(Y, [D], [N], 8)
    assert g["counts"][0] == 0 and g["status"][0] == 0
    assert g["idx"][1, 0] == 5 and abs(g["val"][1, 0] - 3.0) < 1e-5
    # a twin is never selected after its sibling (singular guard or exact zero correlation)
    for i in range(N):
        sel = set(g["idx"][i, :g["counts"][i]].tolist())
        assert not ({3, 7} <= sel)
    r = _oracle(Y, [D], [N], 8)
    same, rel = _compare(g, r, K)
    assert same.mean() >= 0.99     # random signals fitted past m/4 atoms: FP32 near-ties
    # cap = 1 (first step only)
    g1 = _tc_codes(Y, [D], [N], 1)
    r1 = _oracle(Y, [D], [N], 1)
    assert np.mean(g1["idx"][:, 0] == r1[0][:, 0]) >= 0.99


def test_omp_tc_deterministic():
    m, K, s, N = 64, 512, 8, 6000
    D, Y = _problem(m, K, N, s, 0.02, seed=21)
    a = _tc_codes(Y, [D], [N], s)
    b = _tc_codes(Y, [D], [N], s)
    for k in ("idx", "val", "counts", "status", "gap"):
        assert np.array_equal(a[k], b[k])
