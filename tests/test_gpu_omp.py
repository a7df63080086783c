"""GPU parity of the OMP path (C-ABI via the Python boundary) against the
reference's golden vectors and the oracle.

FP64 ("exact") mode: bitwise identical selection order, coefficients,
statuses and residual norms. FP32 ("fast") mode: north-star tolerances —
identical supports on >= 99.9% of signals, codes relative Frobenius error
<= 1e-4.
"""

import numpy as np
import pytest

from conftest import case, golden_cases, load_golden

pytestmark = pytest.mark.gpu

OMP = load_golden("omp_golden.npz")


def _run(c, prec):
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import _engine as E
    cap, eps = int(c["cap"]), float(c["eps"])
    Ydev, bad = E.ingest_signals(c["Y"], prec)
    D64 = E.dict_to_device(c["D"])
    codes = E.code_single_dict(Ydev, D64, cap, eps, prec)
    return codes


@pytest.mark.parametrize("name", golden_cases(OMP))
def test_omp_fp64_bitwise(name):
    from paper_1403_4781_b200 import _engine as E
    c = case(OMP, name)
    if c["Y"].shape[1] == 0:
        pytest.skip("empty batch handled at the API boundary")
    codes = _run(c, "fp64")
    counts = E.d2h(codes.counts).astype(np.int64)
    assert np.array_equal(counts, c["counts"])
    assert np.array_equal(E.d2h(codes.status).astype(np.int64), c["status"])
    assert np.array_equal(E.d2h(codes.idx).astype(np.int64), c["idx"])
    assert np.array_equal(E.d2h(codes.val), c["val"])
    assert np.array_equal(E.d2h(codes.rnorm), c["rnorm"])


@pytest.mark.parametrize("name", golden_cases(OMP))
def test_omp_batch_api_fp64_matches_reference_csc(name):
    import paper_1403_4781_b200 as sdb
    c = case(OMP, name)
    cap, eps = int(c["cap"]), float(c["eps"])
    if eps == 0.0:
        X = sdb.omp_batch(c["Y"], c["D"], s=cap, precision="fp64")
    else:
        X = sdb.omp_batch(c["Y"], c["D"], eps=eps, s_max=cap, precision="fp64")
    assert np.array_equal(X.indptr, c["indptr"])
    assert np.array_equal(X.indices, c["indices"])
    assert np.array_equal(X.data, c["data"])


def _fp32_inputs(c):
    # both sides see the same FP32-representable values
    Y = c["Y"].astype(np.float32).astype(np.float64)
    D = c["D"].astype(np.float32).astype(np.float64)
    D = D / np.linalg.norm(D, axis=0)
    return Y, D


@pytest.mark.parametrize("name", [n for n in golden_cases(OMP)
                                  if n.startswith(("fixed", "eps"))])
def test_omp_fp32_tolerance(name):
    import paper_1403_4781_b200 as sdb
    from oracle import oracle as O
    c = case(OMP, name)
    Y, D = _fp32_inputs(c)
    cap, eps = int(c["cap"]), float(c["eps"])
    kw = dict(s=cap) if eps == 0.0 else dict(eps=eps, s_max=cap)
    X = sdb.omp_batch(Y, D, precision="fp32", **kw)
    Xr, _ = O.omp_codes(Y, D, **kw)
    ref = O.csc_matrix(Xr).toarray()
    got = X.to_dense()
    same = np.mean([np.array_equal(np.flatnonzero(ref[:, i]), np.flatnonzero(got[:, i]))
                    for i in range(ref.shape[1])])
    assert same >= 0.999
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-4


@pytest.mark.parametrize("eps_scale", [0.0, 0.3, 0.9])
def test_omp_fp32_precomputed_ysq_is_bitwise_identical(eps_scale):
    """The training path passes sdb_signal_sq's ||y||^2 and requests no
    residual norms: the codes must equal the default call bit for bit."""
    import torch
    from paper_1403_4781_b200 import _engine as E
    rng = np.random.default_rng(7)
    m, K, N, cap = 64, 256, 5000, 16
    D = rng.standard_normal((m, K)); D /= np.linalg.norm(D, axis=0)
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(K, 6, replace=False), i] = rng.standard_normal(6)
    Y = D @ X + 0.05 * rng.standard_normal((m, N))
    eps = eps_scale * float(np.median(np.linalg.norm(Y, axis=0)))
    Ydev, _ = E.ingest_signals(Y, "fp32")
    ysq = E.signal_sq(Ydev)
    ref = (Ydev.float() ** 2).sum(1)
    assert torch.allclose(ysq, ref, rtol=1e-5)
    D64 = E.dict_to_device(D)
    off, mx = E.shard_offsets([N])
    DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
    a = E.code(Ydev, off, mx, DT, G, cap, eps, "fp32")
    b = E.code(Ydev, off, mx, DT, G, cap, eps, "fp32", ysq=ysq, want_rnorm=False)
    for f in ("idx", "val", "counts", "status"):
        assert torch.equal(getattr(a, f), getattr(b, f)), f


def test_fp32_dynamic_chunks_equal_static_ranges():
    """The FP32 OMP kernel claims 32-signal chunks from a counter when the
    sdb_omp scratch is given and the batch is large; the codes must be bitwise
    those of static per-warp ranges (scratch NULL)."""
    import torch
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200 import _lib
    rng = np.random.default_rng(21)
    m, K, N, cap = 64, 256, 200_000, 6
    D = rng.standard_normal((K, m))
    D /= np.linalg.norm(D, axis=1, keepdims=True)
    Y = (rng.standard_normal((N, 4)) @ D[rng.integers(0, K, 4)] + 0.05 * rng.standard_normal((N, m)))
    Yd = torch.from_numpy(Y.astype(np.float32)).cuda()
    D64 = torch.from_numpy(D[None]).cuda()
    DT, G = E.working_dict(D64, "fp32"), E.gram(D64, "fp32")
    off, _ = E.shard_offsets([N])
    alpha = torch.empty((N, K), dtype=torch.float32, device="cuda")
    wb = _lib.load().sdb_correlate_workspace_bytes(0, 1, m, K)
    cws = torch.empty((wb,), dtype=torch.uint8, device="cuda")
    _lib.call("sdb_correlate", 0, N, m, K, 1, off.data_ptr(), N, Yd.data_ptr(), m, DT.data_ptr(),
              alpha.data_ptr(), K, 1, cws.data_ptr(), wb, E.stream())
    outs = []
    for dynamic in (True, False):
        idx = torch.empty((N, cap), dtype=torch.int32, device="cuda")
        val = torch.empty((N, cap), dtype=torch.float32, device="cuda")
        cnt = torch.empty((N,), dtype=torch.int32, device="cuda")
        sts = torch.empty((N,), dtype=torch.int8, device="cuda")
        sb = _lib.load().sdb_omp_scratch_bytes(0, N, m, cap)
        scr = torch.empty((sb,), dtype=torch.uint8, device="cuda") if dynamic else None
        _lib.call("sdb_omp", 0, N, m, K, 1, off.data_ptr(), alpha.data_ptr(), K, Yd.data_ptr(), m,
                  DT.data_ptr(), G.data_ptr(), cap, 0.0, 1e-6, idx.data_ptr(), val.data_ptr(),
                  cnt.data_ptr(), sts.data_ptr(), None, None, None, scr.data_ptr() if dynamic else None,
                  sb if dynamic else 0, E.stream())
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (idx, val, cnt, sts)])
    for a, b in zip(*outs):
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8))
