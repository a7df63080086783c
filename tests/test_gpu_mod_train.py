"""GPU parity of MOD, atom replacement, training and denoising against the
reference's golden vectors (FP64 mode) and the oracle (FP32 mode).

Tolerances: FP64 mode 1e-10 absolute on dictionaries (the reference solves
the normal equations by LAPACK SVD, we by FP64 Cholesky: same solution to
rounding); FP32 mode per the north star — dictionaries relative Frobenius
error <= 1e-3 after a fixed number of iterations from the same init,
denoising PSNR within 0.05 dB.
"""

import numpy as np
import pytest

from conftest import case, golden_cases, load_golden

pytestmark = pytest.mark.gpu

MOD = load_golden("mod_golden.npz")
TRN = load_golden("train_golden.npz")
DN = load_golden("denoise_golden.npz")


def _X(c, K=None):
    import paper_1403_4781_b200 as sdb
    return sdb.SparseCodeMatrix(int(c["K"]) if K is None else K, c["indptr"], c["indices"],
                                c["data"])


@pytest.mark.parametrize("name", golden_cases(MOD))
def test_mod_update_fp64(name):
    import paper_1403_4781_b200 as sdb
    c = case(MOD, name)
    X = _X(c)
    D, dg = sdb.mod_update(c["Y"], X, c["Dprev"], precision="fp64")
    # rank_deficient: the minimum-norm lstsq solution (sdb_minnorm.cu) like the reference
    np.testing.assert_allclose(D, c["D"], rtol=0, atol=1e-10)
    assert dg.residual_fro == pytest.approx(float(c["resid"]), rel=1e-10)
    assert dg.unused_atoms == list(c["unused"])
    assert dg.rank == int(c["rank"])
    if c["scales"].size:
        np.testing.assert_allclose(dg.scales, c["scales"], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("name", golden_cases(MOD))
def test_replace_fp64(name):
    import paper_1403_4781_b200 as sdb
    c = case(MOD, name)
    X = _X(c)
    Dr, rep = sdb.replace_degenerate_atoms(c["D"], c["Y"], X)
    assert rep.replaced == list(c["replaced"])
    assert rep.unreplaced == list(c["unreplaced"])
    np.testing.assert_allclose(Dr, c["Drep"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("K,m,N,dups,prec", [(6, 8, 100, 1, "fp64"), (64, 16, 2000, 3, "fp64"),
                                              (256, 64, 5000, 5, "fp32"), (300, 32, 4000, 4, "fp64"),
                                              (512, 64, 6000, 2, "fp32")])
def test_mod_min_norm_rank_deficient_vs_oracle(K, m, N, dups, prec):
    """Used blocks with exactly dependent code rows (duplicated rows and a
    row that is the sum of two others): the minimum-norm solution
    (dictionary_update.py:100) on both the clustered (K <= 256) and the
    chained (K > 256) Cholesky paths, vs the oracle's numpy lstsq."""
    import paper_1403_4781_b200 as sdb
    from oracle import oracle as O
    rng = np.random.default_rng(K + dups)
    Dp = rng.standard_normal((m, K))
    Dp /= np.linalg.norm(Dp, axis=0)
    res = 8 if K >= 32 else 3                 # reserved atoms for the dependent rows
    Xd = np.zeros((K, N))
    for i in range(N):
        sup = rng.choice(K - res, min(3, K - res), replace=False)
        Xd[sup, i] = rng.standard_normal(sup.size)
    for d in range(dups):
        Xd[K - res + d] = Xd[d]               # a duplicated code row
    if K >= 32:
        Xd[K - 1] = Xd[10] + Xd[11]           # a sum of two rows
    Xd[K - 2] = 0.0                           # an unused atom
    Y = rng.standard_normal((m, N))
    if prec == "fp32":
        Y = Y.astype(np.float32).astype(np.float64)
        Xd = Xd.astype(np.float32).astype(np.float64)
    from scipy import sparse
    Xc = sparse.csc_array(Xd)
    X = sdb.SparseCodeMatrix(K, Xc.indptr.astype(np.int64), Xc.indices.astype(np.int64), Xc.data)
    D, dg = sdb.mod_update(Y, X, Dp, precision=prec)
    Dr, resid, unused, rank, scales = O.mod_update(Y, (K, Xc.indptr.astype(np.int64),
                                                       Xc.indices.astype(np.int64), Xc.data), Dp)
    np.testing.assert_allclose(D, Dr, rtol=0, atol=1e-9)
    assert dg.rank == rank
    assert dg.unused_atoms == list(unused)
    assert dg.residual_fro == pytest.approx(resid, rel=1e-9)


def test_replace_twins():
    import paper_1403_4781_b200 as sdb
    X = sdb.SparseCodeMatrix(5, MOD["twin__indptr"], MOD["twin__indices"], MOD["twin__data"])
    Dr, rep = sdb.replace_degenerate_atoms(MOD["twin__D"], MOD["twin__Y"], X)
    assert rep.replaced == list(MOD["twin__replaced"])
    np.testing.assert_allclose(Dr, MOD["twin__Drep"], rtol=0, atol=1e-12)


def test_normalize_columns():
    import paper_1403_4781_b200 as sdb
    M = np.array([[0.0, 3.0, 1.0], [0.0, 4.0, 2.0]])
    out, sc = sdb.normalize_columns(M)
    assert np.array_equal(out[:, 0], [0.0, 0.0]) and sc[0] == 0.0
    np.testing.assert_allclose(out[:, 1], [0.6, 0.8], atol=1e-15)
    np.testing.assert_allclose(sc, np.linalg.norm(M, axis=0), rtol=1e-15)


def test_train_standard_fp64():
    import paper_1403_4781_b200 as sdb
    cfg = sdb.TrainConfig(K=32, s=3, iterations=6, seed=5)
    D, X, rep = sdb.train_standard(TRN["std__Y"], cfg)
    np.testing.assert_allclose(D, TRN["std__D"], rtol=0, atol=1e-9)
    np.testing.assert_allclose(rep.per_iteration_residuals, TRN["std__resid"], rtol=1e-9)
    assert np.array_equal(X.indptr, TRN["std__indptr"])
    assert np.array_equal(X.indices, TRN["std__indices"])
    np.testing.assert_allclose(X.data, TRN["std__data"], rtol=0, atol=1e-8)
    assert rep.final_mse_db == pytest.approx(float(TRN["std__mse"]), abs=1e-7)


def test_split_local_merge_fp64():
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200.trainer import _derive_seeds
    L, K1, s1, its, K, s2, mits, seed = (int(v) for v in TRN["sm__params"])
    Y = TRN["sm__Y"]
    shards = sdb.split_dataset(Y, L, seed)
    seeds = _derive_seeds(seed, L + 1)
    locs = [sdb.train_local(shards[t], K1, s1, its, seeds[t]) for t in range(L)]
    for t, (D_t, X_t) in enumerate(locs):
        np.testing.assert_allclose(D_t, TRN[f"sm__D{t}"], rtol=0, atol=1e-9)
    D = sdb.merge_dictionaries(locs, K, s2, mits, seeds[L])
    np.testing.assert_allclose(D, TRN["sm__D"], rtol=0, atol=1e-8)


def test_batched_split_merge_matches_per_shard_loop_fp64():
    """All locals trained in one batched device loop == the reference's
    per-shard composition."""
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device
    L, K1, s1, its, K, s2, mits, seed = (int(v) for v in TRN["sm__params"])
    Ydev, _ = E.ingest_signals(TRN["sm__Y"], "fp64")
    r = split_merge_device(Ydev, L, K1, s1, 0.0, its, K, s2, mits, seed, prec="fp64")
    for t in range(L):
        np.testing.assert_allclose(E.d2h(r.local_D[t]).T, TRN[f"sm__D{t}"], rtol=0, atol=1e-9)
        assert r.weights[t] == pytest.approx(float(TRN[f"sm__w{t}"]), rel=1e-10)
    np.testing.assert_allclose(r.D, TRN["sm__D"], rtol=0, atol=1e-8)


def test_train_split_merge_api_fp64():
    import paper_1403_4781_b200 as sdb
    cfg = sdb.TrainConfig(K=24, s=4, iterations=4, seed=21, mode="split-merge", L=3, K1=16,
                          s1=2, s2=2)
    D, rep = sdb.train_split_merge(TRN["sm__Y"], cfg)
    np.testing.assert_allclose(D, TRN["tsm__D"], rtol=0, atol=1e-8)
    assert rep.final_mse_db == pytest.approx(float(TRN["tsm__mse"]), abs=1e-6)
    assert rep.critical_path_s == pytest.approx(
        rep.split_time_s + max(rep.local_wall_times_s) + rep.merge_wall_time_s)


def test_mse_db_fp64():
    import paper_1403_4781_b200 as sdb
    Y, D = TRN["sm__Y"], TRN["sm__D"]
    X = sdb.omp_batch(Y, D, s=2)
    assert sdb.mse_db(Y, D, X) == pytest.approx(float(TRN["mse__val"]), abs=1e-9)


def test_determinism_fp32_and_fp64():
    import paper_1403_4781_b200 as sdb
    for prec in ("fp64", "fp32"):
        cfg = sdb.TrainConfig(K=32, s=3, iterations=4, seed=5, precision=prec)
        D1, X1, _ = sdb.train_standard(TRN["std__Y"], cfg)
        D2, X2, _ = sdb.train_standard(TRN["std__Y"], cfg)
        assert np.array_equal(D1, D2) and X1 == X2


def test_train_standard_fp32_tolerance():
    """FP32 mode vs the FP64 oracle from the same init on FP32-representable
    data: dictionary relative Frobenius error <= 1e-3 after the iterations."""
    import paper_1403_4781_b200 as sdb
    from oracle import oracle as O
    Y = TRN["std__Y"].astype(np.float32).astype(np.float64)
    cfg = sdb.TrainConfig(K=32, s=3, iterations=6, seed=5, precision="fp32")
    D, X, rep = sdb.train_standard(Y, cfg)
    Dr, Xr, resid = O.train_standard(Y, 32, 3, 6, seed=5)
    rel = np.linalg.norm(D - Dr) / np.linalg.norm(Dr)
    assert rel <= 1e-3
    np.testing.assert_allclose(rep.per_iteration_residuals, resid, rtol=1e-3)


def test_denoise_fp64():
    import paper_1403_4781_b200 as sdb
    out = sdb.denoise_image(sdb.GrayImage(DN["dn__noisy"]), DN["dct8"],
                            sdb.DenoiseConfig(sigma=20.0)).pixels
    np.testing.assert_allclose(out, DN["dn__out"], rtol=0, atol=1e-9)
    out2 = sdb.denoise_image(sdb.GrayImage(DN["dn2__noisy"]), DN["dct4"],
                             sdb.DenoiseConfig(sigma=25.0, patch_size=4, stride=2, eps_gain=3.0,
                                               s_max=6)).pixels
    np.testing.assert_allclose(out2, DN["dn2__out"], rtol=0, atol=1e-9)


def test_patch_pipeline_exact():
    import paper_1403_4781_b200 as sdb
    P = sdb.extract_patches(sdb.GrayImage(DN["dn2__noisy"]), 5, 2)
    assert np.array_equal(P, DN["patch__P"])
    rec = sdb.reconstruct_from_patches(P * 0.5, 31, 26, 5, 2).pixels
    np.testing.assert_allclose(rec, DN["patch__rec"], rtol=0, atol=1e-12)


def test_denoise_fp32_psnr():
    import paper_1403_4781_b200 as sdb
    from oracle import oracle as O
    # the clean image of tests/golden/make_golden.py:make_denoise
    clean = np.clip(128 + 60 * np.sin(np.arange(40)[:, None] / 5.0) * np.cos(np.arange(36) / 7.0),
                    0, 255)
    noisy = DN["dn__noisy"]
    out = sdb.denoise_image(sdb.GrayImage(noisy), DN["dct8"], sdb.DenoiseConfig(sigma=20.0),
                            precision="fp32").pixels
    ref = O.denoise(noisy, DN["dct8"], 20.0)
    assert abs(O.psnr(clean, out) - O.psnr(clean, ref)) <= 0.05


@pytest.mark.parametrize("n", [1, 2, 3, 17, 1025, 65537, 200003, 2040200])
def test_device_split_permutation_equals_numpy(n):
    """Host swap targets + parallel device resolution == numpy's permutation."""
    from paper_1403_4781_b200 import _engine as E
    for seed in (0, 1234):
        got = E.d2h(E.split_permutation(n, seed))
        assert np.array_equal(got, np.random.default_rng(seed).permutation(n))


def _c1_like(N=12000, m=32, K=64, seed=3):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K)); D /= np.linalg.norm(D, axis=0)
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(K, 3, replace=False), i] = rng.standard_normal(3)
    return D @ X + 0.01 * rng.standard_normal((m, N))


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_grouped_locals_equal_batched(prec):
    """Shard groups on separate streams == all shards in one batch, bitwise."""
    import torch
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device
    Y = _c1_like()
    Ydev, _ = E.ingest_signals(Y, prec)
    out = []
    for groups in (1, 3, 4):
        r = split_merge_device(Ydev, 6, 64, 3, 0.0, 4, 64, 2, 3, 77, prec=prec, groups=groups)
        out.append((E.d2h(r.local_D), r.weights, r.D))
    for Dl, w, D in out[1:]:
        assert np.array_equal(Dl, out[0][0])
        assert np.array_equal(w, out[0][1])
        assert np.array_equal(D, out[0][2])


def test_pinned_host_input_streams_and_matches():
    """train_split_merge on pinned host memory (rows gathered over PCIe per
    shard group) == the same call on pageable memory."""
    import torch
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import _engine as E
    Y = _c1_like()
    m, N = Y.shape
    pinned = torch.empty((N, m), dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = Y.T
    assert E.host_mapped(pinned.numpy()) is not None
    assert E.host_mapped(np.ascontiguousarray(Y.T)) is None
    cfg = sdb.TrainConfig(K=64, s=6, mode="split-merge", L=6, K1=64, s1=3, s2=2, iterations=4,
                          seed=5, precision="fp32")
    D_pin, rep_pin = sdb.train_split_merge(pinned.numpy().T, cfg)
    D_pag, rep_pag = sdb.train_split_merge(np.asfortranarray(Y), cfg)
    assert np.array_equal(D_pin, D_pag)
    assert rep_pin.final_mse_db == rep_pag.final_mse_db
    bad = pinned.numpy().copy()
    pinned.numpy()[7, 3] = np.nan
    with pytest.raises(sdb.InvalidInputError):
        sdb.train_split_merge(pinned.numpy().T, cfg)
    pinned.numpy()[:] = bad


@pytest.mark.parametrize("K", [100, 130, 200, 255])
@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_mod_cluster_solve_partial_blocks(K, prec):
    """The clustered Cholesky with 2-4 CTAs per shard and a partial last
    64-row block agrees with the oracle's lstsq MOD."""
    import sys
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    from oracle import oracle as O
    import paper_1403_4781_b200 as sdb
    rng = np.random.default_rng(K)
    m, N = 48, 6 * K
    Dp = rng.standard_normal((m, K)); Dp /= np.linalg.norm(Dp, axis=0)
    Y = rng.standard_normal((m, N))
    X, _ = O.omp_codes(Y, Dp, s=6)
    Xs = sdb.SparseCodeMatrix(K, X[1], X[2], X[3])
    D, dg = sdb.mod_update(Y, Xs, Dp, precision=prec)
    Dr, resid, unused, _rank, _norms = O.mod_update(Y, X, Dp)
    tol = 1e-9 if prec == "fp64" else 2e-4
    np.testing.assert_allclose(D, Dr, rtol=0, atol=tol)
    assert dg.unused_atoms == list(unused)
    assert dg.residual_fro == pytest.approx(resid, rel=1e-9 if prec == "fp64" else 1e-5)


def test_split_merge_ranks_nccl_world1_equals_device():
    """The multi-GPU split-and-merge path (NCCL, here with one rank) gives
    bitwise the same dictionary as the single-GPU batched path."""
    import socket

    import torch
    import torch.distributed as dist

    import benchdata
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.distributed import split_merge_ranks
    from paper_1403_4781_b200.trainer import split_merge_device
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        Y = benchdata.make_training_data("c2", 3, N=40000)
        Ydev, _ = E.ingest_signals(Y.T, "fp32")
        a = split_merge_ranks(Ydev, 4, 256, 16, 184.0, 4, 256, 4, 4, 9, prec="fp32")
        b = split_merge_device(Ydev, 4, 256, 16, 184.0, 4, 256, 4, 4, 9, prec="fp32")
        assert np.array_equal(a.D, b.D)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_shard_groups_equal_one_batch(prec):
    """Concurrent shard groups on their own streams (auto for >= 128 shards)
    give bitwise the dictionaries of the single batched launch: shards are
    independent and every kernel's per-shard arithmetic is fixed."""
    import benchdata
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200.trainer import split_merge_device
    Yd = benchdata.make_training_data_device("c4", 5, prec, N=8 * 4000)
    out = []
    for groups in (1, 4):
        r = split_merge_device(Yd, 8, 96, 6, 0.0, 3, 96, 3, 3, 17, prec=prec, groups=groups)
        out.append((E.d2h(r.local_D), r.D))
    assert np.array_equal(out[0][0].view(np.uint8), out[1][0].view(np.uint8))
    assert np.array_equal(out[0][1].view(np.uint8), out[1][1].view(np.uint8))
