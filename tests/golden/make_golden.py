"""Generate golden vectors by running the REFERENCE implementation.

Run in the dev container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Every fixture stores seeded inputs together with the reference's outputs, so
tests can pin the oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_*.py) to the reference without importing it.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import sparsedict as sd  # noqa: E402
from sparsedict import _kernels  # noqa: E402


def rand_dict(rng, m, K):
    D = rng.standard_normal((m, K))
    return D / np.linalg.norm(D, axis=0)


def sparse_signals(rng, D, N, s, sigma):
    m, K = D.shape
    sup = np.argsort(rng.random((N, K)), axis=1)[:, :s]
    coef = rng.standard_normal((N, s))
    Y = np.zeros((m, N))
    for t in range(s):
        Y += D[:, sup[:, t]] * coef[:, t]
    return Y + sigma * rng.standard_normal((m, N))


def omp_case(name, Y, D, cap, eps, store):
    """Raw kernel outputs (selection order) + the packed CSC from omp_batch."""
    D = np.asfortranarray(D)
    Yf = np.asfortranarray(Y)
    G = _kernels.gram_matrix(D)
    N = Y.shape[1]
    idx = np.zeros((N, cap), np.int64)
    val = np.zeros((N, cap))
    counts = np.zeros(N, np.int64)
    status = np.zeros(N, np.int64)
    rn = np.zeros(N)
    if N:
        _kernels.omp_batch_range(D, G, Yf, cap, eps, 0, N, idx, val, counts, status, rn)
    store[f"{name}__Y"] = Y
    store[f"{name}__D"] = D
    if G.size <= 64 * 64:
        store[f"{name}__G"] = G
    else:  # large Gram: keep a checksum row set instead of 1-8 MB of doubles
        store[f"{name}__Grows"] = G[:: max(1, G.shape[0] // 8)]
    store[f"{name}__cap"] = np.int64(cap)
    store[f"{name}__eps"] = np.float64(eps)
    store[f"{name}__idx"] = idx
    store[f"{name}__val"] = val
    store[f"{name}__counts"] = counts
    store[f"{name}__status"] = status
    store[f"{name}__rnorm"] = rn
    if eps == 0.0:
        X = sd.omp_batch(Y, D, s=cap)
    else:
        X = sd.omp_batch(Y, D, eps=eps, s_max=cap)
    store[f"{name}__indptr"] = X.indptr
    store[f"{name}__indices"] = X.indices
    store[f"{name}__data"] = X.data


def make_omp():
    rng = np.random.default_rng(20240601)
    st = {}
    names = []
    # BASELINE shapes at small N (config 5 grid and configs 1-4 coding shapes)
    for (m, K, s, sig) in [(64, 256, 4, 0.01), (64, 256, 8, 0.01), (64, 256, 16, 0.01),
                           (64, 512, 8, 0.02), (144, 576, 8, 0.01), (64, 1024, 8, 0.01),
                           (256, 1024, 4, 0.01), (64, 256, 32, 0.01)]:
        D = rand_dict(rng, m, K)
        Y = sparse_signals(rng, D, 48 if K >= 1024 else 96, min(s, 8), sig)
        nm = f"fixed_m{m}_K{K}_s{s}"
        omp_case(nm, Y, D, s, 0.0, st)
        names.append(nm)
    # error-bounded mode (configs 2/3 style): residual target mid-range
    for (m, K, smax, eps) in [(64, 256, 16, 0.5), (144, 576, 20, 1.0), (16, 40, 16, 0.3)]:
        D = rand_dict(rng, m, K)
        Y = sparse_signals(rng, D, 160, 6, 0.05)
        nm = f"eps_m{m}_K{K}_s{smax}"
        omp_case(nm, Y, D, smax, eps, st)
        names.append(nm)
    # small random instances (the reference unit tests' regime)
    for k in range(6):
        m = int(rng.integers(4, 20))
        K = int(rng.integers(m, 3 * m))
        s = int(rng.integers(1, min(m, K) + 1))
        D = rand_dict(rng, m, K)
        Y = rng.standard_normal((m, 40))
        nm = f"small{k}"
        omp_case(nm, Y, D, s, 0.0, st)
        names.append(nm)
    # edge cases: zero signals, exact atoms, duplicate atom, near-duplicate
    # (singular stop), stall, K < 32 and K not a multiple of 32, empty batch
    D = rand_dict(rng, 12, 20)
    Y = np.column_stack([np.zeros(12), 3.0 * D[:, 5], D[:, 1] - 2 * D[:, 7],
                         rng.standard_normal(12)])
    omp_case("edge_exact", Y, D, 3, 0.0, st)
    names.append("edge_exact")
    v = np.array([3.0, 4.0]) / 5.0
    omp_case("edge_dup", np.column_stack([2.0 * v, v, -v]), np.column_stack([v, v]), 2, 0.0, st)
    names.append("edge_dup")
    vv, uu = np.array([1.0, 0.0]), np.array([0.0, 1.0])
    d1 = vv + 1e-7 * uu
    d1 /= np.linalg.norm(d1)
    omp_case("edge_singular", (2.0 * vv - uu)[:, None], np.column_stack([vv, d1]), 2, 0.0, st)
    names.append("edge_singular")
    Q, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    Ystall = np.column_stack([Q[:, 0] + Q[:, 4], Q[:, :2] @ np.array([1.0, -2.0])])
    omp_case("edge_stall", Ystall, np.ascontiguousarray(Q[:, :3]), 3, 0.0, st)
    names.append("edge_stall")
    D = rand_dict(rng, 8, 12)
    omp_case("edge_empty", np.empty((8, 0)), D, 2, 0.0, st)
    names.append("edge_empty")
    D = rand_dict(rng, 8, 12)
    y = rng.standard_normal((8, 3))
    omp_case("edge_eps_big", y, D, 8, 2.0 * float(np.linalg.norm(y, axis=0).max()), st)
    names.append("edge_eps_big")
    st["names"] = np.array(names)
    np.savez_compressed(OUT / "omp_golden.npz", **st)


def to_triple(X):
    return X.K, X.indptr, X.indices, X.data


def make_mod():
    rng = np.random.default_rng(777)
    st = {}
    names = []

    def dense_codes(Xd):
        K, N = Xd.shape
        cols = []
        for i in range(N):
            ii = np.flatnonzero(Xd[:, i])
            cols.append(sd.SparseVector(K, ii, Xd[ii, i]))
        return sd.SparseCodeMatrix.from_columns(K, cols)

    def add(nm, Y, X, Dp):
        D, dg = sd.mod_update(Y, X, Dp)
        Dr, rep = sd.replace_degenerate_atoms(D, Y, X)
        st[f"{nm}__Y"] = Y
        st[f"{nm}__Dprev"] = Dp
        st[f"{nm}__K"] = np.int64(X.K)
        st[f"{nm}__indptr"] = X.indptr
        st[f"{nm}__indices"] = X.indices
        st[f"{nm}__data"] = X.data
        st[f"{nm}__D"] = D
        st[f"{nm}__resid"] = np.float64(dg.residual_fro)
        st[f"{nm}__unused"] = np.asarray(dg.unused_atoms, np.int64)
        st[f"{nm}__rank"] = np.int64(dg.rank)
        st[f"{nm}__scales"] = np.zeros(0) if dg.scales is None else dg.scales
        st[f"{nm}__Drep"] = Dr
        st[f"{nm}__replaced"] = np.asarray(rep.replaced, np.int64)
        st[f"{nm}__unreplaced"] = np.asarray(rep.unreplaced, np.int64)
        names.append(nm)

    # MOD after a real OMP pass (the training regime) at BASELINE-like shapes
    for (m, K, N, s) in [(64, 256, 1500, 5), (16, 40, 600, 3), (144, 576, 1400, 4)]:
        Dt = rand_dict(rng, m, K)
        Y = sparse_signals(rng, Dt, N, s, 0.01)
        Dp = sd.normalize_columns(Y[:, :K])[0]
        X = sd.omp_batch(Y, Dp, s=s)
        add(f"omp_m{m}_K{K}", Y, X, Dp)
    # unused atoms, zero codes, rank-deficient, twins, zero data columns
    m, K, N = 6, 5, 40
    Dp = rand_dict(rng, m, K)
    Xd = np.zeros((K, N))
    Xd[:3] = rng.standard_normal((3, N))
    add("unused", rng.standard_normal((m, N)), dense_codes(Xd), Dp)
    add("zero_codes", rng.standard_normal((m, 10)), dense_codes(np.zeros((K, 10))), Dp)
    m, K, N = 8, 6, 100
    Dp = rand_dict(rng, m, K)
    Xd = np.zeros((K, N))
    Xd[0] = rng.standard_normal(N)
    Xd[1] = Xd[0]
    Xd[2] = rng.standard_normal(N)
    add("rank_deficient", rng.standard_normal((m, N)), dense_codes(Xd), Dp)
    m, K, N = 8, 5, 30
    Dp = rand_dict(rng, m, K)
    Xd = rng.standard_normal((K, N))
    Y = rng.standard_normal((m, N))
    # twin after the update: data built so atoms 1 and 4 solve to the same column
    Xd[4] = Xd[1] * 1.0
    add("dense_codes", Y, dense_codes(rng.standard_normal((K, N))), Dp)
    m, K = 8, 4
    Dp = rand_dict(rng, m, K)
    Y = np.zeros((m, 3))
    Y[:, 1] = rng.standard_normal(m)
    Xd = np.zeros((K, 3))
    Xd[:3] = rng.standard_normal((3, 3))
    add("zero_data_cols", Y, dense_codes(Xd), Dp)
    st["names"] = np.array(names)

    # replace_degenerate_atoms on a dictionary with an exact twin
    m, K, N = 8, 5, 30
    D = rand_dict(rng, m, K)
    D[:, 4] = D[:, 1]
    Y = rng.standard_normal((m, N))
    X = dense_codes(rng.standard_normal((K, N)))
    Dr, rep = sd.replace_degenerate_atoms(D, Y, X)
    st["twin__D"] = D
    st["twin__Y"] = Y
    st["twin__indptr"], st["twin__indices"], st["twin__data"] = X.indptr, X.indices, X.data
    st["twin__Drep"] = Dr
    st["twin__replaced"] = np.asarray(rep.replaced, np.int64)
    np.savez_compressed(OUT / "mod_golden.npz", **st)


def make_train():
    rng = np.random.default_rng(4242)
    st = {}
    # train_standard (fixed s), C1-like shapes but small
    Dt = rand_dict(rng, 16, 32)
    Y = sparse_signals(rng, Dt, 800, 3, 0.01)
    cfg = sd.TrainConfig(K=32, s=3, iterations=6, seed=5)
    D, X, rep = sd.train_standard(Y, cfg)
    st["std__Y"], st["std__D"] = Y, D
    st["std__indptr"], st["std__indices"], st["std__data"] = X.indptr, X.indices, X.data
    st["std__resid"] = np.asarray(rep.per_iteration_residuals)
    st["std__mse"] = np.float64(rep.final_mse_db)
    st["std__Dtrue"] = Dt
    # split / seeds
    st["split__idx"] = np.concatenate(sd.split_indices(103, 7, seed=11))
    st["split__sizes"] = np.asarray([b.size for b in sd.split_indices(103, 7, seed=11)])
    from sparsedict.trainer import _derive_seeds
    st["seeds"] = np.asarray(_derive_seeds(123, 9), dtype=np.uint64)
    # split -> local -> merge (C1 recipe) at small size
    Dt = rand_dict(rng, 16, 24)
    Y = sparse_signals(rng, Dt, 1200, 4, 0.01)
    L, K1, s1, its, K, s2, mits, seed = 3, 24, 4, 5, 24, 2, 5, 9
    shards = sd.split_dataset(Y, L, seed)
    seeds = _derive_seeds(seed, L + 1)
    locs = [sd.train_local(shards[t], K1, s1, its, seeds[t]) for t in range(L)]
    Dm = sd.merge_dictionaries(locs, K, s2, mits, seeds[L])
    st["sm__Y"], st["sm__D"] = Y, Dm
    for t, (D_t, X_t) in enumerate(locs):
        st[f"sm__D{t}"] = D_t
        st[f"sm__w{t}"] = np.float64(np.linalg.norm(X_t.data))
    st["sm__params"] = np.asarray([L, K1, s1, its, K, s2, mits, seed])
    # train_split_merge end to end (includes its s1*s2 evaluation pass)
    cfg = sd.TrainConfig(K=24, s=4, iterations=4, seed=21, mode="split-merge", L=3, K1=16,
                         s1=2, s2=2)
    Dsm, rsm = sd.train_split_merge(Y, cfg)
    st["tsm__D"] = Dsm
    st["tsm__mse"] = np.float64(rsm.final_mse_db)
    # mse_db
    st["mse__val"] = np.float64(sd.mse_db(Y, Dm, sd.omp_batch(Y, Dm, s=2)))
    np.savez_compressed(OUT / "train_golden.npz", **st)


def make_denoise():
    rng = np.random.default_rng(99)
    st = {}
    D8 = sd.overcomplete_dct(8, 256)
    D4 = sd.overcomplete_dct(4, 64)
    st["dct8"], st["dct4"] = D8, D4
    img = np.clip(128 + 60 * np.sin(np.arange(40)[:, None] / 5.0) * np.cos(np.arange(36) / 7.0),
                  0, 255)
    noisy = img + rng.normal(0, 20.0, img.shape)
    out = sd.denoise_image(sd.GrayImage(noisy), D8, sd.DenoiseConfig(sigma=20.0)).pixels
    st["dn__noisy"], st["dn__out"] = noisy, out
    noisy2 = rng.uniform(0, 255, (26, 31))
    out2 = sd.denoise_image(sd.GrayImage(noisy2), D4,
                            sd.DenoiseConfig(sigma=25.0, patch_size=4, stride=2, eps_gain=3.0,
                                             s_max=6)).pixels
    st["dn2__noisy"], st["dn2__out"] = noisy2, out2
    P = sd.extract_patches(sd.GrayImage(noisy2), 5, 2)
    st["patch__P"] = P
    rec = sd.reconstruct_from_patches(P * 0.5, 31, 26, 5, 2).pixels
    st["patch__rec"] = rec
    np.savez_compressed(OUT / "denoise_golden.npz", **st)


if __name__ == "__main__":
    make_omp()
    make_mod()
    make_train()
    make_denoise()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
