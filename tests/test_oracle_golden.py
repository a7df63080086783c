"""Pin the CPU oracle to vectors produced by the reference implementation.

The oracle (oracle/omp_oracle.c + oracle/oracle.py) is the checker for the
CUDA path; before trusting it, it must reproduce the reference's own outputs:
bitwise for the OMP kernels, to 1e-12 for the LAPACK/scipy-based MOD layer.
CPU only (no GPU needed).
"""

import numpy as np
import pytest

from conftest import case, golden_cases, load_golden
from oracle import oracle as O

OMP = load_golden("omp_golden.npz")
MOD = load_golden("mod_golden.npz")
TRN = load_golden("train_golden.npz")
DN = load_golden("denoise_golden.npz")


@pytest.mark.parametrize("name", golden_cases(OMP))
def test_oracle_omp_bitwise(name):
    c = case(OMP, name)
    G = O.gram(c["D"])
    if "G" in c:
        assert np.array_equal(G, c["G"])
    else:
        assert np.array_equal(G[:: max(1, G.shape[0] // 8)], c["Grows"])
    idx, val, counts, status, rn = O.omp_raw(c["Y"], c["D"], int(c["cap"]), float(c["eps"]))
    assert np.array_equal(counts, c["counts"])
    assert np.array_equal(status, c["status"])
    assert np.array_equal(idx, c["idx"])
    assert np.array_equal(val, c["val"])          # bitwise
    assert np.array_equal(rn, c["rnorm"])
    K, indptr, indices, data = O.pack_csc(c["D"].shape[1], idx, val, counts)
    assert np.array_equal(indptr, c["indptr"])
    assert np.array_equal(indices, c["indices"])
    assert np.array_equal(data, c["data"])


def test_oracle_threads_invariant():
    c = case(OMP, "fixed_m64_K256_s8")
    a = O.omp_raw(c["Y"], c["D"], 8, 0.0, threads=1)
    b = O.omp_raw(c["Y"], c["D"], 8, 0.0, threads=4)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


def test_oracle_edge_statuses():
    assert list(case(OMP, "edge_singular")["status"]) == [O.STATUS_SINGULAR]
    assert O.STATUS_STALLED in set(case(OMP, "edge_stall")["status"].tolist())
    assert case(OMP, "edge_exact")["counts"][0] == 0


@pytest.mark.parametrize("name", golden_cases(MOD))
def test_oracle_mod(name):
    c = case(MOD, name)
    X = (int(c["K"]), c["indptr"], c["indices"], c["data"])
    D, resid, unused, rank, scales = O.mod_update(c["Y"], X, c["Dprev"])
    np.testing.assert_allclose(D, c["D"], rtol=0, atol=1e-12)
    assert resid == pytest.approx(float(c["resid"]), rel=1e-12)
    assert list(unused) == list(c["unused"])
    assert rank == int(c["rank"])
    Dr, rep, unrep = O.replace_degenerate_atoms(D, c["Y"], X)
    np.testing.assert_allclose(Dr, c["Drep"], rtol=0, atol=1e-12)
    assert rep == list(c["replaced"]) and unrep == list(c["unreplaced"])


def test_oracle_twin_replacement():
    X = (5, MOD["twin__indptr"], MOD["twin__indices"], MOD["twin__data"])
    Dr, rep, _ = O.replace_degenerate_atoms(MOD["twin__D"], MOD["twin__Y"], X)
    assert rep == list(MOD["twin__replaced"])
    assert np.array_equal(Dr, MOD["twin__Drep"])


def test_oracle_train_standard():
    D, X, resid = O.train_standard(TRN["std__Y"], 32, 3, 6, seed=5)
    np.testing.assert_allclose(D, TRN["std__D"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(resid, TRN["std__resid"], rtol=1e-10)
    assert np.array_equal(X[1], TRN["std__indptr"])
    assert np.array_equal(X[2], TRN["std__indices"])
    assert O.mse_db(TRN["std__Y"], D, X) == pytest.approx(float(TRN["std__mse"]), abs=1e-9)


def test_oracle_split_and_seeds():
    blocks = O.split_indices(103, 7, 11)
    assert np.array_equal(np.concatenate(blocks), TRN["split__idx"])
    assert [b.size for b in blocks] == list(TRN["split__sizes"])
    assert O.derive_seeds(123, 9) == [int(v) for v in TRN["seeds"]]


def test_oracle_split_merge():
    L, K1, s1, its, K, s2, mits, seed = (int(v) for v in TRN["sm__params"])
    D, locs = O.split_merge(TRN["sm__Y"], L, K1, s1, its, K, s2, mits, seed)
    for t, (D_t, X_t) in enumerate(locs):
        np.testing.assert_allclose(D_t, TRN[f"sm__D{t}"], rtol=0, atol=1e-10)
        assert np.linalg.norm(X_t[3]) == pytest.approx(float(TRN[f"sm__w{t}"]), rel=1e-10)
    np.testing.assert_allclose(D, TRN["sm__D"], rtol=0, atol=1e-9)


def test_oracle_denoise():
    np.testing.assert_allclose(O.overcomplete_dct(8, 256), DN["dct8"], rtol=0, atol=1e-15)
    out = O.denoise(DN["dn__noisy"], DN["dct8"], 20.0)
    np.testing.assert_allclose(out, DN["dn__out"], rtol=0, atol=1e-9)
    out2 = O.denoise(DN["dn2__noisy"], DN["dct4"], 25.0, patch_size=4, stride=2, eps_gain=3.0,
                     s_max=6)
    np.testing.assert_allclose(out2, DN["dn2__out"], rtol=0, atol=1e-9)
    P = O.extract_patches(DN["dn2__noisy"], 5, 2)
    assert np.array_equal(P, DN["patch__P"])
    rec = O.reconstruct_from_patches(P * 0.5, 31, 26, 5, 2)
    np.testing.assert_allclose(rec, DN["patch__rec"], rtol=0, atol=1e-12)
