"""The parity checker itself (oracle/parity.py): identical codes compare as
identical; a forced divergence is located at the right greedy step and its
near-tie gap is the exact correlation gap of that step."""

import numpy as np

from oracle import oracle as O
from oracle import parity as PA


def _data(seed=0, m=16, K=40, N=300, s=4):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K))
    D /= np.linalg.norm(D, axis=0)
    X = np.zeros((K, N))
    for i in range(N):
        X[rng.choice(K, s, replace=False), i] = rng.standard_normal(s)
    return D, D @ X + 0.01 * rng.standard_normal((m, N))


def test_identical_codes_compare_equal():
    D, Y = _data()
    ref = O.omp_raw(Y, D, 4, 0.0)
    r = PA.compare_codes(Y, D, ref[0], ref[1], ref[2], ref)
    assert r["same_support"] == 1.0 and r["same_order"] == 1.0
    assert r["rel_fro"] == 0.0 and r["n_divergent"] == 0 and r["near_ties"] == []


def test_forced_divergence_is_located_and_gap_measured():
    D, Y = _data(1)
    ref = O.omp_raw(Y, D, 4, 0.0)
    gidx, gval, gcnt = ref[0].copy(), ref[1].copy(), ref[2].copy()
    i = 7
    # the "GPU" picked the runner-up at step 2
    S = list(ref[0][i, :2])
    c = np.abs(PA._step_corr(Y[:, i], D, S))
    c[S] = -1
    order = np.argsort(-c)
    assert order[0] == ref[0][i, 2]
    gidx[i, 2] = order[1]
    r = PA.compare_codes(Y, D, gidx, gval, gcnt, ref)
    assert r["n_divergent"] == 1 and r["same_support"] == 1 - 1 / Y.shape[1]
    t = r["near_ties"][0]
    assert t["signal"] == i and t["kind"] == "selection" and t["step"] == 2
    assert t["oracle_atom"] == order[0] and t["gpu_atom"] == order[1]
    assert np.isclose(t["gap"], (c[order[0]] - c[order[1]]) / c[order[0]])
    assert r["max_selection_gap"] == t["gap"]


def test_stop_divergence_reports_eps_margin():
    D, Y = _data(2)
    eps = 0.5
    ref = O.omp_raw(Y, D, 6, eps)
    gidx, gval, gcnt = ref[0].copy(), ref[1].copy(), ref[2].copy()
    i = int(np.flatnonzero(ref[2] >= 2)[0])
    gcnt[i] -= 1
    r = PA.compare_codes(Y, D, gidx, gval, gcnt, ref, eps=eps)
    t = r["near_ties"][0]
    assert t["kind"] == "stop" and t["step"] == gcnt[i] and t["eps_margin"] > 0
