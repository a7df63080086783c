"""The single-signal wrappers, diagnostics and status semantics through the
public API (sparse_coding.py:172-316), in both precisions.

* omp_fixed_sparsity / omp_error_bound / omp_batch(with_diagnostics) agree
  with one another: a batch coded column by column equals the batch call
  bitwise (reference pkg/tests/test_sparse_coding.py:196-214 states this for
  the reference; here it holds for the exact and the certified FP32 mode).
* Status semantics: a near-duplicate atom (tilted by 1e-7) ends the greedy
  loop with SINGULAR in the reference (_kernels.py:109-127). The plain FP32
  kernels cannot resolve that pivot (their guard is 1e-6); certified FP32
  re-codes any signal whose FP32 status is not OK with the exact FP64 kernel,
  so it reports SINGULAR like the reference.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dict(m, K, seed):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K))
    return D / np.linalg.norm(D, axis=0)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_single_signal_wrappers_equal_batch(prec):
    import paper_1403_4781_b200 as sdb
    D = _dict(16, 40, 3)
    rng = np.random.default_rng(4)
    Y = D[:, :6] @ rng.standard_normal((6, 25)) + 0.01 * rng.standard_normal((16, 25))
    if prec == "fp32":
        Y = Y.astype(np.float32).astype(np.float64)
    X, diags = sdb.omp_batch(Y, D, s=4, with_diagnostics=True, precision=prec)
    Xe, diage = sdb.omp_batch(Y, D, eps=0.05, s_max=6, with_diagnostics=True, precision=prec)
    dense, dense_e = X.to_csc().toarray(), Xe.to_csc().toarray()
    for i in range(Y.shape[1]):
        x, dg = sdb.omp_fixed_sparsity(Y[:, i], D, 4, with_diagnostics=True, precision=prec)
        v = np.zeros(40)
        v[x.indices] = x.values
        assert np.array_equal(v, dense[:, i])
        assert dg.residual_norm == diags[i].residual_norm
        assert (dg.singular_stop, dg.stalled) == (diags[i].singular_stop, diags[i].stalled)
        xe, dge = sdb.omp_error_bound(Y[:, i], D, 0.05, 6, with_diagnostics=True, precision=prec)
        v = np.zeros(40)
        v[xe.indices] = xe.values
        assert np.array_equal(v, dense_e[:, i])
        assert dge.cap_hit == diage[i].cap_hit


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_near_duplicate_atom_reports_singular(prec):
    import paper_1403_4781_b200 as sdb
    from paper_1403_4781_b200 import _engine as E
    v = np.array([1.0, 0.0])
    u = np.array([0.0, 1.0])
    d1 = v + 1e-7 * u
    d1 /= np.linalg.norm(d1)
    D = np.column_stack([v, d1])
    y = 2.0 * v - u
    assert prec == "fp64" or E.CERTIFY
    x, dg = sdb.omp_fixed_sparsity(y, D, 2, with_diagnostics=True, precision=prec)
    assert list(x.indices) == [0]
    assert dg.singular_stop and not dg.stalled
