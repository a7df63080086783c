"""Training-error metric on the B200 — drop-in for sparsedict.metrics.mse_db
(/root/reference/pkg/src/sparsedict/metrics.py:30-44), plus the two
host-side quality reports (psnr :64-73, atom_recovery :47-61) the training
scripts print. The residual ||Y - D X||_F is a device reduction.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _engine as E
from .exceptions import InvalidInputError
from .sparse_coding import SparseCodeMatrix

__all__ = ["MSE_DB_FLOOR", "PSNR_CAP", "mse_db", "atom_recovery", "psnr"]

MSE_DB_FLOOR = -300.0
PSNR_CAP = 300.0


def _db(resid_fro: float, y_fro: float) -> float:
    if y_fro == 0.0:
        raise InvalidInputError("||Y||_F is zero")
    ratio = resid_fro / y_fro
    if ratio <= 0.0:
        return MSE_DB_FLOOR
    return float(max(20.0 * np.log10(ratio), MSE_DB_FLOOR))


def mse_db_device(S: E.ShardSet, codes: E.DeviceCodes, D64: torch.Tensor) -> float:
    """20 log10(||Y - D X||_F / ||Y||_F) for device-resident data (P = 1)."""
    rsq, ysq = E.residual_sq(S, codes, D64, want_ysq=True)
    r = E.shard_sum(S, rsq, True)
    y = E.shard_sum(S, ysq, True)
    return _db(float(r[0].item()), float(y[0].item()))


def mse_db(Y, D, X, precision: str | None = None) -> float:
    """Training error in dB, floored at -300 dB (metrics.py:30-44)."""
    Y = np.asarray(Y, dtype=np.float64)
    D = np.asarray(D, dtype=np.float64)
    if not isinstance(X, SparseCodeMatrix):
        from .sparse_coding import SparseVector
        Xd = np.asarray(X, dtype=np.float64)
        cols = [SparseVector(Xd.shape[0], np.flatnonzero(Xd[:, i]), Xd[np.flatnonzero(Xd[:, i]), i])
                for i in range(Xd.shape[1])]
        X = SparseCodeMatrix.from_columns(Xd.shape[0], cols)
    prec = "fp64" if precision is None else E.get_precision(precision)
    prec = "fp64" if E.certifies(prec) else prec      # certified: the FP64 values
    Ydev, _ = E.ingest_signals(Y, prec)
    S = E.ShardSet.single(Ydev, prec)
    codes = E.codes_from_csc(X.indptr, X.indices, X.data, X.K, prec)
    return mse_db_device(S, codes, E.dict_to_device(D))


def atom_recovery(D_true, D_hat, threshold: float = 0.98) -> float:
    """% of true atoms with max_j |d_i^T dhat_j| >= threshold (host report)."""
    D_true = np.asarray(D_true, dtype=np.float64)
    D_hat = np.asarray(D_hat, dtype=np.float64)
    if D_true.ndim != 2 or D_hat.ndim != 2 or D_true.shape[0] != D_hat.shape[0]:
        raise InvalidInputError("dictionaries must share the signal dimension")
    corr = np.abs(D_true.T @ D_hat)
    return 100.0 * float((corr.max(axis=1) >= threshold).sum()) / D_true.shape[1]


def psnr(reference, test) -> float:
    """20 log10(255 / RMSE), capped at +300 dB (host report)."""
    a = np.asarray(reference, dtype=np.float64)
    b = np.asarray(test, dtype=np.float64)
    if a.shape != b.shape:
        raise InvalidInputError("images must have identical dimensions")
    rmse = float(np.sqrt(np.mean((a - b) ** 2)))
    return PSNR_CAP if rmse == 0.0 else float(min(20.0 * np.log10(255.0 / rmse), PSNR_CAP))
