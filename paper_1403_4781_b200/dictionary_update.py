"""MOD dictionary update and atom maintenance on the B200 — drop-in for
sparsedict.dictionary_update (/root/reference/pkg/src/sparsedict/
dictionary_update.py: normalize_columns :56, mod_update :72,
replace_degenerate_atoms :117).

Host side: validation and numpy <-> device marshalling only. The normal
equations, the FP64 Cholesky solve, residual norms, dead-atom handling,
twin detection and the replacement ranking run in libsdb200.so.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _engine as E
from .exceptions import InvalidInputError
from .sparse_coding import SparseCodeMatrix, check_dictionary

__all__ = [
    "UpdateDiagnostics",
    "ReplacementReport",
    "normalize_columns",
    "mod_update",
    "replace_degenerate_atoms",
]

RANK_RCOND = 1e-10
ZERO_NORM_REL = 1e-12
TWIN_COHERENCE = 0.999


@dataclass
class UpdateDiagnostics:
    """Outcome of one MOD step; ``scales`` are the raw (pre-normalisation)
    column norms, so D_out * scales reconstructs the normal-equation solution."""

    residual_fro: float
    unused_atoms: list[int] = field(default_factory=list)
    rank: int = 0
    scales: np.ndarray | None = None


@dataclass
class ReplacementReport:
    replaced: list[int] = field(default_factory=list)
    unreplaced: list[int] = field(default_factory=list)


def normalize_columns(M) -> tuple[np.ndarray, np.ndarray]:
    """Unit-norm every nonzero column; returns (normalised, original norms)."""
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2:
        raise InvalidInputError("expected a 2-D matrix")
    if M.size == 0:
        return M.copy(), np.zeros(M.shape[1])
    out, sc = E.normalize_rows(torch.from_numpy(np.ascontiguousarray(M.T)).to(E.device()))
    return E.d2h(out).T.copy(), E.d2h(sc)


def _prepare(Y, X: SparseCodeMatrix, m: int, prec: str):
    # MOD / replacement arithmetic is FP64 in both modes; certified FP32 also
    # keeps the inputs FP64 (the reference's values)
    prec = "fp64" if E.certifies(prec) else prec
    Ydev, bad = E.ingest_signals(Y, prec)
    codes = E.codes_from_csc(X.indptr, X.indices, X.data, X.K, prec)
    return E.ShardSet.single(Ydev, prec), codes


def mod_update(Y, X: SparseCodeMatrix, D_prev, precision: str | None = None
               ) -> tuple[np.ndarray, UpdateDiagnostics]:
    """One MOD step D = Y X^T (X X^T)^+ then column renormalisation
    (dictionary_update.py:72-114)."""
    Y = np.asarray(Y, dtype=np.float64)
    D_prev = check_dictionary(D_prev)
    m, K = D_prev.shape
    if Y.ndim != 2 or Y.shape[0] != m:
        raise InvalidInputError("Y must be m x N")
    if X.K != K or X.N != Y.shape[1]:
        raise InvalidInputError("code matrix shape does not match Y and D")
    if m > 256:
        raise InvalidInputError("signal dimension m > 256 is outside the GPU path")
    prec = E.get_precision(precision)
    if X.nnz == 0:  # dictionary_update.py:92-95
        return D_prev.copy(), UpdateDiagnostics(residual_fro=float(np.linalg.norm(Y)),
                                                unused_atoms=list(range(K)), rank=0)
    S, codes = _prepare(Y, X, m, prec)
    r = E.mod_update(S, codes, E.dict_to_device(D_prev))
    D = E.d2h(r.D[0]).T.copy()
    dead = E.d2h(r.dead[0]).astype(bool)
    return D, UpdateDiagnostics(residual_fro=float(r.resid[0].item()),
                                unused_atoms=[int(a) for a in np.flatnonzero(dead)],
                                rank=int(r.rank[0].item()), scales=E.d2h(r.scales[0]))


def replace_degenerate_atoms(D, Y, X: SparseCodeMatrix, rng_seed: int = 0,
                             precision: str | None = None
                             ) -> tuple[np.ndarray, ReplacementReport]:
    """Swap unused, zero-norm and twin atoms for the worst-represented data
    columns (dictionary_update.py:117-177). ``rng_seed`` is accepted and
    ignored, as in the reference."""
    del rng_seed
    D = np.asarray(D, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    m, K = D.shape
    if Y.ndim != 2 or Y.shape[0] != m or X.K != K or X.N != Y.shape[1]:
        raise InvalidInputError("inconsistent dimensions")
    if m > 256:
        raise InvalidInputError("signal dimension m > 256 is outside the GPU path")
    prec = E.get_precision(precision)
    S, codes = _prepare(Y, X, m, prec)
    D64 = E.dict_to_device(D).clone()
    usage = E.code_usage(S, codes)
    flags, _nt = E.replace_degenerate(S, codes, D64, usage)
    f = E.d2h(flags[0])
    rep = ReplacementReport(replaced=[int(a) for a in np.flatnonzero(f == 1)],
                            unreplaced=[int(a) for a in np.flatnonzero(f == 2)])
    return E.d2h(D64[0]).T.copy(), rep
