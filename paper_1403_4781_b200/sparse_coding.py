"""OMP sparse coding on the B200 — drop-in for sparsedict.sparse_coding.

Public signatures follow /root/reference/pkg/src/sparsedict/sparse_coding.py
(omp_batch :230, omp_fixed_sparsity :188, omp_error_bound :208, containers
:34-142). Validation runs on the host before any launch and raises
InvalidInputError exactly where the reference does; the arithmetic runs in
libsdb200.so (Gram, correlation GEMM, warp-per-signal Batch-OMP, CSC packing).

Extension (optional kwarg, reference-preserving default): ``precision`` —
"fp64" (default, OMP bitwise identical to the reference) or "fp32" (fast
mode). ``threads`` is accepted and ignored: the GPU partition never changes
results.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp
import torch

from . import _engine as E
from .exceptions import InvalidInputError

__all__ = [
    "SparseVector",
    "SparseCodeMatrix",
    "OmpDiagnostics",
    "check_dictionary",
    "omp_fixed_sparsity",
    "omp_error_bound",
    "omp_batch",
]

UNIT_NORM_TOL = 1e-9
STATUS_OK, STATUS_SINGULAR, STATUS_STALLED = 0, 2, 3


@dataclass(frozen=True)
class SparseVector:
    """One sparse code: strictly increasing int64 indices, float64 values."""

    length: int
    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        ii = np.asarray(self.indices, dtype=np.int64)
        vv = np.asarray(self.values, dtype=np.float64)
        if ii.ndim != 1 or ii.shape != vv.shape:
            raise InvalidInputError("indices and values must be 1-D and equal length")
        if ii.size:
            if ii[0] < 0 or ii[-1] >= self.length:
                raise InvalidInputError("index out of range")
            if ii.size > 1 and (np.diff(ii) <= 0).any():
                raise InvalidInputError("indices must be strictly increasing")
        object.__setattr__(self, "indices", ii)
        object.__setattr__(self, "values", vv)

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    def to_dense(self) -> np.ndarray:
        d = np.zeros(self.length)
        d[self.indices] = self.values
        return d


@dataclass
class OmpDiagnostics:
    """Per-signal outcome (status codes surface as flags, never exceptions)."""

    residual_norm: float
    n_iterations: int
    singular_stop: bool = False
    stalled: bool = False
    cap_hit: bool = False
    selection_order: np.ndarray = field(default_factory=lambda: np.empty(0, np.int64))


class SparseCodeMatrix:
    """K x N codes in CSC form (int64 indices ascending within a column)."""

    def __init__(self, K: int, indptr: np.ndarray, indices: np.ndarray, data: np.ndarray):
        self.K = int(K)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.data = np.asarray(data, dtype=np.float64)
        if self.indptr.ndim != 1 or self.indptr[0] != 0:
            raise InvalidInputError("malformed indptr")
        if self.indices.shape != self.data.shape:
            raise InvalidInputError("indices/data length mismatch")

    @property
    def N(self) -> int:
        return self.indptr.size - 1

    @property
    def nnz(self) -> int:
        return int(self.indices.size)

    @classmethod
    def from_columns(cls, K: int, columns: list[SparseVector]) -> "SparseCodeMatrix":
        for c in columns:
            if c.length != K:
                raise InvalidInputError("column length mismatch")
        sizes = np.fromiter((c.nnz for c in columns), dtype=np.int64, count=len(columns))
        indptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        if columns:
            indices = np.concatenate([c.indices for c in columns]).astype(np.int64)
            data = np.concatenate([c.values for c in columns]).astype(np.float64)
        else:
            indices, data = np.empty(0, np.int64), np.empty(0)
        return cls(K, indptr, indices, data)

    def column(self, i: int) -> SparseVector:
        a, b = self.indptr[i], self.indptr[i + 1]
        return SparseVector(self.K, self.indices[a:b].copy(), self.data[a:b].copy())

    def columns(self) -> list[SparseVector]:
        return [self.column(i) for i in range(self.N)]

    def nnz_per_column(self) -> np.ndarray:
        return np.diff(self.indptr)

    def row_usage(self) -> np.ndarray:
        return np.bincount(self.indices, minlength=self.K).astype(np.int64)

    def to_csc(self) -> sp.csc_array:
        return sp.csc_array((self.data, self.indices.astype(np.int32), self.indptr),
                            shape=(self.K, self.N))

    def to_dense(self) -> np.ndarray:
        return self.to_csc().toarray()

    def __eq__(self, other) -> bool:
        if not isinstance(other, SparseCodeMatrix):
            return False
        return (self.K == other.K and np.array_equal(self.indptr, other.indptr)
                and np.array_equal(self.indices, other.indices)
                and np.array_equal(self.data, other.data))

    __hash__ = None


def check_dictionary(D) -> np.ndarray:
    """Finite, nonempty 2-D, unit-norm columns within 1e-9 (sparse_coding.py:145-155)."""
    D = np.asarray(D, dtype=np.float64)
    if D.ndim != 2 or D.shape[0] < 1 or D.shape[1] < 1:
        raise InvalidInputError("dictionary must be a nonempty 2-D matrix")
    if not np.isfinite(D).all():
        raise InvalidInputError("dictionary contains non-finite entries")
    if (np.abs(np.linalg.norm(D, axis=0) - 1.0) > UNIT_NORM_TOL).any():
        raise InvalidInputError("dictionary columns must have unit norm")
    if D.shape[1] > E.MAX_K:
        raise InvalidInputError(f"K={D.shape[1]} atoms exceeds the GPU path's limit of {E.MAX_K}")
    return D


def _signal_vector(y, m: int) -> np.ndarray:
    y = np.asarray(y, dtype=np.float64).reshape(-1)
    if y.shape[0] != m:
        raise InvalidInputError(f"signal length {y.shape[0]} != dictionary rows {m}")
    if not np.isfinite(y).all():
        raise InvalidInputError("signal contains non-finite entries")
    return y


def resolve_mode(m: int, K: int, s, eps, s_max) -> tuple[int, float, bool]:
    """(cap, eps, error_mode) with the reference's checks (sparse_coding.py:247-264)."""
    if s is not None:
        if eps is not None or s_max is not None:
            raise InvalidInputError("choose either fixed-sparsity or error-bound mode")
        cap = int(s)
        if not 1 <= cap <= min(m, K):
            raise InvalidInputError("sparsity must satisfy 1 <= s <= min(m, K)")
        return cap, 0.0, False
    if eps is None:
        raise InvalidInputError("one of s or eps is required")
    e = float(eps)
    if e < 0 or not np.isfinite(e):
        raise InvalidInputError("eps must be a finite nonnegative real")
    cap = int(s_max) if s_max is not None else m
    if not 1 <= cap <= m:
        raise InvalidInputError("s_max must satisfy 1 <= s_max <= m")
    return cap, e, True


def codes_to_matrix(codes: E.DeviceCodes, prec: str) -> SparseCodeMatrix:
    indptr, indices, data = E.csc(codes, prec)
    return SparseCodeMatrix(codes.K, E.d2h(indptr), E.d2h(indices), E.d2h(data))


def _diagnostics(codes: E.DeviceCodes, err_mode: bool, eps: float, with_order: bool):
    counts = E.d2h(codes.counts).astype(np.int64)
    status = E.d2h(codes.status).astype(np.int64)
    rn = E.d2h(codes.rnorm).astype(np.float64)
    order = E.d2h(codes.idx).astype(np.int64) if with_order else None
    out = []
    for i in range(counts.size):
        n = int(counts[i])
        out.append(OmpDiagnostics(
            residual_norm=float(rn[i]),
            n_iterations=n,
            singular_stop=bool(status[i] == STATUS_SINGULAR),
            stalled=bool(status[i] == STATUS_STALLED),
            cap_hit=bool(err_mode and n == codes.cap and rn[i] > eps),
            selection_order=order[i, :n].copy() if with_order else np.empty(0, np.int64),
        ))
    return out


def _run(Y, D, cap, eps, prec, N_hint=None):
    Ydev, Y64, bad = E.ingest_for(Y, prec)
    if int(bad.item()):
        raise InvalidInputError("batch contains non-finite entries")
    D64 = E.dict_to_device(D)
    return E.code_single_dict(Ydev, D64, cap, eps, prec, Y64=Y64)


def _single(y, D, cap, eps, prec):
    codes = _run(y.reshape(-1, 1), D, cap, eps, prec)
    X = codes_to_matrix(codes, prec)
    diag = _diagnostics(codes, False, eps, with_order=True)[0]
    return X.column(0), diag


def omp_fixed_sparsity(y, D, s, with_diagnostics: bool = False, precision: str | None = None):
    """OMP with a hard budget of s atoms (sparse_coding.py:188-205)."""
    D = check_dictionary(D)
    m, K = D.shape
    y = _signal_vector(y, m)
    s = int(s)
    if not 1 <= s <= min(m, K):
        raise InvalidInputError("sparsity must satisfy 1 <= s <= min(m, K)")
    x, diag = _single(y, D, s, 0.0, E.get_precision(precision))
    return (x, diag) if with_diagnostics else x


def omp_error_bound(y, D, eps, s_max, with_diagnostics: bool = False,
                    precision: str | None = None):
    """OMP until ||r||_2 <= eps or s_max atoms (sparse_coding.py:208-227)."""
    D = check_dictionary(D)
    m, K = D.shape
    y = _signal_vector(y, m)
    eps = float(eps)
    if eps < 0 or not np.isfinite(eps):
        raise InvalidInputError("eps must be a finite nonnegative real")
    s_max = int(s_max)
    if not 1 <= s_max <= m:
        raise InvalidInputError("s_max must satisfy 1 <= s_max <= m")
    x, diag = _single(y, D, s_max, eps, E.get_precision(precision))
    diag.cap_hit = diag.n_iterations == s_max and diag.residual_norm > eps
    return (x, diag) if with_diagnostics else x


def omp_batch(Y, D, s=None, eps=None, s_max=None, threads: int = 1,
              with_diagnostics: bool = False, precision: str | None = None):
    """Column-wise OMP over Y (m x N), one warp per signal on the GPU
    (sparse_coding.py:230-316). ``Y`` may also be a CUDA tensor (m x N)."""
    D = check_dictionary(D)
    m, K = D.shape
    if isinstance(Y, torch.Tensor):
        if Y.ndim != 2 or Y.shape[0] != m:
            raise InvalidInputError(f"batch must be 2-D with {m} rows")
    else:
        Y = np.asarray(Y, dtype=np.float64)
        if Y.ndim != 2 or Y.shape[0] != m:
            raise InvalidInputError(f"batch must be 2-D with {m} rows")
    cap, e, err_mode = resolve_mode(m, K, s, eps, s_max)
    prec = E.get_precision(precision)
    N = Y.shape[1]
    if N == 0:
        X = SparseCodeMatrix(K, np.zeros(1, np.int64), np.empty(0, np.int64), np.empty(0))
        return (X, []) if with_diagnostics else X
    codes = _run(Y, D, cap, e, prec)
    X = codes_to_matrix(codes, prec)
    if not with_diagnostics:
        return X
    return X, _diagnostics(codes, err_mode, e, with_order=False)
