"""Synthetic sparse-model generators (reference synthesis.py:44-79), host and
device.

* ``gen_dictionary`` / ``gen_signals``: the reference's generators, same
  signatures and the same PCG64 draw order (``default_rng(seed)``; per signal
  a sorted ``choice(K, s, replace=False)`` support, then ``standard_normal(s)``),
  so a seed gives the reference's exact arrays. Y = D X is formed on the GPU.
* ``gen_signals_device``: the BASELINE sparse model generated on the GPU
  (sdb_synth_sparse: counter-based Philox stream, each signal a fixed function
  of (seed, index)) with optional additive N(0, sigma^2) noise -- the 4M-signal
  C4 batch in milliseconds instead of tens of seconds on the host. Not the
  PCG64 stream: callers that check against the CPU oracle hand it the same
  array (copied back).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _engine as E
from .exceptions import InvalidInputError
from .sparse_coding import SparseCodeMatrix

__all__ = ["gen_dictionary", "gen_signals", "gen_signals_device"]


def gen_dictionary(m: int, K: int, seed: int) -> np.ndarray:
    """i.i.d. N(0,1) entries, unit-norm columns (synthesis.py:44-53)."""
    if m < 1 or K < 1:
        raise InvalidInputError("m and K must be positive")
    D = np.random.default_rng(seed).standard_normal((m, K))
    nrm = np.linalg.norm(D, axis=0)
    if np.any(nrm == 0):
        raise InvalidInputError("degenerate zero column generated")
    return D / nrm


def gen_signals(D: np.ndarray, N: int, s: int, seed: int) -> tuple[np.ndarray, SparseCodeMatrix]:
    """Noiseless s-sparse signals Y = D X with the ground-truth X
    (synthesis.py:56-79): per column s distinct uniform atoms (sorted),
    standard-normal coefficients."""
    D = np.asarray(D, dtype=np.float64)
    m, K = D.shape
    if s > K:
        raise InvalidInputError("s must not exceed the atom count")
    if N < 0:
        raise InvalidInputError("N must be nonnegative")
    rng = np.random.default_rng(seed)
    indptr = np.arange(0, (N + 1) * s, s, dtype=np.int64)
    indices = np.empty(N * s, dtype=np.int64)
    data = np.empty(N * s)
    for i in range(N):
        indices[i * s:(i + 1) * s] = np.sort(rng.choice(K, size=s, replace=False))
        data[i * s:(i + 1) * s] = rng.standard_normal(s)
    X = SparseCodeMatrix(K, indptr, indices, data)
    if N == 0:
        return np.zeros((m, 0)), X
    # Y = D X on the device (f64; sums in a different order than scipy's,
    # i.e. equal to the reference's Y to rounding)
    Dd = torch.from_numpy(np.ascontiguousarray(D)).to(E.device())
    idx = torch.from_numpy(indices.reshape(N, s)).to(E.device())
    val = torch.from_numpy(data.reshape(N, s)).to(E.device())
    Y = torch.einsum("mns,ns->mn", Dd[:, idx], val)
    return E.d2h(Y), X


def gen_signals_device(D: np.ndarray, N: int, s: int, sigma: float = 0.0, seed: int = 0,
                       precision: str | None = None, want_support: bool = False):
    """The sparse model on the GPU (sdb_synth_sparse): (N, m) device rows in
    the working precision (signal-major == F-order m x N), optionally with the
    (N, s) int32 supports in draw order."""
    D = np.asarray(D, dtype=np.float64)
    if D.ndim != 2 or s < 1 or s > D.shape[1] or s > 64 or N < 0 or sigma < 0:
        raise InvalidInputError("bad generator arguments")
    return E.synth_sparse(D, N, s, sigma, seed, E.get_precision(precision), want_support)
