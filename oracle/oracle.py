"""CPU ORACLE — test infrastructure only, never part of the product path.

A restatement of the reference ``sparsedict`` hot path (``/root/reference/
pkg/src/sparsedict``) used to check the B200 implementation. Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline``
leg and ``--impl reference``) may import this module.

* The OMP inner loops run in ``omp_oracle.c`` (bit-exact restatement of the
  Numba kernels ``_kernels.py:23-173``), loaded through ctypes.
* Everything above them (CSC packing, MOD, atom replacement, the training
  loops, the patch pipeline, mse) is restated here with numpy / scipy — the
  same third-party arithmetic the reference calls (``numpy.linalg.lstsq``,
  ``scipy.sparse``).

Pinned against vectors produced by the reference itself
(``tests/golden/make_golden.py`` → ``tests/golden/*.npz``), checked by
``tests/test_oracle_golden.py``.

Codes are carried as a plain CSC triple ``(K, indptr, indices, data)``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libomp_oracle.so"

STATUS_OK, STATUS_SINGULAR, STATUS_STALLED = 0, 2, 3   # _kernels.py:13-15
UNIT_NORM_TOL = 1e-9                                    # sparse_coding.py:31
RANK_RCOND = 1e-10                                      # dictionary_update.py:27
ZERO_NORM_REL = 1e-12                                   # dictionary_update.py:30
TWIN_COHERENCE = 0.999                                  # dictionary_update.py:32
MSE_DB_FLOOR = -300.0                                   # metrics.py:26

_lib = None


class OracleInputError(ValueError):
    """Precondition violation (the reference raises InvalidInputError)."""


def build() -> Path:
    """Compile omp_oracle.c (idempotent)."""
    src = _HERE / "omp_oracle.c"
    if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int64)
        i64 = ctypes.c_int64
        L.orc_gram_matrix.argtypes = [dp, i64, i64, dp]
        L.orc_gram_matrix.restype = None
        L.orc_omp_batch_threads.argtypes = [dp, dp, dp, i64, i64, i64, i64, ctypes.c_double,
                                            ctypes.c_int, ip, dp, ip, ip, dp]
        L.orc_omp_batch_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# ---------------------------------------------------------------- OMP layer
def gram(D: np.ndarray) -> np.ndarray:
    """_kernels.gram_matrix (_kernels.py:23-35), bit-exact."""
    D = np.asfortranarray(D, dtype=np.float64)
    m, K = D.shape
    G = np.empty((K, K))
    lib().orc_gram_matrix(_dptr(D), m, K, _dptr(G))
    return G


def omp_raw(Y: np.ndarray, D: np.ndarray, cap: int, eps: float, threads: int = 1,
            G: np.ndarray | None = None):
    """_kernels.omp_batch_range over all columns (sparse_coding.py:266-292).

    Returns (idx[N,cap] selection order, val[N,cap], counts, status, rnorm).
    """
    D = np.asfortranarray(D, dtype=np.float64)
    Y = np.asfortranarray(Y, dtype=np.float64)
    m, K = D.shape
    N = Y.shape[1]
    if G is None:
        G = gram(D)
    G = np.ascontiguousarray(G)
    idx = np.zeros((N, cap), dtype=np.int64)
    val = np.zeros((N, cap))
    counts = np.zeros(N, dtype=np.int64)
    status = np.zeros(N, dtype=np.int64)
    rnorm = np.zeros(N)
    if N:
        rc = lib().orc_omp_batch_threads(_dptr(D), _dptr(G), _dptr(Y), m, K, N, cap, float(eps),
                                         int(threads), _iptr(idx), _dptr(val), _iptr(counts),
                                         _iptr(status), _dptr(rnorm))
        if rc != 0:
            raise MemoryError("oracle OMP scratch allocation failed")
    return idx, val, counts, status, rnorm


def pack_csc(K: int, idx, val, counts):
    """Codes (selection order) -> CSC with indices ascending per column
    (sparse_coding.py:294-303)."""
    N, cap = idx.shape
    indptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    keep = np.arange(cap)[None, :] < counts[:, None]
    col = np.repeat(np.arange(N, dtype=np.int64), counts)
    fi, fv = idx[keep], val[keep]
    order = np.lexsort((fi, col))
    return K, indptr, fi[order], fv[order]


def check_dictionary(D) -> np.ndarray:
    """sparse_coding.py:145-155."""
    D = np.asarray(D, dtype=np.float64)
    if D.ndim != 2 or min(D.shape) < 1:
        raise OracleInputError("dictionary must be a nonempty 2-D matrix")
    if not np.isfinite(D).all():
        raise OracleInputError("dictionary contains non-finite entries")
    if (np.abs(np.linalg.norm(D, axis=0) - 1.0) > UNIT_NORM_TOL).any():
        raise OracleInputError("dictionary columns must have unit norm")
    return D


def omp_codes(Y, D, s=None, eps=None, s_max=None, threads=1):
    """omp_batch (sparse_coding.py:230-316) as a CSC triple plus per-signal
    (counts, status, rnorm, cap, err_mode)."""
    D = check_dictionary(D)
    m, K = D.shape
    Y = np.asarray(Y, dtype=np.float64)
    if Y.ndim != 2 or Y.shape[0] != m:
        raise OracleInputError("batch shape")
    if s is not None:
        cap, e, err_mode = int(s), 0.0, False
    else:
        e = float(eps)
        cap = int(s_max) if s_max is not None else m
        err_mode = True
    idx, val, counts, status, rnorm = omp_raw(Y, D, cap, e, threads)
    X = pack_csc(K, idx, val, counts)
    return X, dict(idx=idx, counts=counts, status=status, rnorm=rnorm, cap=cap,
                   err_mode=err_mode, eps=e)


def csc_matrix(X):
    K, indptr, indices, data = X
    return sp.csc_array((data, indices.astype(np.int32), indptr), shape=(K, indptr.size - 1))


# ---------------------------------------------------------------- MOD layer
def normalize_columns(M):
    """dictionary_update.py:56-69."""
    M = np.asarray(M, dtype=np.float64)
    scales = np.linalg.norm(M, axis=0)
    out = M.copy()
    nz = scales > 0
    out[:, nz] = out[:, nz] / scales[nz]
    return out, scales


def mod_update(Y, X, D_prev):
    """dictionary_update.py:72-114. Returns (D, residual_fro, unused, rank, scales)."""
    Y = np.asarray(Y, dtype=np.float64)
    D_prev = check_dictionary(D_prev)
    K = D_prev.shape[1]
    usage = np.bincount(X[2], minlength=K)
    if X[2].size == 0:
        return D_prev.copy(), float(np.linalg.norm(Y)), list(range(K)), 0, None
    Xc = csc_matrix(X)
    XXT = (Xc @ Xc.T).toarray()
    YXT = Y @ Xc.T
    sol, _r, rank, _sv = np.linalg.lstsq(XXT, YXT.T, rcond=RANK_RCOND)
    Dn = sol.T
    resid = float(np.linalg.norm(Y - Dn @ Xc))
    norms = np.linalg.norm(Dn, axis=0)
    top = norms.max() if norms.size else 0.0
    dead = (usage == 0) | (norms <= ZERO_NORM_REL * max(top, 1.0))
    Dn[:, dead] = D_prev[:, dead]
    Dout, _ = normalize_columns(Dn)
    return Dout, resid, list(np.flatnonzero(dead)), int(rank), norms


def replace_degenerate_atoms(D, Y, X):
    """dictionary_update.py:117-177. Returns (D, replaced, unreplaced)."""
    D = np.asarray(D, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    K = D.shape[1]
    usage = np.bincount(X[2], minlength=K)
    norms = np.linalg.norm(D, axis=0)
    bad = (usage == 0) | (norms <= ZERO_NORM_REL)
    Dn, _ = normalize_columns(D)
    C = np.abs(Dn.T @ Dn)
    np.fill_diagonal(C, 0.0)
    ii, jj = np.nonzero(np.triu(C > TWIN_COHERENCE, k=1))
    for i, j in zip(ii, jj):
        if not bad[i]:
            bad[j] = True
    targets = np.flatnonzero(bad)
    if targets.size == 0:
        return D.copy(), [], []
    res = np.linalg.norm(Y - D @ csc_matrix(X), axis=0)
    order = np.lexsort((np.arange(res.size), -res))
    ynorm = np.linalg.norm(Y, axis=0)
    out = D.copy()
    replaced, unreplaced = [], []
    pos = 0
    for a in targets:
        while pos < order.size and ynorm[order[pos]] == 0.0:
            pos += 1
        if pos >= order.size:
            unreplaced.append(int(a))
            continue
        c = order[pos]
        pos += 1
        out[:, a] = Y[:, c] / ynorm[c]
        replaced.append(int(a))
    return out, replaced, unreplaced


# ---------------------------------------------------------------- training
def overcomplete_dct(p: int, K: int) -> np.ndarray:
    """denoising.py:166-195 (an init option of the trainer)."""
    q = int(round(np.sqrt(K)))
    grid = np.arange(p)
    base = np.empty((q, p))
    for k in range(q):
        v = np.cos(np.pi * k * grid / q)
        if k > 0:
            v = v - v.mean()
        base[k] = v / np.linalg.norm(v)
    D = np.empty((p * p, K))
    for k in range(q):
        for l in range(q):
            D[:, k * q + l] = np.outer(base[k], base[l]).flatten(order="F")
    return D / np.linalg.norm(D, axis=0)


def init_dictionary(Y, K, init, seed):
    """trainer.py:138-162."""
    m, N = Y.shape
    if not isinstance(init, str):
        D0, _ = normalize_columns(np.asarray(init, dtype=np.float64))
    elif init == "first-columns":
        if N < K:
            raise OracleInputError("first-columns init needs N >= K")
        D0, _ = normalize_columns(Y[:, :K])
    else:
        p = int(round(np.sqrt(m)))
        D0 = overcomplete_dct(p, K)
    zero = np.linalg.norm(D0, axis=0) == 0
    if zero.any():
        rng = np.random.default_rng(np.random.SeedSequence(seed).spawn(1)[0])
        fill = rng.standard_normal((m, int(zero.sum())))
        D0[:, zero] = fill / np.linalg.norm(fill, axis=0)
    return D0


def train_standard(Y, K, s, iterations, init="first-columns", seed=0, eps=None, s_max=None,
                   threads=1):
    """trainer.py:165-197, plus the error-bounded coding extension used by
    BASELINE configs 2/3 (``eps``/``s_max``; SURVEY.md §7 hard part 9 and
    Appendix A: the same loop composed from omp_batch(eps, s_max))."""
    Y = np.asarray(Y, dtype=np.float64)
    D = init_dictionary(Y, K, init, seed)
    residuals = []
    kw = dict(s=s) if eps is None else dict(eps=eps, s_max=s_max)
    for it in range(iterations):
        X, _ = omp_codes(Y, D, threads=threads, **kw)
        D, resid, _u, _r, _sc = mod_update(Y, X, D)
        D, _rep, _unr = replace_degenerate_atoms(D, Y, X)
        residuals.append(resid)
    X, _ = omp_codes(Y, D, threads=threads, **kw)
    return D, X, residuals


def split_indices(N, L, seed):
    """trainer.py:200-217."""
    perm = np.random.default_rng(seed).permutation(N)
    base, extra = divmod(N, L)
    bounds = np.concatenate([[0], np.cumsum([base + (t < extra) for t in range(L)])])
    return [perm[bounds[t]:bounds[t + 1]] for t in range(L)]


def derive_seeds(seed, count):
    """trainer.py:263-265."""
    return [int(c.generate_state(1, np.uint64)[0])
            for c in np.random.SeedSequence(seed).spawn(count)]


def merge_dataset(locals_):
    """trainer.py:248-256: [||X_t||_F D_t] over locals with nonzero codes."""
    blocks = []
    for D_t, X_t in locals_:
        w = float(np.linalg.norm(X_t[3]))
        if w > 0.0:
            blocks.append(w * np.asarray(D_t, dtype=np.float64))
    if not blocks:
        raise OracleInputError("all local code matrices are zero")
    return np.concatenate(blocks, axis=1)


def _local_job(args):
    """One train_local in a worker process (1 BLAS thread, like the
    reference's process pool, trainer.py:301-305)."""
    Yt, K1, s1, its, seed_t, eps, s_max = args
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        D_t, X_t, _ = train_standard(Yt, K1, s1, its, "first-columns", seed_t, eps=eps, s_max=s_max)
    return D_t, X_t


def train_locals(Y, L, K1, s1, local_iters, seed, eps=None, s_max=None, threads=1, procs=1,
                 only=None):
    """split_dataset -> train_local for every shard (or the shard indices in
    ``only``); ``procs`` > 1 trains shards in a process pool."""
    Y = np.asarray(Y, dtype=np.float64)
    seeds = derive_seeds(seed, L + 1)
    parts = split_indices(Y.shape[1], L, seed)
    todo = list(range(L)) if only is None else list(only)
    jobs = [(np.ascontiguousarray(Y[:, parts[t]]), K1, s1, local_iters, seeds[t], eps, s_max) for t in todo]
    if procs > 1 and len(jobs) > 1:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(min(procs, len(jobs))) as pool:
            return pool.map(_local_job, jobs, chunksize=1)
    out = []
    for j in jobs:
        D_t, X_t, _ = train_standard(j[0], K1, s1, local_iters, "first-columns", j[4], eps=eps,
                                     s_max=s_max, threads=threads)
        out.append((D_t, X_t))
    return out


def split_merge(Y, L, K1, s1, local_iters, K, s2, merge_iters, seed, init="first-columns",
                eps=None, s_max=None, merge_eps=None, merge_s_max=None, threads=1, procs=1):
    """split_dataset -> train_local -> merge_dictionaries (trainer.py:220-260,
    295-311), i.e. train_split_merge without its evaluation pass (SURVEY
    Appendix A). Returns (D, locals)."""
    Y = np.asarray(Y, dtype=np.float64)
    seeds = derive_seeds(seed, L + 1)
    locals_ = train_locals(Y, L, K1, s1, local_iters, seed, eps, s_max, threads, procs)
    Ym = merge_dataset(locals_)
    kw = {} if merge_eps is None else dict(eps=merge_eps, s_max=merge_s_max)
    D, _X, _ = train_standard(Ym, K, s2, merge_iters, init, seeds[L], threads=threads, **kw)
    return D, locals_


# ---------------------------------------------------------------- denoising
def extract_patches(px, p, stride=1):
    """denoising.py:118-135: column-major vectorised windows, row-offset major."""
    H, W = px.shape
    R, C = (H - p) // stride + 1, (W - p) // stride + 1
    out = np.empty((p * p, R * C))
    for j in range(p):          # patch column offset
        for i in range(p):      # patch row offset
            out[i + j * p] = px[i:i + R * stride:stride, j:j + C * stride:stride].reshape(-1)
    return out


def reconstruct_from_patches(P, width, height, p, stride=1):
    """denoising.py:138-163: mean of all covering patch estimates."""
    R, C = (height - p) // stride + 1, (width - p) // stride + 1
    acc = np.zeros((height, width))
    cnt = np.zeros((height, width))
    for j in range(p):
        for i in range(p):
            acc[i:i + R * stride:stride, j:j + C * stride:stride] += P[i + j * p].reshape(R, C)
            cnt[i:i + R * stride:stride, j:j + C * stride:stride] += 1.0
    out = np.zeros((height, width))
    hit = cnt > 0
    out[hit] = acc[hit] / cnt[hit]
    return out


def denoise(noisy_px, D, sigma, patch_size=8, stride=1, eps_gain=8.5, s_max=None, threads=1):
    """denoising.py:223-239."""
    D = np.asarray(D, dtype=np.float64)
    p = patch_size
    cap = s_max if s_max is not None else p * p
    P = extract_patches(np.asarray(noisy_px, dtype=np.float64), p, stride)
    X, _ = omp_codes(P, D, eps=eps_gain * sigma, s_max=cap, threads=threads)
    est = np.asarray(D @ csc_matrix(X))
    H, W = noisy_px.shape
    return np.clip(reconstruct_from_patches(est, W, H, p, stride), 0.0, 255.0)


def mse_db(Y, D, X):
    """metrics.py:30-44."""
    Y = np.asarray(Y, dtype=np.float64)
    yf = np.linalg.norm(Y)
    R = Y - np.asarray(D, dtype=np.float64) @ csc_matrix(X)
    ratio = np.linalg.norm(R) / yf
    if ratio <= 0.0:
        return MSE_DB_FLOOR
    return float(max(20.0 * np.log10(ratio), MSE_DB_FLOOR))


def psnr(a, b):
    rmse = np.sqrt(np.mean((np.asarray(a, float) - np.asarray(b, float)) ** 2))
    return 300.0 if rmse == 0 else float(min(20 * np.log10(255.0 / rmse), 300.0))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def timed(fn, *a, **k):
    t0 = time.perf_counter()
    out = fn(*a, **k)
    return out, time.perf_counter() - t0
