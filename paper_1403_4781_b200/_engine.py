"""Device-resident primitives over the C-ABI (torch is plumbing only:
device memory, the current CUDA stream and pinned host buffers).

Every function here launches sm_100a kernels from libsdb200.so; nothing
computes on the host.
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import SDB_F32, SDB_F32X, SDB_F64

PRECISIONS = ("fp64", "fp32")
# Singular-support guard on the Cholesky pivot (_kernels.py:18). FP64 keeps the
# reference's 1e-12; in FP32 that threshold is below the arithmetic's
# resolution (unit-norm atoms give pivots accurate to ~1e-7), so the FP32 mode
# uses 1e-6 ("FP32 divergences").
GUARD = {"fp64": 1e-12, "fp32": 1e-6}
MAX_K = 1024

_precision = os.environ.get("SPARSEDICT_B200_PRECISION", "fp64")


def set_precision(p: str) -> None:
    """Select the arithmetic of the GPU path: "fp64" (default; OMP bitwise
    identical to the reference) or "fp32" (fast mode, tcgen05 3xTF32
    correlation GEMM, tolerance-based parity)."""
    global _precision
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    _precision = p


def get_precision(override: str | None = None) -> str:
    p = override or _precision
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {PRECISIONS}")
    return p


def sdb_dtype(p: str) -> int:
    return SDB_F64 if p == "fp64" else SDB_F32


def torch_dtype(p: str):
    return torch.float64 if p == "fp64" else torch.float32


_dev_checked = False

# Optional per-call CUDA-event timers (bench.py roofline): name -> list of
# (start_event, end_event, algorithmic_bytes, flops). None = disabled.
KTIMER: dict | None = None
# with KTIMER on: device counters of the fused coding path (signals coded by
# sdb_code_step1, signals it deferred to sdb_omp_deferred)
KSTAT: dict = {}
# error-bounded FP32 coding through sdb_code_step1 + sdb_omp_deferred (False:
# sdb_correlate + sdb_omp; the codes are bitwise the same, tests compare both)
FUSE_STEP1 = True
# certified FP32 coding (sdb_certify): the FP32/TF32 kernels decide, signals
# whose decision margin is within CERT_TAU * ||y|| (or whose FP32 status is not
# OK) are re-coded by the exact FP64 kernel, every other signal's coefficients
# are refitted in FP64 on its support -> the reference's FP64 codes; MOD and
# replacement then run in FP64 on an FP64 copy of the signals
CERTIFY = os.environ.get("SDB_CERTIFY", "1") != "0"
CERT_TAU = float(os.environ.get("SDB_CERT_TAU", "4e-6"))
# FP32 coding with m <= 64, K <= 512, cap <= 8 through the fused tensor-core
# Batch-OMP (sdb_omp_tc: per-step D^T r on tcgen05, no alpha0 in HBM); False:
# sdb_correlate + sdb_omp (k_omp_fast)
OMP_TC = os.environ.get("SDB_OMP_TC", "1") != "0"
# the kernels' 32-bit chunk counters overshoot N by < 2^22 (sdb_capi.cu OMP_DYN_MAX_N)
DYN_MAX_N = (1 << 31) - (1 << 22)


def timed_call(name: str, nbytes: float, flops: float, fn, *args):
    if KTIMER is None or torch.cuda.is_current_stream_capturing():
        return _lib.call(fn, *args)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = _lib.call(fn, *args)
    e1.record()
    KTIMER.setdefault(name, []).append((e0, e1, float(nbytes), float(flops)))
    return rc


def device() -> torch.device:
    """The CUDA device; raises NativeUnavailable without an sm_100 GPU."""
    global _dev_checked
    if not _dev_checked:
        if not torch.cuda.is_available():
            raise _lib.NativeUnavailable("no CUDA device: the sparsedict-B200 path has no CPU fallback")
        _lib.load()
        torch.cuda.init()
        cc = _lib.load().sdb_device_cc()
        if cc < 100:
            raise _lib.NativeUnavailable(f"compute capability {cc / 10:.1f} < 10.0 (sm_100a build)")
        _dev_checked = True
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def empty(shape, dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=device())


# ---------------------------------------------------------------- ingest
def h2d_f64(a: np.ndarray) -> torch.Tensor:
    """Copy a host float64 array (any layout) to the device unchanged."""
    t = torch.from_numpy(np.ascontiguousarray(a) if not (a.flags.c_contiguous or a.flags.f_contiguous)
                         else a)
    return t.to(device(), non_blocking=False)


UPLOAD_CHUNK = 8 << 20      # f64 elements per staged chunk (64 MB)
UPLOAD_THREADS = int(os.environ.get("SDB_UPLOAD_THREADS", "8"))
_upload_ring: list | None = None
_upload_pool = None
_upload_lock = threading.Lock()      # one staged upload at a time (the ring is shared)


def upload_pageable(Yh: np.ndarray) -> torch.Tensor:
    """Contiguous pageable f64 host array -> device tensor of the same shape
    and strides. A plain cudaMemcpy from pageable memory runs at ~10 GB/s
    (the driver stages it on one thread); here host threads copy 64 MB chunks
    into a ring of three pinned buffers and every chunk crosses PCIe
    asynchronously while the next one is being staged."""
    global _upload_ring, _upload_pool
    flat = Yh.ravel(order="K")                       # a view: Yh is C- or F-contiguous
    n = flat.size
    out = empty((max(n, 1),), torch.float64)[:n]
    if n < 2 * UPLOAD_CHUNK or not flat.flags.c_contiguous:
        out.copy_(torch.from_numpy(np.ascontiguousarray(flat)))
        return torch.as_strided(out, Yh.shape, tuple(st // 8 for st in Yh.strides))
    with _upload_lock:
        if _upload_ring is None:
            from concurrent.futures import ThreadPoolExecutor
            _upload_ring = [[torch.empty((UPLOAD_CHUNK,), dtype=torch.float64, pin_memory=True), None]
                            for _ in range(3)]
            _upload_pool = ThreadPoolExecutor(max_workers=UPLOAD_THREADS)
        nt = UPLOAD_THREADS
        for k, lo in enumerate(range(0, n, UPLOAD_CHUNK)):
            hi = min(n, lo + UPLOAD_CHUNK)
            slot = _upload_ring[k % 3]
            if slot[1] is not None:
                slot[1].synchronize()                # the copy out of this buffer has finished
            dst = slot[0].numpy()
            step = -(-(hi - lo) // nt)
            futs = [_upload_pool.submit(np.copyto, dst[a:min(a + step, hi - lo)], flat[lo + a:min(lo + a + step, hi)])
                    for a in range(0, hi - lo, step)]
            for f in futs:
                f.result()
            out[lo:hi].copy_(slot[0][:hi - lo], non_blocking=True)
            if slot[1] is None:
                slot[1] = torch.cuda.Event()
            slot[1].record()
    return torch.as_strided(out, Yh.shape, tuple(st // 8 for st in Yh.strides))


def ingest_signals(Y, prec: str) -> tuple[torch.Tensor, int]:
    """m x N host (numpy f64, any order) or device tensor -> device N x m
    signal-major in the working precision. Returns (Ydev, nonfinite_flag)."""
    dt = sdb_dtype(prec)
    if isinstance(Y, torch.Tensor) and Y.is_cuda:
        src = Y.to(torch.float64) if Y.dtype != torch.float64 else Y
        m, N = src.shape
        s_row, s_col = src.stride()
    else:
        Yh = np.asarray(Y, dtype=np.float64)
        m, N = Yh.shape
        if not (Yh.flags.c_contiguous or Yh.flags.f_contiguous):
            Yh = np.asfortranarray(Yh)
        src = upload_pageable(Yh)
        s_row, s_col = (Yh.strides[0] // 8, Yh.strides[1] // 8)
    out = empty((N, m), torch_dtype(prec))
    bad = zeros((1,), torch.int32)
    _lib.call("sdb_ingest", dt, m, N, ptr(src), s_row, s_col, ptr(out), m, ptr(bad), stream())
    return out, bad


def ingest_for(Y, prec: str):
    """Host / device m x N signals -> (working-precision rows, FP64 rows or
    None, nonfinite flag). In certified FP32 mode the FP64 rows are kept as the
    authoritative data (the FP32 rows are their rounding, the kernels' input)."""
    if certifies(prec):
        Y64, bad = ingest_signals(Y, "fp64")
        return Y64.to(torch.float32), Y64, bad
    Yw, bad = ingest_signals(Y, prec)
    return Yw, None, bad


def dict_to_device(D: np.ndarray) -> torch.Tensor:
    """Host m x K f64 dictionary -> device (1, K, m) f64 atom-major."""
    D = np.asarray(D, dtype=np.float64)
    return torch.from_numpy(np.ascontiguousarray(D.T)).to(device()).unsqueeze(0)


def working_dict(D64: torch.Tensor, prec: str) -> torch.Tensor:
    if prec == "fp64":
        return D64
    out = empty(D64.shape, torch.float32)
    _lib.call("sdb_cast", SDB_F32, D64.numel(), ptr(D64), ptr(out), stream())
    return out


def gram(D64: torch.Tensor, prec: str) -> torch.Tensor:
    P, K, m = D64.shape
    G = empty((P, K, K), torch_dtype(prec))
    _lib.call("sdb_gram", sdb_dtype(prec), P, m, K, ptr(D64), ptr(G), stream())
    return G


def gram_pair(D64: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    """(G32, G64) of one pass over the dictionaries (certified FP32 mode); G32 is
    bitwise gram(D64, "fp32")."""
    P, K, m = D64.shape
    G64 = empty((P, K, K), torch.float64)
    G32 = empty((P, K, K), torch.float32)
    _lib.call("sdb_gram_pair", P, m, K, ptr(D64), ptr(G64), ptr(G32), stream())
    return G32, G64


# ---------------------------------------------------------------- coding
@dataclass
class DeviceCodes:
    """OMP results on the device (selection order)."""

    K: int
    cap: int
    idx: torch.Tensor      # (N, cap) int32
    val: torch.Tensor      # (N, cap) working precision
    counts: torch.Tensor   # (N,) int32
    status: torch.Tensor   # (N,) int8
    rnorm: torch.Tensor    # (N,) working precision (fp64 when certified)
    gap: torch.Tensor | None = None   # (N,) fp32 decision margin / ||y|| (sdb_omp_tc, when requested)
    vprec: str | None = None          # precision of val / rnorm when not the working one
    nfrag: torch.Tensor | None = None  # (1,) int32: signals re-decided in FP64 (certified codes)

    @property
    def N(self) -> int:
        return self.counts.shape[0]


class _PinnedRing:
    """Two pinned staging buffers used in turn. The H2D copy out of a buffer
    is asynchronous, so before the host overwrites a buffer it waits for the
    copy issued from it two calls ago (an event); back-to-back trainings
    without a device sync keep their host/device overlap and never race."""

    def __init__(self, dtype):
        self.dtype = dtype
        self.buf = [None, None]
        self.ev = [None, None]
        self.k = 0

    def take(self, n: int) -> torch.Tensor:
        k = self.k = self.k ^ 1
        if self.ev[k] is not None:
            self.ev[k].synchronize()
        if self.buf[k] is None or self.buf[k].numel() < n:
            self.buf[k] = torch.empty((max(n, 1),), dtype=self.dtype, pin_memory=True)
        return self.buf[k][:n]

    def to_device(self, host: torch.Tensor) -> torch.Tensor:
        out = host.to(device(), non_blocking=True)
        if self.ev[self.k] is None:
            self.ev[self.k] = torch.cuda.Event()
        self.ev[self.k].record()
        return out


_pinned_perm = _PinnedRing(torch.int64)
_pinned_js = _PinnedRing(torch.int32)


def split_permutation(N: int, seed) -> torch.Tensor:
    """Device int64 numpy.random.default_rng(seed).permutation(N), bit-identical.

    The host parses the PCG64 stream into the Fisher-Yates swap targets
    (native, multi-threaded, streamed into a pinned buffer); the device
    resolves the swaps in parallel (sdb_permutation_from_targets). Falls back
    to the all-host routine when the 32-bit draw path does not apply."""
    if 2 <= N <= 0x7fffffff:
        host = _pinned_js.take(N - 1)
        if _lib.swap_targets(N, seed, host.numpy()):
            js = _pinned_js.to_device(host)
            wsb = _lib.load().sdb_permutation_workspace_bytes(N)
            ws = empty((wsb,), torch.uint8)
            perm = empty((N,), torch.int64)
            _lib.call("sdb_permutation_from_targets", N, ptr(js), ptr(perm), ptr(ws), wsb, stream())
            return perm
    host = _pinned_perm.take(N)
    _lib.permutation(N, seed, out=host.numpy())
    return _pinned_perm.to_device(host)


def shard_offsets(sizes) -> tuple[torch.Tensor, int]:
    off = np.concatenate([[0], np.cumsum(np.asarray(sizes, dtype=np.int64))]).astype(np.int64)
    return torch.from_numpy(off).to(device()), int(max(sizes) if len(sizes) else 0)


def alpha_chunk_rows(K: int, prec: str) -> int:
    """Signals per coding chunk so that alpha0 stays <= 4 GiB."""
    return max(1, (4 << 30) // (K * (8 if prec == "fp64" else 4)))


def omp_tc_applies(m: int, K: int, cap: int, prec: str, use_tc: bool = True) -> bool:
    return (OMP_TC and use_tc and prec == "fp32"
            and bool(_lib.load().sdb_omp_tc_supported(m, K, cap)))


def code(Ydev: torch.Tensor, off: torch.Tensor, max_rows: int, DT: torch.Tensor, G: torch.Tensor,
         cap: int, eps: float, prec: str, use_tc: bool = True, out: DeviceCodes | None = None,
         ysq: torch.Tensor | None = None, want_rnorm: bool = True, want_gap: bool = False) -> DeviceCodes:
    """OMP over every row of Ydev; row i uses the dictionary of its shard.

    ysq: optional per-signal FP32 ||y||^2 from signal_sq (fp32 only; the
    codes are bitwise the same with or without it). want_rnorm=False leaves
    out.rnorm unwritten (the training loop never reads it)."""
    N, m = Ydev.shape
    P, K, _ = DT.shape
    dt = sdb_dtype(prec)
    tdt = torch_dtype(prec)
    if out is None:
        out = DeviceCodes(K, cap, empty((N, cap), torch.int32), empty((N, cap), tdt),
                          empty((N,), torch.int32), empty((N,), torch.int8), empty((N,), tdt))
    if N == 0:
        return out
    es = 8 if prec == "fp64" else 4
    fused1 = (FUSE_STEP1 and prec == "fp32" and use_tc and ysq is not None and eps > 0.0 and not want_rnorm
              and K <= 256 and m <= 256 and cap <= 32 and K % 4 == 0 and m % 4 == 0 and N <= DYN_MAX_N)
    if want_gap and prec == "fp32" and out.gap is None:
        out.gap = empty((N,), torch.float32)
    if not fused1 and N <= DYN_MAX_N and omp_tc_applies(m, K, cap, prec, use_tc):
        wb = _lib.load().sdb_omp_tc_workspace_bytes(P, m, K)
        ws = empty((wb,), torch.uint8)
        # algorithmic HBM bytes per signal: y row in, code row + count + status out
        timed_call("omp_tc", N * (4 * m + cap * 8 + 5 + (4 if want_rnorm else 0)), 2.0 * N * m * K * cap,
                   "sdb_omp_tc", N, m, K, P, ptr(off), ptr(Ydev), Ydev.stride(0), ptr(DT), ptr(G), cap,
                   float(eps), GUARD[prec], ptr(out.idx), ptr(out.val), ptr(out.counts), ptr(out.status),
                   ptr(out.rnorm) if want_rnorm else None, ptr(out.gap), ptr(ws), int(wb), stream())
        return out
    alpha = empty((N, K), tdt)
    if fused1:
        # error-bounded mode: GEMM + first greedy step fused, OMP only for the
        # signals that need more (bitwise the same codes as the path below)
        wb = _lib.load().sdb_code_step1_workspace_bytes(P, m, K)
        ws = empty((wb,), torch.uint8)
        ndef = ws[wb - 256:wb - 252].view(torch.int32)   # deferred count (written by the launch)
        timed_call("step1", N * (4 * m + 4), 2.0 * N * m * K, "sdb_code_step1", N, m, K, P, ptr(off),
                   ptr(Ydev), m, ptr(DT), ptr(G), ptr(ysq), cap, float(eps), GUARD[prec], ptr(alpha), K,
                   ptr(out.idx), ptr(out.val), ptr(out.counts), ptr(out.status),
                   ptr(out.gap) if want_gap else None, ptr(ws), int(wb), stream())
        timed_call("omp_deferred", 0.0, 0.0, "sdb_omp_deferred", N, m, K, P, ptr(off), ptr(alpha), K,
                   ptr(Ydev), m, ptr(DT), ptr(G), ptr(ysq), cap, float(eps), GUARD[prec], ptr(out.idx),
                   ptr(out.val), ptr(out.counts), ptr(out.status), ptr(out.gap) if want_gap else None,
                   ptr(ws), int(wb), stream())
        if KTIMER is not None and not torch.cuda.is_current_stream_capturing():
            if "deferred" not in KSTAT:
                KSTAT["deferred"] = zeros((1,), torch.int64)
                KSTAT["coded"] = 0
            KSTAT["deferred"].add_(ndef)
            KSTAT["coded"] += N
        return out
    cwb = _lib.load().sdb_correlate_workspace_bytes(dt, P, m, K) if use_tc else 0
    cws = empty((cwb,), torch.uint8) if cwb > 0 else None
    timed_call("correlate", N * (m + K) * es, 2.0 * N * m * K,
               "sdb_correlate", dt, N, m, K, P, ptr(off), max_rows, ptr(Ydev), m, ptr(DT),
               ptr(alpha), K, int(use_tc), ptr(cws), int(cwb), stream())
    sb = _lib.load().sdb_omp_scratch_bytes(dt, N, m, cap)
    scratch = empty((max(sb, 1),), torch.uint8) if sb > 0 else None
    # algorithmic HBM bytes per signal: alpha0 row + code row (idx+val) + count/status, plus
    # either ||y||^2 (precomputed) or y, plus rnorm when requested
    yb = 4 if (ysq is not None and prec == "fp32") else m * es
    timed_call("omp", N * (K * es + yb + cap * (4 + es) + 5 + (es if want_rnorm else 0)), 0.0,
               "sdb_omp", dt, N, m, K, P, ptr(off), ptr(alpha), K, ptr(Ydev), m, ptr(DT), ptr(G),
               cap, float(eps), GUARD[prec], ptr(out.idx), ptr(out.val), ptr(out.counts),
               ptr(out.status), ptr(out.rnorm) if want_rnorm else None,
               ptr(ysq) if (ysq is not None and prec == "fp32") else None,
               ptr(out.gap) if (want_gap and prec == "fp32") else None, ptr(scratch), int(sb), stream())
    return out


def certify(Y32: torch.Tensor, off: torch.Tensor, D64: torch.Tensor, G64: torch.Tensor, codes: DeviceCodes,
            eps: float, want_rnorm: bool = False, Y64: torch.Tensor | None = None) -> DeviceCodes:
    """FP64 certification of FP32 codes (sdb_certify): returns codes with FP64
    values (vprec "fp64"); idx / counts / status are updated in place for the
    re-decided signals. Y64: authoritative FP64 rows when Y32 rounds them.
    Shapes outside the certification kernels (cap > 32) return the FP32
    codes unchanged."""
    N, m = Y32.shape
    if codes.cap > 32 or m > 256 or D64.shape[1] > 1024:
        return codes
    P, K, _ = D64.shape
    cap = codes.cap
    val = empty((N, cap), torch.float64)
    rn = empty((N,), torch.float64) if want_rnorm else codes.rnorm
    lst = empty((max(N, 1),), torch.int32)
    nl = empty((1,), torch.int32)
    if N:
        assert Y64 is None or (Y64.shape == Y32.shape and Y64.stride(0) == Y32.stride(0))
        Dt64 = D64.transpose(1, 2).contiguous()      # P x m x K: coalesced c0 of the re-coded signals
        timed_call("certify", N * ((8 if Y64 is not None else 4) * m + cap * 12 + 9), 0.0, "sdb_certify", N, m, K,
                   P, ptr(off), ptr(Y32), ptr(Y64), Y32.stride(0), ptr(D64), ptr(Dt64), ptr(G64), cap, float(eps), CERT_TAU, ptr(codes.idx), ptr(val),
                   ptr(codes.counts), ptr(codes.status), ptr(rn) if want_rnorm else None, ptr(codes.gap),
                   ptr(lst), ptr(nl), stream())
        if KTIMER is not None and not torch.cuda.is_current_stream_capturing():
            if "fragile" not in KSTAT:
                KSTAT["fragile"] = zeros((1,), torch.int64)
                KSTAT["certified"] = 0
            KSTAT["fragile"].add_(nl)
            KSTAT["certified"] += N
    else:
        nl.zero_()
    return DeviceCodes(K, cap, codes.idx, val, codes.counts, codes.status, rn, gap=codes.gap,
                       vprec="fp64", nfrag=nl)


def certifies(prec: str) -> bool:
    return prec == "fp32" and CERTIFY


def code_shards(S: "ShardSet", D64: torch.Tensor, cap: int, eps: float, use_tc: bool = True,
                want_rnorm: bool = False) -> DeviceCodes:
    """The training loop's coding pass over every shard: FP32 kernels plus the
    FP64 certification in certified mode, the plain kernels otherwise."""
    prec = S.prec
    if certifies(prec):
        G, G64 = gram_pair(D64)
    else:
        G, G64 = gram(D64, prec), None
    codes = code(S.Y, S.off, S.max_rows, working_dict(D64, prec), G, cap, eps, prec, use_tc,
                 ysq=S.signal_sq(), want_rnorm=want_rnorm and not certifies(prec),
                 want_gap=certifies(prec))
    if not certifies(prec):
        return codes
    return certify(S.Y, S.off, D64, G64, codes, eps, want_rnorm,
                   Y64=S._exact.Y if (S._exact is not None and S._exact_auth) else None)


def signal_sq(Ydev: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-signal FP32 ||y||^2 with the fast OMP kernel's own arithmetic."""
    N, m = Ydev.shape
    if out is None:
        out = empty((max(N, 1),), torch.float32)
    _lib.call("sdb_signal_sq", N, m, ptr(Ydev), Ydev.stride(0), ptr(out), stream())
    return out[:N]


def code_single_dict(Ydev, D64, cap, eps, prec, use_tc=True, want_rnorm=True, Y64=None) -> DeviceCodes:
    """Code all rows of Ydev against one dictionary (P = 1), chunked.
    want_rnorm=False (callers that never read the residual norms, e.g. the
    denoiser) lets FP32 error-bounded coding take the fused path. Y64: the
    authoritative FP64 rows when Ydev rounds them (certified mode)."""
    N = Ydev.shape[0]
    DT = working_dict(D64, prec)
    cert = certifies(prec)
    if cert:
        G, G64 = gram_pair(D64)
    else:
        G = gram(D64, prec)
    K = D64.shape[1]
    rows = alpha_chunk_rows(K, prec)
    ysq = None
    if not want_rnorm and prec == "fp32" and eps > 0.0:
        ysq = signal_sq(Ydev)
    if N <= rows:
        off, mx = shard_offsets([N])
        c = code(Ydev, off, mx, DT, G, cap, eps, prec, use_tc, ysq=ysq, want_rnorm=want_rnorm and not cert,
                 want_gap=cert)
        return certify(Ydev, off, D64, G64, c, eps, want_rnorm, Y64=Y64) if cert else c
    tdt = torch_dtype(prec)
    res = DeviceCodes(K, cap, empty((N, cap), torch.int32), empty((N, cap), tdt),
                      empty((N,), torch.int32), empty((N,), torch.int8), empty((N,), tdt))
    if cert:
        res.val = empty((N, cap), torch.float64)
        res.rnorm = empty((N,), torch.float64)
        res.vprec = "fp64"
        res.nfrag = zeros((1,), torch.int32)
    for lo in range(0, N, rows):
        hi = min(N, lo + rows)
        off, mx = shard_offsets([hi - lo])
        if cert:
            view = DeviceCodes(K, cap, res.idx[lo:hi], empty((hi - lo, cap), tdt), res.counts[lo:hi],
                               res.status[lo:hi], empty((hi - lo,), tdt))
            c = code(Ydev[lo:hi], off, mx, DT, G, cap, eps, prec, use_tc, out=view,
                     ysq=None if ysq is None else ysq[lo:hi], want_rnorm=False, want_gap=True)
            cc = certify(Ydev[lo:hi], off, D64, G64, c, eps, want_rnorm,
                         Y64=None if Y64 is None else Y64[lo:hi])
            res.val[lo:hi].copy_(cc.val)
            if want_rnorm:
                res.rnorm[lo:hi].copy_(cc.rnorm)
            res.nfrag.add_(cc.nfrag)
            continue
        view = DeviceCodes(K, cap, res.idx[lo:hi], res.val[lo:hi], res.counts[lo:hi],
                           res.status[lo:hi], res.rnorm[lo:hi])
        code(Ydev[lo:hi], off, mx, DT, G, cap, eps, prec, use_tc, out=view,
             ysq=None if ysq is None else ysq[lo:hi], want_rnorm=want_rnorm)
    return res


def csc(codes: DeviceCodes, prec: str):
    """Device CSC packing -> (indptr, indices int64, data f64) device tensors."""
    prec = codes.vprec or prec
    N = codes.N
    indptr = empty((N + 1,), torch.int64)
    ws = empty((max(_lib.load().sdb_csc_workspace_bytes(N), 8),), torch.uint8)
    _lib.call("sdb_csc_indptr", N, ptr(codes.counts), ptr(indptr), ptr(ws), stream())
    nnz = int(indptr[N].item()) if N else 0
    indices = empty((max(nnz, 1),), torch.int64)
    data = empty((max(nnz, 1),), torch.float64)
    if N:
        _lib.call("sdb_csc_fill", sdb_dtype(prec), N, codes.cap, ptr(codes.idx), ptr(codes.val),
                  ptr(codes.counts), ptr(indptr), ptr(indices), ptr(data), stream())
    return indptr, indices[:nnz], data[:nnz]


def synth_sparse(D: np.ndarray, N: int, s: int, sigma: float, seed: int, prec: str,
                 want_support: bool = False):
    """On-device sparse-model signals (sdb_synth_sparse; synthesis.py:56-79
    plus additive noise): (N, m) device rows in the working precision, and
    optionally the (N, s) int32 supports in draw order."""
    D = np.asarray(D, dtype=np.float64)
    m, K = D.shape
    Dd = torch.from_numpy(np.ascontiguousarray(D.T)).to(device())
    Y = empty((N, m), torch_dtype(prec))
    sup = empty((N, s), torch.int32) if want_support else None
    _lib.call("sdb_synth_sparse", sdb_dtype(prec), N, m, K, s, ptr(Dd), float(sigma),
              int(seed) & ((1 << 64) - 1), ptr(Y), m, ptr(sup), stream())
    return (Y, sup) if want_support else Y


def d2h(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu").numpy()


# ---------------------------------------------------------------- MOD layer
RANK_RCOND = 1e-10   # dictionary_update.py:27 (used as the relative pivot tolerance)


@dataclass
class ShardSet:
    """Signals on the device, shard-contiguous: rows off[p]..off[p+1] of Y."""

    Y: torch.Tensor        # (N, m) working precision
    off: torch.Tensor      # (P+1,) int64 device
    sizes: list            # host copy of the shard sizes
    prec: str

    @property
    def P(self) -> int:
        return len(self.sizes)

    @property
    def N(self) -> int:
        return self.Y.shape[0]

    @property
    def m(self) -> int:
        return self.Y.shape[1]

    @property
    def max_rows(self) -> int:
        return int(max(self.sizes)) if self.sizes else 0

    _ysq: torch.Tensor | None = None
    _sig_sq: torch.Tensor | None = None

    def signal_sq(self) -> torch.Tensor | None:
        """Per-signal FP32 ||y||^2 for the fast OMP path (computed once; None
        in fp64 mode)."""
        if self.prec != "fp32":
            return None
        if self._sig_sq is None:
            self._sig_sq = signal_sq(self.Y)
        return self._sig_sq

    def energy(self) -> torch.Tensor:
        """||Y_p||_F^2 per shard (computed once, reused by every MOD step)."""
        if self._ysq is None:
            self._ysq = empty((self.P,), torch.float64)
            self._energy_into(self._ysq)
        return self._ysq

    def _energy_into(self, out: torch.Tensor):
        tmp = empty((max(self.N, 1),), torch.float64)
        _lib.call("sdb_shard_energy", sdb_dtype(self.prec), self.P, self.N, self.m,
                  ptr(self.off), ptr(self.Y), self.m, ptr(tmp), ptr(out), stream())

    _exact: "ShardSet | None" = None
    _exact_auth: bool = False   # the FP64 copy is the authoritative data (Y rounds it)

    def exact(self) -> "ShardSet":
        """FP64 copy of the signals (same shards) for the certified mode's
        FP64 MOD / replacement; created once, refreshed with the signals."""
        if self.prec == "fp64":
            return self
        if self._exact is None:
            self._exact = ShardSet(self.Y.double(), self.off, self.sizes, "fp64")
        return self._exact

    @classmethod
    def with_exact(cls, Y64: torch.Tensor, off: torch.Tensor, sizes: list, prec: str) -> "ShardSet":
        """Shards whose data are FP64 (e.g. the merge phase's scaled atoms):
        the working-precision copy for the coding kernels plus the FP64
        original for certification, MOD and replacement."""
        if prec == "fp64":
            return cls(Y64, off, sizes, "fp64")
        S = cls(Y64.to(torch_dtype(prec)), off, sizes, prec)
        S._exact = cls(Y64, off, sizes, "fp64")
        S._exact_auth = True
        return S

    def refresh(self):
        """Recompute the cached per-signal / per-shard quantities in place
        after Y was overwritten (their storage is kept: captured graphs
        hold these addresses)."""
        if self._sig_sq is not None:
            signal_sq(self.Y, out=self._sig_sq)
        if self._ysq is not None:
            self._energy_into(self._ysq)
        if self._exact is not None:
            if not self._exact_auth:
                self._exact.Y.copy_(self.Y)
            self._exact.refresh()

    @classmethod
    def single(cls, Y: torch.Tensor, prec: str) -> "ShardSet":
        off, _ = shard_offsets([Y.shape[0]])
        return cls(Y, off, [Y.shape[0]], prec)


@dataclass
class ModResult:
    D: torch.Tensor          # (P, K, m) f64, normalised
    scales: torch.Tensor     # (P, K) raw column norms
    usage: torch.Tensor      # (P, K) int32
    dead: torch.Tensor       # (P, K) int8
    resid: torch.Tensor      # (P,) f64
    rank: torch.Tensor       # (P,) int32
    deficient: torch.Tensor  # (P,) int32


def _for_codes(S: "ShardSet", codes: DeviceCodes) -> "ShardSet":
    """The shard set whose precision matches the codes' values (certified FP32
    codes carry FP64 values: MOD / replacement / residuals run in FP64 on the
    FP64 copy of the signals)."""
    if codes.vprec == "fp64" and S.prec != "fp64":
        return S.exact()
    return S


def mod_update(S: ShardSet, codes: DeviceCodes, D64: torch.Tensor) -> ModResult:
    Yrows = None
    if codes.vprec == "fp64" and S.prec == "fp32" and not S._exact_auth:
        # certified FP32: the FP32 rows hold the exact values of the FP64
        # copy -- read them (half the gather bytes), compute in FP64
        Yrows = S.Y
    S = _for_codes(S, codes)
    P, K, m = D64.shape
    dt = sdb_dtype(S.prec) if Yrows is None else SDB_F32X
    r = ModResult(empty((P, K, m), torch.float64), empty((P, K), torch.float64),
                  empty((P, K), torch.int32), empty((P, K), torch.int8),
                  empty((P,), torch.float64), empty((P,), torch.int32), empty((P,), torch.int32))
    wsb = _lib.load().sdb_mod_workspace_bytes(P, S.N, m, K, codes.cap)
    ws = empty((wsb,), torch.uint8)
    es = 8 if S.prec == "fp64" else 4
    if Yrows is not None:
        es = 4
    vb = 8 if (codes.vprec == "fp64" or S.prec == "fp64") else 4
    timed_call("mod_update", S.N * (2 * m * es + codes.cap * (4 + vb) + 4), 0.0, "sdb_mod_update", dt, P, S.N, m, K,
               codes.cap, ptr(S.off), ptr(S.Y if Yrows is None else Yrows), m,
              ptr(codes.idx), ptr(codes.val), ptr(codes.counts), ptr(D64), ptr(r.D),
              ptr(r.scales), ptr(r.usage), ptr(r.dead), ptr(r.resid), ptr(r.rank),
              ptr(r.deficient), RANK_RCOND, ptr(S.energy()), ptr(ws), wsb, stream())
    return r


def replace_degenerate(S: ShardSet, codes: DeviceCodes, D64: torch.Tensor, usage: torch.Tensor):
    """In place on D64; returns (flags (P,K) int8, ntarget (P,) int32)."""
    S = _for_codes(S, codes)
    P, K, m = D64.shape
    flags = empty((P, K), torch.int8)
    ntarget = empty((P,), torch.int32)
    wsb = _lib.load().sdb_replace_workspace_bytes(P, S.N, m, K)
    ws = empty((wsb,), torch.uint8)
    es = 8 if S.prec == "fp64" else 4
    # algorithmic bytes of the part that always runs (normalised copy of D,
    # |Dn^T Dn| twins, flags); the residual ranking pass over Y runs only for
    # shards with replacement targets and is not counted
    timed_call("replace", P * K * (2 * m + 2 * K) * 8 + P * K * 6, 0.0, "sdb_replace_degenerate", sdb_dtype(S.prec), P, S.N, m, K, codes.cap, ptr(S.off),
              ptr(S.Y), m, ptr(codes.idx), ptr(codes.val), ptr(codes.counts), ptr(usage),
              ptr(D64), ptr(flags), ptr(ntarget), ptr(ws), wsb, stream())
    return flags, ntarget


def code_usage(S: ShardSet, codes: DeviceCodes) -> torch.Tensor:
    u = empty((S.P, codes.K), torch.int32)
    _lib.call("sdb_code_usage", S.P, S.N, codes.K, codes.cap, ptr(S.off), ptr(codes.idx),
              ptr(codes.counts), ptr(u), stream())
    return u


def residual_sq(S: ShardSet, codes: DeviceCodes, D64: torch.Tensor, want_ysq=False):
    S = _for_codes(S, codes)
    P, K, m = D64.shape
    rsq = empty((max(S.N, 1),), torch.float64)
    ysq = empty((max(S.N, 1),), torch.float64) if want_ysq else None
    if S.N:
        _lib.call("sdb_residual_sq", sdb_dtype(S.prec), S.N, m, K, codes.cap, P, ptr(S.off),
                  ptr(S.Y), m, ptr(codes.idx), ptr(codes.val), ptr(codes.counts), ptr(D64),
                  ptr(rsq), ptr(ysq), stream())
    return rsq, ysq


def shard_sum(S: ShardSet, v: torch.Tensor, do_sqrt: bool) -> torch.Tensor:
    out = empty((S.P,), torch.float64)
    _lib.call("sdb_shard_sum", S.P, ptr(S.off), ptr(v), ptr(out), int(do_sqrt), stream())
    return out


def code_energy(S: ShardSet, codes: DeviceCodes) -> torch.Tensor:
    """||X_p||_F per shard (trainer.py:250)."""
    S = _for_codes(S, codes)
    e = empty((max(S.N, 1),), torch.float64)
    if S.N:
        _lib.call("sdb_code_energy", sdb_dtype(S.prec), S.N, codes.cap, ptr(codes.val),
                  ptr(codes.counts), ptr(e), stream())
    return shard_sum(S, e, True)


def codes_from_csc(indptr, indices, data, K: int, prec: str) -> DeviceCodes:
    N = indptr.size - 1
    counts = np.diff(indptr)
    cap = max(1, int(counts.max()) if N else 1)
    dip = torch.from_numpy(np.ascontiguousarray(indptr, dtype=np.int64)).to(device())
    dii = torch.from_numpy(np.ascontiguousarray(indices, dtype=np.int64)).to(device()) \
        if indices.size else zeros((1,), torch.int64)
    dd = torch.from_numpy(np.ascontiguousarray(data, dtype=np.float64)).to(device()) \
        if data.size else zeros((1,), torch.float64)
    tdt = torch_dtype(prec)
    c = DeviceCodes(K, cap, empty((max(N, 1), cap), torch.int32), empty((max(N, 1), cap), tdt),
                    empty((max(N, 1),), torch.int32), zeros((max(N, 1),), torch.int8),
                    zeros((max(N, 1),), tdt))
    if N:
        _lib.call("sdb_csc_to_codes", sdb_dtype(prec), N, cap, ptr(dip), ptr(dii), ptr(dd),
                  ptr(c.idx), ptr(c.val), ptr(c.counts), stream())
    c.idx, c.val, c.counts, c.status, c.rnorm = (c.idx[:N], c.val[:N], c.counts[:N],
                                                 c.status[:N], c.rnorm[:N])
    return c


def normalize_rows(D64: torch.Tensor):
    """normalize_columns on atom-major rows (any leading shape)."""
    m = D64.shape[-1]
    rows = D64.numel() // m
    out = empty(D64.shape, torch.float64)
    sc = empty(D64.shape[:-1], torch.float64)
    _lib.call("sdb_normalize", rows, m, ptr(D64), ptr(out), ptr(sc), stream())
    return out, sc


def host_mapped(arr) -> int | None:
    """Device address of a pinned, device-mapped host numpy array, else None."""
    dev = ctypes.c_void_p()
    if arr.size == 0 or _lib.load().sdb_host_mapped(arr.ctypes.data, ctypes.byref(dev)) != 0:
        return None
    return dev.value


def ingest_gather(src_ptr: int, ldi: int, perm: torch.Tensor, lo: int, hi: int, m: int, prec: str,
                  bad: torch.Tensor, head=(None, 0)) -> torch.Tensor:
    """Rows perm[lo:hi] of an f64 row-major source (device or mapped host
    address) -> device (hi-lo) x m in the working precision; bad |= non-finite.
    head = (device copy of the source's first rows, their number)."""
    rows = hi - lo
    out = empty((max(rows, 1), m), torch_dtype(prec))[:rows]
    dsrc, drows = head
    if dsrc is not None and drows > 0:
        _lib.call("sdb_ingest_gather_split", sdb_dtype(prec), rows, m, src_ptr, ldi, ptr(perm) + 8 * lo,
                  ptr(dsrc), drows, ptr(out), m, ptr(bad), stream())
    else:
        _lib.call("sdb_ingest_gather", sdb_dtype(prec), rows, m, src_ptr, ldi, ptr(perm) + 8 * lo,
                  ptr(out), m, ptr(bad), stream())
    return out


def gather_rows(Y: torch.Tensor, perm: torch.Tensor, prec: str) -> torch.Tensor:
    rows, m = perm.shape[0], Y.shape[1]
    out = empty((rows, m), Y.dtype)
    _lib.call("sdb_gather_rows", sdb_dtype(prec), rows, m, ptr(Y), Y.stride(0), ptr(perm),
              ptr(out), m, stream())
    return out


def first_columns(S: ShardSet, K: int):
    D = empty((S.P, K, S.m), torch.float64)
    zf = empty((S.P, K), torch.int32)
    _lib.call("sdb_first_columns", sdb_dtype(S.prec), S.P, K, S.m, ptr(S.off), ptr(S.Y), S.m,
              ptr(D), ptr(zf), stream())
    return D, zf


def scale_rows(D64: torch.Tensor, w: torch.Tensor, group: int, prec: str) -> torch.Tensor:
    rows, m = D64.shape[0] * D64.shape[1], D64.shape[2]
    out = empty((rows, m), torch_dtype(prec))
    _lib.call("sdb_scale_rows", sdb_dtype(prec), rows, group, m, ptr(D64), ptr(w), ptr(out),
              stream())
    return out
