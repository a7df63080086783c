"""Standard and split-and-merge dictionary training on the B200 — drop-in for
sparsedict.trainer (/root/reference/pkg/src/sparsedict/trainer.py).

The alternating loop (OMP coding, MOD update, atom replacement) is
device-resident: Y is uploaded once, every iteration is a fixed sequence of
stream-ordered launches with no host synchronisation, and the split phase
trains ALL L shards in the same launches (shard-batched kernels), instead of
the reference's process pool (trainer.py:301-305). Only the seeded host
pieces the reference defines through numpy's RNG stay on the host: the split
permutation (trainer.py:208-209), the seed derivation (:263-265) and the
random fill of zero init columns (:157-161).

Extensions (optional, reference-preserving defaults): ``TrainConfig.eps`` /
``s_max`` select error-bounded coding for standard / local training
(BASELINE configs 2-3; SURVEY.md §7 hard part 9), ``precision`` selects the
arithmetic ("fp64" default, "fp32" fast mode).
"""

from __future__ import annotations

import os
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _engine as E
from .dictionary_update import normalize_columns
from .exceptions import InvalidInputError
from .metrics import mse_db_device
from .sparse_coding import SparseCodeMatrix, codes_to_matrix

__all__ = [
    "TrainConfig",
    "TrainReport",
    "train_standard",
    "split_indices",
    "split_dataset",
    "train_local",
    "merge_dictionaries",
    "train_split_merge",
]

INIT_MODES = ("first-columns", "overcomplete-dct")
_CONFIG_FIELDS = {"K", "s", "iterations", "init", "seed", "mode", "L", "K1", "s1", "s2",
                  "local_iterations", "merge_iterations", "eps", "s_max", "precision"}


@dataclass
class TrainConfig:
    """Parameters of either training mode (trainer.py:44-111)."""

    K: int
    s: int
    iterations: int = 100
    init: str | np.ndarray = "first-columns"
    seed: int = 0
    mode: str = "standard"
    L: int = 1
    K1: int | None = None
    s1: int | None = None
    s2: int | None = None
    local_iterations: int | None = None
    merge_iterations: int | None = None
    threads: int = 1
    eps: float | None = None        # extension: error-bounded coding (standard / locals)
    s_max: int | None = None        # extension: support cap in error-bounded mode
    precision: str | None = None    # extension: "fp64" | "fp32"

    def validate(self) -> None:
        if self.K < 1 or self.s < 1 or self.iterations < 1:
            raise InvalidInputError("K, s, iterations must be positive")
        if isinstance(self.init, str):
            if self.init not in INIT_MODES:
                raise InvalidInputError(f"unknown init mode {self.init!r}")
        else:
            M = np.asarray(self.init, dtype=np.float64)
            if M.ndim != 2 or M.shape[1] != self.K:
                raise InvalidInputError("explicit init must be an (m, K) matrix")
        if self.eps is not None:
            e = float(self.eps)
            if e < 0 or not np.isfinite(e):
                raise InvalidInputError("eps must be a finite nonnegative real")
            if self.s_max is not None and int(self.s_max) < 1:
                raise InvalidInputError("s_max must be positive")
        if self.precision is not None:
            E.get_precision(self.precision)
        if self.mode == "standard":
            return
        if self.mode != "split-merge":
            raise InvalidInputError(f"unknown mode {self.mode!r}")
        if self.L < 1:
            raise InvalidInputError("L must be >= 1")
        if self.K1 is None or self.s1 is None or self.s2 is None:
            raise InvalidInputError("split-merge mode requires K1, s1 and s2")
        if self.s1 * self.s2 != self.s:
            raise InvalidInputError(
                f"sparsity levels must compose: s1*s2 = {self.s1}*{self.s2} != s = {self.s}")
        if self.K1 > self.K:
            raise InvalidInputError("K1 must not exceed K")

    @classmethod
    def from_dict(cls, d: dict) -> "TrainConfig":
        unknown = set(d) - _CONFIG_FIELDS
        if unknown:
            raise InvalidInputError(f"unknown config fields: {sorted(unknown)}")
        cfg = cls(**d)
        cfg.validate()
        return cfg

    def to_dict(self) -> dict:
        d = {"K": self.K, "s": self.s, "iterations": self.iterations, "seed": self.seed,
             "mode": self.mode,
             "init": self.init if isinstance(self.init, str) else "explicit-matrix"}
        if self.mode == "split-merge":
            d.update(L=self.L, K1=self.K1, s1=self.s1, s2=self.s2,
                     local_iterations=self.local_iterations,
                     merge_iterations=self.merge_iterations)
        for k in ("eps", "s_max", "precision"):
            if getattr(self, k) is not None:
                d[k] = getattr(self, k)
        return d


@dataclass
class TrainReport:
    """Timing and quality summary (trainer.py:114-135).

    local_wall_times_s: one entry per local, as in the reference; the locals
    of train_split_merge run concurrently in one batched launch sequence on
    the GPU (not in a process pool), so every entry is the same batched
    local-phase wall time (no per-shard timeline exists to report)."""

    final_mse_db: float
    per_iteration_residuals: list[float] = field(default_factory=list)
    wall_time_s: float = 0.0
    split_time_s: float = 0.0
    local_wall_times_s: list[float] = field(default_factory=list)
    merge_wall_time_s: float = 0.0
    critical_path_s: float = 0.0

    def to_dict(self) -> dict:
        return {
            "final_mse_db": self.final_mse_db,
            "per_iteration_residuals": list(self.per_iteration_residuals),
            "wall_time_s": self.wall_time_s,
            "split_time_s": self.split_time_s,
            "local_wall_times_s": list(self.local_wall_times_s),
            "merge_wall_time_s": self.merge_wall_time_s,
            "critical_path_s": self.critical_path_s,
        }


# ============================================================ device engine
def _zero_fill(D: torch.Tensor, zero_flags: np.ndarray, seeds) -> None:
    """Seeded N(0,1) atoms for zero init columns (trainer.py:156-161); the
    columns come from numpy's PCG64 so they match the reference exactly."""
    P, K, m = D.shape
    for p in range(P):
        z = np.flatnonzero(zero_flags[p])
        if z.size == 0:
            continue
        rng = np.random.default_rng(np.random.SeedSequence(int(seeds[p])).spawn(1)[0])
        fill = rng.standard_normal((m, z.size))
        cols = torch.from_numpy(np.ascontiguousarray((fill / np.linalg.norm(fill, axis=0)).T))
        D[p, torch.from_numpy(z)] = cols.to(D.device)


def init_dictionaries(S: E.ShardSet, K: int, init, seeds) -> torch.Tensor:
    """_init_dictionary (trainer.py:138-162) for every shard: (P, K, m) f64."""
    if S._exact is not None and S._exact_auth:
        S = S.exact()          # first columns of the authoritative FP64 data
    m = S.m
    if isinstance(init, str) and init == "first-columns":
        if min(S.sizes) < K:
            raise InvalidInputError("first-columns init needs N >= K")
        D, zf = E.first_columns(S, K)
        zfh = E.d2h(zf)
        if zfh.any():
            _zero_fill(D, zfh, seeds)
        return D
    if isinstance(init, str):  # overcomplete-dct
        from .denoising import overcomplete_dct
        p = int(round(np.sqrt(m)))
        if p * p != m:
            raise InvalidInputError("overcomplete-dct init needs a square patch dimension")
        D0 = overcomplete_dct(p, K)
    else:
        D0 = np.asarray(init, dtype=np.float64)
        if D0.shape != (m, K):
            raise InvalidInputError("explicit init has wrong shape")
        D0, _ = normalize_columns(D0)
    D = E.dict_to_device(D0).repeat(S.P, 1, 1).contiguous()
    zero = (np.linalg.norm(D0, axis=0) == 0)
    if zero.any():
        _zero_fill(D, np.tile(zero, (S.P, 1)), seeds)
    return D


def coding_mode(m: int, K: int, s: int, eps, s_max) -> tuple[int, float]:
    """(cap, eps) for the training loop (fixed s unless eps is given)."""
    if eps is None:
        if not 1 <= s <= min(m, K):
            raise InvalidInputError("sparsity must satisfy 1 <= s <= min(m, K)")
        return int(s), 0.0
    cap = int(s_max) if s_max is not None else m
    if not 1 <= cap <= m:
        raise InvalidInputError("s_max must satisfy 1 <= s_max <= m")
    return cap, float(eps)


USE_GRAPHS = True   # small jobs replay a cached graph (captured once per shape)
# jobs up to this many signals replay a graph per iteration (the static copy of
# the signals costs one device copy per training; larger jobs launch eagerly)
GRAPH_MAX_N = int(os.environ.get("SDB_GRAPH_MAX_N", str(1 << 23)))


def _iteration(S: E.ShardSet, D: torch.Tensor, cap: int, eps: float, use_tc: bool):
    """One alternating step (trainer.py:184-187): code, MOD, replace.
    Returns (new D, residual_fro per shard)."""
    codes = E.code_shards(S, D, cap, eps, use_tc)
    r = E.mod_update(S, codes, D)
    E.replace_degenerate(S, codes, r.D, r.usage)
    return r.D, r.resid


class _GraphedLoop:
    """One captured alternating iteration on static buffers, reused by every
    later call with the same shapes: the inputs (signals, initial
    dictionary) are copied in, ||y||^2 recomputed in place, and the graph is
    replayed once per iteration. The merge phase is host-launch bound
    (~40 small launches per iteration), which a replay removes; in the local
    phase it removes the inter-launch gaps and most of the host enqueue."""

    def __init__(self, S: E.ShardSet, D0: torch.Tensor, cap: int, eps: float, use_tc: bool):
        if S._exact is not None and S._exact_auth:
            self.S = E.ShardSet.with_exact(S._exact.Y.clone(), S.off.clone(), list(S.sizes), S.prec)
        else:
            self.S = E.ShardSet(S.Y.clone(), S.off.clone(), list(S.sizes), S.prec)
        self.S.signal_sq()
        self.D = D0.clone()
        # warm-up outside capture (first launches set kernel attributes and
        # fill the ShardSet's lazily computed per-signal / per-shard caches)
        _iteration(self.S, self.D.clone(), cap, eps, use_tc)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(self.graph, stream=s):
                D_new, self.rr = _iteration(self.S, self.D, cap, eps, use_tc)
                self.D.copy_(D_new)
        torch.cuda.current_stream().wait_stream(s)

    def load(self, S: E.ShardSet, D0: torch.Tensor):
        self.S.Y.copy_(S.Y)
        if self.S._exact_auth:
            self.S._exact.Y.copy_(S._exact.Y)
        self.S.refresh()
        self.D.copy_(D0)


_GRAPH_CACHE: "OrderedDict" = OrderedDict()
GRAPH_CACHE_MAX = 16
# total bytes the cached graphs may pin (static signal copy + the captured
# iteration's private pool: alpha, codes, MOD workspaces); LRU beyond that.
# Default: 40% of the device's memory (SDB_GRAPH_CACHE_GB overrides)
GRAPH_CACHE_BYTES = int(float(os.environ.get("SDB_GRAPH_CACHE_GB", "0")) * (1 << 30))


def _graph_cache_limit() -> int:
    if GRAPH_CACHE_BYTES > 0:
        return GRAPH_CACHE_BYTES
    return int(0.4 * torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)


def _graph_bytes(S: E.ShardSet, D0: torch.Tensor, cap: int) -> int:
    """Estimate of what one cached graph keeps resident."""
    P, K, m = D0.shape
    es = 8 if S.prec == "fp64" else 4
    N = S.N
    # the alpha0 matrix exists only on the paths that materialise it (not the
    # fused tensor-core OMP)
    alpha = 0 if E.omp_tc_applies(m, K, cap, S.prec) else N * K * es
    return (N * m * es * 2            # static Y copy + split/tf32 staging
            + (N * m * 8 + N * cap * 8 if E.certifies(S.prec) else 0)   # FP64 copy + FP64 code values
            + alpha                   # alpha0 (the coding pass's largest buffer)
            + N * cap * (4 + es) + N * 16
            + P * (K * K + 4 * K * m) * 8)


def _evict_one() -> None:
    key, g = _GRAPH_CACHE.popitem(last=False)
    dev = key[-3]
    torch.cuda.synchronize(dev)   # nothing may still replay it
    del g


def _graphed(S: E.ShardSet, D0: torch.Tensor, cap: int, eps: float, use_tc: bool,
             tag=None) -> "_GraphedLoop":
    # tag: callers that run several trainings of equal shape concurrently (shard
    # groups on their own streams) get one graph -- and static buffers -- each
    key = (S.prec, tuple(S.Y.shape), tuple(S.sizes), tuple(D0.shape), cap, float(eps), bool(use_tc),
           E.get_precision(None), E.FUSE_STEP1, E.CERTIFY, E.CERT_TAU, bool(S._exact_auth), torch.cuda.current_device(), _graph_bytes(S, D0, cap), tag)
    g = _GRAPH_CACHE.get(key)
    if g is not None:
        _GRAPH_CACHE.move_to_end(key)   # LRU: the hot shapes stay
        return g
    need = key[-2]
    limit = _graph_cache_limit()
    while _GRAPH_CACHE and (len(_GRAPH_CACHE) >= GRAPH_CACHE_MAX or
                            sum(k[-2] for k in _GRAPH_CACHE) + need > limit):
        _evict_one()
    while True:
        try:
            g = _GraphedLoop(S, D0, cap, eps, use_tc)
            break
        except torch.cuda.OutOfMemoryError:
            if not _GRAPH_CACHE:
                raise
            _evict_one()
            torch.cuda.empty_cache()
    _GRAPH_CACHE[key] = g
    return g


def train_device(S: E.ShardSet, D0: torch.Tensor, cap: int, eps: float, iterations: int,
                 use_tc: bool = True, use_graph: bool | None = None, graph_tag=None):
    """The alternating loop (trainer.py:183-188) on every shard at once.

    Returns (D (P,K,m) f64, final codes, residuals (iterations, P) f64 device).
    Stream-ordered; nothing here synchronises with the host. Small jobs (the
    merge phase: N <= GRAPH_MAX_N signals) replay a cached CUDA graph of one
    iteration (see _GraphedLoop); large ones launch eagerly (GPU bound).
    """
    prec = S.prec
    P = D0.shape[0]
    resid = E.empty((iterations, P), torch.float64)
    graph = (USE_GRAPHS and S.N <= GRAPH_MAX_N) if use_graph is None else use_graph
    if E.KTIMER is not None:
        graph = False   # per-call kernel timing (bench breakdown) needs eager launches
    if graph and iterations > 0:
        g = _graphed(S, D0, cap, eps, use_tc, graph_tag)
        g.load(S, D0)
        for it in range(iterations):
            g.graph.replay()
            resid[it].copy_(g.rr)
        D = g.D.clone()
    else:
        D = D0
        for it in range(iterations):
            D, rr = _iteration(S, D, cap, eps, use_tc)
            resid[it].copy_(rr)
    codes = E.code_shards(S, D, cap, eps, use_tc)
    return D, codes, resid


def _check_Y(Y) -> np.ndarray:
    Y = np.asarray(Y, dtype=np.float64)
    if Y.ndim != 2 or Y.shape[0] < 1:
        raise InvalidInputError("Y must be a nonempty m x N matrix")
    if Y.shape[0] > 256:
        raise InvalidInputError("signal dimension m > 256 is outside the GPU path")
    return Y


def _ingest_checked2(Y, prec):
    """(working-precision rows, authoritative FP64 rows or None)."""
    Yw, Y64, bad = E.ingest_for(Y, prec)
    if int(bad.item()):
        raise InvalidInputError("batch contains non-finite entries")
    return Yw, Y64


def _ingest_checked(Y, prec):
    Ydev, bad = E.ingest_signals(Y, prec)
    if int(bad.item()):
        raise InvalidInputError("batch contains non-finite entries")
    return Ydev


def _sync():
    torch.cuda.synchronize()


# ============================================================ public API
def train_standard(Y, cfg: TrainConfig) -> tuple[np.ndarray, SparseCodeMatrix, TrainReport]:
    """Alternating OMP / MOD / replacement on the whole dataset
    (trainer.py:165-197); returns (D, codes against the final D, report)."""
    cfg.validate()
    if cfg.mode != "standard":
        raise InvalidInputError("train_standard requires mode='standard'")
    Y = _check_Y(Y)
    m, N = Y.shape
    if cfg.K > E.MAX_K:
        raise InvalidInputError(f"K={cfg.K} exceeds the GPU path's limit of {E.MAX_K}")
    prec = E.get_precision(cfg.precision)
    cap, eps = coding_mode(m, cfg.K, cfg.s, cfg.eps, cfg.s_max)
    t0 = time.perf_counter()
    Yw, Y64 = _ingest_checked2(Y, prec)
    S = (E.ShardSet.with_exact(Y64, E.shard_offsets([N])[0], [N], prec) if Y64 is not None
         else E.ShardSet.single(Yw, prec))
    D0 = init_dictionaries(S, cfg.K, cfg.init, [cfg.seed])
    D, codes, resid = train_device(S, D0, cap, eps, cfg.iterations)
    _sync()
    wall = time.perf_counter() - t0
    report = TrainReport(final_mse_db=mse_db_device(S, codes, D),
                         per_iteration_residuals=[float(v) for v in E.d2h(resid[:, 0])],
                         wall_time_s=wall, critical_path_s=wall)
    return E.d2h(D[0]).T.copy(), codes_to_matrix(codes, prec), report


def split_indices(N: int, L: int, seed: int) -> list[np.ndarray]:
    """Seeded partition of range(N) into L blocks (trainer.py:200-217): a
    PCG64 permutation cut into consecutive blocks, the first N mod L one longer."""
    if L < 1 or L > N:
        raise InvalidInputError("require 1 <= L <= N")
    perm = E._lib.permutation(N, seed)
    base, extra = divmod(N, L)
    ends = np.cumsum([base + (1 if t < extra else 0) for t in range(L)])
    return np.split(perm, ends[:-1])


def split_dataset(Y, L: int, seed: int) -> list[np.ndarray]:
    """Column shards of Y (trainer.py:220-223)."""
    Y = np.asarray(Y, dtype=np.float64)
    return [Y[:, ids] for ids in split_indices(Y.shape[1], L, seed)]


def train_local(Y_t, K1: int, s1: int, iterations: int, seed: int,
                init: str | np.ndarray = "first-columns", threads: int = 1,
                precision: str | None = None, eps: float | None = None,
                s_max: int | None = None) -> tuple[np.ndarray, SparseCodeMatrix]:
    """One local dictionary: train_standard with (K1, s1) (trainer.py:226-233)."""
    cfg = TrainConfig(K=K1, s=s1, iterations=iterations, init=init, seed=seed, threads=threads,
                      precision=precision, eps=eps, s_max=s_max)
    D, X, _ = train_standard(Y_t, cfg)
    return D, X


def _merge_weights(local_results, prec) -> list[float]:
    """w_t = ||X_t||_F (trainer.py:250-251) as device reductions."""
    ws = []
    for _D, X_t in local_results:
        data = X_t.data if isinstance(X_t, SparseCodeMatrix) else np.asarray(X_t).reshape(-1)
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.size == 0:
            ws.append(0.0)
            continue
        v = torch.from_numpy(data).to(E.device())
        n = data.size
        off, _ = E.shard_offsets([n])
        e = E.empty((n,), torch.float64)
        counts = torch.ones((n,), dtype=torch.int32, device=E.device())
        E._lib.call("sdb_code_energy", E.SDB_F64, n, 1, E.ptr(v), E.ptr(counts), E.ptr(e), E.stream())
        out = E.empty((1,), torch.float64)
        E._lib.call("sdb_shard_sum", 1, E.ptr(off), E.ptr(e), E.ptr(out), 1, E.stream())
        ws.append(float(out.item()))
    return ws


def merge_dictionaries(local_results: list, K: int, s2: int, merge_iterations: int, seed: int,
                       init: str | np.ndarray = "first-columns", threads: int = 1,
                       precision: str | None = None) -> np.ndarray:
    """Global dictionary from the scaled local atoms (trainer.py:236-260)."""
    if not local_results:
        raise InvalidInputError("empty list of local dictionaries")
    prec = E.get_precision(precision)
    ws = _merge_weights(local_results, prec)
    keep = [t for t, w in enumerate(ws) if w > 0.0]
    if not keep:
        raise InvalidInputError("all local code matrices are zero")
    Dl = torch.stack([E.dict_to_device(np.asarray(local_results[t][0], dtype=np.float64))[0]
                      for t in keep])
    w = torch.tensor([ws[t] for t in keep], dtype=torch.float64, device=E.device())
    Ym = E.scale_rows(Dl.contiguous(), w, Dl.shape[1], prec)
    return _train_merge(Ym, K, s2, merge_iterations, seed, init, prec)[0]


def _train_merge(Ym: torch.Tensor, K: int, s2: int, iters: int, seed: int, init, prec: str):
    m = Ym.shape[1]
    cfg = TrainConfig(K=K, s=s2, iterations=iters, init=init, seed=seed)
    cfg.validate()
    cap, eps = coding_mode(m, K, s2, None, None)
    S = E.ShardSet.single(Ym, prec)
    D0 = init_dictionaries(S, K, init, [seed])
    D, codes, _ = train_device(S, D0, cap, eps, iters)
    return E.d2h(D[0]).T.copy(), D, codes


def _derive_seeds(seed: int, count: int) -> list[int]:
    """trainer.py:263-265."""
    return [int(c.generate_state(1, np.uint64)[0])
            for c in np.random.SeedSequence(seed).spawn(count)]


@dataclass
class SplitMergeResult:
    D: np.ndarray
    D_dev: torch.Tensor            # (1, K, m) f64
    local_D: torch.Tensor          # (L, K1, m) f64
    weights: np.ndarray            # (L,)
    split_s: float
    local_s: float
    merge_s: float
    wall_s: float
    codings: int                   # OMP signal-codings performed


_STREAMS: dict = {}


def _group_streams(G: int) -> tuple:
    """(copy stream, [work stream per shard group]) with priorities: the row
    gathers highest (PCIe is the bottleneck while rows arrive), then later
    groups above earlier ones — the last group to land has the longest
    remaining chain of iterations, the earlier groups have slack to fill the
    gaps (makespan ordering)."""
    key = G
    if key not in _STREAMS:
        lo, hi = torch.cuda.Stream.priority_range()   # (least, greatest); greatest is numerically lower
        levels = list(range(lo, hi - 1, -1))         # least ... greatest
        copy = torch.cuda.Stream(priority=levels[-1])
        work_levels = levels[:-1] or levels
        work = [torch.cuda.Stream(priority=work_levels[min(len(work_levels) - 1,
                                                           (g * len(work_levels)) // max(G, 1))])
                for g in range(G)]
        _STREAMS[key] = (copy, work)
    return _STREAMS[key]


def _split_locals(src, N: int, m: int, L: int, K1: int, local_cap: int, local_eps: float,
                  local_iters: int, seeds, perm: torch.Tensor, prec: str, use_tc: bool, groups: int,
                  host_f64: int | None = None, bad: torch.Tensor | None = None, head=(None, 0),
                  src64: torch.Tensor | None = None):
    """split_dataset + every train_local (trainer.py:291-305), in G groups of
    consecutive shards, each on its own CUDA stream. The group's rows are
    gathered in permuted order (all gathers in order on one copy stream, so
    group 0's rows land first), then the group trains as soon as they are
    there, overlapping later groups' gathers and each other's latency-bound
    MOD steps. src: device (N, m) working-precision signals, or ``host_f64``:
    the device address of pinned, mapped host f64 rows (the transfer over
    PCIe then is the gather itself). Shards are independent, so the result
    equals the one-group (batched) computation. Returns (Dl, w) on the
    caller's stream."""
    base, extra = divmod(N, L)
    sizes = [base + (1 if t < extra else 0) for t in range(L)]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if min(sizes) < K1:
        raise InvalidInputError("first-columns init needs N >= K")
    G = max(1, min(int(groups), L))
    # certified FP32 with FP64 input: the shards keep the authoritative FP64
    # rows (the FP32 copy feeds the coding kernels)
    exact_in = E.certifies(prec) and (src64 is not None or host_f64 is not None)

    def shardset(Yg, off, sz):
        if exact_in:
            return E.ShardSet.with_exact(Yg, off, sz, prec)
        return E.ShardSet(Yg, off, sz, prec)

    gprec = "fp64" if exact_in else prec
    gsrc = src64 if (exact_in and src64 is not None) else src
    if G == 1 and host_f64 is None:
        # one batch on the caller's stream (no cross-stream allocations)
        Ys = E.gather_rows(gsrc, perm, gprec)
        off, _ = E.shard_offsets(sizes)
        S = shardset(Ys, off, sizes)
        D0 = init_dictionaries(S, K1, "first-columns", seeds[:L])
        Dl, codes, _ = train_device(S, D0, local_cap, local_eps, local_iters, use_tc)
        return Dl, E.code_energy(S, codes)
    bounds = [(g * L) // G for g in range(G + 1)]   # (unequal splits measured no better)
    main = torch.cuda.current_stream()
    copy, work = _group_streams(G)
    ready = []
    copy.wait_stream(main)   # perm (and a device source) are ready
    with torch.cuda.stream(copy):
        for g in range(G):
            r0, r1 = int(offs[bounds[g]]), int(offs[bounds[g + 1]])
            if host_f64 is not None:
                Ys = E.ingest_gather(host_f64, m, perm, r0, r1, m, gprec, bad[g:g + 1], head=head)
            else:
                Ys = E.gather_rows(gsrc, perm[r0:r1], gprec)
            ev = torch.cuda.Event()
            ev.record(copy)
            ready.append((Ys, ev))
    outD, outw = [], []
    for g in range(G):
        a, b = bounds[g], bounds[g + 1]
        s = work[g]
        Ys, ev = ready[g]
        if host_f64 is not None:
            ev.synchronize()  # validate the group's rows before any compute on them
            if int(bad[g].item()):
                # later gathers (copy stream) and earlier groups (work streams)
                # still use perm / bad / the head rows: drain them before the
                # allocator may hand those blocks out again
                copy.synchronize()
                for w_s in work:
                    w_s.synchronize()
                raise InvalidInputError("batch contains non-finite entries")
        s.wait_event(ev)
        Ys.record_stream(s)
        with torch.cuda.stream(s):
            off, _ = E.shard_offsets(sizes[a:b])
            S = shardset(Ys, off, sizes[a:b])
            D0 = init_dictionaries(S, K1, "first-columns", seeds[a:b])
            # one graph per group: equal-shaped groups run concurrently on their
            # own streams and must not share a graph's static buffers
            Dl, codes, _ = train_device(S, D0, local_cap, local_eps, local_iters, use_tc,
                                        graph_tag=("group", g, G))
            w = E.code_energy(S, codes)
        Dl.record_stream(main)
        w.record_stream(main)
        outD.append(Dl)
        outw.append(w)
    for s in work:
        main.wait_stream(s)
    if G == 1:
        return outD[0], outw[0]
    return torch.cat(outD), torch.cat(outw)


def _merge(Dl: torch.Tensor, w: torch.Tensor, K1: int, m: int, K: int, s2: int, merge_iters: int,
           seed_merge: int, init, prec: str, use_tc: bool):
    """merge_dictionaries (trainer.py:236-260) on the device-resident locals."""
    L = Dl.shape[0]
    w_h = E.d2h(w)
    keep = np.flatnonzero(w_h > 0.0)
    if keep.size == 0:
        raise InvalidInputError("all local code matrices are zero")
    if keep.size < L:
        kt = torch.from_numpy(keep).to(E.device())
        Dk, wk = Dl.index_select(0, kt).contiguous(), w.index_select(0, kt).contiguous()
    else:
        Dk, wk = Dl, w
    cap2, _ = coding_mode(m, K, s2, None, None)
    Sm, D0m = merge_data(Dk, wk, K1, K, init, seed_merge, prec)
    Dm, _codes_m, _ = train_device(Sm, D0m, cap2, 0.0, merge_iters, use_tc)
    return Dm, w_h, Sm.N


def merge_data(Dk: torch.Tensor, wk: torch.Tensor, K1: int, K: int, init, seed_merge: int, prec: str):
    """The merge training set [w_t D_t] (trainer.py:248-256) as shards plus
    the merge's initial dictionary. Certified mode keeps the pooled scaled
    atoms in FP64 (the FP32 copy only feeds the coding kernels), like the
    reference's merge data."""
    if E.certifies(prec):
        Ym64 = E.scale_rows(Dk, wk, K1, "fp64")
        Sm = E.ShardSet.with_exact(Ym64, E.shard_offsets([Ym64.shape[0]])[0], [Ym64.shape[0]], prec)
        return Sm, init_dictionaries(Sm.exact(), K, init, [seed_merge])
    Sm = E.ShardSet.single(E.scale_rows(Dk, wk, K1, prec), prec)
    return Sm, init_dictionaries(Sm, K, init, [seed_merge])


def split_merge_device(Ydev: torch.Tensor, L: int, K1: int, local_cap: int, local_eps: float,
                       local_iters: int, K: int, s2: int, merge_iters: int, seed: int,
                       init="first-columns", prec: str = "fp64", use_tc: bool = True,
                       t_start: float | None = None, perm: torch.Tensor | None = None,
                       groups: int = 1, src64: torch.Tensor | None = None) -> SplitMergeResult:
    """split_dataset -> locals (all shards batched, optionally in ``groups``
    concurrent shard groups) -> merge (trainer.py:291-313). ``Ydev`` is
    (N, m) device, signal-major."""
    if t_start is None:
        _sync()
        t_start = time.perf_counter()
    N, m = Ydev.shape
    if not 1 <= L <= N:
        raise InvalidInputError("require 1 <= L <= N")
    # split_indices' blocks are consecutive slices of one PCG64 permutation
    # (native, bit-identical to numpy; ``perm`` may be precomputed by the caller)
    if perm is None:
        perm = E.split_permutation(N, seed)
    t_split = time.perf_counter()
    seeds = _derive_seeds(seed, L + 1)
    Dl, w = _split_locals(Ydev, N, m, L, K1, local_cap, local_eps, local_iters, seeds, perm, prec,
                          use_tc, groups, src64=src64)
    w_h = E.d2h(w)                       # synchronises: end of the split phase
    t_local = time.perf_counter()
    Dm, w_h, n_merge = _merge(Dl, w, K1, m, K, s2, merge_iters, seeds[L], init, prec, use_tc)
    _sync()
    t_end = time.perf_counter()
    codings = (local_iters + 1) * N + (merge_iters + 1) * n_merge
    return SplitMergeResult(E.d2h(Dm[0]).T.copy(), Dm, Dl, w_h, t_split - t_start,
                            t_local - t_split, t_end - t_local, t_end - t_start, codings)


HOST_GROUPS = int(os.environ.get("SDB_HOST_GROUPS", "2"))  # shard groups streamed from pinned host memory (C4 e2e: 253 ms with 2, 258 with 3, 262 with 4)


def auto_groups(L: int) -> int:
    """Concurrent shard groups for device-resident split phases. One batch:
    every phase kernel now fills the SMs by itself (the fused OMP and the
    dictionary-resident refit take a whole SM's shared memory), so groups on
    their own streams no longer overlap anything (C4 job: 227.7 ms with one
    batch, 225 ms +- outliers with two, 236 ms with four, 242 ms with eight;
    four was best, 301.6 vs 316.0 ms, before those kernels)."""
    return 1
# 1/HEAD_DIV of a host batch is copied ahead (during the host permutation)
HEAD_DIV = int(os.environ.get("SDB_HEAD_DIV", "8"))


def _split_merge_host(src: int, N: int, m: int, cfg, cap1: int, eps1: float, local_iters: int,
                      merge_iters: int, prec: str, t0: float) -> SplitMergeResult:
    """train_split_merge's device pipeline for pinned host input (``src``:
    device address of the f64 N x m rows). While the host forms the split
    permutation, the first rows of the batch (in source order) are copied to
    the device; the group gathers then read those from HBM and only the rest
    over PCIe."""
    G = max(1, min(int(HOST_GROUPS), cfg.L))
    copy, _ = _group_streams(G)
    head = N // HEAD_DIV if HEAD_DIV > 0 else 0
    Yhead = None
    if head > 0:
        Yhead = E.empty((head, m), torch.float64)
        copy.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(copy):
            E._lib.call("sdb_copy_async", E.ptr(Yhead), src, head * m * 8, E.stream())
    perm = E.split_permutation(N, cfg.seed)
    t_split = time.perf_counter()
    seeds = _derive_seeds(cfg.seed, cfg.L + 1)
    bad = E.zeros((max(1, cfg.L),), torch.int32)  # one non-finite flag per group (<= L groups)
    Dl, w = _split_locals(None, N, m, cfg.L, cfg.K1, cap1, eps1, local_iters, seeds, perm, prec,
                          True, HOST_GROUPS, host_f64=src, bad=bad, head=(Yhead, head))
    t_local = time.perf_counter()
    Dm, w_h, n_merge = _merge(Dl, w, cfg.K1, m, cfg.K, cfg.s2, merge_iters, seeds[cfg.L],
                              cfg.init, prec, True)
    _sync()
    t_end = time.perf_counter()
    codings = (local_iters + 1) * N + (merge_iters + 1) * n_merge
    return SplitMergeResult(E.d2h(Dm[0]).T.copy(), Dm, Dl, w_h, t_split - t0, t_local - t_split,
                            t_end - t_local, t_end - t0, codings)


def train_split_merge(Y, cfg: TrainConfig, evaluate: bool = True) -> tuple[np.ndarray, TrainReport]:
    """Split / all-locals-at-once / merge pipeline (trainer.py:275-326),
    followed by the s1*s2 evaluation pass that is not counted in wall time
    (``evaluate=False``, an extension, skips it: final_mse_db is then nan)."""
    cfg.validate()
    if cfg.mode != "split-merge":
        raise InvalidInputError("train_split_merge requires mode='split-merge'")
    Y = _check_Y(Y)
    m, N = Y.shape
    if max(cfg.K, cfg.K1) > E.MAX_K:
        raise InvalidInputError(f"K exceeds the GPU path's limit of {E.MAX_K}")
    if cfg.L > N:
        raise InvalidInputError("require 1 <= L <= N")
    prec = E.get_precision(cfg.precision)
    local_iters = cfg.local_iterations or cfg.iterations
    merge_iters = cfg.merge_iterations or cfg.iterations
    cap1, eps1 = coding_mode(m, cfg.K1, cfg.s1, cfg.eps, cfg.s_max)
    _sync()
    t0 = time.perf_counter()
    src = E.host_mapped(Y.T) if Y.T.flags.c_contiguous else None
    Ydev = Ydev64 = None
    if src is not None:
        # pinned, signal-major host input: each shard group's rows cross PCIe
        # directly in permuted order and the group trains as soon as they land
        r = _split_merge_host(src, N, m, cfg, cap1, eps1, local_iters, merge_iters, prec, t0)
    else:
        # the split permutation (host, native) runs while Y streams to the device
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=1) as ex:
            fut = ex.submit(E.split_permutation, N, cfg.seed)
            Ydev, Ydev64 = _ingest_checked2(Y, prec)
            perm = fut.result()
        r = split_merge_device(Ydev, cfg.L, cfg.K1, cap1, eps1, local_iters, cfg.K, cfg.s2,
                               merge_iters, cfg.seed, cfg.init, prec, t_start=t0, perm=perm, src64=Ydev64,
                               groups=auto_groups(cfg.L))
    # evaluation pass (trainer.py:315-319), outside wall_time_s
    mse = float("nan")
    if evaluate:
        if Ydev is None:
            Ydev, Ydev64 = _ingest_checked2(Y, prec)
        S = (E.ShardSet.with_exact(Ydev64, E.shard_offsets([N])[0], [N], prec) if Ydev64 is not None
             else E.ShardSet.single(Ydev, prec))
        cap_e, _ = coding_mode(m, cfg.K, cfg.s, None, None)
        codes = E.code_single_dict(S.Y, r.D_dev, cap_e, 0.0, prec,
                                   Y64=Ydev64 if Ydev64 is not None else None)
        mse = mse_db_device(S, codes, r.D_dev)
    report = TrainReport(final_mse_db=mse, wall_time_s=r.wall_s,
                         # the L locals run concurrently in one batched launch sequence: they
                         # start and finish together, so each local's wall time is the local
                         # phase's (the reference's pool workers each report their own; here
                         # there is no per-shard timeline to report)
                         split_time_s=r.split_s, local_wall_times_s=[r.local_s] * cfg.L,
                         merge_wall_time_s=r.merge_s,
                         critical_path_s=r.split_s + r.local_s + r.merge_s)
    return r.D, report
