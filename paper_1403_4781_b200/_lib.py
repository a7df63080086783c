"""ctypes binding of the C-ABI library (include/sparsedict_b200.h).

The CUDA library is the ONLY compute path: there is no CPU fallback. If the
library is missing or no sm_100 device is present, every compute entry point
raises ``NativeUnavailable`` loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
# SDB_LIB: an alternative build of the same ABI (A/B comparisons of kernel versions)
LIB_PATH = Path(os.environ["SDB_LIB"]) if os.environ.get("SDB_LIB") else PKG / "libsdb200.so"

SDB_F32, SDB_F64, SDB_F32X = 0, 1, 2

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p

# name -> (restype, argtypes); mirrors include/sparsedict_b200.h
SIGNATURES = {
    "sdb_abi_version": (c_int, []),
    "sdb_last_error": (ctypes.c_char_p, []),
    "sdb_device_cc": (c_int, []),
    "sdb_ingest": (c_int, [c_int, c_i64, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "sdb_cast": (c_int, [c_int, c_i64, c_vp, c_vp, c_vp]),
    "sdb_gram": (c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "sdb_gram_pair": (c_int, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdb_correlate_workspace_bytes": (c_i64, [c_int, c_i64, c_i64, c_i64]),
    "sdb_correlate": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp,
                              c_vp, c_i64, c_int, c_vp, c_i64, c_vp]),
    "sdb_omp_scratch_bytes": (c_i64, [c_int, c_i64, c_i64, c_i64]),
    "sdb_omp": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                        c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                        c_i64, c_vp]),
    "sdb_signal_sq": (c_int, [c_i64, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "sdb_code_step1_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64]),
    "sdb_code_step1": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                               c_i64, c_dbl, c_dbl, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                               c_i64, c_vp]),
    "sdb_omp_deferred": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                 c_vp, c_vp, c_i64, c_dbl, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                                 c_i64, c_vp]),
    "sdb_certify": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl,
                            c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sdb_omp_tc_supported": (c_int, [c_i64, c_i64, c_i64]),
    "sdb_omp_tc_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64]),
    "sdb_omp_tc": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_i64, c_dbl, c_dbl,
                           c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sdb_csc_workspace_bytes": (c_i64, [c_i64]),
    "sdb_csc_indptr": (c_int, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdb_csc_fill": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sdb_mod_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64, c_i64, c_i64]),
    "sdb_mod_update": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp,
                               c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_dbl,
                               c_vp, c_vp, c_i64, c_vp]),
    "sdb_shard_energy": (c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "sdb_replace_workspace_bytes": (c_i64, [c_i64, c_i64, c_i64, c_i64]),
    "sdb_replace_degenerate": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64,
                                       c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sdb_code_usage": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sdb_residual_sq": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sdb_shard_sum": (c_int, [c_i64, c_vp, c_vp, c_vp, c_int, c_vp]),
    "sdb_code_energy": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdb_first_columns": (c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "sdb_scale_rows": (c_int, [c_int, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdb_gather_rows": (c_int, [c_int, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "sdb_csc_to_codes": (c_int, [c_int, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sdb_normalize": (c_int, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sdb_extract_patches": (c_int, [c_int, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "sdb_reconstruct": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp,
                                c_dbl, c_dbl, c_vp, c_vp]),
    "sdb_reconstruct_dense": (c_int, [c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "sdb_ingest_gather": (c_int, [c_int, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "sdb_ingest_gather_split": (c_int, [c_int, c_i64, c_i64, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64,
                                        c_vp, c_vp]),
    "sdb_copy_async": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "sdb_host_mapped": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "sdb_synth_sparse": (c_int, [c_int, c_i64, c_i64, c_i64, c_i64, c_vp, c_dbl, ctypes.c_uint64, c_vp, c_i64,
                                 c_vp, c_vp]),
    "sdb_pcg64_swap_targets": (c_int, [c_i64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_uint64, c_vp]),
    "sdb_permutation_workspace_bytes": (c_i64, [c_i64]),
    "sdb_permutation_from_targets": (c_int, [c_i64, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "sdb_pcg64_permutation": (c_int, [c_i64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_uint64, c_int, ctypes.c_uint32, c_vp]),
}


class NativeUnavailable(RuntimeError):
    """The sm_100a CUDA library or device is not available (no fallback)."""


class NativeError(RuntimeError):
    """A C-ABI call returned an error code."""


_lib = None
# must equal sdb_abi_version() in csrc/sdb_capi.cu (bumped whenever exports change)
ABI_VERSION = 12


def load():
    """Load (building first if needed) and bind the library."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        if os.environ.get("SDB_NO_BUILD"):
            raise NativeUnavailable(f"{LIB_PATH} is missing (run python -m paper_1403_4781_b200.build)")
        from . import build as _build
        _build.build()
    lib = ctypes.CDLL(str(LIB_PATH))
    lib.sdb_abi_version.restype = c_int
    got = lib.sdb_abi_version()
    if got != ABI_VERSION:
        raise NativeUnavailable(f"{LIB_PATH} has ABI {got}, expected {ABI_VERSION}: stale build "
                                "(run python -m paper_1403_4781_b200.build --force)")
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().sdb_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def permutation(n: int, seed, out=None):
    """numpy.random.default_rng(seed).permutation(n), bit-identical, computed
    by the native host routine (prefetched Fisher-Yates). ``out``: optional
    int64 buffer (e.g. a pinned torch tensor's numpy view)."""
    import numpy as np
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = st["state"]["state"], st["state"]["inc"]
    M = (1 << 64) - 1
    arr = np.empty(n, dtype=np.int64) if out is None else out
    check(load().sdb_pcg64_permutation(n, s >> 64, s & M, inc >> 64, inc & M,
                                       int(st["has_uint32"]), int(st["uinteger"]),
                                       arr.ctypes.data if n else None), "sdb_pcg64_permutation")
    return arr


def swap_targets(n: int, seed, out):
    """Fisher-Yates swap targets of numpy.random.default_rng(seed).permutation(n)
    into ``out`` (n - 1 uint32, e.g. a pinned tensor's numpy view). Returns
    False when the 32-bit fast path does not apply (caller falls back)."""
    import numpy as np
    st = np.random.default_rng(seed).bit_generator.state
    if n < 2 or n - 1 > 0xffffffff or int(st["has_uint32"]):
        return False
    s, inc = st["state"]["state"], st["state"]["inc"]
    M = (1 << 64) - 1
    check(load().sdb_pcg64_swap_targets(n, s >> 64, s & M, inc >> 64, inc & M, out.ctypes.data),
          "sdb_pcg64_swap_targets")
    return True


def call(name: str, *args) -> int:
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc
