"""The C-ABI library loads without a GPU and exports exactly what
include/sparsedict_b200.h declares (no compute calls: CPU-only test)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "sparsedict_b200.h"


def declared():
    src = HEADER.read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entries():
    names = declared()
    assert "sdb_omp" in names and "sdb_mod_update" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    from paper_1403_4781_b200 import _lib
    lib = _lib.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert missing == []


def test_python_binding_covers_header():
    from paper_1403_4781_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared()


def test_abi_version_and_no_device():
    from paper_1403_4781_b200 import _lib
    lib = _lib.load()
    assert lib.sdb_abi_version() == _lib.ABI_VERSION
    import torch
    if not torch.cuda.is_available():
        assert lib.sdb_device_cc() < 0
        assert b"device" in lib.sdb_last_error()


def test_bad_args_rejected_without_launch():
    from paper_1403_4781_b200 import _lib
    lib = _lib.load()
    rc = lib.sdb_omp(7, 1, 1, 1, 1, None, None, 1, None, 1, None, None, 1, 0.0, 1e-12,
                     None, None, None, None, None, None, None, None, 0, None)
    assert rc == -22
    assert b"bad args" in lib.sdb_last_error()
    assert lib.sdb_signal_sq(-1, 64, None, 64, None, None) == -22


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    import paper_1403_4781_b200 as sdb
    D = np.eye(4)
    with pytest.raises(sdb._lib.NativeUnavailable if hasattr(sdb, "_lib") else RuntimeError):
        sdb.omp_batch(np.ones((4, 3)), D, s=1)
