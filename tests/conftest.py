import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def random_dictionary(rng, m, K):
    D = rng.standard_normal((m, K))
    return D / np.linalg.norm(D, axis=0)


def orthonormal_dictionary(rng, m, K):
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    return np.ascontiguousarray(Q[:, :K])


def load_golden(name):
    return np.load(GOLDEN / name, allow_pickle=False)


def golden_cases(z):
    return [str(n) for n in z["names"]]


def case(z, name):
    pre = name + "__"
    return {k[len(pre):]: z[k] for k in z.files if k.startswith(pre)}
