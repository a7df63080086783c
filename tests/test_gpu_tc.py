"""tcgen05 3xTF32 correlation GEMM vs an FP64 reference of the same op.

alpha0[i, j] = <y_i, d_j> over ragged shards; tolerance: |err| <= 4e-6 *
||y_i|| ||d_j|| (FP32-level, 3xTF32 split precision), plus every shape edge
the kernel tiles: m not a multiple of 32 (TMA zero fill), K not a multiple
of 256 (partial N chunk), K < 32, tiles straddling shard ends.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _alpha(Y, Ds, sizes, use_tc):
    from paper_1403_4781_b200 import _engine as E
    from paper_1403_4781_b200 import _lib
    N, m = Y.shape
    P, K, _ = Ds.shape
    Yd = torch.from_numpy(Y.astype(np.float32)).cuda()
    Dd = torch.from_numpy(Ds.astype(np.float32)).cuda()
    off, mx = E.shard_offsets(sizes)
    out = torch.full((N, K), float("nan"), dtype=torch.float32, device="cuda")
    wb = _lib.load().sdb_correlate_workspace_bytes(0, P, m, K)
    ws = torch.empty((wb,), dtype=torch.uint8, device="cuda")
    _lib.call("sdb_correlate", 0, N, m, K, P, off.data_ptr(), mx, Yd.data_ptr(), m, Dd.data_ptr(),
              out.data_ptr(), K, int(use_tc), ws.data_ptr(), wb, E.stream())
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("m,K,sizes", [
    (64, 256, [1000, 777, 1]),
    (64, 512, [300, 300]),
    (144, 576, [513, 129]),
    (256, 1024, [200]),
    (64, 1024, [130, 127, 260]),
    (16, 24, [50, 70]),
    (12, 20, [7]),
    # several items per CTA, the walks cross shard and chunk boundaries and skip empty shards
    (64, 512, [9000, 0, 7000, 130, 0, 12000]),
    (64, 256, [0, 20000, 0, 0, 1, 15000, 0]),
    (144, 576, [6000, 0, 5000]),
])
def test_tc_correlation_matches_fp64(m, K, sizes):
    rng = np.random.default_rng(m * 1000 + K)
    P = len(sizes)
    N = sum(sizes)
    Y = rng.standard_normal((N, m)) * rng.uniform(0.1, 100, (N, 1))
    Ds = rng.standard_normal((P, K, m))
    Ds /= np.linalg.norm(Ds, axis=2, keepdims=True)
    Y32 = Y.astype(np.float32).astype(np.float64)
    D32 = Ds.astype(np.float32).astype(np.float64)
    got = _alpha(Y, Ds, sizes, use_tc=True)
    off = np.concatenate([[0], np.cumsum(sizes)])
    ref = np.empty((N, K))
    for p in range(P):
        ref[off[p]:off[p + 1]] = Y32[off[p]:off[p + 1]] @ D32[p].T
    scale = np.linalg.norm(Y32, axis=1)[:, None]
    err = np.abs(got - ref) / scale
    assert np.isfinite(got).all()
    assert err.max() <= 4e-6, err.max()


def test_tc_and_simt_agree():
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((4000, 64))
    D = rng.standard_normal((2, 256, 64))
    D /= np.linalg.norm(D, axis=2, keepdims=True)
    a = _alpha(Y, D, [2500, 1500], True)
    b = _alpha(Y, D, [2500, 1500], False)
    assert np.abs(a - b).max() <= 1e-4
