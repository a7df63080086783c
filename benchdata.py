"""Seeded synthetic inputs for the BASELINE.json configurations (harness only).

No public dataset is involved: the reference's own corpus (skimage sample
images) is absent, and BASELINE.json defines every config synthetically.
Generated once in float64 with PCG64; the GPU path and the CPU oracle get
the same values (FP32 runs see FP32-representable values on both sides).

  C1  sparse model m=64, K=256, N=20,000, s=5, sigma=0.01; split P=4
  C2  8 synthetic 512x512 images (20 edges / sinusoids / blobs each, scaled
      to [0,255]) + N(0, 20^2) noise; all 8x8 patches stride 1, DC removed
      (2,040,200 x 64); split P=16, eps = 1.15*20*8 = 184, s <= 16
  C3  same generator, sigma=25, 12x12 patches stride 2 (504,008 x 144)
  C4  sparse model m=64, K=512, N=4,000,000, s=8, sigma=0.02; P=256
  C5  coding sweep, N=1,000,000, (m,K) in {(64,256),(64,1024),(144,576),(256,1024)}
"""

from __future__ import annotations

import numpy as np


def gen_dictionary(m: int, K: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((m, K))
    return D / np.linalg.norm(D, axis=0)


def sparse_signals(D: np.ndarray, N: int, s: int, sigma: float, seed: int,
                   chunk: int = 1 << 18) -> np.ndarray:
    """Y (N x m, signal-major == F-order m x N): s distinct uniform atoms per
    signal with N(0,1) coefficients plus N(0, sigma^2) noise (vectorised)."""
    m, K = D.shape
    rng = np.random.default_rng(seed)
    Y = np.empty((N, m))
    Dt = np.ascontiguousarray(D.T)
    for lo in range(0, N, chunk):
        n = min(chunk, N - lo)
        # s distinct atoms per signal: partial Fisher-Yates via argpartition of uniforms
        sup = np.argpartition(rng.random((n, K)), s - 1, axis=1)[:, :s] if s < K else \
            np.tile(np.arange(K), (n, 1))
        coef = rng.standard_normal((n, s))
        blk = np.einsum("ns,nsm->nm", coef, Dt[sup])
        blk += sigma * rng.standard_normal((n, m))
        Y[lo:lo + n] = blk
    return Y


def sparse_signals_device(D: np.ndarray, N: int, s: int, sigma: float, seed: int, prec: str = "fp32"):
    """The same sparse model generated on the GPU (sdb_synth_sparse, counter-
    based Philox stream): (N, m) device tensor. The oracle is fed the very same
    values (copy back the rows it needs)."""
    from paper_1403_4781_b200 import _engine as E
    return E.synth_sparse(D, N, s, sigma, seed, prec)


def synthetic_image(rng, size: int = 512, n_components: int = 20) -> np.ndarray:
    """Sum of random-oriented step edges, 2-D sinusoids (0.01-0.2 cyc/px) and
    Gaussian blobs, min-max scaled to [0, 255]."""
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    img = np.zeros((size, size))
    for _ in range(n_components):
        kind = rng.integers(0, 3)
        amp = rng.uniform(0.3, 1.0) * rng.choice([-1.0, 1.0])
        th = rng.uniform(0, np.pi)
        u = xx * np.cos(th) + yy * np.sin(th)
        if kind == 0:    # step edge
            img += amp * (u > rng.uniform(0.1, 0.9) * size * (abs(np.cos(th)) + abs(np.sin(th))))
        elif kind == 1:  # sinusoid
            f = rng.uniform(0.01, 0.2)
            img += amp * 0.5 * np.sin(2 * np.pi * f * u + rng.uniform(0, 2 * np.pi))
        else:            # Gaussian blob
            cy, cx = rng.uniform(0, size, 2)
            sg = rng.uniform(5, 60)
            img += amp * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * sg * sg))
    lo, hi = img.min(), img.max()
    return 255.0 * (img - lo) / (hi - lo if hi > lo else 1.0)


def patches_dc_removed(img: np.ndarray, p: int, stride: int) -> np.ndarray:
    """(n_patches, p*p) signal-major rows in extract_patches order
    (denoising.py:118-135), each with its mean subtracted."""
    win = np.lib.stride_tricks.sliding_window_view(img, (p, p))[::stride, ::stride]
    R, C = win.shape[:2]
    P = win.transpose(0, 1, 3, 2).reshape(R * C, p * p).astype(np.float64)
    P -= P.mean(axis=1, keepdims=True)
    return P


def image_patches(n_images: int, sigma: float, p: int, stride: int, seed: int,
                  size: int = 512):
    rng = np.random.default_rng(seed)
    clean, noisy, rows = [], [], []
    for _ in range(n_images):
        c = synthetic_image(rng, size)
        nz = c + rng.normal(0.0, sigma, c.shape)
        clean.append(c)
        noisy.append(nz)
        rows.append(patches_dc_removed(nz, p, stride))
    return np.concatenate(rows, axis=0), clean, noisy


CONFIGS = {
    # name: dict(kind, data params, split/train params)
    "c1": dict(kind="sparse", m=64, K_true=256, N=20_000, s_true=5, sigma=0.01, L=4, K1=256,
               s1=5, eps=None, s_max=None, local_iters=10, K=256, s2=3, merge_iters=10),
    "c2": dict(kind="image", n_images=8, sigma=20.0, p=8, stride=1, L=16, K1=256, s1=16,
               eps=1.15 * 20.0 * 8.0, s_max=16, local_iters=15, K=256, s2=4, merge_iters=15),
    "c3": dict(kind="image", n_images=8, sigma=25.0, p=12, stride=2, L=32, K1=576, s1=20,
               eps=1.15 * 25.0 * 12.0, s_max=20, local_iters=10, K=576, s2=4, merge_iters=10),
    "c4": dict(kind="sparse", m=64, K_true=512, N=4_000_000, s_true=8, sigma=0.02, L=256,
               K1=512, s1=8, eps=None, s_max=None, local_iters=8, K=512, s2=4, merge_iters=8),
}


def make_training_data_device(name: str, seed: int = 1234, prec: str = "fp32", N: int | None = None):
    """Device (N, m) training signals of config ``name``: sparse-model configs
    are generated on the GPU (sdb_synth_sparse); image configs are made on the
    host (3 s for C2) and ingested."""
    c = CONFIGS[name]
    if c["kind"] == "sparse":
        D = gen_dictionary(c["m"], c["K_true"], seed)
        return sparse_signals_device(D, N or c["N"], c["s_true"], c["sigma"], seed + 1, prec)
    from paper_1403_4781_b200 import _engine as E
    Y = make_training_data(name, seed, N)
    return E.ingest_signals(Y.T, prec)[0]


def make_training_data(name: str, seed: int = 1234, N: int | None = None) -> np.ndarray:
    """Signal-major (N, m) float64 training signals of config ``name``."""
    c = CONFIGS[name]
    if c["kind"] == "sparse":
        D = gen_dictionary(c["m"], c["K_true"], seed)
        return sparse_signals(D, N or c["N"], c["s_true"], c["sigma"], seed + 1)
    Y, _, _ = image_patches(c["n_images"], c["sigma"], c["p"], c["stride"], seed)
    return Y if N is None else Y[:N]
