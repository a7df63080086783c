"""Patch-based denoising on the B200 — drop-in for the hot part of
sparsedict.denoising (/root/reference/pkg/src/sparsedict/denoising.py:
extract_patches :118, reconstruct_from_patches :138, denoise_image :223).

The image goes to the device once; patch extraction, error-bounded OMP over
every patch, the patch estimates D x_k and the overlap averaging (a
deterministic per-pixel gather in the reference's summation order) plus the
final clip run in libsdb200.so. ``overcomplete_dct`` (an init option,
:166-195) is built on the host like any other user-supplied dictionary.
PGM I/O and corpus sampling are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _engine as E
from .exceptions import InvalidInputError
from .sparse_coding import check_dictionary

__all__ = [
    "GrayImage",
    "DenoiseConfig",
    "add_gaussian_noise",
    "extract_patches",
    "reconstruct_from_patches",
    "overcomplete_dct",
    "denoise_image",
]


@dataclass
class GrayImage:
    """Grayscale image, float64 pixels (height, width)."""

    pixels: np.ndarray

    def __post_init__(self):
        px = np.asarray(self.pixels, dtype=np.float64)
        if px.ndim != 2 or px.size == 0:
            raise InvalidInputError("pixels must be a nonempty 2-D array")
        self.pixels = px

    @property
    def width(self) -> int:
        return self.pixels.shape[1]

    @property
    def height(self) -> int:
        return self.pixels.shape[0]


@dataclass
class DenoiseConfig:
    """Denoiser parameters (denoising.py:54-75)."""

    sigma: float
    patch_size: int = 8
    stride: int = 1
    eps_gain: float = 8.5
    s_max: int | None = None

    def validate(self) -> None:
        p = self.patch_size
        if p < 1:
            raise InvalidInputError("patch_size must be positive")
        if not 1 <= self.stride <= p:
            raise InvalidInputError("require 1 <= stride <= patch_size")
        if self.sigma < 0:
            raise InvalidInputError("sigma must be nonnegative")
        if self.eps_gain < 0:
            raise InvalidInputError("eps_gain must be nonnegative")
        if self.s_max is not None and not 1 <= self.s_max <= p * p:
            raise InvalidInputError("require 1 <= s_max <= patch_size**2")


def add_gaussian_noise(img: GrayImage, sigma: float, seed: int) -> GrayImage:
    """i.i.d. N(0, sigma^2) per pixel from PCG64(seed), no clamping."""
    if sigma < 0:
        raise InvalidInputError("sigma must be nonnegative")
    rng = np.random.default_rng(seed)
    return GrayImage(img.pixels + rng.normal(0.0, sigma, img.pixels.shape))


def _grid(H: int, W: int, p: int, stride: int) -> tuple[int, int]:
    return (H - p) // stride + 1, (W - p) // stride + 1


def patches_device(px: torch.Tensor, p: int, stride: int, prec: str) -> torch.Tensor:
    """Device image (H, W) f64 -> (R*C, p^2) signal-major patches."""
    H, W = px.shape
    R, C = _grid(H, W, p, stride)
    out = E.empty((R * C, p * p), E.torch_dtype(prec))
    E._lib.call("sdb_extract_patches", E.sdb_dtype(prec), E.ptr(px), H, W, p, stride,
                E.ptr(out), E.stream())
    return out


def extract_patches(img: GrayImage, p: int, stride: int = 1) -> np.ndarray:
    """All p x p windows at stride, one column each, column-major vectorised,
    row-offset-major column order (denoising.py:118-135)."""
    H, W = img.pixels.shape
    if p > min(H, W):
        raise InvalidInputError("patch size exceeds image dimensions")
    if stride < 1:
        raise InvalidInputError("stride must be positive")
    px = torch.from_numpy(np.ascontiguousarray(img.pixels)).to(E.device())
    return E.d2h(patches_device(px, p, stride, "fp64")).T.copy()


def reconstruct_from_patches(patches, width: int, height: int, p: int,
                             stride: int = 1) -> GrayImage:
    """Mean of all patch estimates covering each pixel; uncovered pixels 0
    (denoising.py:138-163)."""
    patches = np.asarray(patches, dtype=np.float64)
    R, C = _grid(height, width, p, stride)
    if patches.ndim != 2 or patches.shape != (p * p, R * C):
        raise InvalidInputError(
            f"expected a ({p * p}, {R * C}) patch matrix, got {patches.shape}")
    P = torch.from_numpy(np.ascontiguousarray(patches.T)).to(E.device())
    out = E.empty((height, width), torch.float64)
    E._lib.call("sdb_reconstruct_dense", height, width, p, stride, E.ptr(P), E.ptr(out), E.stream())
    return GrayImage(E.d2h(out))


def overcomplete_dct(p: int, K: int) -> np.ndarray:
    """Separable overcomplete DCT dictionary (p*p, K = q*q), atom k*q + l
    (denoising.py:166-195)."""
    if p < 1 or K < 1:
        raise InvalidInputError("p and K must be positive")
    q = int(round(np.sqrt(K)))
    if q * q != K:
        raise InvalidInputError("K must be a perfect square")
    if q < p:
        raise InvalidInputError("require sqrt(K) >= p")
    t = np.arange(p)
    base = np.cos(np.pi * np.arange(q)[:, None] * t[None, :] / q)
    base[1:] -= base[1:].mean(axis=1, keepdims=True)
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    # atom (k, l) = outer(base[k], base[l]) vectorised column-major
    D = np.einsum("ki,lj->klji", base, base).reshape(q * q, p * p).T.copy()
    return D / np.linalg.norm(D, axis=0)


def denoise_device(px: torch.Tensor, D64: torch.Tensor, p: int, stride: int, eps: float,
                   cap: int, prec: str) -> torch.Tensor:
    """Device-resident denoise: (H, W) f64 image -> (H, W) f64 clipped."""
    H, W = px.shape
    Pt64 = None
    if E.certifies(prec):
        Pt64 = patches_device(px, p, stride, "fp64")     # the authoritative patch values
        Pt = Pt64.to(torch.float32)
    else:
        Pt = patches_device(px, p, stride, prec)
    codes = E.code_single_dict(Pt, D64, cap, eps, prec, want_rnorm=False, Y64=Pt64)   # norms are never read
    out = E.empty((H, W), torch.float64)
    E._lib.call("sdb_reconstruct", E.sdb_dtype(codes.vprec or prec), H, W, p, stride, E.ptr(D64), codes.cap,
                E.ptr(codes.idx), E.ptr(codes.val), E.ptr(codes.counts), 0.0, 255.0,
                E.ptr(out), E.stream())
    return out


def denoise_image(noisy: GrayImage, D, cfg: DenoiseConfig, threads: int = 1,
                  precision: str | None = None) -> GrayImage:
    """Error-bounded OMP per patch (eps = eps_gain * sigma, s_max default
    p^2), overlap averaging, one clip to [0, 255] (denoising.py:223-239)."""
    cfg.validate()
    p = cfg.patch_size
    D = np.asarray(D, dtype=np.float64)
    if D.shape[0] != p * p:
        raise InvalidInputError(f"dictionary rows {D.shape[0]} != patch dimension {p * p}")
    D = check_dictionary(D)
    if p > min(noisy.height, noisy.width):
        raise InvalidInputError("patch size exceeds image dimensions")
    if p * p > 256:
        raise InvalidInputError("patch dimension p*p > 256 is outside the GPU path")
    cap = cfg.s_max if cfg.s_max is not None else p * p
    eps = cfg.eps_gain * cfg.sigma
    prec = E.get_precision(precision)
    px = torch.from_numpy(np.ascontiguousarray(noisy.pixels)).to(E.device())
    if not bool(torch.isfinite(px).all()):
        raise InvalidInputError("batch contains non-finite entries")
    out = denoise_device(px, E.dict_to_device(D), p, cfg.stride, eps, cap, prec)
    return GrayImage(E.d2h(out))
