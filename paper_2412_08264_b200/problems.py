"""Seeded synthetic inputs for the BASELINE configs (data generation, not the hot path).

Piecewise-constant images (6 rectangles + 4 disks, U[0,1] intensities, clipped
to [0,1]), b x b Gaussian blur with zero boundary, noise scaled to the exact
relative level (the experiments.py:160-167 recipe), theta_0 with alpha_j =
alpha0 and std*N(0,1) filters with the mean removed.  The draws are identical
to ``oracle.cpu_imaging.deblur_sample`` (checked by tests/test_problems.py).

``synthetic_sequence`` produces a frozen sequence of upper-level systems
(theta_i, xhat_i) with small consecutive changes -- the replay protocol's
input (experiments.py:390-463) -- without running lower-level solves.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.signal import convolve2d

from .operators import Model, as_device

__all__ = ["CONFIGS", "DeblurConfig", "gaussian_taps", "make_batch", "piecewise_constant", "synthetic_sequence",
           "theta0"]


@dataclass(frozen=True)
class DeblurConfig:
    size: int = 64
    batch: int = 1
    blur_size: int = 9
    blur_sigma: float = 1.5
    noise: float = 0.01
    reg: str = "tv"
    num_filters: int = 0
    kernel_size: int = 0
    eps: float = 1e-2
    alpha0: float = -3.0
    filter_std: float = 0.1
    seed: int = 0
    recycle_dim: int = 10
    max_iter: int = 100
    upper_steps: int = 20
    method: str = "minres"  # Krylov method of the Hessian solves: "minres" (RMINRES) or "cg" (recycled CG)


CONFIGS = {
    # BASELINE.json configs[0..4]
    "C1": DeblurConfig(64, 1, 9, 1.5, 0.01, "tv", recycle_dim=10, max_iter=100, upper_steps=20, method="cg"),
    "C2": DeblurConfig(128, 8, 9, 1.5, 0.01, "filters", 8, 5, recycle_dim=20, max_iter=200, upper_steps=30),
    "C3": DeblurConfig(256, 64, 15, 2.5, 0.02, "filters", 8, 5, recycle_dim=30, max_iter=300, upper_steps=30),
    "C4": DeblurConfig(512, 128, 21, 3.5, 0.01, "filters", 24, 7, recycle_dim=40, max_iter=500, upper_steps=20),
    "C5": DeblurConfig(1024, 1, 15, 2.5, 0.01, "filters", 8, 5, recycle_dim=40, max_iter=500, upper_steps=50),
}


def gaussian_taps(size: int, sigma: float) -> np.ndarray:
    r = size // 2
    t = np.exp(-(np.arange(-r, r + 1, dtype=float) ** 2) / (2.0 * sigma * sigma))
    return t / t.sum()


def piecewise_constant(size: int, rng: np.random.Generator, rects: int = 6, disks: int = 4) -> np.ndarray:
    img = np.zeros((size, size))
    lo, hi = max(1, size // 8), max(2, size // 2)
    for _ in range(rects):
        h = int(rng.integers(lo, hi + 1))
        w = int(rng.integers(lo, hi + 1))
        r0 = int(rng.integers(0, size - h + 1))
        c0 = int(rng.integers(0, size - w + 1))
        img[r0 : r0 + h, c0 : c0 + w] += rng.uniform(0.0, 1.0)
    yy, xx = np.mgrid[0:size, 0:size]
    rlo, rhi = max(1.0, size / 16.0), max(2.0, size / 6.0)
    for _ in range(disks):
        cy, cx = rng.uniform(0, size), rng.uniform(0, size)
        rad = rng.uniform(rlo, rhi)
        img[(yy - cy) ** 2 + (xx - cx) ** 2 <= rad * rad] += rng.uniform(0.0, 1.0)
    return np.clip(img, 0.0, 1.0)


def sample_arrays(cfg: DeblurConfig, index: int):
    """(x_true, y) of sample ``index``: rng(seed + index) draws the image then the noise."""
    rng = np.random.default_rng(cfg.seed + index)
    x_true = piecewise_constant(cfg.size, rng).ravel()
    taps = gaussian_taps(cfg.blur_size, cfg.blur_sigma)
    ax = convolve2d(x_true.reshape(cfg.size, cfg.size), np.outer(taps, taps), mode="same", boundary="fill").ravel()
    e = rng.standard_normal(ax.size)
    e *= cfg.noise * np.linalg.norm(ax) / np.linalg.norm(e)
    return x_true, ax + e


def theta0(cfg: DeblurConfig) -> np.ndarray:
    if cfg.reg == "tv":
        return np.array([cfg.alpha0])
    rng = np.random.default_rng(cfg.seed)
    parts = []
    for _ in range(cfg.num_filters):
        k = cfg.filter_std * rng.standard_normal((cfg.kernel_size, cfg.kernel_size))
        parts += [[cfg.alpha0], (k - k.mean()).ravel()]
    return np.concatenate(parts)


def make_batch(cfg: DeblurConfig, first: int = 0, count: int | None = None, device=None) -> Model:
    """Device model of samples [first, first + count)."""
    count = cfg.batch if count is None else count
    xs, ys = zip(*[sample_arrays(cfg, first + k) for k in range(count)])
    return Model(shape=(cfg.size, cfg.size), batch=count, data_kind="blur", data_scale=2.0, ridge=0.0,
                 y=as_device(np.stack(ys), device), x_true=as_device(np.stack(xs), device),
                 taps=gaussian_taps(cfg.blur_size, cfg.blur_sigma), reg_kind=cfg.reg,
                 potential="smooth_abs", eps=cfg.eps, num_filters=cfg.num_filters, ksize=cfg.kernel_size)


def synthetic_sequence(cfg: DeblurConfig, x_trues: np.ndarray, steps: int, seed: int = 1234, first: int = 0):
    """Frozen systems i = 0..steps-1: theta_i = theta_0 + i * dtheta and
    xhat_i = x_true + smooth_i, with smooth_i a blurred 3%-level field that drifts
    slowly with i (consecutive-system relative changes O(1e-2)).

    The fields of sample k (global index first + b) come from their own generator
    default_rng([seed, kind, k]), so a rank that owns samples [first, first + B)
    sees exactly the systems the single-process batch holds for them."""
    rng = np.random.default_rng(seed)
    th0 = theta0(cfg)
    dth = 0.002 * rng.standard_normal(th0.size)
    B, n = x_trues.shape
    size = cfg.size
    taps = gaussian_taps(9, 2.0)
    k2 = np.outer(taps, taps)

    def field(kind, b):
        f = np.random.default_rng([seed, kind, first + b]).standard_normal((size, size))
        return convolve2d(f, k2, mode="same", boundary="fill").ravel()

    base = np.stack([field(0, b) for b in range(B)])
    drift = np.stack([field(1, b) for b in range(B)])
    scale = 0.03 / np.maximum(np.abs(base).max(axis=1, keepdims=True), 1e-12)
    thetas, xhats = [], []
    for i in range(steps):
        thetas.append(th0 + i * dth)
        xhats.append(x_trues + scale * (base + 0.05 * i * drift))
    return thetas, xhats
