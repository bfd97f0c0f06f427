"""CPU restatement of the lower-level imaging operators (TEST ORACLE ONLY).

Two model families share one code path:

* the reference's Fields-of-Experts inpainting model
  (``operators.py:1-17``): ``L = 1/2||Mx - y||^2 + eps/2||x||^2 +
  sum_i e^{th_i} ||K_i x||^2``, i.e. data = row mask, data scale 1, ridge,
  quadratic potential phi(t) = t^2;
* the BASELINE configs' deblurring model: ``L = ||Ax - y||^2 + R(x)`` with A
  a b x b Gaussian blur (true convolution, zero boundary), no ridge, and R
  either smoothed TV ``e^a sum sqrt(Dh^2 + Dv^2 + eps^2)`` (Neumann forward
  differences) or learned filters ``sum_j e^{a_j} sum phi_eps(c_j * x)``
  with phi_eps(t) = sqrt(t^2 + eps^2).

Convolution convention: true convolution, zero boundary, same-size output
(``operators.py:19-22,309-326``); the adjoint is correlation.
theta layout: blocks ``[a_j, c_j row-major]`` (``operators.py:150-172``);
TV has theta = [a].
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
from scipy.signal import convolve2d, correlate2d

LOG_CLAMP = 30.0  # operators.py:52


class ClampWarning(UserWarning):
    """operators.py:55-56"""


# --------------------------------------------------------------------------
# convolution primitives (operators.py:309-326)


def conv_same(img: np.ndarray, k: np.ndarray) -> np.ndarray:
    return convolve2d(img, k, mode="same", boundary="fill")


def corr_same(img: np.ndarray, k: np.ndarray) -> np.ndarray:
    return correlate2d(img, k, mode="same", boundary="fill")


def shift_corr(v: np.ndarray, x: np.ndarray, q: int) -> np.ndarray:
    """out[a, b] = sum_p v[p] * x[p - (a - c), p - (b - c)]  (operators.py:386-408):
    the gradient of <conv(k, x), v> with respect to k[a, b]."""
    c = q // 2
    rows, cols = v.shape
    out = np.zeros((q, q))
    for a in range(q):
        da = a - c
        r_lo, r_hi = max(0, da), min(rows, rows + da)
        for b in range(q):
            db = b - c
            c_lo, c_hi = max(0, db), min(cols, cols + db)
            if r_lo < r_hi and c_lo < c_hi:
                out[a, b] = float(
                    np.sum(v[r_lo:r_hi, c_lo:c_hi] * x[r_lo - da : r_hi - da, c_lo - db : c_hi - db])
                )
    return out


def gaussian_taps(size: int, sigma: float) -> np.ndarray:
    """1-D normalised Gaussian; the b x b blur is outer(taps, taps)."""
    if size % 2 == 0 or size < 1:
        raise ValueError(f"blur size must be odd and positive, got {size}")
    r = size // 2
    t = np.exp(-(np.arange(-r, r + 1, dtype=float) ** 2) / (2.0 * sigma * sigma))
    return t / t.sum()


# Neumann forward differences: last column / last row difference is zero.


def diff_h(x: np.ndarray) -> np.ndarray:
    out = np.zeros_like(x)
    out[:, :-1] = x[:, 1:] - x[:, :-1]
    return out


def diff_v(x: np.ndarray) -> np.ndarray:
    out = np.zeros_like(x)
    out[:-1, :] = x[1:, :] - x[:-1, :]
    return out


def diff_h_adj(p: np.ndarray) -> np.ndarray:
    out = np.zeros_like(p)
    out[:, :-1] -= p[:, :-1]
    out[:, 1:] += p[:, :-1]
    return out


def diff_v_adj(p: np.ndarray) -> np.ndarray:
    out = np.zeros_like(p)
    out[:-1, :] -= p[:-1, :]
    out[1:, :] += p[:-1, :]
    return out


# --------------------------------------------------------------------------
# operator protocol (operators.py:238-301)


class SymOp:
    """Matrix-free symmetric operator with a declared model cost (operators.py:238-266)."""

    def __init__(self, dim: int, fn, cost: int | None = None):
        self.dim = int(dim)
        self._fn = fn
        self.apply_cost = int(cost) if cost is not None else 2 * self.dim * self.dim - self.dim

    def __call__(self, v):
        v = np.asarray(v, dtype=float)
        if v.shape != (self.dim,):
            raise ValueError(f"operator of dim {self.dim} applied to shape {v.shape}")
        return self._fn(v)

    def apply_matrix(self, M):
        return np.column_stack([self(M[:, j]) for j in range(M.shape[1])])

    def to_dense(self):
        return self.apply_matrix(np.eye(self.dim))


def dense_op(M, cost=None) -> SymOp:
    M = np.asarray(M, dtype=float)
    return SymOp(M.shape[0], lambda v: M @ v, cost)


class JacOp:
    """Adjoint action w -> J w, J = -(D^2_{theta x} L)^T (operators.py:277-301)."""

    def __init__(self, num_params: int, dim: int, fn, cost: int = 0):
        self.num_params = int(num_params)
        self.dim = int(dim)
        self._fn = fn
        self.adjoint_cost = int(cost)

    def apply_adjoint(self, w):
        w = np.asarray(w, dtype=float)
        if w.shape != (self.dim,):
            raise ValueError(f"expected an n-vector of length {self.dim}, got shape {w.shape}")
        return self._fn(w)

    def apply_adjoint_matrix(self, W):
        return np.column_stack([self.apply_adjoint(W[:, j]) for j in range(W.shape[1])])

    def to_dense(self):
        return self.apply_adjoint_matrix(np.eye(self.dim))


# --------------------------------------------------------------------------
# model description


@dataclass(frozen=True)
class DataTerm:
    """cost = scale/2 ||A x - y||^2 + ridge/2 ||x||^2.

    kind "mask": A keeps ``mask_rows`` (operators.py:187-235), y has m entries;
    kind "blur": A = conv with outer(taps, taps), y has n entries.
    """

    kind: str
    shape: tuple[int, int]
    y: np.ndarray
    scale: float = 2.0
    ridge: float = 0.0
    mask_rows: np.ndarray | None = None
    taps: np.ndarray | None = None
    x_true: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.shape[0] * self.shape[1]

    def kernel2d(self) -> np.ndarray:
        return np.outer(self.taps, self.taps)

    def mask_diag(self) -> np.ndarray:
        d = np.zeros(self.n)
        d[self.mask_rows] = 1.0
        return d

    def A(self, x: np.ndarray) -> np.ndarray:
        if self.kind == "mask":
            return x[self.mask_rows]
        return conv_same(x.reshape(self.shape), self.kernel2d()).ravel()

    def At(self, r: np.ndarray) -> np.ndarray:
        if self.kind == "mask":
            out = np.zeros(self.n)
            out[self.mask_rows] = r
            return out
        return corr_same(r.reshape(self.shape), self.kernel2d()).ravel()

    def AtA(self, v: np.ndarray) -> np.ndarray:
        if self.kind == "mask":
            return self.mask_diag() * v
        return self.At(self.A(v))


@dataclass(frozen=True)
class Regularizer:
    """kind "filters": blocks [a_j, c_j]; potential "quadratic" (phi = t^2,
    the reference FoE) or "smooth_abs" (phi = sqrt(t^2+eps^2)).
    kind "tv": theta = [a], R = e^a sum sqrt(Dh^2 + Dv^2 + eps^2)."""

    kind: str = "filters"
    num_filters: int = 0
    ksize: int = 0
    potential: str = "quadratic"
    eps: float = 1e-2

    @property
    def num_params(self) -> int:
        if self.kind == "tv":
            return 1
        return self.num_filters * (1 + self.ksize * self.ksize)

    def split(self, theta: np.ndarray):
        theta = np.asarray(theta, dtype=float).ravel()
        if theta.size != self.num_params:
            raise ValueError(f"theta has {theta.size} entries, expected {self.num_params}")
        if self.kind == "tv":
            return theta[:1].copy(), None
        blk = theta.reshape(self.num_filters, 1 + self.ksize * self.ksize)
        return blk[:, 0].copy(), blk[:, 1:].reshape(self.num_filters, self.ksize, self.ksize).copy()

    def phi(self, t):
        if self.potential == "quadratic":
            return t * t
        return np.sqrt(t * t + self.eps * self.eps)

    def dphi(self, t):
        if self.potential == "quadratic":
            return 2.0 * t
        return t / np.sqrt(t * t + self.eps * self.eps)

    def ddphi(self, t):
        if self.potential == "quadratic":
            return np.full_like(t, 2.0)
        e2 = self.eps * self.eps
        return e2 / (t * t + e2) ** 1.5


def pack_theta(alphas, kernels) -> np.ndarray:
    """Flat layout [a_j, c_j row-major] (operators.py:150-155)."""
    parts = []
    for a, k in zip(np.atleast_1d(alphas), kernels):
        parts.append([a])
        parts.append(np.asarray(k, dtype=float).ravel())
    return np.concatenate(parts)


def filter_weights(alphas: np.ndarray) -> np.ndarray:
    """exp with +/-30 clamp and ClampWarning (operators.py:174-184)."""
    a = np.asarray(alphas, dtype=float)
    if np.any(np.abs(a) > LOG_CLAMP):
        warnings.warn("log-weights clamped to +/-30 before exponentiation", ClampWarning, stacklevel=2)
        a = np.clip(a, -LOG_CLAMP, LOG_CLAMP)
    return np.exp(a)


@dataclass(frozen=True)
class Model:
    data: DataTerm
    reg: Regularizer

    @property
    def n(self) -> int:
        return self.data.n

    @property
    def shape(self):
        return self.data.shape

    @property
    def p(self) -> int:
        return self.reg.num_params


# --------------------------------------------------------------------------
# lower-level cost, gradient, Hessian, mixed Jacobian


def _tv_parts(reg: Regularizer, x_img: np.ndarray):
    gh, gv = diff_h(x_img), diff_v(x_img)
    s = np.sqrt(gh * gh + gv * gv + reg.eps * reg.eps)
    return gh, gv, s


def lower_cost(model: Model, theta, x) -> float:
    """operators.py:329-342 generalised."""
    d, reg = model.data, model.reg
    x = np.asarray(x, dtype=float)
    res = d.A(x) - d.y
    val = 0.5 * d.scale * float(res @ res) + 0.5 * d.ridge * float(x @ x)
    alphas, kernels = reg.split(theta)
    w = filter_weights(alphas)
    img = x.reshape(d.shape)
    if reg.kind == "tv":
        _, _, s = _tv_parts(reg, img)
        val += w[0] * float(np.sum(s))
    else:
        for wj, kj in zip(w, kernels):
            u = conv_same(img, kj).ravel()
            if reg.potential == "quadratic":
                val += wj * float(u @ u)
            else:
                val += wj * float(np.sum(reg.phi(u)))
    if not np.isfinite(val):
        raise FloatingPointError("non-finite lower-level cost")
    return val


def lower_grad(model: Model, theta, x) -> np.ndarray:
    """operators.py:345-353 generalised: scale A^T(Ax-y) + ridge x + sum w C^T phi'(C x)."""
    d, reg = model.data, model.reg
    x = np.asarray(x, dtype=float)
    g = d.scale * d.At(d.A(x) - d.y) if d.scale != 1.0 else d.At(d.A(x) - d.y)
    g = g + d.ridge * x
    alphas, kernels = reg.split(theta)
    w = filter_weights(alphas)
    img = x.reshape(d.shape)
    if reg.kind == "tv":
        gh, gv, s = _tv_parts(reg, img)
        g = g + w[0] * (diff_h_adj(gh / s) + diff_v_adj(gv / s)).ravel()
    else:
        for wj, kj in zip(w, kernels):
            u = conv_same(img, kj)
            if reg.potential == "quadratic":
                g += (2.0 * wj) * corr_same(u, kj).ravel()
            else:
                g += wj * corr_same(reg.dphi(u), kj).ravel()
    return g


def data_cost_model(model: Model) -> int:
    d = model.data
    n = d.n
    if d.kind == "mask":
        return 4 * n  # operators.py:357
    b = d.taps.size
    return 2 * n * (2 * b * b - 1) + 4 * n


def hessian_cost(model: Model) -> int:
    """Declared model FLOPs per application (operators.py:356-360 for the FoE
    model; the blur and TV terms use the same dense-convolution counting)."""
    n, reg = model.n, model.reg
    base = data_cost_model(model)
    if reg.kind == "tv":
        return base + n * 16
    conv = n * (2 * reg.ksize**2 - 1)
    return base + reg.num_filters * (2 * conv + 2 * n)


def hessian(model: Model, theta, x_hat=None) -> SymOp:
    """H v = scale A^T A v + ridge v + sum_j w_j C_j^T(phi''(C_j xhat) . C_j v)
    (operators.py:363-383; the configs' curvature-weighted generalisation)."""
    d, reg = model.data, model.reg
    shape = d.shape
    alphas, kernels = reg.split(theta)
    w = filter_weights(alphas)
    mask = d.mask_diag() if d.kind == "mask" else None
    k2 = d.kernel2d() if d.kind == "blur" else None
    scale, ridge = d.scale, d.ridge

    if reg.kind == "tv":
        gh, gv, s = _tv_parts(reg, np.asarray(x_hat, dtype=float).reshape(shape))
        m11 = (1.0 - gh * gh / (s * s)) / s
        m12 = -(gh * gv) / (s * s * s)
        m22 = (1.0 - gv * gv / (s * s)) / s
        wa = w[0]

        def apply(v):
            img = v.reshape(shape)
            if mask is not None:
                out = (scale * mask) * v + ridge * v
            else:
                out = scale * corr_same(conv_same(img, k2), k2).ravel() + ridge * v
            dh, dv = diff_h(img), diff_v(img)
            ph = m11 * dh + m12 * dv
            pv = m12 * dh + m22 * dv
            ph[:, -1] = 0.0
            pv[-1, :] = 0.0
            return out + wa * (diff_h_adj(ph) + diff_v_adj(pv)).ravel()

        return SymOp(d.n, apply, hessian_cost(model))

    if reg.potential == "quadratic":
        curv = None
    else:
        xi = np.asarray(x_hat, dtype=float).reshape(shape)
        curv = [reg.ddphi(conv_same(xi, kj)) for kj in kernels]

    def apply(v):
        img = v.reshape(shape)
        if mask is not None:
            out = mask * v + ridge * v if scale == 1.0 else (scale * mask) * v + ridge * v
        else:
            out = scale * corr_same(conv_same(img, k2), k2).ravel() + ridge * v
        for j, (wj, kj) in enumerate(zip(w, kernels)):
            u = conv_same(img, kj)
            if curv is None:
                out += (2.0 * wj) * corr_same(u, kj).ravel()
            else:
                out += wj * corr_same(curv[j] * u, kj).ravel()
        return out

    return SymOp(d.n, apply, hessian_cost(model))


def jacobian(model: Model, theta, x_hat) -> JacOp:
    """J w per filter j (operators.py:411-444 generalised):
      a_j  entry : -w_j <phi'(C_j xhat), C_j w>
      c_j[a]     : -w_j (shift(phi'(C_j xhat), w) + shift(phi''(C_j xhat) . C_j w, xhat))[a]
    TV: -e^a <D xhat / s, D w>."""
    d, reg = model.data, model.reg
    shape = d.shape
    alphas, kernels = reg.split(theta)
    w = filter_weights(alphas)
    xi = np.asarray(x_hat, dtype=float).reshape(shape)
    n = d.n

    if reg.kind == "tv":
        gh, gv, s = _tv_parts(reg, xi)
        nh, nv = gh / s, gv / s

        def apply_tv(wv):
            img = wv.reshape(shape)
            return np.array([-w[0] * float(np.sum(nh * diff_h(img) + nv * diff_v(img)))])

        return JacOp(1, n, apply_tv, 4 * n)

    q = reg.ksize
    cx = [conv_same(xi, kj) for kj in kernels]
    if reg.potential == "quadratic":
        slope = cx  # phi' = 2 C x; the factor 2 is folded below as in operators.py:434-438
        curv = None
    else:
        slope = [reg.dphi(u) for u in cx]
        curv = [reg.ddphi(u) for u in cx]

    def apply(wv):
        img = wv.reshape(shape)
        out = []
        for j, (wj, kj) in enumerate(zip(w, kernels)):
            cw = conv_same(img, kj)
            if curv is None:
                head = -2.0 * wj * float(slope[j].ravel() @ cw.ravel())
                gk = shift_corr(slope[j], img, q) + shift_corr(cw, xi, q)
                out.append(np.concatenate(([head], (-2.0 * wj) * gk.ravel())))
            else:
                head = -wj * float(slope[j].ravel() @ cw.ravel())
                gk = shift_corr(slope[j], img, q) + shift_corr(curv[j] * cw, xi, q)
                out.append(np.concatenate(([head], (-wj) * gk.ravel())))
        return np.concatenate(out)

    conv = n * (2 * q * q - 1)
    return JacOp(reg.num_params, n, apply, reg.num_filters * (2 * conv + 2 * n * q * q))


# --------------------------------------------------------------------------
# problem generators


def builtin_glyph(size: int = 28) -> np.ndarray:
    """Deterministic blocky glyph (images.py:20-44): rectangles on a 28x28
    design grid rescaled with integer rounding."""
    if size < 8:
        raise ValueError(f"glyph needs at least an 8 x 8 canvas, got {size}")
    img = np.zeros((size, size))
    f = size / 28.0
    design = [
        (3, 7, 4, 24, 1.0),
        (7, 12, 19, 24, 1.0),
        (12, 16, 12, 21, 1.0),
        (16, 21, 8, 15, 1.0),
        (21, 25, 5, 12, 1.0),
        (9, 12, 5, 9, 0.5),
    ]
    for r0, r1, c0, c1, val in design:
        ra = int(round(r0 * f))
        rb = max(ra + 1, int(round(r1 * f)))
        ca = int(round(c0 * f))
        cb = max(ca + 1, int(round(c1 * f)))
        img[ra:rb, ca:cb] = val
    return img


def foe_inpainting(
    image_size: int = 16,
    intensity: float = 0.25,
    rate: float = 0.3,
    noise: float = 0.3,
    num_filters: int = 3,
    kernel_size: int = 5,
    seed: int = 0,
    ridge: float = 1e-6,
    kernel_init_std: float = 0.1,
):
    """Seeded FoE inpainting instance (experiments.py:139-177): glyph scaled to
    peak ``intensity``, ceil(rate n) retained pixels, noise scaled to the exact
    relative level, zero log-weights, N(0, std^2) kernels -- all from one rng."""
    raw = builtin_glyph(image_size).ravel()
    peak = float(np.max(np.abs(raw)))
    x_true = raw if peak == 0 else (intensity / peak) * raw
    n = x_true.size
    m = int(np.ceil(rate * n))
    rng = np.random.default_rng(seed)
    mask = np.sort(rng.permutation(n)[:m])
    clean = x_true[mask]
    if noise > 0:
        e = rng.standard_normal(m)
        e *= noise * np.linalg.norm(clean) / np.linalg.norm(e)
        y = clean + e
    else:
        y = clean.copy()
    data = DataTerm("mask", (image_size, image_size), y, scale=1.0, ridge=ridge, mask_rows=mask, x_true=x_true)
    reg = Regularizer("filters", num_filters, kernel_size, "quadratic")
    kernels = [kernel_init_std * rng.standard_normal((kernel_size, kernel_size)) for _ in range(num_filters)]
    theta0 = pack_theta(np.zeros(num_filters), kernels)
    return Model(data, reg), theta0


def piecewise_constant(size: int, rng: np.random.Generator, rects: int = 6, disks: int = 4) -> np.ndarray:
    """Seeded piecewise-constant test image (BASELINE configs): ``rects``
    axis-aligned rectangles and ``disks`` disks with U[0,1] intensities added
    on a zero canvas, clipped to [0, 1]."""
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


@dataclass(frozen=True)
class DeblurConfig:
    """One BASELINE config (configs[0..4])."""

    size: int = 64
    batch: int = 1
    blur_size: int = 9
    blur_sigma: float = 1.5
    noise: float = 0.01
    reg: str = "tv"  # "tv" | "filters"
    num_filters: int = 0
    kernel_size: int = 0
    eps: float = 1e-2
    alpha0: float = -3.0
    filter_std: float = 0.1
    seed: int = 0


CONFIGS = {
    "C1": DeblurConfig(64, 1, 9, 1.5, 0.01, "tv"),
    "C2": DeblurConfig(128, 8, 9, 1.5, 0.01, "filters", 8, 5),
    "C3": DeblurConfig(256, 64, 15, 2.5, 0.02, "filters", 8, 5),
    "C4": DeblurConfig(512, 128, 21, 3.5, 0.01, "filters", 24, 7),
    "C5": DeblurConfig(1024, 1, 15, 2.5, 0.01, "filters", 8, 5),
}


def deblur_sample(cfg: DeblurConfig, index: int) -> tuple[Model, np.ndarray]:
    """Sample ``index`` of a config: rng(seed + index) draws the image then the
    noise; y = A x + e with ||e|| / ||A x|| == noise exactly (experiments.py:160-167)."""
    rng = np.random.default_rng(cfg.seed + index)
    x_true = piecewise_constant(cfg.size, rng).ravel()
    taps = gaussian_taps(cfg.blur_size, cfg.blur_sigma)
    shape = (cfg.size, cfg.size)
    ax = conv_same(x_true.reshape(shape), np.outer(taps, taps)).ravel()
    e = rng.standard_normal(ax.size)
    e *= cfg.noise * np.linalg.norm(ax) / np.linalg.norm(e)
    data = DataTerm("blur", shape, ax + e, scale=2.0, ridge=0.0, taps=taps, x_true=x_true)
    if cfg.reg == "tv":
        reg = Regularizer("tv", eps=cfg.eps)
    else:
        reg = Regularizer("filters", cfg.num_filters, cfg.kernel_size, "smooth_abs", cfg.eps)
    return Model(data, reg), x_true


def deblur_theta0(cfg: DeblurConfig) -> np.ndarray:
    """theta_0 from one rng(seed): a_j = alpha0, filters std*N(0,1) with the
    per-filter mean removed."""
    if cfg.reg == "tv":
        return np.array([cfg.alpha0])
    rng = np.random.default_rng(cfg.seed)
    kernels = []
    for _ in range(cfg.num_filters):
        k = cfg.filter_std * rng.standard_normal((cfg.kernel_size, cfg.kernel_size))
        kernels.append(k - k.mean())
    return pack_theta(np.full(cfg.num_filters, cfg.alpha0), kernels)


def perturbed(H: SymOp, rel: float = 2e-16, seed: int = 0) -> SymOp:
    """H with each output entry multiplied by (1 + rel * N(0,1)): a roundoff-level
    perturbation used to measure the reference algorithm's own sensitivity
    (its "roundoff floor") -- the SURVEY App. B roundoff-sensitivity probe."""
    rng = np.random.default_rng(seed)
    return SymOp(H.dim, lambda v: H(v) * (1.0 + rel * rng.standard_normal(v.size)), H.apply_cost)
