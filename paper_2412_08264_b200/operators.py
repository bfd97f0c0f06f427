"""Device operators mirroring ``krecycle.operators`` (reference operators.py).

The reference's duck-typed protocol is kept: ``SymmetricOperator`` with
``dim``, ``__call__``, ``apply_matrix``, ``to_dense``, ``apply_cost``
(operators.py:238-266) and ``MixedJacobianOperator`` with ``apply_adjoint``
and ``apply_adjoint_matrix`` (operators.py:277-301).  Vectors are CUDA fp64
tensors; an n x t block is an (n, t) tensor whose columns are contiguous
(stride (1, ld)), i.e. the reference's numpy matrix stored column-major.

Behind them sits one model family (``Model``): data term (row mask as in the
reference's inpainting problem, or a separable Gaussian blur as in the
BASELINE configs), ridge, and a regulariser (learned filters with a
quadratic or phi_eps potential, or smoothed TV).  Every application is one
call into ``libkrecycle_b200`` (no CPU path).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import KrOp

LOG_WEIGHT_CLAMP = 30.0  # operators.py:52

__all__ = [
    "ClampWarning", "FoEParams", "ImageVector", "InpaintingProblem", "Kernel", "Model",
    "MixedJacobianOperator", "SymmetricOperator", "HessianOperator", "StencilJacobian",
    "dense_operator", "foe_cost", "foe_gradient", "foe_hessian", "mixed_jacobian",
    "naive_apply_cost", "operators_at", "columns", "new_columns",
]


class ClampWarning(UserWarning):
    """Log-weights clamped before exponentiation (operators.py:55-56)."""


def naive_apply_cost(n: int) -> int:
    return 2 * n * n - n


def _dev(device=None):
    return torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)


def as_device(x, device=None) -> torch.Tensor:
    """fp64 CUDA tensor (copy from numpy / host if needed)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(device), dtype=torch.float64)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=_dev(device))


def columns(M: torch.Tensor) -> torch.Tensor:
    """Return M (.., n, t) with contiguous columns (stride(-2) == 1)."""
    if M.stride(-2) == 1 and (M.shape[-1] <= 1 or M.stride(-1) >= M.shape[-2]):
        return M
    return M.transpose(-1, -2).contiguous().transpose(-1, -2)


def new_columns(*shape, device=None) -> torch.Tensor:
    """Uninitialised (.., n, t) tensor with contiguous columns."""
    *lead, n, t = shape
    return torch.empty(*lead, t, n, dtype=torch.float64, device=_dev(device)).transpose(-1, -2)


# --------------------------------------------------------------------------
# reference value types (operators.py:64-235)


@dataclass(frozen=True)
class ImageVector:
    """operators.py:64-92; ``data`` may be numpy or a tensor."""

    data: object
    shape: tuple[int, int]

    def __post_init__(self):
        d = self.data
        if isinstance(d, torch.Tensor):
            d = d.reshape(-1).to(torch.float64)
            ok = bool(torch.isfinite(d).all())
        else:
            d = np.asarray(d, dtype=float).ravel()
            ok = bool(np.all(np.isfinite(d)))
        object.__setattr__(self, "data", d)
        rows, cols = self.shape
        if rows * cols != d.numel() if isinstance(d, torch.Tensor) else rows * cols != d.size:
            raise ValueError(f"shape {self.shape} inconsistent with vector of length {len(d)}")
        if not ok:
            raise ValueError("image contains non-finite entries")

    @classmethod
    def from_matrix(cls, mat):
        if isinstance(mat, torch.Tensor):
            return cls(mat.reshape(-1), tuple(mat.shape))
        mat = np.asarray(mat, dtype=float)
        return cls(mat.ravel(), mat.shape)

    def as_matrix(self):
        return self.data.reshape(self.shape)

    @property
    def size(self) -> int:
        return self.shape[0] * self.shape[1]


@dataclass(frozen=True)
class Kernel:
    """operators.py:95-111"""

    weights: np.ndarray

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=float)
        if w.ndim != 2 or w.shape[0] != w.shape[1]:
            raise ValueError(f"kernel must be square, got shape {w.shape}")
        if w.shape[0] % 2 == 0:
            raise ValueError(f"kernel size must be odd, got {w.shape[0]}")
        object.__setattr__(self, "weights", w)

    @property
    def size(self) -> int:
        return self.weights.shape[0]


def _clamped_exp(lw: np.ndarray) -> np.ndarray:
    lw = np.asarray(lw, dtype=float)
    if np.any(np.abs(lw) > LOG_WEIGHT_CLAMP):
        warnings.warn("log-weights clamped to +/-%g before exponentiation" % LOG_WEIGHT_CLAMP,
                      ClampWarning, stacklevel=3)
        lw = np.clip(lw, -LOG_WEIGHT_CLAMP, LOG_WEIGHT_CLAMP)
    return np.exp(lw)


@dataclass(frozen=True)
class FoEParams:
    """One log-weight and one kernel per filter; flat layout [a_i, k_i row-major]
    (operators.py:114-184)."""

    log_weights: np.ndarray
    kernels: tuple

    def __post_init__(self):
        lw = np.asarray(self.log_weights, dtype=float).ravel()
        ks = tuple(self.kernels)
        if lw.size != len(ks):
            raise ValueError(f"{lw.size} log-weights but {len(ks)} kernels")
        if len({k.size for k in ks}) > 1:
            raise ValueError("kernels have mixed sizes")
        object.__setattr__(self, "log_weights", lw)
        object.__setattr__(self, "kernels", ks)

    @property
    def num_filters(self) -> int:
        return self.log_weights.size

    @property
    def kernel_size(self) -> int:
        return self.kernels[0].size

    @property
    def num_params(self) -> int:
        return self.num_filters * (1 + self.kernel_size**2)

    def flatten(self) -> np.ndarray:
        parts = []
        for a, k in zip(self.log_weights, self.kernels):
            parts += [[a], k.weights.ravel()]
        return np.concatenate(parts)

    @classmethod
    def unflatten(cls, theta, num_filters: int, kernel_size: int) -> "FoEParams":
        theta = np.asarray(theta, dtype=float).ravel()
        blk = 1 + kernel_size**2
        if theta.size != num_filters * blk:
            raise ValueError(f"parameter vector of length {theta.size} does not match "
                             f"{num_filters} filters of size {kernel_size}")
        t = theta.reshape(num_filters, blk)
        return cls(t[:, 0].copy(), tuple(Kernel(r[1:].reshape(kernel_size, kernel_size)) for r in t))

    def filter_weights(self) -> np.ndarray:
        return _clamped_exp(self.log_weights)


@dataclass(frozen=True)
class InpaintingProblem:
    """operators.py:187-235 (mask rows, y, ridge, shape, x_true)."""

    mask_rows: np.ndarray
    y: np.ndarray
    ridge: float
    shape: tuple[int, int]
    x_true: ImageVector | None = None

    def __post_init__(self):
        mask = np.asarray(self.mask_rows, dtype=np.int64).ravel()
        y = np.asarray(self.y, dtype=float).ravel()
        n = self.shape[0] * self.shape[1]
        if mask.size != np.unique(mask).size:
            raise ValueError("mask indices must be distinct")
        if mask.size and (mask.min() < 0 or mask.max() >= n):
            raise ValueError(f"mask indices must lie in [0, {n})")
        if y.size != mask.size:
            raise ValueError(f"y has length {y.size}, mask has {mask.size} rows")
        if not self.ridge > 0:
            raise ValueError(f"ridge must be positive, got {self.ridge}")
        object.__setattr__(self, "mask_rows", mask)
        object.__setattr__(self, "y", y)

    @property
    def n(self) -> int:
        return self.shape[0] * self.shape[1]

    @property
    def m(self) -> int:
        return self.mask_rows.size

    def mask_diagonal(self) -> np.ndarray:
        d = np.zeros(self.n)
        d[self.mask_rows] = 1.0
        return d

    def model(self, device=None) -> "Model":
        ys = np.zeros(self.n)
        ys[self.mask_rows] = self.y
        xt = None
        if self.x_true is not None:
            xt = as_device(self.x_true.data, device).reshape(1, -1)
        return Model(shape=tuple(self.shape), batch=1, data_kind="mask", data_scale=1.0, ridge=self.ridge,
                     mask=as_device(self.mask_diagonal(), device).reshape(1, -1),
                     y=as_device(ys, device).reshape(1, -1), x_true=xt, reg_kind="filters",
                     potential="quadratic", num_filters=0, ksize=0)


# --------------------------------------------------------------------------
# the device model


@dataclass
class Model:
    """A batch of lower-level problems sharing theta.

    cost_b(x) = data_scale/2 ||A x - y_b||^2 + ridge/2 ||x||^2 + R_theta(x)
    data_kind "mask": A = row mask (reference inpainting); y stored scattered (A^T y).
    data_kind "blur": A = conv with outer(taps, taps), true convolution, zero boundary.
    reg_kind "filters": R = sum_j e^{a_j} sum phi((c_j * x)_p), potential "quadratic"
    (phi = t^2) or "smooth_abs" (phi = sqrt(t^2 + eps^2)); reg_kind "tv":
    R = e^a sum sqrt(Dh x^2 + Dv x^2 + eps^2).  theta = [a_j, c_j row-major]...
    (filters, operators.py:150-172) or [a] (tv).  num_filters / ksize of 0 are
    inferred from theta at the first use for the FoE mirror.
    """

    shape: tuple
    batch: int
    data_kind: str
    data_scale: float
    ridge: float
    y: torch.Tensor
    x_true: torch.Tensor | None = None
    mask: torch.Tensor | None = None
    taps: np.ndarray | None = None
    reg_kind: str = "filters"
    potential: str = "smooth_abs"
    eps: float = 1e-2
    num_filters: int = 0
    ksize: int = 0

    @property
    def n(self) -> int:
        return self.shape[0] * self.shape[1]

    @property
    def num_params(self) -> int:
        if self.reg_kind == "tv":
            return 1
        return self.num_filters * (1 + self.ksize**2)

    @property
    def device(self):
        return self.y.device

    def split(self, theta):
        theta = np.asarray(theta, dtype=float).ravel()
        if theta.size != self.num_params:
            raise ValueError(f"theta has {theta.size} entries, expected {self.num_params}")
        if self.reg_kind == "tv":
            return theta[:1].copy(), None
        blk = theta.reshape(self.num_filters, 1 + self.ksize**2)
        return blk[:, 0].copy(), blk[:, 1:].reshape(self.num_filters, self.ksize, self.ksize).copy()

    def sample(self, b: int) -> "Model":
        """Single-sample view (shares device storage)."""
        return self.slice(b, b + 1)

    def slice(self, lo: int, hi: int) -> "Model":
        """View of samples [lo, hi) (shares device storage)."""
        sl = slice(lo, hi)
        return Model(self.shape, hi - lo, self.data_kind, self.data_scale, self.ridge, self.y[sl],
                     None if self.x_true is None else self.x_true[sl],
                     None if self.mask is None else (self.mask[sl] if self.mask.shape[0] > 1 else self.mask),
                     self.taps, self.reg_kind, self.potential, self.eps, self.num_filters, self.ksize)

    def select(self, idx) -> "Model":
        """Samples idx (any order), gathered into new storage."""
        it = torch.as_tensor(list(idx), dtype=torch.long, device=self.y.device)
        return Model(self.shape, len(idx), self.data_kind, self.data_scale, self.ridge, self.y.index_select(0, it),
                     None if self.x_true is None else self.x_true.index_select(0, it),
                     None if self.mask is None else (self.mask.index_select(0, it) if self.mask.shape[0] > 1
                                                     else self.mask),
                     self.taps, self.reg_kind, self.potential, self.eps, self.num_filters, self.ksize)

    def hessian_cost(self) -> int:
        """Declared model FLOPs per H v (operators.py:356-360 for the FoE family)."""
        n = self.n
        base = 4 * n if self.data_kind == "mask" else 2 * n * (2 * len(self.taps) ** 2 - 1) + 4 * n
        if self.reg_kind == "tv":
            return base + 16 * n
        conv = n * (2 * self.ksize**2 - 1)
        return base + self.num_filters * (2 * conv + 2 * n)

    def jacobian_cost(self) -> int:
        n, q = self.n, self.ksize
        if self.reg_kind == "tv":
            return 4 * n
        return self.num_filters * (2 * n * (2 * q * q - 1) + 2 * n * q * q)

    # -- kr_op construction ------------------------------------------------

    def _kr_op(self, theta, x_hat, keep: dict) -> KrOp:
        op = KrOp()
        op.rows, op.cols = int(self.shape[0]), int(self.shape[1])
        op.batch = int(self.batch)
        op.data_scale = float(self.data_scale)
        op.ridge = float(self.ridge)
        if self.data_kind == "mask":
            op.data_kind = _lib.DATA_MASK
            keep["mask"] = self.mask
            op.mask = self.mask.data_ptr()
            op.mask_bstride = self.n if self.mask.shape[0] > 1 else 0
        elif self.data_kind == "blur":
            op.data_kind = _lib.DATA_BLUR
            taps = np.asarray(self.taps, dtype=float)
            if taps.size > _lib.KR_MAX_BLUR or taps.size % 2 == 0:
                raise ValueError("blur size must be odd and <= 31")
            op.blur_size = taps.size
            for i, v in enumerate(taps):
                op.blur_taps[i] = float(v)
        else:
            raise ValueError(f"unknown data kind {self.data_kind!r}")
        alphas, kernels = self.split(theta)
        fw = _clamped_exp(alphas)
        keep["fweights"] = as_device(fw, self.device)
        op.fweights = keep["fweights"].data_ptr()
        op.eps = float(self.eps)
        n, B = self.n, self.batch
        if self.reg_kind == "tv":
            op.reg_kind = _lib.REG_TV
            keep["curv"] = torch.empty(B, 3, n, dtype=torch.float64, device=self.device)
            keep["slope"] = torch.empty(B, 2, n, dtype=torch.float64, device=self.device)
        else:
            op.reg_kind = _lib.REG_FILTERS
            op.potential = _lib.POT_QUADRATIC if self.potential == "quadratic" else _lib.POT_SMOOTH_ABS
            op.num_filters, op.ksize = self.num_filters, self.ksize
            keep["kernels"] = as_device(kernels, self.device).contiguous()
            op.kernels = keep["kernels"].data_ptr()
            J = self.num_filters
            keep["slope"] = torch.empty(B, J, n, dtype=torch.float64, device=self.device)
            if self.potential != "quadratic":
                keep["curv"] = torch.empty(B, J, n, dtype=torch.float64, device=self.device)
        if "curv" in keep:
            op.curv = keep["curv"].data_ptr()
        op.slope = keep["slope"].data_ptr()
        if x_hat is not None:
            xh = as_device(x_hat, self.device).reshape(B, n).contiguous()
            keep["xhat"] = xh
            op.xhat = xh.data_ptr()
        return op

    def at(self, theta, x_hat):
        """(H, J) at (theta, xhat): one kr_op_prepare shared by both (operators.py:363-444)."""
        if self.num_filters == 0 and self.reg_kind == "filters":
            raise ValueError("model has no filters configured")
        keep: dict = {}
        op = self._kr_op(theta, x_hat, keep)
        if x_hat is not None:
            _lib.check(_lib.lib().kr_op_prepare(ctypes.byref(op), _lib.stream_ptr()), "kr_op_prepare")
            _lib.note_launch("kr_op_prepare")
        H = HessianOperator(self, op, keep)
        J = StencilJacobian(self, op, keep) if x_hat is not None else None
        return H, J

    # -- lower level ---------------------------------------------------------

    def cost_grad(self, theta, X: torch.Tensor, work: dict | None = None):
        """Lower-level cost [B] and gradient [B, n] at X (operators.py:329-353)."""
        keep: dict = {}
        op = self._kr_op(theta, None, keep)
        L = _lib.lib()
        X = X.reshape(self.batch, self.n).contiguous()
        cost = torch.empty(self.batch, dtype=torch.float64, device=self.device)
        grad = torch.empty_like(X)
        wl = L.kr_lower_workspace(ctypes.byref(op))
        ws = torch.empty(max(wl, 1), dtype=torch.float64, device=self.device)
        _lib.check(L.kr_lower_eval(ctypes.byref(op), X.data_ptr(), self.y.data_ptr(), cost.data_ptr(),
                                   grad.data_ptr(), ws.data_ptr(), wl, _lib.stream_ptr()), "kr_lower_eval")
        _lib.note_launch("kr_lower_eval", 2)
        return cost, grad


# --------------------------------------------------------------------------
# operator protocol (operators.py:238-301)


class SymmetricOperator:
    """Matrix-free symmetric map on n-vectors with a declared apply cost."""

    batch = 1

    def __init__(self, dim, apply, apply_cost=None):
        self.dim = int(dim)
        self._apply = apply
        self.apply_cost = int(apply_cost) if apply_cost is not None else naive_apply_cost(self.dim)
        if self.apply_cost < 0:
            raise ValueError("apply_cost must be nonnegative")

    def __call__(self, v):
        v = as_device(v)
        if v.shape != (self.dim,):
            raise ValueError(f"operator of dim {self.dim} applied to shape {tuple(v.shape)}")
        return self._apply(v)

    def apply_matrix(self, M):
        M = as_device(M)
        return torch.stack([self(M[:, j]) for j in range(M.shape[1])], dim=1) if M.shape[1] else M.clone()

    def to_dense(self):
        return self.apply_matrix(torch.eye(self.dim, dtype=torch.float64, device=_dev()))


class HessianOperator(SymmetricOperator):
    """Stencil Hessian of a ``Model`` at (theta, xhat); batched over samples.

    ``__call__`` takes (n,) when batch == 1 or (B, n); ``apply_matrix`` takes
    (n, t) or (B, n, t).  Each call is one ``kr_hvp`` launch.
    """

    def __init__(self, model: Model, op: KrOp, keep: dict):
        self.model = model
        self.op = op
        self._keep = keep
        self.dim = model.n
        self.batch = model.batch
        self.apply_cost = model.hessian_cost()

    def sample(self, b: int) -> "HessianOperator":
        if not 0 <= b < self.batch:
            raise IndexError(f"sample {b} out of range for batch {self.batch}")
        return self.slice(b, b + 1)

    def slice(self, lo: int, hi: int) -> "HessianOperator":
        """Operator over samples [lo, hi): the same kr_op with shifted per-sample pointers."""
        if not 0 <= lo < hi <= self.batch:
            raise IndexError(f"samples [{lo}, {hi}) out of range for batch {self.batch}")
        op = KrOp.from_buffer_copy(self.op)
        op.batch = hi - lo
        k = self._keep
        if op.mask_bstride:
            op.mask = k["mask"][lo].data_ptr()
        if "curv" in k:
            op.curv = k["curv"][lo].data_ptr()
        if "slope" in k:
            op.slope = k["slope"][lo].data_ptr()
        if "xhat" in k:
            op.xhat = k["xhat"][lo].data_ptr()
        return HessianOperator(self.model.slice(lo, hi), op, self._keep)

    def select(self, idx) -> "HessianOperator":
        """Operator over the samples idx (any order): the per-sample tables (curvature,
        slope, xhat, mask) gathered into new buffers; theta's filter bank is shared."""
        idx = list(idx)
        if not idx or min(idx) < 0 or max(idx) >= self.batch:
            raise IndexError(f"samples {idx} out of range for batch {self.batch}")
        op = KrOp.from_buffer_copy(self.op)
        op.batch = len(idx)
        k = dict(self._keep)
        dev = self.model.y.device
        it = torch.as_tensor(idx, dtype=torch.long, device=dev)
        if op.mask_bstride and "mask" in k:
            k["mask"] = k["mask"].index_select(0, it)
            op.mask = k["mask"].data_ptr()
        for key in ("curv", "slope", "xhat"):
            if key in k:
                k[key] = k[key].index_select(0, it)
                setattr(op, key, k[key].data_ptr())
        return HessianOperator(self.model.select(idx), op, k)

    def _apply_cols(self, M: torch.Tensor) -> torch.Tensor:
        # M: (B, n, t) with contiguous columns
        B, n, t = M.shape
        out = new_columns(B, n, t, device=M.device)
        if t == 0:
            return out
        _lib.check(_lib.lib().kr_hvp(ctypes.byref(self.op), M.data_ptr(), M.stride(2) if t > 1 else n,
                                     M.stride(0), t, out.data_ptr(), out.stride(2) if t > 1 else n,
                                     out.stride(0), _lib.stream_ptr()), "kr_hvp")
        _lib.note_launch("kr_hvp")
        return out

    def __call__(self, v):
        v = as_device(v)
        if v.dim() == 1:
            if self.batch != 1 or v.shape[0] != self.dim:
                raise ValueError(f"operator of dim {self.dim} applied to shape {tuple(v.shape)}")
            return self._apply_cols(v.contiguous().reshape(1, -1, 1)).reshape(-1)
        if v.shape != (self.batch, self.dim):
            raise ValueError(f"batched operator ({self.batch}, {self.dim}) applied to {tuple(v.shape)}")
        return self._apply_cols(v.contiguous().unsqueeze(-1)).squeeze(-1)

    def apply_matrix(self, M):
        M = as_device(M)
        if M.dim() == 2:
            if self.batch != 1 or M.shape[0] != self.dim:
                raise ValueError(f"operator of dim {self.dim} applied to shape {tuple(M.shape)}")
            return self._apply_cols(columns(M).unsqueeze(0))[0]
        if M.shape[0] != self.batch or M.shape[1] != self.dim:
            raise ValueError(f"batched operator applied to {tuple(M.shape)}")
        return self._apply_cols(columns(M))


class DenseOperator(HessianOperator):
    """Explicit symmetric matrix on the device (operators.py:269-274)."""

    def __init__(self, M: torch.Tensor, apply_cost=None):
        M = as_device(M)
        if M.dim() == 2:
            M = M.unsqueeze(0)
        if M.dim() != 3 or M.shape[1] != M.shape[2]:
            raise ValueError(f"expected a square matrix, got shape {tuple(M.shape)}")
        M = M.contiguous()
        op = KrOp()
        op.rows, op.cols, op.batch = 1, M.shape[1], M.shape[0]
        op.data_kind = _lib.DATA_DENSE
        op.dense = M.data_ptr()
        op.dense_bstride = M.shape[1] * M.shape[2]
        self.op = op
        self._keep = {"dense": M}
        self.matrix = M
        self.model = None
        self.dim = M.shape[1]
        self.batch = M.shape[0]
        self.apply_cost = int(apply_cost) if apply_cost is not None else naive_apply_cost(self.dim)

    def sample(self, b: int) -> "DenseOperator":
        return DenseOperator(self.matrix[b], self.apply_cost)

    def slice(self, lo: int, hi: int) -> "DenseOperator":
        return DenseOperator(self.matrix[lo:hi], self.apply_cost)


def dense_operator(M, apply_cost=None) -> DenseOperator:
    return DenseOperator(M, apply_cost)


class MixedJacobianOperator:
    """w -> J w with J = -(D^2_{theta x} L)^T (operators.py:277-301); generic callable form."""

    batch = 1

    def __init__(self, num_params, dim, apply_adjoint, adjoint_cost=0):
        self.num_params = int(num_params)
        self.dim = int(dim)
        self._apply_adjoint = apply_adjoint
        self.adjoint_cost = int(adjoint_cost)

    def apply_adjoint(self, w):
        w = as_device(w)
        if w.shape != (self.dim,):
            raise ValueError(f"expected an n-vector of length {self.dim}, got shape {tuple(w.shape)}")
        return self._apply_adjoint(w)

    def apply_adjoint_matrix(self, W):
        W = as_device(W)
        return torch.stack([self.apply_adjoint(W[:, j]) for j in range(W.shape[1])], dim=1)

    def to_dense(self):
        return self.apply_adjoint_matrix(torch.eye(self.dim, dtype=torch.float64, device=_dev()))


class StencilJacobian(MixedJacobianOperator):
    """Mixed Jacobian of a ``Model`` at (theta, xhat): one ``kr_jadj`` launch per call."""

    def __init__(self, model: Model, op: KrOp, keep: dict):
        self.model = model
        self.op = op
        self._keep = keep
        self.num_params = model.num_params
        self.dim = model.n
        self.batch = model.batch
        self.adjoint_cost = model.jacobian_cost()

    def sample(self, b: int) -> "StencilJacobian":
        H = HessianOperator(self.model, self.op, self._keep).sample(b)
        return StencilJacobian(H.model, H.op, self._keep)

    def slice(self, lo: int, hi: int) -> "StencilJacobian":
        H = HessianOperator(self.model, self.op, self._keep).slice(lo, hi)
        return StencilJacobian(H.model, H.op, self._keep)

    def select(self, idx, hessian: "HessianOperator | None" = None) -> "StencilJacobian":
        """Jacobian over the samples idx; pass the matching ``HessianOperator.select`` to
        share its gathered tables."""
        H = hessian if hessian is not None else HessianOperator(self.model, self.op, self._keep).select(idx)
        return StencilJacobian(H.model, H.op, H._keep)

    def _apply_cols(self, W: torch.Tensor) -> torch.Tensor:
        B, n, t = W.shape
        p = self.num_params
        out = new_columns(B, p, t, device=W.device)
        if t == 0:
            return out
        L = _lib.lib()
        wl = L.kr_jadj_workspace(ctypes.byref(self.op), t)
        ws = torch.empty(max(wl, 1), dtype=torch.float64, device=W.device)
        _lib.check(L.kr_jadj(ctypes.byref(self.op), W.data_ptr(), W.stride(2) if t > 1 else n, W.stride(0), t,
                             out.data_ptr(), out.stride(2) if t > 1 else p, out.stride(0), ws.data_ptr(), wl,
                             _lib.stream_ptr()), "kr_jadj")
        _lib.note_launch("kr_jadj", 2)
        return out

    def apply_adjoint(self, w):
        w = as_device(w)
        if w.dim() == 1:
            if self.batch != 1 or w.shape[0] != self.dim:
                raise ValueError(f"expected an n-vector of length {self.dim}, got shape {tuple(w.shape)}")
            return self._apply_cols(w.contiguous().reshape(1, -1, 1)).reshape(-1)
        if w.shape != (self.batch, self.dim):
            raise ValueError(f"batched Jacobian ({self.batch}, {self.dim}) applied to {tuple(w.shape)}")
        return self._apply_cols(w.contiguous().unsqueeze(-1)).squeeze(-1)

    def apply_adjoint_matrix(self, W):
        W = as_device(W)
        if W.dim() == 2:
            if self.batch != 1:
                raise ValueError("use a (B, n, t) block for a batched Jacobian")
            return self._apply_cols(columns(W).unsqueeze(0))[0]
        return self._apply_cols(columns(W))


def operators_at(model: Model, theta, x_hat):
    return model.at(theta, x_hat)


# --------------------------------------------------------------------------
# reference entry points (operators.py:329-444)


def _foe_model(params: FoEParams, prob: InpaintingProblem) -> Model:
    m = prob.model()
    m.num_filters, m.ksize = params.num_filters, params.kernel_size
    return m


def foe_hessian(params: FoEParams, prob: InpaintingProblem) -> HessianOperator:
    """operators.py:363-383 on the device."""
    H, _ = _foe_model(params, prob).at(params.flatten(), None)
    return H


def mixed_jacobian(params: FoEParams, x_hat: ImageVector, prob: InpaintingProblem) -> StencilJacobian:
    """operators.py:411-444 on the device."""
    if tuple(x_hat.shape) != tuple(prob.shape):
        raise ValueError(f"image shape {x_hat.shape} does not match expected {prob.shape}")
    _, J = _foe_model(params, prob).at(params.flatten(), x_hat.data)
    return J


def foe_cost(x: ImageVector, params: FoEParams, prob: InpaintingProblem) -> float:
    """operators.py:329-342 on the device."""
    if tuple(x.shape) != tuple(prob.shape):
        raise ValueError(f"image shape {x.shape} does not match expected {prob.shape}")
    c, _ = _foe_model(params, prob).cost_grad(params.flatten(), as_device(x.data))
    v = float(c[0])
    if not np.isfinite(v):
        raise FloatingPointError("non-finite lower-level cost; exp(log-weight) overflowed the filter term")
    return v


def foe_gradient(x: ImageVector, params: FoEParams, prob: InpaintingProblem) -> torch.Tensor:
    """operators.py:345-353 on the device."""
    if tuple(x.shape) != tuple(prob.shape):
        raise ValueError(f"image shape {x.shape} does not match expected {prob.shape}")
    _, g = _foe_model(params, prob).cost_grad(params.flatten(), as_device(x.data))
    return g[0]
