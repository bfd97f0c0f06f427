"""Fast CPU restatement of the deblurring operators -- TEST INFRASTRUCTURE ONLY.

``hessian`` / ``jacobian`` here compute exactly what ``cpu_imaging.hessian`` /
``cpu_imaging.jacobian`` compute for the BASELINE configs' blur + phi_eps learned
filter models (operators.py:363-444 generalised; see cpu_imaging), through the
plain-C restatement ``cpu_stencil.c`` (OpenMP over rows) instead of scipy's direct
``convolve2d``: at 512^2 with J = 24 7x7 filters and a 21x21 blur scipy takes ~3.5 s
per Hessian product, which puts a config-sized oracle sequence out of reach.  Only
the summation order differs (tests/test_oracle.py checks both against each other).
Used by ``tests/golden/make_config_fixtures.py``; never by the product.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

from . import cpu_imaging as im

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "cpu_stencil.c"
_SO = _HERE / "_lib" / "libcpu_stencil.so"
_LIB = None

_D = ctypes.POINTER(ctypes.c_double)


def build() -> Path:
    """Compile cpu_stencil.c (gcc -O2 -fopenmp) into oracle/_lib/ (git-ignored)."""
    _SO.parent.mkdir(exist_ok=True)
    if not _SO.exists() or _SO.stat().st_mtime < _SRC.stat().st_mtime:
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", str(_SO), str(_SRC)])
    return _SO


def _lib():
    global _LIB
    if _LIB is None:
        build()
        L = ctypes.CDLL(str(_SO))
        i, d = ctypes.c_int, ctypes.c_double
        L.oc_hvp.argtypes = [_D, _D, i, i, _D, i, d, d, i, i, _D, _D, _D]
        L.oc_jadj.argtypes = [_D, _D, i, i, _D, i, i, _D, _D, _D, _D]
        L.oc_conv_same.argtypes = [_D, _D, i, i, _D, i]
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _parts(model: im.Model, theta, x_hat):
    d, reg = model.data, model.reg
    if d.kind != "blur" or reg.kind != "filters" or reg.potential != "smooth_abs":
        raise ValueError("cpu_fast covers the blur + phi_eps learned-filter models (BASELINE C2-C5)")
    alphas, kernels = reg.split(theta)
    w = _c(im.filter_weights(alphas))
    R, Cc = d.shape
    xi = _c(np.asarray(x_hat, dtype=float).reshape(R, Cc))
    L = _lib()
    J, q = reg.num_filters, reg.ksize
    kern = _c(kernels)
    cx = np.empty((J, R * Cc))
    for j in range(J):
        kj = _c(kernels[j])
        L.oc_conv_same(_p(xi), _p(cx[j]), R, Cc, _p(kj), q)
    return w, kern, xi, cx, R, Cc, J, q


def hessian(model: im.Model, theta, x_hat) -> im.SymOp:
    """cpu_imaging.hessian for the filter models, through cpu_stencil.oc_hvp."""
    w, kern, xi, cx, R, Cc, J, q = _parts(model, theta, x_hat)
    reg, d = model.reg, model.data
    curv = _c(reg.ddphi(cx))
    taps = _c(d.taps)
    L = _lib()

    def apply(v):
        v = _c(v)
        out = np.empty_like(v)
        L.oc_hvp(_p(v), _p(out), R, Cc, _p(taps), taps.size, float(d.scale), float(d.ridge), J, q, _p(kern), _p(w),
                 _p(curv))
        return out

    return im.SymOp(d.n, apply, im.hessian_cost(model))


def jacobian(model: im.Model, theta, x_hat) -> im.JacOp:
    """cpu_imaging.jacobian for the filter models, through cpu_stencil.oc_jadj."""
    w, kern, xi, cx, R, Cc, J, q = _parts(model, theta, x_hat)
    reg = model.reg
    slope, curv = _c(reg.dphi(cx)), _c(reg.ddphi(cx))
    L = _lib()

    def apply(wv):
        wv = _c(wv)
        out = np.empty(reg.num_params)
        L.oc_jadj(_p(wv), _p(out), R, Cc, _p(xi), J, q, _p(kern), _p(w), _p(slope), _p(curv))
        return out

    conv = model.n * (2 * q * q - 1)
    return im.JacOp(reg.num_params, model.n, apply, reg.num_filters * (2 * conv + 2 * model.n * q * q))


def threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
