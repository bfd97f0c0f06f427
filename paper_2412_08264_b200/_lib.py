"""ctypes binding of ``include/krecycle_b200.h`` (the C ABI of the CUDA path).

There is no CPU fallback: if the shared library is missing, was built for the
wrong ABI, or no CUDA device is visible, every entry point raises.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import torch

from ._build import lib_path

KR_OK, KR_EINVAL, KR_ECUDA, KR_ENONSPD, KR_ENOMEM = 0, -1, -2, -3, -4
KR_MAX_BLUR = 31
DATA_NONE, DATA_MASK, DATA_BLUR, DATA_DENSE = 0, 1, 2, 3
REG_NONE, REG_FILTERS, REG_TV = 0, 1, 2
POT_QUADRATIC, POT_SMOOTH_ABS = 0, 1
REASONS = {0: "tolerance", 1: "max_iter", 2: "breakdown", 3: "nonspd"}

_c_i32, _c_i64, _c_f64, _c_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class KrOp(ctypes.Structure):
    """Mirror of ``kr_op`` (include/krecycle_b200.h)."""

    _fields_ = [
        ("rows", _c_i32), ("cols", _c_i32), ("batch", _c_i32), ("data_kind", _c_i32),
        ("data_scale", _c_f64), ("ridge", _c_f64),
        ("mask", _c_p), ("mask_bstride", _c_i64),
        ("dense", _c_p), ("dense_bstride", _c_i64),
        ("blur_size", _c_i32), ("blur_taps", _c_f64 * KR_MAX_BLUR),
        ("reg_kind", _c_i32), ("potential", _c_i32), ("eps", _c_f64),
        ("num_filters", _c_i32), ("ksize", _c_i32),
        ("kernels", _c_p), ("fweights", _c_p), ("curv", _c_p), ("slope", _c_p), ("xhat", _c_p),
    ]


ABI_VERSION = 6  # KR_ABI_VERSION of include/krecycle_b200.h


class KrSolveArgs(ctypes.Structure):
    """Mirror of ``kr_solve_args``."""

    _fields_ = [
        ("max_iter", _c_i32), ("s", _c_i32),
        ("g", _c_p), ("w0", _c_p), ("U", _c_p), ("C", _c_p), ("ld_uc", _c_i64), ("bs_uc", _c_i64),
        ("stop_kind", _c_i32), ("delta", _c_f64), ("nsc_s", _c_i32),
        ("Z", _c_p), ("ld_z", _c_i64), ("bs_z", _c_i64), ("ZtC", _c_p),
        ("track_residual", _c_i32),
        ("w", _c_p), ("r", _c_p), ("basis", _c_p), ("ld_basis", _c_i64), ("bs_basis", _c_i64),
        ("res_norms", _c_p), ("stop_vals", _c_p), ("iters", _c_p), ("reasons", _c_p),
        ("Minv", _c_p), ("nsc_r0", _c_p),
    ]


class KrRecycleArgs(ctypes.Structure):
    """Mirror of ``kr_recycle_args``."""

    _fields_ = [
        ("batch", _c_i32), ("T", _c_i32), ("s", _c_i32), ("vec_type", _c_i32), ("size_code", _c_i32),
        ("side", _c_i32), ("reuse_products", _c_i32),
        ("V", _c_p), ("ld_v", _c_i64), ("bs_v", _c_i64), ("kdims", _c_p),
        ("Uprev", _c_p), ("ld_u", _c_i64), ("bs_u", _c_i64), ("sdims", _c_p),
        ("W", _c_p), ("HW", _c_p), ("U", _c_p), ("C", _c_p), ("mu", _c_p), ("VH", _c_p), ("Z", _c_p),
        ("tdims", _c_p), ("nsel", _c_p), ("status", _c_p), ("op_proj", _c_p),
    ]


class KrError(RuntimeError):
    pass


class NonSPDError(RuntimeError):
    """CG met non-positive curvature (krylov.py:53-54)."""


_LOCK = threading.Lock()
_LIB = None


def _declare(lib):
    P = ctypes.POINTER
    sig = {
        "kr_abi_version": (_c_i32, []),
        "kr_last_error": (ctypes.c_char_p, []),
        "kr_device_info": (_c_i32, [P(_c_i32), P(_c_i32), P(_c_i32)]),
        "kr_struct_sizes": (_c_i32, [P(_c_i64), P(_c_i64)]),
        "kr_op_prepare": (_c_i32, [P(KrOp), _c_p]),
        "kr_hvp": (_c_i32, [P(KrOp), _c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i64, _c_p]),
        "kr_jadj_workspace": (_c_i64, [P(KrOp), _c_i32]),
        "kr_jadj": (_c_i32, [P(KrOp), _c_p, _c_i64, _c_i64, _c_i32, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_p]),
        "kr_lower_workspace": (_c_i64, [P(KrOp)]),
        "kr_lower_eval": (_c_i32, [P(KrOp), _c_p, _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
        "kr_rminres_workspace": (_c_i64, [P(KrOp), P(KrSolveArgs)]),
        "kr_rminres": (_c_i32, [P(KrOp), P(KrSolveArgs), _c_p, _c_i64, _c_p]),
        "kr_cg_workspace": (_c_i64, [P(KrOp), P(KrSolveArgs)]),
        "kr_cg": (_c_i32, [P(KrOp), P(KrSolveArgs), _c_p, _c_i64, _c_p]),
        "kr_syev_select_workspace": (_c_i64, [_c_i32, _c_i32]),
        "kr_syev_select": (_c_i32, [_c_p, _c_i64, _c_i64, _c_p, _c_i32, _c_i32, _c_i32, _c_i32, _c_p, _c_i64,
                                    _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_i64, _c_p]),
        "kr_chol_inv_workspace": (_c_i64, [_c_i32, _c_i32]),
        "kr_chol_inv": (_c_i32, [_c_p, _c_i64, _c_i64, _c_p, _c_i32, _c_i32, _c_i32, _c_p, _c_p, _c_i64, _c_i64,
                                 _c_p, _c_p, _c_p, _c_p, _c_i64, _c_p]),
        "kr_qrcp_small": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, ctypes.c_double, _c_p, _c_p, _c_p, _c_p, _c_i64,
                                   _c_p]),
        "kr_qrcp_small_cluster": (_c_i32, [_c_p, _c_p, _c_i32, _c_i32, ctypes.c_double, _c_p, _c_p, _c_p, _c_p,
                                           _c_i64, _c_p]),
        "kr_recycle_workspace": (_c_i64, [P(KrOp), P(KrRecycleArgs)]),
        "kr_thread_warmup": (ctypes.c_int, []),
        "kr_recycle_update": (_c_i32, [P(KrOp), P(KrRecycleArgs), _c_p, _c_i64, _c_p]),
        "kr_ordered_sum": (_c_i32, [_c_p, _c_i32, _c_i32, _c_i64, _c_p, _c_p]),
        "kr_gram_workspace": (_c_i64, [_c_i32, _c_i32, _c_i64]),
        "kr_gram": (_c_i32, [_c_p, _c_p, _c_i64, _c_i64, _c_i32, _c_i32, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64,
                             _c_p]),
        "kr_rows_mul": (_c_i32, [_c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_p, _c_i64, _c_i64, _c_i32, _c_i32,
                                 _c_i64, _c_i32, ctypes.c_double, ctypes.c_double, _c_i32, _c_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return sig


EXPORTED = (
    "kr_abi_version", "kr_last_error", "kr_device_info", "kr_struct_sizes", "kr_op_prepare",
    "kr_hvp", "kr_jadj_workspace", "kr_jadj", "kr_lower_workspace", "kr_lower_eval",
    "kr_rminres_workspace", "kr_rminres", "kr_cg_workspace", "kr_cg",
    "kr_syev_select_workspace", "kr_syev_select", "kr_chol_inv_workspace", "kr_chol_inv", "kr_qrcp_small", "kr_qrcp_small_cluster",
    "kr_gram_workspace", "kr_gram", "kr_recycle_workspace", "kr_recycle_update", "kr_thread_warmup",
    "kr_ordered_sum", "kr_rows_mul",
)


def load_library(path: Path | None = None):
    """Load and verify the shared library (no device needed)."""
    global _LIB
    with _LOCK:
        if _LIB is not None and path is None:
            return _LIB
        p = Path(path) if path is not None else lib_path()
        if not p.exists():
            raise ImportError(
                f"CUDA extension {p} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(str(p))
        _declare(lib)
        if lib.kr_abi_version() != ABI_VERSION:
            raise ImportError("libkrecycle_b200 ABI version mismatch")
        a, b = _c_i64(), _c_i64()
        lib.kr_struct_sizes(ctypes.byref(a), ctypes.byref(b))
        if a.value != ctypes.sizeof(KrOp) or b.value != ctypes.sizeof(KrSolveArgs):
            raise ImportError(
                f"struct layout mismatch: kr_op {a.value} vs {ctypes.sizeof(KrOp)}, "
                f"kr_solve_args {b.value} vs {ctypes.sizeof(KrSolveArgs)}"
            )
        if path is None:
            _LIB = lib
        return lib


def lib():
    """The library, on a machine with a CUDA device (raises otherwise)."""
    L = load_library()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2412_08264_b200 needs a CUDA device; there is no CPU fallback")
    return L


def check(rc: int, what: str = ""):
    if rc == KR_OK:
        return
    msg = (_LIB.kr_last_error() or b"").decode() if _LIB is not None else ""
    text = f"{what}: {msg}" if what else msg
    if rc == KR_EINVAL:
        raise ValueError(text)
    if rc == KR_ENONSPD:
        raise NonSPDError(text)
    raise KrError(text)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# --------------------------------------------------------------------------
# instrumentation used by bench.py: launch counts and CUDA-event kernel timing

LAUNCHES: dict = {}
PROFILE: list | None = None  # when a list, solver launches append (start_event, end_event, info)


def note_launch(name: str, count: int = 1) -> None:
    LAUNCHES[name] = LAUNCHES.get(name, 0) + count


def total_launches() -> int:
    return sum(LAUNCHES.values())
