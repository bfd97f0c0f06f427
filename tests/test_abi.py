"""CPU tests of the C ABI boundary: the library loads without a GPU, exports every
symbol include/krecycle_b200.h declares, its struct layout matches the binding,
and argument validation maps onto the reference's exceptions without touching
the device."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2412_08264_b200 import _lib
from paper_2412_08264_b200._build import lib_path

HEADER = Path(__file__).resolve().parents[1] / "include" / "krecycle_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(kr_\w+)\s*\(", text, flags=re.M)))


def test_library_builds_and_loads():
    assert lib_path().exists(), "run __graft_entry__.build() first"
    L = _lib.load_library()
    assert L.kr_abi_version() == _lib.ABI_VERSION == 6


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 14
    L = ctypes.CDLL(str(lib_path()))
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_struct_layout_matches_binding():
    L = _lib.load_library()
    a, b = ctypes.c_int64(), ctypes.c_int64()
    assert L.kr_struct_sizes(ctypes.byref(a), ctypes.byref(b)) == 0
    assert a.value == ctypes.sizeof(_lib.KrOp)
    assert b.value == ctypes.sizeof(_lib.KrSolveArgs)


def test_argument_validation_without_device():
    L = _lib.load_library()
    assert L.kr_hvp(None, None, 0, 0, 1, None, 0, 0, None) == _lib.KR_EINVAL
    assert b"null operator" in L.kr_last_error()
    op = _lib.KrOp()
    op.rows, op.cols, op.batch = 8, 8, 1
    op.data_kind = _lib.DATA_BLUR
    op.blur_size = 4  # even: invalid
    assert L.kr_op_prepare(ctypes.byref(op), None) == _lib.KR_EINVAL
    assert b"odd" in L.kr_last_error()
    op.blur_size = 9
    op.reg_kind = _lib.REG_FILTERS
    op.num_filters, op.ksize = 2, 4
    assert L.kr_op_prepare(ctypes.byref(op), None) == _lib.KR_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.KR_EINVAL, "x")
    with pytest.raises(_lib.NonSPDError):
        _lib.check(_lib.KR_ENONSPD, "x")


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="CUDA"):
        _lib.lib()


def test_product_never_imports_the_oracle():
    pkg = Path(__file__).resolve().parents[1] / "paper_2412_08264_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "from oracle" not in src, f
