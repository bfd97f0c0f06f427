"""The fp64 tensor-core products of the recycle update (kr_gemm.cu) against torch.matmul.

Oracle: the dense products the reference writes with numpy (`W.T @ HW`, recycling.py:230, 250;
`A @ coeffs`, recycling.py:362-383) evaluated by torch in fp64.  The kernels sum in a different
order (k-steps of 4 inside mma.m8n8k4, split-K partials in fixed order), so the bar is a
relative 1e-13 of ||x_i|| ||y_j||; repeated launches must be bitwise identical (deterministic
split-K), and a true Gram must come back exactly symmetric (mirrored lower tile blocks).
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _rand(*shape, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, dtype=torch.float64, device="cuda", generator=g)


@pytest.mark.parametrize("B,T,n", [(1, 1, 4096), (2, 7, 4098), (3, 64, 8192), (2, 65, 5000), (2, 130, 16384),
                                   (1, 331, 65536)])
def test_gram_matches_matmul(cuda, B, T, n):
    from paper_2412_08264_b200.batched import gram

    A = _rand(B, T, n, seed=B * 1000 + T)
    G = gram(A)
    ref = A @ A.transpose(1, 2)
    scale = (A.norm(dim=2)[:, :, None] * A.norm(dim=2)[:, None, :]).clamp_min(1e-300)
    assert float(((G - ref).abs() / scale).max()) < 1e-13
    assert torch.equal(G, G.transpose(1, 2))  # mirrored lower tile blocks
    assert torch.equal(G, gram(A))            # deterministic split-K
    Bm = _rand(B, T, n, seed=7)
    G2 = gram(A, Bm)
    ref2 = A @ Bm.transpose(1, 2)
    scale2 = (A.norm(dim=2)[:, :, None] * Bm.norm(dim=2)[:, None, :]).clamp_min(1e-300)
    assert float(((G2 - ref2).abs() / scale2).max()) < 1e-13


def test_gram_odd_strides(cuda):
    """Rows of odd length and an odd leading dimension take the 8-byte copy path."""
    from paper_2412_08264_b200 import _lib

    B, T, n, ld = 2, 37, 4097, 4099
    buf = _rand(B, T, ld, seed=3)
    A = buf[:, :, :n]
    G = torch.empty(B, T, T, dtype=torch.float64, device="cuda")
    L = _lib.lib()
    wl = int(L.kr_gram_workspace(B, T, n))
    ws = torch.empty(wl, dtype=torch.float64, device="cuda")
    _lib.check(L.kr_gram(buf.data_ptr(), buf.data_ptr(), ld, T * ld, B, T, n, G.data_ptr(), T, T * T, ws.data_ptr(), wl,
                         _lib.stream_ptr()), "kr_gram")
    ref = A @ A.transpose(1, 2)
    assert float((G - ref).abs().max() / ref.abs().max()) < 1e-13


@pytest.mark.parametrize("B,R2,R1,L", [(1, 1, 1, 130), (2, 30, 200, 4096), (2, 33, 64, 4098), (3, 64, 64, 1000),
                                       (2, 130, 130, 16384), (1, 331, 331, 65536), (2, 100, 40, 331)])
def test_rows_mul_matches_matmul(cuda, B, R2, R1, L):
    from paper_2412_08264_b200.gemm import rows_mul

    F = _rand(B, R2, R1, seed=R2)
    X = _rand(B, R1, L, seed=L % 1000)
    Y = rows_mul(F, X)
    ref = F @ X
    scale = (F.norm(dim=2)[:, :, None] * X.norm(dim=1)[:, None, :]).clamp_min(1e-300)
    assert float(((Y - ref).abs() / scale).max()) < 1e-13
    # accumulate: Y <- -0.5 F X + 2 Y0
    Y0 = _rand(B, R2, L, seed=11)
    Y1 = rows_mul(F, X, out=Y0.clone(), alpha=-0.5, beta=2.0)
    assert float(((Y1 - (-0.5 * ref + 2.0 * Y0)).abs() / (scale + Y0.abs())).max()) < 1e-13


@pytest.mark.parametrize("B,T,L", [(2, 50, 4096), (2, 130, 8192), (1, 331, 65536), (2, 200, 200)])
def test_rows_mul_lower_triangular(cuda, B, T, L):
    """lower = True must not read the strict upper triangle beyond the diagonal tile: the
    result equals tril(F) @ X, and garbage above the diagonal tiles is ignored."""
    from paper_2412_08264_b200.gemm import rows_mul

    F = torch.tril(_rand(B, T, T, seed=T))
    X = _rand(B, T, L, seed=5)
    ref = F @ X
    Fg = F.clone()
    for i0 in range(0, T, 64):  # NaN above the 64-row diagonal tiles
        Fg[:, i0:i0 + 64, i0 + 64:] = float("nan")
    Y = rows_mul(Fg, X, lower=True)
    scale = (F.norm(dim=2)[:, :, None] * X.norm(dim=1)[:, None, :]).clamp_min(1e-300)
    assert float(((Y - ref).abs() / scale).max()) < 1e-13
