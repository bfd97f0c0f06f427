"""Host bindings of the fp64 tensor-core products of the recycle update (kr_gemm.cu).

``gram`` lives in ``batched.py`` (it predates this module); ``rows_mul`` is the
row-block product Y = alpha F X + beta Y behind the W <- R^-T A passes of the
Cholesky-QRs (reference recycling.py:194, 369) and the basis recombinations
U~ = W X, H U~ = (H W) X (recycling.py:362-383).
"""

from __future__ import annotations

import torch

from . import _lib


def rows_mul(F: torch.Tensor, X: torch.Tensor, out: torch.Tensor | None = None, alpha: float = 1.0,
             beta: float = 0.0, lower: bool = False) -> torch.Tensor:
    """(B, R2, L) = alpha F (B, R2, R1) @ X (B, R1, L) + beta out.  ``lower``: F is lower
    triangular (its strict upper triangle is not read past the diagonal tile)."""
    if F.dim() != 3 or X.dim() != 3 or F.shape[0] != X.shape[0] or F.shape[2] != X.shape[1]:
        raise ValueError("rows_mul: F (B, R2, R1) and X (B, R1, L) expected")
    if not (F.is_cuda and X.is_cuda and F.dtype == torch.float64 and X.dtype == torch.float64):
        raise ValueError("rows_mul: float64 CUDA tensors expected")
    F = F.contiguous()
    X = X.contiguous()
    B, R2, R1 = F.shape
    L = X.shape[2]
    if out is None:
        if beta != 0.0:
            raise ValueError("rows_mul: beta needs an output to accumulate into")
        out = torch.empty(B, R2, L, dtype=torch.float64, device=X.device)
    elif out.shape != (B, R2, L) or not out.is_contiguous():
        raise ValueError("rows_mul: out must be a contiguous (B, R2, L) tensor")
    _lib.check(_lib.lib().kr_rows_mul(F.data_ptr(), R1, R2 * R1, X.data_ptr(), L, R1 * L, out.data_ptr(), L, R2 * L,
                                      R2, R1, L, B, float(alpha), float(beta), int(lower), _lib.stream_ptr()),
               "kr_rows_mul")
    _lib.note_launch("kr_rows_mul", 1)
    return out
