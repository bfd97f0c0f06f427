"""Recycle update batched over samples (the B200 layout of ``next_recycle``).

The reference updates one sample at a time through numpy/LAPACK
(recycling.py:386-465).  Here every step of the update runs once for the whole
batch: sample b's t_b candidate vectors are the rows [0, t_b) of a (B, T, n)
block (T = max t_b, zero rows beyond), the n x t products are strided-batched
GEMMs, the t x t factorizations are batched Cholesky (cuSOLVER) and the
selected-eigenpair kernel ``kr_syev_select`` (one CTA per sample).  Padding is
exact: pad rows are zero and the pad block of every Gram matrix is the identity,
so the leading t_b block of each factor is the per-sample factor.

Vectors are stored as ROWS here ((B, t, n): sample b, vector j, n entries), i.e.
the column-major n x t blocks of the reference with one contiguous vector per
row; the per-sample views handed back are the reference's n x t column blocks.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

SIZE_CODES = {"S": 0, "L": 1, "M": 2}
EIG_TMAX = 228


def syev_select(M: torch.Tensor, dims: torch.Tensor, size: str, s: int):
    """Selected eigenpairs of the leading dims[b] x dims[b] blocks of M (B, T, T).

    Returns (lam (B, s), Z (B, s, T), nsel (B,) int32), all on the device:
    eigenvector q of sample b is Z[b, q] (zero beyond dims[b]); see kr_syev_select."""
    B, T, T2 = M.shape
    if T != T2:
        raise ValueError(f"expected square blocks, got {tuple(M.shape)}")
    if M.stride(2) != 1 and M.stride(1) != 1:
        M = M.contiguous()
    M = M.contiguous()
    dims = dims.to(device=M.device, dtype=torch.int32).contiguous()
    lam = torch.zeros(B, max(s, 1), dtype=torch.float64, device=M.device)
    Z = torch.empty(B, max(s, 1), T, dtype=torch.float64, device=M.device)
    nsel = torch.zeros(B, dtype=torch.int32, device=M.device)
    L = _lib.lib()
    wl = int(L.kr_syev_select_workspace(B, T))
    ws = torch.empty(max(wl, 1), dtype=torch.float64, device=M.device)
    # M is symmetrised inside, so row- or column-major reading gives the same matrix
    _lib.check(L.kr_syev_select(M.data_ptr(), T, T * T, dims.data_ptr(), B, T, SIZE_CODES[size], s,
                                lam.data_ptr(), lam.stride(0), Z.data_ptr(), T, Z.stride(0), nsel.data_ptr(),
                                ws.data_ptr(), wl, _lib.stream_ptr()), "kr_syev_select")
    _lib.note_launch("kr_syev_select")
    return lam[:, :s], Z[:, :s], nsel
