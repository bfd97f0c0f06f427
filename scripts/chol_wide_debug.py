"""kr_chol_inv at t > 228 (global workspace) vs the shared-memory variant (flag 16
forces the workspace path at any t: bitwise equal expected) and vs torch.linalg."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2412_08264_b200 import _lib, batched  # noqa: E402


def run(G, dims, flags, force_ws=False):
    B, T, _ = G.shape
    L = _lib.lib()
    wl = B * T * (T + 1) // 2 if force_ws else int(L.kr_chol_inv_workspace(B, T))
    ws = torch.empty(max(wl, 1), dtype=torch.float64, device="cuda")
    F = torch.empty_like(G)
    st = torch.empty(B, 4, dtype=torch.float64, device="cuda")
    info = torch.empty(B, dtype=torch.int32, device="cuda")
    _lib.check(L.kr_chol_inv(G.data_ptr(), T, T * T, dims.data_ptr(), B, T, flags | (16 if force_ws else 0), 0,
                             F.data_ptr(), T, T * T, st.data_ptr(), info.data_ptr(), 0, ws.data_ptr(), wl,
                             _lib.stream_ptr()), "chol")
    return F, info, st


for T in (200, 228, 229, 330):
    g = torch.Generator(device="cuda").manual_seed(T)
    B = 3
    X = torch.randn(B, T, 3 * T + 4, generator=g, dtype=torch.float64, device="cuda")
    G = (X @ X.transpose(1, 2)).contiguous()
    dims = torch.tensor([T, T - 3, 7], dtype=torch.int32, device="cuda")
    for flags in (2, 3):
        F1, i1, _ = run(G, dims, flags)
        F2, i2, _ = run(G, dims, flags, force_ws=True)
        Ft, it, _ = batched._chol_inv.__wrapped__(G, dims, bool(flags & 1)) if hasattr(batched._chol_inv, "__wrapped__") else (None, None, None)
        old = batched.CHOL_TMAX
        batched.CHOL_TMAX = -1
        Ft, it, _ = batched._chol_inv(G, dims, bool(flags & 1))
        batched.CHOL_TMAX = old
        for b in range(B):
            e12 = float((F1[b] - F2[b]).abs().max())
            e1t = float((F1[b] - Ft[b]).abs().max() / Ft[b].abs().max())
            print(f"T={T} flags={flags} b={b} info={int(i1[b])},{int(i2[b])},{int(it[b])} smem-vs-ws {e12:.3e} vs-torch {e1t:.3e}")
