"""Time kr_chol_inv / kr_syev_select at the recycle update's size (B=8, t=220)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import batched

B, T = 8, int(sys.argv[1]) if len(sys.argv) > 1 else 220
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(B, T, 2 * T, generator=g, dtype=torch.float64, device="cuda")
G = X @ X.transpose(1, 2)
dims = torch.full((B,), T, dtype=torch.int32, device="cuda")


def tm(name, fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name:40s} {a.elapsed_time(b) / reps * 1e3:9.1f} us", flush=True)


tm("chol_inv scale+inverse", lambda: batched._chol_inv(G, dims, True))
tm("chol_inv factor only", lambda: batched._chol_inv(G, dims, True, inverse=False))
tm("syev_select L 20", lambda: batched.syev_select(G / T, dims, "L", 20))
tm("syev_select M 2", lambda: batched.syev_select(G / T, dims, "M", 2))
tm("torch cholesky_ex", lambda: torch.linalg.cholesky_ex(G))
R = torch.linalg.cholesky(G).transpose(1, 2).contiguous()  # upper triangular, stored so rows = columns of R^T
tm("qrcp_small", lambda: batched.qrcp_small(R, dims, 1e-10))
tm("gram (B,T,16384)", lambda: torch.randn(1, device="cuda") if False else None)
