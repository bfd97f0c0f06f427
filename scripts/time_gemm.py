"""Time the DMMA products of the recycle update (kr_gemm.cu) against torch (cuBLAS) at the
C3 group shape: 16 samples x T candidate rows x 256^2 pixels."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200.batched import gram
from paper_2412_08264_b200.gemm import rows_mul

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T = int(sys.argv[2]) if len(sys.argv) > 2 else 330
n = int(sys.argv[3]) if len(sys.argv) > 3 else 65536
A = torch.randn(B, T, n, dtype=torch.float64, device="cuda")
F = torch.tril(torch.randn(B, T, T, dtype=torch.float64, device="cuda"))
C = torch.randn(B, 30, T, dtype=torch.float64, device="cuda")
out = torch.empty_like(A)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


full = 2.0 * B * T * T * n
for name, fn, flops in [
    ("gram sym (dmma)", lambda: gram(A), full),
    ("gram A,B (dmma, lower mirrored)", lambda: gram(A, out), full),
    ("gram torch bmm", lambda: torch.bmm(A, A.transpose(1, 2)), full),
    ("rows_mul lower (dmma)", lambda: rows_mul(F, A, out=out, lower=True), full),
    ("rows_mul full (dmma)", lambda: rows_mul(F, A, out=out), full),
    ("rows_mul torch bmm", lambda: torch.bmm(F, A, out=out), full),
    ("rows_mul 30 rows (dmma)", lambda: rows_mul(C, A), 2.0 * B * 30 * T * n),
    ("rows_mul 30 rows torch", lambda: torch.bmm(C, A), 2.0 * B * 30 * T * n),
]:
    ms = timeit(fn)
    print(f"{name:34s} {ms:8.3f} ms   {flops / ms / 1e9:7.2f} TF/s (full-GEMM flop count)")
