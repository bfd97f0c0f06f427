"""Latency probe of the small dense decompositions the recycle update needs (fp64, B200)."""

import time

import torch

dev = "cuda"
torch.manual_seed(0)


def t(name, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    print(f"{name:45s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms")


tt = 220
A = torch.randn(tt, tt, dtype=torch.float64, device=dev)
S = A @ A.T + tt * torch.eye(tt, dtype=torch.float64, device=dev)
S8 = S.expand(8, tt, tt).contiguous()
W = torch.randn(16384, tt, dtype=torch.float64, device=dev)
J = torch.randn(428, tt, dtype=torch.float64, device=dev)
P = torch.randn(208, tt, dtype=torch.float64, device=dev)
t("eigh 220", lambda: torch.linalg.eigh(S))
t("eigh 8x220 batched", lambda: torch.linalg.eigh(S8))
t("eigvalsh 220", lambda: torch.linalg.eigvalsh(S))
t("svdvals 220", lambda: torch.linalg.svdvals(S))
t("svd 208x220 reduced", lambda: torch.linalg.svd(P, full_matrices=False))
t("svd 220x220 gesvdj", lambda: torch.linalg.svd(S, full_matrices=False, driver="gesvdj"))
t("qr 428x220", lambda: torch.linalg.qr(J))
t("qr 16384x220", lambda: torch.linalg.qr(W))
t("cholesky 220", lambda: torch.linalg.cholesky(S))
t("cholesky_ex 220", lambda: torch.linalg.cholesky_ex(S))
t("solve_triangular 220", lambda: torch.linalg.solve_triangular(S.triu(), S, upper=True))
t("gram W^T W 16384x220", lambda: W.T @ W)
t("W @ X 16384x220x20", lambda: W @ S[:, :20])
t("eigh 220 (cpu)", lambda: torch.linalg.eigh(S.cpu()))
t("svd 208x220 (cpu)", lambda: torch.linalg.svd(P.cpu(), full_matrices=False))
