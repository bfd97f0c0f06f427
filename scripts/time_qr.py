"""Time the tall Householder QR shapes of the rank-drop path."""
import os
import sys
import time

import torch

x = torch.randn(16384, 220, dtype=torch.float64, device="cuda")
for name, fn in (("linalg.qr", lambda: torch.linalg.qr(x)), ("geqrf", lambda: torch.geqrf(x)),
                 ("geqrf+householder_product", lambda: torch.linalg.householder_product(*torch.geqrf(x)))):
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        print(f"{name:28s} rep {rep}: {(time.perf_counter() - t0) * 1e3:8.2f} ms", flush=True)
