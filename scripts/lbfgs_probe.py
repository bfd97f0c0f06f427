"""Device L-BFGS (lower.lower_solve) convergence and speed at a config:  python scripts/lbfgs_probe.py C2"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2412_08264_b200.lower import lower_solve
from paper_2412_08264_b200.problems import CONFIGS, make_batch, theta0

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
model = make_batch(cfg)
th = theta0(cfg)
x = None
for gtol, mi in ((1e-2, 2000), (1e-4, 4000), (1e-6, 8000), (1e-8, 8000)):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, st = lower_solve(model, th, x, gtol=gtol, max_iter=mi)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it = int(st.iterations.max())
    print(f"gtol {gtol:g}: iters max {it} mean {st.iterations.mean():.0f}, |g| max {st.gradient_norm.max():.3e}, "
          f"evals {int(st.cost_evaluations.max())}, {dt:.2f} s ({1e3 * dt / max(it, 1):.2f} ms/iter)", flush=True)
