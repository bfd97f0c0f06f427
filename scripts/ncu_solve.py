"""One config-sized sequence (default C3, 64 samples) through SequenceSolver: systems 0..2;
the persistent solve of the last system is the kernel to capture with
    ncu -k regex:rminres -s 2 -c 1 ... python scripts/ncu_solve.py C3
(the first two rminres launches are systems 0 and 1)."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
systems = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = CONFIGS[name]
model = make_batch(cfg)
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), systems)
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
for i in range(systems):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    hg, res, _ = hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    torch.cuda.synchronize()
    its = [r.iterations for r in res]
    print(f"system {i}: {1e3 * (time.perf_counter() - t0):.1f} ms, iterations mean {sum(its) / len(its):.1f} "
          f"max {max(its)}", flush=True)
