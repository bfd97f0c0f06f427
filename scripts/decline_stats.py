"""Count samples the batched recycle update declines on the C2 bench sequence, per check."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
model = make_batch(cfg)
steps = 8
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), steps)
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
batched.STATS = {}
for i in range(steps):
    hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    print(i, dict(batched.STATS), flush=True)
