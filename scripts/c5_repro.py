import sys, torch
sys.path.insert(0,'/root/repo')
from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence
import os
cfg = CONFIGS["C5"]; model = make_batch(cfg)
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 3)
seq = SequenceSolver(HessianSolveConfig.from_strategy(sys.argv[1], recycle_dim=int(sys.argv[2]), delta=float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6, max_iter=500))
for i in range(3):
    hg, res, _ = hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    print(i, [r.iterations for r in res], flush=True)
