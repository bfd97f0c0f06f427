"""cProfile of the host side of bench steps (C2): where the Python time goes."""

import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[name]
model = make_batch(cfg)
n = model.n
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 8, seed=1234)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      method=cfg.method, max_iter=cfg.max_iter))
torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
t_max = cfg.max_iter + cfg.recycle_dim
seq.reserve(cfg.batch, 8 * n * t_max * 6, shape=(n, t_max))
for i in range(4):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for i in range(4, 8):
    hg, _, _ = hypergradients(model, thetas[i], X[i], seq)
    hg.sum().item()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumtime").print_stats(40)
