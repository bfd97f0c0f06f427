"""Per-phase wall-clock breakdown of one C2 hypergradient step (synchronising after each phase)."""

import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

import paper_2412_08264_b200.recycling as rc
from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

T = defaultdict(float)
N = defaultdict(int)


def timed(name, fn):
    def wrap(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        N[name] += 1
        return out
    return wrap


cfg_name = sys.argv[1] if len(sys.argv) > 1 else "C2"
cfg = CONFIGS[cfg_name]
model = make_batch(cfg)
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 6)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
for i in range(3):
    hypergradients(model, thetas[i], X[i], seq)

import paper_2412_08264_b200.bilevel as bl
import paper_2412_08264_b200.krylov as kr
import paper_2412_08264_b200.operators as op

rc.build_candidate_basis = timed("candidate_basis(QR)", rc.build_candidate_basis)
rc.gsvd_pair = timed("gsvd_pair(t x t)", rc.gsvd_pair)
rc.prepare_recycle = timed("prepare_recycle", rc.prepare_recycle)
op.HessianOperator._apply_cols = timed("H.apply (kr_hvp)", op.HessianOperator._apply_cols)
op.StencilJacobian._apply_cols = timed("J.apply (kr_jadj)", op.StencilJacobian._apply_cols)
op.Model.at = timed("Model.at (prepare)", op.Model.at)
bl.next_recycle = timed("next_recycle total", bl.next_recycle)
bl.rminres = timed("rminres (persistent kernel + setup)", bl.rminres)
torch.cuda.synchronize()
t0 = time.perf_counter()
steps = 3
for i in range(3, 3 + steps):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"{cfg_name}: {steps} steps, {wall / steps * 1e3:.1f} ms/step")
for k in sorted(T, key=lambda k: -T[k]):
    print(f"  {k:40s} {T[k] / steps * 1e3:9.2f} ms/step   ({N[k] // steps} calls/step)")
