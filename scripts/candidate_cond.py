"""Conditioning of the candidate blocks [V_prev, U_prev] on the C2 sequence: the
reference's pivoted-QR drop ratio vs. cond(A) vs. the batched path's bound."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import scipy.linalg as sl
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

cfg = CONFIGS["C2"]
model = make_batch(cfg)
steps = 6
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), steps)
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
seq.batched_update = False
for i in range(steps):
    _, res, _ = hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    for b in range(model.batch):
        V = seq._prev_basis[b].cpu().numpy()
        U = seq._prev_recycle[b].U.cpu().numpy()
        A = np.concatenate([V, U], axis=1)
        _, R, _ = sl.qr(A, mode="economic", pivoting=True)
        d = np.abs(np.diag(R))
        sv = np.linalg.svd(A, compute_uv=False)
        cn = np.linalg.norm(A, axis=0)
        As = A / cn
        svs = np.linalg.svd(As, compute_uv=False)
        bound = np.linalg.norm(A) * np.sqrt(np.sum(1.0 / sv ** 2))
        print(f"step {i} sample {b} k={V.shape[1]} s={U.shape[1]} piv_ratio={d.min() / d[0]:.2e} "
              f"dropped={int((d <= 1e-10 * d[0]).sum())} cond={sv[0] / sv[-1]:.2e} cond_scaled={svs[0] / svs[-1]:.2e} "
              f"bound={bound:.2e} colnorm[{cn.min():.2e},{cn.max():.2e}] VtV-I={np.abs(V.T @ V - np.eye(V.shape[1])).max():.1e}",
              flush=True)
