"""Batched vs per-sample recycle update on the smoke's deblur case (n = 576, heavy loss of orthogonality)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from oracle import cpu_imaging as im
from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.operators import Model, as_device
from paper_2412_08264_b200.recycling import next_recycle

cfg = im.DeblurConfig(24, 2, 9, 1.5, 0.01, "filters", 2, 5, eps=0.1, alpha0=-1.0)
models, xts = zip(*[im.deblur_sample(cfg, k) for k in range(cfg.batch)])
theta0 = im.deblur_theta0(cfg)
rng = np.random.default_rng(0)
xs = [np.stack([xt + 0.02 * rng.standard_normal(xt.size) for xt in xts]) for _ in range(2)]
thetas = [theta0, theta0 + 0.01 * rng.standard_normal(theta0.size)]
d0 = models[0].data
dm = Model(shape=d0.shape, batch=cfg.batch, data_kind="blur", data_scale=2.0, ridge=0.0,
           y=as_device(np.stack([m.data.y for m in models])), x_true=as_device(np.stack(xts)), taps=d0.taps,
           reg_kind="filters", potential="smooth_abs", eps=cfg.eps, num_filters=2, ksize=5)
for batched_update in (False, True):
    seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)", recycle_dim=6, delta=1e-10, max_iter=400))
    seq.batched_update = batched_update
    batched.STATS = {}
    its = []
    for step in range(2):
        hg, res, recs = hypergradients(dm, thetas[step], as_device(xs[step]), seq)
        its.append([r.iterations for r in res])
        if step == 0:
            H, J = dm.at(thetas[1], as_device(xs[1]))
            st = seq.cfg.strategy
            b_recs = batched.recycle_update(st, 6, H, J, seq._prev_basis, seq._prev_recycle)
            for b in range(2):
                ref = next_recycle(st, h_current=H.sample(b), jac_current=J.sample(b), prev_basis=seq._prev_basis[b],
                                   prev_recycle=seq._prev_recycle[b], s=6)
                Pg = torch.linalg.qr(b_recs[b].C)[0]
                Pr = torch.linalg.qr(ref.C)[0]
                V = seq._prev_basis[b]
                sv = torch.linalg.svdvals(torch.cat([V, seq._prev_recycle[b].U], 1))
                print(f"sample {b}: |P_C diff| {torch.dist(Pg @ Pg.T, Pr @ Pr.T):.2e}  mu batched "
                      f"{b_recs[b].nsc_data.values.cpu().numpy()} ref {ref.nsc_data.values.cpu().numpy()} "
                      f"k={V.shape[1]} cond(cands)={float(sv[0] / sv[-1]):.2e}", flush=True)
    print("batched" if batched_update else "per-sample", its, batched.STATS, flush=True)
