"""Debug: which samples lose their NSC data in the C2 sequence, and why."""

import sys
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

import paper_2412_08264_b200.recycling as rc
from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

orig_prepare = rc.prepare_recycle


def prepare(H, Ut, nsc=None, HU=None):
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        out = orig_prepare(H, Ut, nsc, HU)
    if out.nsc_data is None or out.dim < Ut.shape[1]:
        hn = None if HU is None else float(torch.linalg.vector_norm(HU))
        print(f"prepare: dim {out.dim} of {Ut.shape[1]}, nsc {out.nsc_data is not None}, |HU| {hn}, "
              f"|Ut| {float(torch.linalg.vector_norm(Ut))}, warnings {[str(x.message) for x in w]}", flush=True)
    return out


rc.prepare_recycle = prepare
orig_next = rc.next_recycle


def next_recycle(*a, **k):
    out = orig_next(*a, **k)
    if out.nsc_data is None:
        print("next_recycle returned no nsc data; dim", out.dim, flush=True)
    return out


import paper_2412_08264_b200.bilevel as bl

bl.next_recycle = next_recycle
cfg = CONFIGS["C2"]
model = make_batch(cfg)
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 14)
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=20, delta=1e-6, max_iter=200))
if len(sys.argv) > 1:
    seq.max_workers = int(sys.argv[1])
for i in range(14):
    try:
        hg, res, recs = hypergradients(model, thetas[i], torch.as_tensor(xh[i], device="cuda"), seq)
        print(i, [r.iterations for r in res], [r.dim for r in recs], [r.nsc_data is not None for r in recs], flush=True)
    except Exception as e:
        print("step", i, "failed:", type(e).__name__, e, flush=True)
        break
