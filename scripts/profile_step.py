"""Where does a C2 bench step go?  (1) torch.profiler kernel table over 3 steps with
the production threading; (2) per-phase host timing of one sample's recycle update
with a device sync after every phase (serialised, so absolute numbers are upper bounds)."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, recycling as R
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
model = make_batch(cfg)
steps = 8
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), steps)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
seq.reserve(cfg.batch, 8 * model.n * (cfg.max_iter + cfg.recycle_dim) * 6)
for i in range(4):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()

# ---- (2) phase timing, one sample, serialised ----
phases = {}


def timed(name, fn, *a, **k):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn(*a, **k)
    torch.cuda.synchronize()
    phases[name] = phases.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return out


H, J = model.at(thetas[4], X[4])
hb, jb = H.sample(0), J.sample(0)
Vp = seq._prev_basis[0]
Up = seq._prev_recycle[0].U
for rep in range(3):
    W = timed("candidate_basis (cat + CholQR2)", R.build_candidate_basis, Vp, Up).W
    HW = timed("H W (kr_hvp)", hb.apply_matrix, W)
    Jt = timed("J W (kr_jadj)", jb.apply_adjoint_matrix, W)
    Ht = timed("W^T H W", lambda: R._sym(W.T @ HW))
    t = W.shape[1]
    Jt2 = torch.cat([Jt, torch.zeros(max(0, t - Jt.shape[0]), t, dtype=Jt.dtype, device=Jt.device)], 0)
    timed("cond screen", R._hessian_condition, Ht, True)
    S = torch.cat([Jt2, Ht], 0)
    QRs = timed("CholQR2 [Jt;Ht]", R._cholqr2, S)
    Q1 = QRs[0][: Jt2.shape[0]]
    timed("eigh t x t", torch.linalg.eigh, R._sym(Q1.T @ Q1))
    f = timed("gsvd_pair total", R.gsvd_pair, Jt2, Ht, True)
    timed("rgen_select total", R.rgen_select, W, hb, jb, cfg.recycle_dim, "L", "R", HW=HW, Jt=Jt,
          return_coeffs=True)
    timed("next_recycle total", seq._recycle_one, H, J, cfg.batch, 0)
print(f"t = {W.shape[1]}, n = {model.n}")
for k, v in phases.items():
    print(f"  {k:36s} {v / 3:8.3f} ms")

# ---- (1) profiler over whole steps ----
from torch.profiler import ProfilerActivity, profile

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    for i in range(4, 7):
        hypergradients(model, thetas[i], X[i], seq)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / 3
print(f"wall per step under profiler: {wall:.2f} ms")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
Path("gpurun_out").mkdir(exist_ok=True)
prof.export_chrome_trace("gpurun_out/step_trace.json")
