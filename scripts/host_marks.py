"""Host-side wall time of the pieces of one C2 step (no device syncs added except
at the step end): where the Python / orchestrator time goes."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched, bilevel, krylov
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

cfg = CONFIGS["C2"]
model = make_batch(cfg)
n = model.n
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 10, seed=1234)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
t_max = cfg.max_iter + cfg.recycle_dim
seq.reserve(cfg.batch, 8 * n * t_max * 6, shape=(n, t_max))
T0 = [0.0]
log = []


def wrap(obj, name, label):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        log.append((f"{label} start", (t - T0[0]) * 1e3))
        r = f(*a, **k)
        log.append((f"{label} end", (time.perf_counter() - T0[0]) * 1e3))
        return r

    setattr(obj, name, g)


wrap(model, "at", "model.at")
wrap(SequenceSolver, "_recycle_all", "recycle_all")
wrap(SequenceSolver, "_options", "options")
wrap(batched, "recycle_update_native", "native")
bilevel.recycle_update_native = batched.recycle_update_native
wrap(krylov._Launch, "__init__", "launch.init")
wrap(krylov._Launch, "run", "launch.run")
wrap(krylov._Launch, "results", "launch.results")
for i in range(4):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
for i in range(4, 7):
    log.clear()
    T0[0] = time.perf_counter()
    hg, _, _ = hypergradients(model, thetas[i], X[i], seq)
    log.append(("hypergradients returned", (time.perf_counter() - T0[0]) * 1e3))
    torch.cuda.synchronize()
    log.append(("synced", (time.perf_counter() - T0[0]) * 1e3))
    print(f"--- step {i}")
    for k, v in log:
        print(f"  {v:8.3f} ms  {k}")
