"""Time the whole-batch recycle update alone (python vs native orchestrator, 1 or 2
sample groups) on a C2 state reached by a few recycled solves."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
model = make_batch(cfg)
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 6)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      max_iter=cfg.max_iter))
seq.reserve(cfg.batch, 8 * model.n * (cfg.max_iter + cfg.recycle_dim) * 6, model.x_true.shape)
for i in range(4):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
H, J = model.at(thetas[4], X[4])
B = model.batch
print("kdims", [int(v.shape[1]) for v in seq._prev_basis])
import os
grp = [int(x) for x in os.environ.get("UPD_GROUPS", "1,2").split(",")]
for native in (False, True):
    for groups in grp:
        if not native and groups > 2:
            continue
        seq.native_update, seq.groups = native, groups
        if seq._gstreams is not None and len(seq._gstreams) < groups:
            seq._gstreams = None
            seq.reserve(cfg.batch, 8 * model.n * (cfg.max_iter + cfg.recycle_dim) * 6, model.x_true.shape)
        ts = []
        for r in range(8):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            seq._recycle_batched(H, J, B)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort()
        print(f"native={native} groups={groups}: min {ts[0]:.2f} med {ts[len(ts) // 2]:.2f} max {ts[-1]:.2f} ms")
seq.native_update, seq.groups = True, 1
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    for r in range(3):
        seq._recycle_batched(H, J, B)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
prof.export_chrome_trace("gpurun_out/update_trace.json")
