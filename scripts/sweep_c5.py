"""BASELINE config 5, the recycling-stress sweep: one 1024^2 sample (J = 8 5x5 filters,
15x15 blur sigma 2.5), a frozen sequence of lower-level solutions along the theta path
(sequence.solve_path), recycle dimension s in {0, 10, 20, 40, 80}, Ritz vs RGen recycling,
residual vs NSC stopping (experiments.dimension_sweep), plus cold/warm CG vs MINRES
(experiments.cg_vs_minres); hypergradient errors against MINRES-to-1e-13 references.

    python scripts/sweep_c5.py [systems] [out.json]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200.experiments import cg_vs_minres, compute_references, dimension_sweep
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence
from paper_2412_08264_b200.sequence import solve_path

systems = int(sys.argv[1]) if len(sys.argv) > 1 else 50
out = Path(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/sweep_c5.json")
cfg = CONFIGS["C5"]
DELTA, DIMS = 1e-6, [0, 10, 20, 40, 80]
t0 = time.perf_counter()
model = make_batch(cfg)
thetas, _ = synthetic_sequence(cfg, model.x_true.cpu().numpy(), systems, seed=1234)
seq = solve_path(cfg, thetas, lower_gtol=1e-6)
xhats = [s.x_hats for s in seq.systems]
print(f"sequence: {systems} systems in {time.perf_counter() - t0:.1f} s", flush=True)
t0 = time.perf_counter()
refs = compute_references(model, thetas, xhats)
torch.cuda.synchronize()
print(f"references: {time.perf_counter() - t0:.1f} s", flush=True)
result = {"config": "C5", "systems": systems, "delta": DELTA, "max_inner": cfg.max_iter, "dims": DIMS, "sweeps": [],
          "seconds": {}}
for strat, stop in (("Ritz-L", "res"), ("RGen-L(R)", "res"), ("RGen-L(R)-NSC", "nsc")):
    t0 = time.perf_counter()
    rows = dimension_sweep(model, thetas, xhats, strat, DIMS, stop=stop, delta=DELTA, max_inner=cfg.max_iter,
                           refs=refs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    result["seconds"][f"{strat}/{stop}"] = dt
    for r in rows:
        result["sweeps"].append({"strategy": r[0], "stop": stop, "recycle_dim": r[1], "total_iterations": r[2],
                                 "total_flops": r[3], "max_hg_rel_error": r[4], "mean_hg_rel_error": r[5]})
        print(f"{strat:14s} {stop:3s} s={r[1]:3d}: iterations {r[2]:6d} ({r[2] / systems:6.1f}/solve) "
              f"hg error max {r[4]:.2e} mean {r[5]:.2e}", flush=True)
    print(f"  [{dt:.1f} s]", flush=True)
t0 = time.perf_counter()
cvm = cg_vs_minres(model, thetas, xhats, delta=DELTA, max_inner=cfg.max_iter, refs=refs)
result["cg_vs_minres"] = [dict(zip(["solver", "start", "system", "sample", "iterations", "cum_iterations", "flops",
                                    "final_residual", "hg_rel_error"], r)) for r in cvm]
for name in ("minres", "cg"):
    for start in ("cold", "warm"):
        tot = sum(r[4] for r in cvm if r[0] == name and r[1] == start)
        print(f"{name:6s} {start}: total iterations {tot}", flush=True)
result["seconds"]["cg_vs_minres"] = time.perf_counter() - t0
out.parent.mkdir(exist_ok=True)
out.write_text(json.dumps(result, indent=1))
print("wrote", out)
