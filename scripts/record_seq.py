"""Record a frozen sequence on the device and time it:  python scripts/record_seq.py C2 6 1e-8 [out_dir]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2412_08264_b200.problems import CONFIGS
from paper_2412_08264_b200.sequence import load_sequence, record, save_sequence

name, systems, gtol = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
out = sys.argv[4] if len(sys.argv) > 4 else f"gpurun_out/seq_{name}"
t0 = time.perf_counter()
seq = record(CONFIGS[name], systems, lower_gtol=gtol)
torch.cuda.synchronize()
print(f"{name}: recorded {len(seq)} systems in {time.perf_counter() - t0:.1f} s")
for r in seq.systems:
    print(f"  system {r.index}: cost {r.cost:.6e} |hg| {r.grad_norm:.3e} beta {r.beta_init} iters mean "
          f"{np.mean(r.iterations):.1f} max {max(r.iterations)}")
save_sequence(seq, out)
back = load_sequence(out)
assert all(np.array_equal(a.x_hats, b.x_hats) for a, b in zip(seq.systems, back.systems))
print("saved", out)
