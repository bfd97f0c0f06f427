"""Time the recycle update's H W (kr_hvp) alone at a config's size, e.g.
    python scripts/hvp_probe.py C3 64          # 64 columns of every sample
and capture it with
    ncu -k regex:hvp_kernel -s 2 -c 1 --set full ... python scripts/hvp_probe.py C3 64 1
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
cfg = CONFIGS[name]
model = make_batch(cfg)
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 1)
H, _ = model.at(th[0], torch.as_tensor(xh[0], device="cuda"))
B, n = model.batch, model.n
g = torch.Generator(device="cuda").manual_seed(7)
W = torch.randn(B, cols, n, dtype=torch.float64, device="cuda", generator=g).transpose(1, 2)
HW = H._apply_cols(W)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    H._apply_cols(W)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
F = 8 * cfg.blur_size + cfg.num_filters * (4 * cfg.kernel_size ** 2 + 2) + 2
tf = B * cols * n * F / (ms / 1e3) / 1e12
print(f"{name}: H W of {B} x {cols} columns: {ms:.3f} ms, {tf:.2f} TFLOP/s (F = {F} flops/pixel), "
      f"checksum {float(HW.double().square().sum()):.17e}", flush=True)
