"""Timeline of one bench step (C2 by default): every kernel with its stream, start
offset and duration (torch.profiler / CUPTI), GPU-idle gaps (no kernel on any
stream: host decisions, syncs, launch latency) and per-stream busy time.

    python scripts/timeline.py [C2] [steps_before=4] > gpurun_out/timeline.txt
"""

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
before = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = CONFIGS[name]
model = make_batch(cfg)
n = model.n
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), before + 2, seed=1234)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6,
                                                      method=cfg.method, max_iter=cfg.max_iter))
torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
t_max = cfg.max_iter + cfg.recycle_dim
seq.reserve(cfg.batch, 8 * n * t_max * 6, shape=(n, t_max))
for i in range(before):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()

from torch.profiler import ProfilerActivity, profile

out = Path("gpurun_out")
out.mkdir(exist_ok=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    hypergradients(model, thetas[before], X[before], seq)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
trace = out / f"timeline_{name}.json"
prof.export_chrome_trace(str(trace))
ev = json.loads(trace.read_text())["traceEvents"]
ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
ks.sort(key=lambda e: e["ts"])
t_first = ks[0]["ts"]
print(f"{name}: wall {wall:.2f} ms (under profiler), {len(ks)} device activities, "
      f"span {(ks[-1]['ts'] + ks[-1]['dur'] - t_first) / 1e3:.2f} ms")
busy = 0.0
end = t_first
gaps = []
for e in ks:
    if e["ts"] > end:
        gaps.append((end - t_first, e["ts"] - end, e["name"][:60]))
    new_end = max(end, e["ts"] + e["dur"])
    busy += new_end - max(end, e["ts"]) if e["ts"] + e["dur"] > end else 0.0
    end = new_end
print(f"union busy {busy / 1e3:.2f} ms, idle {sum(g[1] for g in gaps) / 1e3:.2f} ms in {len(gaps)} gaps")
print("largest idle gaps (offset us, gap us, next activity):")
for g in sorted(gaps, key=lambda g: -g[1])[:25]:
    print(f"  {g[0]:10.1f} {g[1]:8.1f}  {g[2]}")
per_stream = {}
for e in ks:
    st = e.get("args", {}).get("stream", -1)
    per_stream.setdefault(st, []).append(e)
for st, lst in per_stream.items():
    print(f"stream {st}: {len(lst)} activities, busy {sum(e['dur'] for e in lst) / 1e3:.2f} ms, "
          f"first {(lst[0]['ts'] - t_first) / 1e3:.2f} last end {(lst[-1]['ts'] + lst[-1]['dur'] - t_first) / 1e3:.2f} ms")
print("activities (offset us, dur us, stream, name):")
for e in ks:
    print(f"  {e['ts'] - t_first:10.1f} {e['dur']:9.1f} {e.get('args', {}).get('stream', -1):4} {e['name'][:90]}")
