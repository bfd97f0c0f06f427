import sys, time, cProfile, pstats, threading
sys.path.insert(0, "/root/repo")
import torch
from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched, bilevel
from paper_2412_08264_b200.bilevel import hypergradients
from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence
import os
os.environ["KR_RECYCLE_GROUPS"] = "1"
cfg = CONFIGS["C2"]
model = make_batch(cfg)
thetas, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 10, seed=1234)
X = [torch.as_tensor(x, device="cuda") for x in xh]
seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=1e-6, max_iter=cfg.max_iter))
seq.groups = 1
torch.empty(3 * 1024**3 // 8, dtype=torch.float64, device="cuda")
for i in range(4):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
orig = batched.recycle_update_native
prof = cProfile.Profile()
from paper_2412_08264_b200 import _lib
real_call = _lib.lib().kr_recycle_update
def wrapped(*a, **k):
    prof.enable()
    try:
        return orig(*a, **k)
    finally:
        prof.disable()
bilevel.recycle_update_native = wrapped
for i in range(4, 8):
    hypergradients(model, thetas[i], X[i], seq)
torch.cuda.synchronize()
st = pstats.Stats(prof)
st.sort_stats("tottime").print_stats(18)
