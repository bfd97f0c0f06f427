"""Single batched rminres launch on a deblur model: B samples, recycle dim s, NSC columns ns."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2412_08264_b200 import RecycleSpace, SolveOptions, ResidualNormRule, NscRule, NscData, rminres
from paper_2412_08264_b200.problems import DeblurConfig, make_batch, synthetic_sequence

size, B, s, ns, maxit = (int(a) for a in sys.argv[1:6])
cfg = DeblurConfig(size, B, 9, 1.5, 0.01, "filters", 8, 5)
model = make_batch(cfg)
th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 1)
X = torch.as_tensor(xh[0], device="cuda")
H, J = model.at(th[0], X)
G = X - model.x_true
n = model.n
torch.manual_seed(0)
recs, rules = [], []
for b in range(B):
    if s:
        Ut = torch.randn(n, s, dtype=torch.float64, device="cuda")
        HU = H.sample(b).apply_matrix(Ut)
        C, R = torch.linalg.qr(HU)
        U = torch.linalg.solve_triangular(R, Ut, upper=True, left=False)
        data = None
        if ns:
            W = torch.linalg.qr(torch.randn(n, 3 * ns, dtype=torch.float64, device="cuda"))[0]
            data = NscData(torch.rand(ns, dtype=torch.float64, device="cuda"),
                           torch.linalg.qr(torch.randn(3 * ns, ns, dtype=torch.float64, device="cuda"))[0], W)
        recs.append(RecycleSpace(U.T.contiguous().T, C.T.contiguous().T, data))
        rules.append(NscRule(1e-6, data) if ns else ResidualNormRule(1e-6))
    else:
        recs.append(RecycleSpace.empty(n))
        rules.append(ResidualNormRule(1e-6))
res = rminres(H, G, recs, SolveOptions(max_iter=maxit, stop_rule=rules, track_basis=True))
torch.cuda.synchronize()
print(sys.argv[1:], "ok", [r.iterations for r in res], flush=True)
