import sys, torch, time
sys.path.insert(0, "/root/repo")
from paper_2412_08264_b200.batched import qrcp_small
B, T = 4, 220
M = torch.randn(B, T, T, dtype=torch.float64, device="cuda")
dims = torch.full((B,), T, dtype=torch.int32)
for _ in range(3): qrcp_small(M, dims, 1e-10)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): qrcp_small(M, dims, 1e-10)
e1.record(); torch.cuda.synchronize()
print("qrcp ms", e0.elapsed_time(e1) / 10)
