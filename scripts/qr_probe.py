import torch, time
for m in (16, 25, 32, 48, 220):
    A = torch.randn(16384, m, dtype=torch.float64, device="cuda")
    for _ in range(3): torch.linalg.qr(A)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(10): torch.linalg.qr(A)
    torch.cuda.synchronize(); print(m, (time.perf_counter()-t)/10*1e3, "ms")
