"""Bitwise regression check of kr_syev_select: run a fixed set of symmetric
matrices (random, clustered, rank-deficient Q1^T Q1 with a null cluster as in
config 1) through the library named by KR_LIB_NAME and save / compare outputs.

    KR_LIB_NAME=libkrecycle_b200_old.so python scripts/eig_bitwise.py save gpurun_out/eig_ref.npz
    python scripts/eig_bitwise.py compare gpurun_out/eig_ref.npz
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2412_08264_b200.batched import syev_select


def cases():
    rng = np.random.default_rng(7)
    out = []
    for t in (20, 57, 155, 213, 220):
        A = rng.standard_normal((t, t))
        out.append(("rand", A + A.T))
        Q, _ = np.linalg.qr(rng.standard_normal((t, t)))
        ev = np.concatenate([np.full(t // 3, 1.0), np.linspace(2, 3, t - t // 3)])
        out.append(("cluster", (Q * ev) @ Q.T))
        q1 = rng.standard_normal((1, t))  # config-1 GSVD: one nonzero mu, null cluster
        S = np.vstack([q1, np.zeros((t - 1, t)), rng.standard_normal((t, t))])
        Qs, _ = np.linalg.qr(S)
        Q1 = Qs[:t]
        out.append(("nullclu", Q1.T @ Q1))
    return out


def run():
    res = {}
    for ci, (name, A) in enumerate(cases()):
        t = A.shape[0]
        T = 228 if t > 200 else t
        M = torch.zeros(2, T, T, dtype=torch.float64, device="cuda")
        M[:, :t, :t] = torch.as_tensor(A, device="cuda")
        dims = torch.tensor([t, t], dtype=torch.int32)
        for size in ("S", "L", "M"):
            lam, Z, ns = syev_select(M, dims, size, min(20, t))
            res[f"{ci}_{name}_{size}_lam"] = lam.cpu().numpy()
            res[f"{ci}_{name}_{size}_Z"] = Z.cpu().numpy()
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    r = run()
    if mode == "save":
        np.savez(path, **r)
        print(f"saved {len(r)} arrays")
    else:
        ref = np.load(path)
        bad = [k for k in r if not np.array_equal(r[k].view(np.uint64), ref[k].view(np.uint64))]
        print(f"compared {len(r)} arrays: {len(bad)} differ" + (f": {bad[:6]}" if bad else " (bitwise identical)"))
        for k in bad[:6]:
            print(k, np.max(np.abs(r[k] - ref[k])))
        sys.exit(1 if bad else 0)
