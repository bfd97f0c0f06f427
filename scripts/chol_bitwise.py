"""Bitwise regression check of kr_chol_inv (as eig_bitwise.py): Grams of random,
ill-conditioned and rank-deficient row blocks, scaled / shifted / skip modes, through
the library named by KR_LIB_NAME; save or compare F, info, stats."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2412_08264_b200.batched import _chol_inv


def run():
    rng = np.random.default_rng(11)
    out = {}
    for t in (20, 57, 150, 213, 220):
        T = 228 if t > 200 else t
        mats = []
        A = rng.standard_normal((t, 600))
        mats.append(A @ A.T)
        U, _ = np.linalg.qr(rng.standard_normal((600, t)))
        sv = np.logspace(0, -9, t)
        B = (U * sv) @ rng.standard_normal((t, t))
        mats.append(B.T @ B)
        C = rng.standard_normal((t, 600))
        C[t // 2] = C[1] + C[2]  # dependent row
        mats.append(C @ C.T)
        G = torch.zeros(len(mats), T, T, dtype=torch.float64, device="cuda")
        for i, M in enumerate(mats):
            G[i, :t, :t] = torch.as_tensor(M, device="cuda")
            if T > t:
                G[i, t:, t:] = torch.eye(T - t, dtype=torch.float64, device="cuda")
        dims = torch.full((len(mats),), t, dtype=torch.int32)
        for mode in ("plain", "scaled", "shifted", "skip"):
            sh = torch.full((len(mats),), 1e-6, dtype=torch.float64, device="cuda") if mode == "shifted" else None
            r = _chol_inv(G, dims, scale=mode != "plain", shift=sh, skip=mode == "skip")
            for j, v in enumerate(r):
                if v is not None:
                    out[f"{t}_{mode}_{j}"] = v.cpu().numpy()
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    r = run()
    if mode == "save":
        np.savez(path, **r)
        print(f"saved {len(r)} arrays")
    else:
        ref = np.load(path)
        def bits(a):
            a = np.ascontiguousarray(a)
            return a.view(np.uint8)
        bad = [k for k in r if not np.array_equal(bits(r[k]), bits(ref[k]))]
        print(f"compared {len(r)} arrays: {len(bad)} differ" + (f": {bad[:6]}" if bad else " (bitwise identical)"))
        sys.exit(1 if bad else 0)
