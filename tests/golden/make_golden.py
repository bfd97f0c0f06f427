"""Generate the golden fixtures in tests/golden/ by running the REFERENCE package.

Run in the build container only (the reference is not present on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Outputs (small .npz files, committed):
  foe12_seq.npz   -- record_sequence(RunConfig(image="builtin:12", seed=3,
                     max_upper=6, recycle_dim=10)) + compute_references: the
                     frozen systems behind pkg/plots/sample_data/replay.csv,
                     plus the reference replay of None / Ritz-S / RGen-L(R) /
                     RGen-L(R)-NSC (iterations, stop values, hypergradients).
  foe16_seq.npz   -- the acceptance "desk" sequence (RunConfig() defaults,
                     builtin:16, 25 systems) with the reference replay totals
                     (test_acceptance.py:261-298).
  spd_solves.npz  -- random SPD systems (test_krylov.py:19-30 recipe) solved by
                     the reference minres / rminres / cg.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def _seq_arrays(seq):
    prob = seq.problem
    out = {
        "shape": np.array(prob.shape),
        "mask_rows": prob.mask_rows,
        "y": prob.y,
        "ridge": np.array(prob.ridge),
        "x_true": prob.x_true.data,
        "num_filters": np.array(seq.config.num_filters),
        "kernel_size": np.array(seq.config.kernel_size),
        "theta": np.stack([r.theta for r in seq.systems]),
        "x_hat": np.stack([r.x_hat for r in seq.systems]),
        "g": np.stack([r.g for r in seq.systems]),
        "ref_hg": np.stack([r.ref_hg for r in seq.systems]),
        "w_star": np.stack([r.w_star for r in seq.systems]),
    }
    return out


def _replay(seq, strategies, recycle_dim):
    import warnings

    from krecycle.bilevel import HessianSolveConfig, SequenceSolver
    from krecycle.recycling import StrategyDescriptor

    out = {}
    for name in strategies:
        strat = StrategyDescriptor.parse(name)
        solver = SequenceSolver(HessianSolveConfig.from_strategy(
            strat, recycle_dim=recycle_dim, delta=seq.config.delta, max_iter=seq.config.max_inner))
        its, hgs, finals, svals, dims = [], [], [], [], []
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            for i, rec in enumerate(seq.systems):
                H, J = seq.hessian(i), seq.jacobian(i)
                res, rc = solver.solve(H, rec.g, J)
                hgs.append(J.apply_adjoint(res.solution))
                its.append(res.iterations)
                finals.append(res.residual_norms[-1])
                svals.append(res.stop_values[-1])
                dims.append(rc.dim)
        key = name.replace("(", "_").replace(")", "_").replace("-", "_")
        out[f"{key}__iters"] = np.array(its)
        out[f"{key}__hg"] = np.stack(hgs)
        out[f"{key}__final_residual"] = np.array(finals)
        out[f"{key}__final_stop_value"] = np.array(svals)
        out[f"{key}__recycle_dim"] = np.array(dims)
    return out


def main():
    from krecycle.experiments import RunConfig, compute_references, record_sequence
    from krecycle.krylov import SolveOptions, cg, minres, rminres
    from krecycle.operators import dense_operator
    from krecycle.recycling import RecycleSpace
    from krecycle.stopping import ResidualNormRule

    strategies = ["None", "Ritz-S", "RGen-L(R)", "RGen-L(R)-NSC"]
    seq = record_sequence(RunConfig(image="builtin:12", seed=3, max_upper=6, recycle_dim=10))
    compute_references(seq)
    np.savez_compressed(HERE / "foe12_seq.npz", **_seq_arrays(seq), **_replay(seq, strategies, 10))

    desk = record_sequence(RunConfig())
    compute_references(desk)
    np.savez_compressed(HERE / "foe16_seq.npz", **_seq_arrays(desk), **_replay(desk, strategies, 30))

    rng = np.random.default_rng(20240817)
    mats, gs, us = [], [], []
    rec = {}
    for trial in range(6):
        n = int(rng.integers(20, 48))
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        M = Q @ np.diag(np.geomspace(1.0, 100.0, n)) @ Q.T
        g = rng.standard_normal(n)
        Ut = rng.standard_normal((n, 3))
        HU = M @ Ut
        C, R = np.linalg.qr(HU)
        U = Ut @ np.linalg.inv(R)
        opts = SolveOptions(stop_rule=ResidualNormRule(1e-9), max_iter=400, track_basis=True)
        r_m = minres(dense_operator(M), g, opts)
        r_r = rminres(dense_operator(M), g, RecycleSpace(U=U, C=C), opts)
        r_c = cg(dense_operator(M), g, SolveOptions(stop_rule=ResidualNormRule(1e-9), max_iter=400))
        for tag, r in (("minres", r_m), ("rminres", r_r), ("cg", r_c)):
            rec[f"{trial}_{tag}_iters"] = np.array(r.iterations)
            rec[f"{trial}_{tag}_solution"] = r.solution
            rec[f"{trial}_{tag}_residual_norms"] = r.residual_norms
            rec[f"{trial}_{tag}_flops"] = np.array(r.flops)
        rec[f"{trial}_M"] = M
        rec[f"{trial}_g"] = g
        rec[f"{trial}_U"] = U
        rec[f"{trial}_C"] = C
    np.savez_compressed(HERE / "spd_solves.npz", **rec)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    if "/root/reference/pkg/src" not in sys.path:
        sys.path.insert(0, "/root/reference/pkg/src")
    main()
