"""Oracle upper-level trajectory of BASELINE config 1 (VERDICT r1 item 9 / north star:
"the same upper-level theta trajectory within 1e-6 relative after the configured number of
steps").  The CPU oracle (oracle/cpu_bilevel.gradient_descent: the reference's
bilevel.py:392-502 with its L-BFGS lower solve :81-167 and Armijo backtracking :326-358)
runs config 1 -- 64^2 piecewise-constant image, 9x9 sigma 1.5 blur, 1 % noise, smoothed TV
(eps 1e-2, alpha0 = -3), L-BFGS to gradient norm 1e-8, 20 upper steps, recycled CG with
RGen-L(R)-NSC, s = 10, max 100 iterations, NSC tolerance 1e-6 -- and stores theta_i,
the upper cost F_i, ||hypergradient||, the line-search trial counts and the Krylov
iteration counts per step; plus three control trajectories whose Hessian products are
perturbed at 2e-16 relative (the algorithm's own roundoff spread: with p = 1 < s = 10 the
RGen-L selection takes 9 vectors from the GSVD's mu = 0 null cluster, whose basis is
arbitrary in the reference too), and the same for the well-posed s = 1.

    python tests/golden/make_trajectory_fixture.py      ->  tests/golden/traj_C1.npz
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import cpu_bilevel as ob  # noqa: E402
from oracle import cpu_imaging as im  # noqa: E402

STEPS, GTOL = 20, 1e-8


def run(recycle_dim, perturb_seed=None):
    """One oracle trajectory; with perturb_seed every Hessian product of the hypergradient
    solves is perturbed at 2e-16 relative (cpu_imaging.perturbed): a control run measuring
    the reference algorithm's own sensitivity to roundoff."""
    cfg = im.CONFIGS["C1"]
    model, xt = im.deblur_sample(cfg, 0)
    theta0 = im.deblur_theta0(cfg)
    hess = im.hessian
    if perturb_seed is not None:
        calls = [0]

        def perturbed_hessian(*a, **k):
            calls[0] += 1
            return im.perturbed(hess(*a, **k), 2e-16, seed=1000 * perturb_seed + calls[0])

        ob.im.hessian = perturbed_hessian
    try:
        scfg = ob.SolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=recycle_dim, delta=1e-6, max_iter=100,
                                            method="cg")
        state, trace, reason = ob.gradient_descent(theta0, ob.Batch([model], [xt]), 1e-300, solver_cfg=scfg,
                                                   lower_gtol=GTOL, lower_max_iter=20000, max_upper=STEPS)
    finally:
        ob.im.hessian = hess
    return state, trace


def main():
    out = {}
    for tag, s in (("", 10), ("s1_", 1)):
        t0 = time.time()
        state, trace = run(s)
        print(f"s={s}: {len(trace)} steps in {time.time() - t0:.0f} s")
        for r in trace:
            print(f"  step {r.index}: theta {r.theta} F {r.cost:.10e} |hg| {r.grad_norm:.3e} "
                  f"trials {r.linesearch_trials} iters {r.iterations} {r.stop_reasons}")
        ctl = [np.array([r.theta for r in run(s, seed)[1]]) for seed in (1, 2, 3)]
        out.update({
            f"{tag}thetas": np.array([r.theta for r in trace]), f"{tag}theta_final": state.theta,
            f"{tag}costs": np.array([r.cost for r in trace]), f"{tag}grad_norms": np.array([r.grad_norm for r in trace]),
            f"{tag}trials": np.array([r.linesearch_trials for r in trace]),
            f"{tag}iterations": np.array([r.iterations for r in trace]),
            f"{tag}ctl_thetas": np.stack(ctl)})
        spread = max(np.abs(c - out[f"{tag}thetas"]).max() for c in ctl) / np.abs(out[f"{tag}thetas"]).max()
        print(f"  control spread (max relative theta difference): {spread:.3e}")
    np.savez_compressed(ROOT / "tests" / "golden" / "traj_C1.npz", gtol=GTOL, steps=STEPS, **out)


if __name__ == "__main__":
    main()
