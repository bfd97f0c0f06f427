"""Oracle fixtures at the BASELINE configs' sizes ("parity at the benchmarked sizes").

For each case below, the CPU oracle's SequenceSolver (oracle/cpu_bilevel.py, the
reference's bilevel.py:225-288 / recycling.py / krylov.py restated) runs RGen-L(R)-NSC
over consecutive systems of the seeded synthetic sequence the bench replays
(paper_2412_08264_b200.problems: sample_arrays + synthetic_sequence, numpy only), with
the config's operators (oracle/cpu_fast.py: the C restatement of cpu_imaging's
deblurring operators, for speed at 256^2 / 512^2).  It stores, per system and sample:
iterations, stop reason, final stop value, the hypergradient J w, the candidate width
t = k_prev + s_prev the recycle update saw -- and the same for P control runs whose
Hessian products are perturbed at roundoff level (cpu_imaging.perturbed, 2e-16
relative, per-run seeds) and whose carried Lanczos basis is perturbed by 1e-15 relative
before each recycle update: the reference algorithm's own roundoff floor, against which
the GPU results are judged (tests/test_gpu_configs.py).

    python tests/golden/make_config_fixtures.py [C2|C3s|C4s ...]

Writes tests/golden/cfg_<case>.npz (a few KB each).  Run in the build container.
"""

from __future__ import annotations

import dataclasses
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import cpu_bilevel as ob  # noqa: E402
from oracle import cpu_fast as cf  # noqa: E402
from oracle import cpu_imaging as im  # noqa: E402
from oracle import cpu_krylov as ok  # noqa: E402

STRATEGY = "RGen-L(R)-NSC"
DELTA = 1e-6

# case -> (BASELINE config, image size, global sample indices, systems, s, max_iter, control runs[, delta])
CASES = {
    # C2 exactly: 8 x 128^2, 9x9 blur, J=8 q=5, s=20, max 200, delta 1e-6
    "C2": ("C2", 128, list(range(8)), 5, 20, 200, 4),
    # C3's operators (256^2, 15x15 sigma 2.5 blur, 2 % noise) on two of its samples:
    # s=30, max 300 -> candidate widths up to 330 (> 228, the round-1 shared-memory limit)
    "C3s": ("C3", 256, [0, 1], 5, 30, 300, 2),
    # C4's operators (512^2, J=24 7x7 filters, 21x21 sigma 3.5 blur) on one sample, s=40
    "C4s": ("C4", 512, [0], 3, 40, 500, 1),
    # C3 sample 41, whose solves run to max_iter on this sequence: the recycle updates see the
    # config's widest candidate blocks, t = 300 + 30 = 330
    "C3t": ("C3", 256, [41], 4, 30, 300, 1),
}


def run_case(name: str):
    from paper_2412_08264_b200.problems import CONFIGS, sample_arrays, synthetic_sequence

    base, size, samples, systems, s, max_iter, ncontrol = CASES[name][:7]
    delta = CASES[name][7] if len(CASES[name]) > 7 else DELTA
    pcfg = dataclasses.replace(CONFIGS[base], size=size)
    ocfg = dataclasses.replace(im.CONFIGS[base], size=size)
    xts = []
    models = []
    for gi in samples:
        m, xt = im.deblur_sample(ocfg, gi)
        xt2, y2 = sample_arrays(pcfg, gi)
        assert np.array_equal(xt, xt2) and np.array_equal(m.data.y, y2), "oracle / product generators disagree"
        models.append(m)
        xts.append(xt)
    xts = np.stack(xts)
    # the sequence fields are per global sample index (problems.synthetic_sequence(first=...))
    thetas, xh_cols = [], []
    per = [synthetic_sequence(pcfg, xts[i: i + 1], systems, first=gi) for i, gi in enumerate(samples)]
    thetas = per[0][0]
    xhats = [np.concatenate([per[i][1][k] for i in range(len(samples))]) for k in range(systems)]
    mk = lambda: ob.SequenceSolver(ob.SolveConfig.from_strategy(STRATEGY, recycle_dim=s, delta=delta,
                                                                 max_iter=max_iter))
    B, P = len(samples), models[0].reg.num_params
    out = {k: [] for k in ("iters", "reasons", "stopval", "hg", "tdim", "hg_adj", "kept")}
    ctl = {k: [] for k in ("iters", "hg")}
    solvers = [mk() for _ in range(B)]
    controls = [[mk() for _ in range(B)] for _ in range(ncontrol)]
    t0 = time.time()
    for k in range(systems):
        row = {key: [] for key in out}
        crow = {key: [[] for _ in range(ncontrol)] for key in ctl}
        for b in range(B):
            H = cf.hessian(models[b], thetas[k], xhats[k][b])
            J = cf.jacobian(models[b], thetas[k], xhats[k][b])
            g = xhats[k][b] - xts[b]
            sv = solvers[b]
            t = 0 if sv.prev_basis is None else sv.prev_basis.shape[1] + sv.prev_recycle.dim
            r, rec = sv.solve(H, g, J)
            # the hypergradients one iteration before / after the stop (same recycle space, same
            # iterates: the stop rule does not change w): a solve whose NSC value crosses delta
            # one iteration apart from the oracle's is compared at the same iteration count
            kk = r.iterations
            adj = np.full((3, P), np.nan)
            if 0 < kk < max_iter:
                rr = ok.rminres(H, g, rec, ok.Options(max_iter=kk + 1, stop_rule=ok.ResidualRule(1e-300),
                                                      collect_iterates=True))
                for d in range(3):
                    if 0 <= kk - 1 + d < len(rr.iterates):
                        adj[d] = J.apply_adjoint(rr.iterates[kk - 1 + d])
            row["hg_adj"].append(adj)
            # candidate columns kept by the pivoted-QR rank drop (recycling.py:187-199)
            row["kept"].append(0 if rec.nsc_data is None or rec.nsc_data.w is None else int(rec.nsc_data.w.shape[1]))
            row["iters"].append(r.iterations)
            row["reasons"].append(r.stop_reason)
            row["stopval"].append(r.stop_values[-1])
            row["hg"].append(J.apply_adjoint(r.solution))
            row["tdim"].append(t)
            for c in range(ncontrol):
                rc, _ = controls[c][b].solve(im.perturbed(H, 2e-16, seed=1000 * c + 10 * k + b), g, J)
                # ... and its carried Lanczos basis perturbed at 1e-15 relative: the roundoff an
                # implementation that orthonormalises the candidates differently (CholQR2 /
                # projected eigenproblem instead of pivoted Householder QR / SVD) puts into the
                # next recycle space
                prng = np.random.default_rng([7, c, k, b])
                cb = controls[c][b]
                cb.prev_basis = cb.prev_basis * (1.0 + 1e-15 * prng.standard_normal(cb.prev_basis.shape))
                crow["iters"][c].append(rc.iterations)
                crow["hg"][c].append(J.apply_adjoint(rc.solution))
            print(f"{name} system {k} sample {b}: t={t} iters {r.iterations} ({r.stop_reason}) control "
                  f"{[crow['iters'][c][-1] for c in range(ncontrol)]}  [{time.time() - t0:.0f} s]", flush=True)
        for key in out:
            out[key].append(row[key])
        for key in ctl:
            ctl[key].append(crow[key])
    np.savez_compressed(
        ROOT / "tests" / "golden" / f"cfg_{name}.npz",
        config=base, size=size, samples=np.array(samples), systems=systems, recycle_dim=s, max_iter=max_iter,
        delta=delta, strategy=STRATEGY,
        iters=np.array(out["iters"]), reasons=np.array(out["reasons"]), stopval=np.array(out["stopval"]),
        hg=np.array(out["hg"]).reshape(systems, B, P), tdim=np.array(out["tdim"]),
        hg_adj=np.array(out["hg_adj"]).reshape(systems, B, 3, P),  # iterations k-1, k, k+1
        kept=np.array(out["kept"]),
        ctl_iters=np.array(ctl["iters"]).transpose(1, 0, 2),  # (control, system, sample)
        ctl_hg=np.array(ctl["hg"]).transpose(1, 0, 2, 3),
    )


if __name__ == "__main__":
    for case in sys.argv[1:] or list(CASES):
        run_case(case)
