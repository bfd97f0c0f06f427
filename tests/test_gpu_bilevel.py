"""GPU parity of the next rows of SURVEY 8(f): the device L-BFGS lower solve
(bilevel.py:81-167) and the upper gradient-descent loop (bilevel.py:326-502).

* The reference's own record_sequence trajectory (tests/golden/foe12_seq.npz:
  theta_i, xhat_i of builtin:12 seed 3) is reproduced by the device upper loop:
  theta within 1e-6 relative after every step (the north-star bar).
* A small deblurring batch: device lower solves and two upper steps vs the
  oracle's batch gradient descent.
"""

import numpy as np
import pytest
import torch

from oracle import cpu_bilevel as ob
from oracle import cpu_imaging as im
from tests.conftest import golden
from tests.helpers import device_model, rel, to_np

pytestmark = pytest.mark.gpu


def _foe_device_model(d):
    from paper_2412_08264_b200 import ImageVector, InpaintingProblem

    shape = tuple(int(v) for v in d["shape"])
    prob = InpaintingProblem(d["mask_rows"], d["y"], float(d["ridge"]), shape, ImageVector(d["x_true"], shape))
    m = prob.model()
    m.num_filters, m.ksize = int(d["num_filters"]), int(d["kernel_size"])
    return m


def test_lower_solve_matches_oracle(cuda):
    from paper_2412_08264_b200.lower import lower_solve

    d = golden("foe12_seq.npz")
    dm = _foe_device_model(d)
    model, _ = im.foe_inpainting(12, seed=3)
    for i in (0, 3):
        x_gpu, st = lower_solve(dm, d["theta"][i], None, gtol=1e-3)
        x_cpu, st_cpu = ob.lower_solve(model, d["theta"][i], None, gtol=1e-3)
        assert int(st.iterations[0]) == st_cpu.iterations
        assert rel(to_np(x_gpu[0]), x_cpu) <= 1e-9
        # the recorded lower solution of the reference (x_hat_0 starts from zeros)
        if i == 0:
            assert rel(to_np(x_gpu[0]), d["x_hat"][0]) <= 1e-9


def test_upper_trajectory_matches_reference_record(cuda):
    """record_sequence(builtin:12, seed 3, max_upper 6) on the device == the reference's recording."""
    from paper_2412_08264_b200.lower import record_sequence

    d = golden("foe12_seq.npz")
    dm = _foe_device_model(d)
    trace = record_sequence(dm, d["theta"][0], delta=1e-2, max_inner=500, lower_gtol=1e-3, eps_stop=1e-4,
                            max_upper=d["theta"].shape[0])
    assert len(trace) == d["theta"].shape[0]
    for i, rec in enumerate(trace):
        assert rel(rec.theta, d["theta"][i]) <= 1e-6, (i, rel(rec.theta, d["theta"][i]))
        assert rel(to_np(rec.x_hats[0]), d["x_hat"][i]) <= 1e-6
        assert rec.iterations[0] == int(d["None__iters"][i])


def test_batched_deblur_gradient_descent_matches_oracle(cuda):
    """Two upper steps of a 2-sample deblurring batch sharing theta (F = sum_k)."""
    from paper_2412_08264_b200.lower import gradient_descent, LowerConfig
    from paper_2412_08264_b200 import HessianSolveConfig, StrategyDescriptor

    cfg = im.DeblurConfig(16, 2, 5, 1.0, 0.01, "filters", 2, 3, eps=0.2, alpha0=-1.0)
    pairs = [im.deblur_sample(cfg, k) for k in range(2)]
    models = [m for m, _ in pairs]
    xts = [x for _, x in pairs]
    th0 = im.deblur_theta0(cfg)
    _, trace_cpu, _ = ob.gradient_descent(th0, ob.Batch(models, xts), 1e-12,
                                          solver_cfg=ob.SolveConfig(delta=1e-10, max_iter=2000),
                                          lower_gtol=1e-9, max_upper=3)
    dm = device_model(models)
    _, trace_gpu = gradient_descent(dm, th0, 1e-12,
                                    solver_cfg=HessianSolveConfig(StrategyDescriptor("None"), delta=1e-10,
                                                                  max_iter=2000),
                                    lower_cfg=LowerConfig(gtol=1e-9), max_upper=3)
    assert len(trace_gpu) == len(trace_cpu)
    for a, b in zip(trace_gpu, trace_cpu):
        assert rel(a.theta, b.theta) <= 1e-6
        assert abs(a.cost - b.cost) <= 1e-8 * abs(b.cost)
        assert abs(a.grad_norm - b.grad_norm) <= 1e-6 * b.grad_norm


def _tv_problem(size, cuda):
    import numpy as np

    from oracle import cpu_imaging as im
    from paper_2412_08264_b200.problems import DeblurConfig, make_batch

    model = make_batch(DeblurConfig(size, 1, 9, 1.5, 0.01, "tv", 1, 1))
    om, xt = im.deblur_sample(im.DeblurConfig(size, 1, 9, 1.5, 0.01, "tv", 1, 1), 0)
    assert np.allclose(model.x_true[0].cpu().numpy(), xt)
    return model, om, xt


def test_recycled_cg_sequence_matches_oracle(cuda):
    """Recycled CG (method="cg") through SequenceSolver on a reduced config-1
    problem (smoothed TV, 9x9 blur) against the oracle's sequence, with a
    well-posed selection (Ritz-S): iterations within the oracle's own roundoff
    spread (+-1 minimum), hypergradients within max(1e-8, 10 x that floor)."""
    import numpy as np

    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
    from paper_2412_08264_b200.bilevel import hypergradients

    model, om, xt = _tv_problem(32, cuda)
    rng = np.random.default_rng(3)
    kw = dict(recycle_dim=6, delta=1e-7, max_iter=300, method="cg")
    gpu = SequenceSolver(HessianSolveConfig.from_strategy("Ritz-S", **kw))
    cpu = ob.SequenceSolver(ob.SolveConfig.from_strategy("Ritz-S", **kw))
    cpu_p = ob.SequenceSolver(ob.SolveConfig.from_strategy("Ritz-S", **kw))
    for step in range(4):
        th = np.array([-3.0 + 0.05 * step])
        xh = xt + 0.02 * rng.standard_normal(xt.size)
        hg, res, _ = hypergradients(model, th, torch.as_tensor(xh[None], device=cuda), gpu)
        H, J = im.hessian(om, th, xh), im.jacobian(om, th, xh)
        r, _ = cpu.solve(H, xh - xt, J)
        rp, _ = cpu_p.solve(im.perturbed(H, seed=step), xh - xt, J)
        # the control run also carries a 1e-15-perturbed basis into its next recycle
        # update: Ritz-S picks from clustered small eigenvalues of W^T H W, whose
        # eigenvectors (and so the next recycle space) move with any roundoff
        cpu_p.prev_basis = cpu_p.prev_basis * (1 + 1e-15 * rng.standard_normal(cpu_p.prev_basis.shape))
        ref = J.apply_adjoint(r.solution)
        floor = np.linalg.norm(J.apply_adjoint(rp.solution) - ref) / np.linalg.norm(ref)
        slack = max(1, abs(rp.iterations - r.iterations) + 1)
        assert abs(res[0].iterations - r.iterations) <= slack, (step, res[0].iterations, r.iterations, rp.iterations)
        err = np.linalg.norm(hg[0].cpu().numpy() - ref) / np.linalg.norm(ref)
        assert err <= max(1e-8, 10.0 * floor), (step, err, floor)


def test_config1_solver_hypergradient_accuracy(cuda):
    """Config 1's exact solver -- recycled CG, RGen-L(R)-NSC, hypergradient-error
    stop -- on a reduced problem.  With p = 1 the GSVD has one nonzero mu and a
    mu = 0 null cluster, so L-size selection beyond one vector picks an arbitrary
    basis of that cluster (in the reference too: LAPACK's order of zero singular
    values); iteration counts are not comparable and the check is the outcome:
    the NSC estimate reaches delta and the hypergradient error against an exact
    solve is within the reference algorithm's own spread.  That spread is measured
    here: the oracle re-run with its Hessian product perturbed at roundoff level
    (2e-16 relative, several seeds) -- on this problem its error moves by up to
    ~30x at step 2 and ~700x at step 3 (a different arbitrary null-cluster basis
    each time), so one unperturbed oracle run is not a meaningful bar."""
    import numpy as np

    from oracle import cpu_imaging as im
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
    from paper_2412_08264_b200.bilevel import hypergradients

    from oracle import cpu_bilevel as ob

    model, om, xt = _tv_problem(32, cuda)
    rng = np.random.default_rng(3)
    kw = dict(recycle_dim=6, delta=1e-6, max_iter=100, method="cg")
    gpu = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", **kw))
    seeds = [None, 0, 1, 2, 3]
    cpus = [ob.SequenceSolver(ob.SolveConfig.from_strategy("RGen-L(R)-NSC", **kw)) for _ in seeds]
    for step in range(4):
        th = np.array([-3.0 + 0.05 * step])
        xh = xt + 0.02 * rng.standard_normal(xt.size)
        hg, res, _ = hypergradients(model, th, torch.as_tensor(xh[None], device=cuda), gpu)
        H, J = im.hessian(om, th, xh), im.jacobian(om, th, xh)
        Hd = np.column_stack([H(e) for e in np.eye(xt.size)])
        exact = J.apply_adjoint(np.linalg.solve(Hd, xh - xt))
        e_gpu = np.linalg.norm(hg[0].cpu().numpy() - exact)
        e_cpu = []
        for seed, cpu in zip(seeds, cpus):
            Hs = H if seed is None else im.perturbed(H, 2e-16, 10 * seed + step)
            r, _ = cpu.solve(Hs, xh - xt, J)
            e_cpu.append(np.linalg.norm(J.apply_adjoint(r.solution) - exact))
            if seed is None:
                r0 = r
        # first system: residual rule, both may stop at max_iter; later: NSC
        assert res[0].stop_reason == r0.stop_reason or step > 0, (step, res[0].stop_reason, r0.stop_reason)
        if res[0].stop_reason == "tolerance":
            assert res[0].stop_values[-1] < 1e-6
        assert e_gpu <= 10 * max(e_cpu) + 1e-6 * np.linalg.norm(exact), (step, e_gpu, e_cpu)
