"""Golden replay on the GPU: the reference's own frozen sequences replayed through
the device SequenceSolver must reproduce the reference's iteration counts
(pkg/plots/sample_data/replay.csv and the acceptance desk totals
371 / 177 / 179 / 163, test_acceptance.py:261-298) and hypergradients.

Bars: iterations equal to the reference per solve (+-1 allowed by the north
star, the observed counts are exact), hypergradients within 1e-8 relative of
the reference's for None / Ritz-S / RGen-L(R) / RGen-L(R)-NSC.
"""

import numpy as np
import pytest
import torch

from tests.conftest import golden
from tests.helpers import rel, to_np

pytestmark = pytest.mark.gpu

STRATS = ["None", "Ritz-S", "RGen-L(R)", "RGen-L(R)-NSC"]


def _key(name):
    return name.replace("(", "_").replace(")", "_").replace("-", "_")


def _replay(d, strategy, recycle_dim, reuse_products=True):
    from paper_2412_08264_b200 import HessianSolveConfig, InpaintingProblem, ImageVector, SequenceSolver
    from paper_2412_08264_b200 import StrategyDescriptor
    from paper_2412_08264_b200.operators import Model, as_device

    shape = tuple(int(v) for v in d["shape"])
    prob = InpaintingProblem(d["mask_rows"], d["y"], float(d["ridge"]), shape, ImageVector(d["x_true"], shape))
    model = prob.model()
    model.num_filters, model.ksize = int(d["num_filters"]), int(d["kernel_size"])
    solver = SequenceSolver(HessianSolveConfig.from_strategy(
        StrategyDescriptor.parse(strategy), recycle_dim=recycle_dim, delta=1e-2, max_iter=500,
        reuse_products=reuse_products))
    its, hgs = [], []
    for i in range(d["theta"].shape[0]):
        H, J = model.at(d["theta"][i], d["x_hat"][i])
        res, rec = solver.solve(H, as_device(d["g"][i]), J)
        hgs.append(to_np(J.apply_adjoint(res.solution)))
        its.append(res.iterations)
    return np.array(its), np.stack(hgs)


@pytest.mark.parametrize("strategy", STRATS)
@pytest.mark.parametrize("reuse", [True, False])
def test_replay_csv_golden(cuda, strategy, reuse):
    d = golden("foe12_seq.npz")
    its, hgs = _replay(d, strategy, 10, reuse)
    ref_its = d[f"{_key(strategy)}__iters"]
    assert np.array_equal(its, ref_its), (its, ref_its)
    ref_hg = d[f"{_key(strategy)}__hg"]
    for i in range(len(its)):
        assert rel(hgs[i], ref_hg[i]) <= 1e-8, (i, rel(hgs[i], ref_hg[i]))


@pytest.mark.parametrize("strategy", STRATS)
def test_desk_sequence_totals(cuda, strategy):
    d = golden("foe16_seq.npz")
    its, hgs = _replay(d, strategy, 30)
    ref_its = d[f"{_key(strategy)}__iters"]
    assert np.max(np.abs(its - ref_its)) <= 1, (its, ref_its)
    expected_total = {"None": 371, "Ritz-S": 177, "RGen-L(R)": 179, "RGen-L(R)-NSC": 163}[strategy]
    assert abs(int(its.sum()) - expected_total) <= 1
    ref_hg = d[f"{_key(strategy)}__hg"]
    worst = max(rel(hgs[i], ref_hg[i]) for i in range(len(its)) if its[i] == ref_its[i])
    assert worst <= 1e-8, worst


# pkg/plots/sample_data/sweep.csv (the reference's dimension_sweep of the foe12 sequence,
# experiments.py:505-535): Ritz-S, recycle dims 0 / 2 / 4 / 8 / 12 ->
# (total iterations, total flops, max and mean relative hypergradient error vs J w*)
SWEEP_GOLDEN = {
    0: (76, 3768192, 0.033694827195256682, 0.016520784270208023),
    2: (72, 3741718, 0.026326296642218004, 0.013062908269928819),
    4: (66, 3554132, 0.024341119751564732, 0.01341575650779959),
    8: (63, 3600160, 0.020297843837332619, 0.010121535657028299),
    12: (60, 3618571, 0.023730413966896402, 0.011710216193678263),
}


def test_dimension_sweep_matches_reference_sweep_csv(cuda):
    """experiments.dimension_sweep on the device over the reference's frozen foe12
    sequence reproduces the reference's sweep.csv: total iterations and flops exactly,
    the hypergradient error statistics against the stored J w* to 1e-6 relative."""
    from paper_2412_08264_b200 import ImageVector, InpaintingProblem
    from paper_2412_08264_b200.experiments import dimension_sweep

    d = golden("foe12_seq.npz")
    shape = tuple(int(v) for v in d["shape"])
    prob = InpaintingProblem(d["mask_rows"], d["y"], float(d["ridge"]), shape, ImageVector(d["x_true"], shape))
    model = prob.model()
    model.num_filters, model.ksize = int(d["num_filters"]), int(d["kernel_size"])
    refs = [torch.as_tensor(r, device=cuda).reshape(1, -1) for r in d["ref_hg"]]
    rows = dimension_sweep(model, list(d["theta"]), list(d["x_hat"]), "Ritz-S", sorted(SWEEP_GOLDEN), delta=1e-2,
                           max_inner=500, refs=refs)
    for strat, s, its, flops, emax, emean in rows:
        g_its, g_flops, g_max, g_mean = SWEEP_GOLDEN[s]
        assert (its, flops) == (g_its, g_flops), (s, its, flops)
        assert abs(emax - g_max) <= 1e-6 * g_max and abs(emean - g_mean) <= 1e-6 * g_mean, (s, emax, emean)


@pytest.mark.parametrize("strategy", ["Eig-S", "Eig-L", "GSVD-L(R)", "GSVD-L(R)-NSC", "inner:Eig-S",
                                      "HRitz-S", "inner:RGen-L(R)-NSC"])
def test_remaining_strategies_match_oracle(cuda, strategy):
    """The strategies outside the bench path: dense Eig / GSVD
    (recycling.py:416-445, the n x n projections through the library eigensolver), harmonic
    Ritz (:239-272, native batched update) and inner placement (:409-415, native with the
    previous operator) replayed over the reference's foe12 sequence against the CPU oracle:
    iterations within +-1, hypergradients within 1e-8 where the iteration counts agree."""
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im

    d = golden("foe12_seq.npz")
    its, hgs = _replay(d, strategy, 10)
    shape = tuple(int(v) for v in d["shape"])
    data = im.DataTerm("mask", shape, d["y"], scale=1.0, ridge=float(d["ridge"]), mask_rows=d["mask_rows"],
                       x_true=d["x_true"])
    model = im.Model(data, im.Regularizer("filters", int(d["num_filters"]), int(d["kernel_size"]), "quadratic"))
    solver = ob.SequenceSolver(ob.SolveConfig.from_strategy(strategy, recycle_dim=10, delta=1e-2, max_iter=500))
    for i in range(d["theta"].shape[0]):
        H = im.hessian(model, d["theta"][i], d["x_hat"][i])
        J = im.jacobian(model, d["theta"][i], d["x_hat"][i])
        res, _ = solver.solve(H, d["g"][i], J)
        ref = J.apply_adjoint(res.solution)
        assert abs(int(its[i]) - res.iterations) <= 1, (i, its[i], res.iterations)
        if its[i] == res.iterations:
            assert rel(hgs[i], ref) <= 1e-8, (i, rel(hgs[i], ref))


@pytest.mark.parametrize("strategy", ["None", "Ritz-S", "RGen-L(R)"])
def test_true_hypergradient_stop_matches_oracle(cuda, strategy):
    """The true-hypergradient-error stop rule (stopping.py:121-185, bilevel.py:267-268),
    evaluated every iteration inside the persistent solver (s-space recurrence of
    J H^-1 r_k), over the reference's foe12 sequence against the CPU oracle's TrueHgRule
    (dense Cholesky per iteration): iterations within +-1, stop values and hypergradients
    within 1e-8 where the counts agree."""
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im
    from paper_2412_08264_b200 import HessianSolveConfig, ImageVector, InpaintingProblem, SequenceSolver
    from paper_2412_08264_b200.operators import as_device

    d = golden("foe12_seq.npz")
    shape = tuple(int(v) for v in d["shape"])
    prob = InpaintingProblem(d["mask_rows"], d["y"], float(d["ridge"]), shape, ImageVector(d["x_true"], shape))
    model = prob.model()
    model.num_filters, model.ksize = int(d["num_filters"]), int(d["kernel_size"])
    kw = dict(recycle_dim=10, delta=1e-4, max_iter=500, stop="true-hg")
    gpu = SequenceSolver(HessianSolveConfig.from_strategy(strategy, **kw))
    data = im.DataTerm("mask", shape, d["y"], scale=1.0, ridge=float(d["ridge"]), mask_rows=d["mask_rows"],
                       x_true=d["x_true"])
    om = im.Model(data, im.Regularizer("filters", int(d["num_filters"]), int(d["kernel_size"]), "quadratic"))
    cpu = ob.SequenceSolver(ob.SolveConfig.from_strategy(strategy, **kw))
    for i in range(d["theta"].shape[0]):
        H, J = model.at(d["theta"][i], d["x_hat"][i])
        res, _ = gpu.solve(H, as_device(d["g"][i]), J)
        hg = to_np(J.apply_adjoint(res.solution))
        Ho, Jo = im.hessian(om, d["theta"][i], d["x_hat"][i]), im.jacobian(om, d["theta"][i], d["x_hat"][i])
        r, _ = cpu.solve(Ho, d["g"][i], Jo)
        ref = Jo.apply_adjoint(r.solution)
        assert abs(res.iterations - r.iterations) <= 1, (i, res.iterations, r.iterations)
        if res.iterations == r.iterations:
            assert rel(hg, ref) <= 1e-8, (i, rel(hg, ref))
            assert rel(res.stop_values, r.stop_values) <= 1e-8, (i, res.stop_values[-3:], r.stop_values[-3:])
