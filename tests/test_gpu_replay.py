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
