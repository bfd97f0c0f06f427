"""GPU parity of the operator kernels (kr_hvp, kr_jadj, kr_lower_eval) against the CPU oracle.

Oracle styles from the reference suite: loop/dense oracles, adjointness and
symmetry probes, finite differences (test_operators.py:52-326).  Bar: fp64
roundoff, relative error <= 1e-12 (stencil sums in a different order).
"""

import numpy as np
import pytest
import torch

from oracle import cpu_imaging as im
from tests.helpers import device_model, oracle_models, rel, to_np

pytestmark = pytest.mark.gpu

CASES = [
    ("foe", 12, 12, 1, dict(J=3, q=5)),
    ("foe", 21, 45, 2, dict(J=2, q=3)),
    ("filters", 20, 37, 2, dict(blur=9, J=3, q=5)),
    ("filters", 33, 70, 1, dict(blur=15, sigma=2.5, J=2, q=7)),
    ("filters", 16, 32, 3, dict(blur=21, sigma=3.5, J=1, q=3)),
    ("tv", 19, 41, 2, dict(blur=9)),
    ("tv", 64, 64, 1, dict(blur=9)),
]


@pytest.mark.parametrize("kind,rows,cols,batch,kw", CASES)
def test_hvp_matches_oracle(cuda, kind, rows, cols, batch, kw):
    models, theta, xh, _ = oracle_models(kind, rows, cols, batch, seed=rows * cols, **kw)
    dm = device_model(models)
    H, _ = dm.at(theta, xh)
    rng = np.random.default_rng(1)
    t = 4
    V = rng.standard_normal((batch, rows * cols, t))
    HV = to_np(H.apply_matrix(torch.as_tensor(V, device=cuda)))
    for b in range(batch):
        Ho = im.hessian(models[b], theta, xh[b])
        for j in range(t):
            ref = Ho(V[b, :, j])
            assert rel(HV[b, :, j], ref) <= 1e-12, (b, j, rel(HV[b, :, j], ref))


@pytest.mark.parametrize("t", [3, 70, 260])  # 3: per-tile kernel; 70, 260: conv + split-K DGEMM (1 and 2 column chunks)
@pytest.mark.parametrize("kind,rows,cols,batch,kw", CASES)
def test_jadj_matches_oracle(cuda, kind, rows, cols, batch, kw, t):
    models, theta, xh, _ = oracle_models(kind, rows, cols, batch, seed=7 + rows, **kw)
    dm = device_model(models)
    _, J = dm.at(theta, xh)
    rng = np.random.default_rng(2)
    W = rng.standard_normal((batch, rows * cols, t))
    JW = to_np(J.apply_adjoint_matrix(torch.as_tensor(W, device=cuda)))
    for b in range(batch):
        Jo = im.jacobian(models[b], theta, xh[b])
        for j in range(t):
            ref = Jo.apply_adjoint(W[b, :, j])
            assert rel(JW[b, :, j], ref) <= 1e-12, (b, j, rel(JW[b, :, j], ref))


@pytest.mark.parametrize("kind,rows,cols,batch,kw", CASES)
def test_lower_cost_grad_matches_oracle(cuda, kind, rows, cols, batch, kw):
    models, theta, xh, _ = oracle_models(kind, rows, cols, batch, seed=11 + cols, **kw)
    dm = device_model(models)
    cost, grad = dm.cost_grad(theta, torch.as_tensor(xh, device=cuda))
    cost, grad = to_np(cost), to_np(grad)
    for b in range(batch):
        c_ref = im.lower_cost(models[b], theta, xh[b])
        g_ref = im.lower_grad(models[b], theta, xh[b])
        assert abs(cost[b] - c_ref) <= 1e-12 * abs(c_ref)
        assert rel(grad[b], g_ref) <= 1e-12


def test_hessian_symmetric_and_pd(cuda):
    models, theta, xh, _ = oracle_models("filters", 10, 11, 1, seed=3, blur=9, J=2, q=5)
    H, _ = device_model(models).at(theta, xh)
    D = to_np(H.to_dense())
    assert np.max(np.abs(D - D.T)) <= 1e-12 * np.max(np.abs(D))
    assert np.min(np.linalg.eigvalsh(0.5 * (D + D.T))) > 0


def test_hvp_is_gradient_derivative(cuda):
    """H v = d/dt grad(xhat + t v) (central differences of the device gradient)."""
    models, theta, xh, _ = oracle_models("filters", 17, 23, 1, seed=5, blur=9, J=2, q=5, eps=0.3)
    dm = device_model(models)
    H, _ = dm.at(theta, xh)
    v = np.random.default_rng(3).standard_normal(17 * 23)
    h = 1e-6
    xp = torch.as_tensor(xh + h * v, device=cuda)
    xm = torch.as_tensor(xh - h * v, device=cuda)
    _, gp = dm.cost_grad(theta, xp)
    _, gm = dm.cost_grad(theta, xm)
    fd = to_np((gp - gm) / (2 * h))[0]
    hv = to_np(H(torch.as_tensor(v, device=cuda)))
    assert rel(hv, fd) <= 1e-6


def test_dense_operator_gemv(cuda):
    from paper_2412_08264_b200 import dense_operator

    rng = np.random.default_rng(4)
    for n in (5, 300, 600):
        M = rng.standard_normal((n, n))
        M = M + M.T
        v = rng.standard_normal(n)
        out = to_np(dense_operator(torch.as_tensor(M, device=cuda))(torch.as_tensor(v, device=cuda)))
        assert rel(out, M @ v) <= 1e-13


def test_foe_reference_entry_points(cuda):
    """foe_hessian / mixed_jacobian / foe_cost / foe_gradient vs the oracle FoE model."""
    from paper_2412_08264_b200 import FoEParams, ImageVector, InpaintingProblem, Kernel
    from paper_2412_08264_b200 import foe_cost, foe_gradient, foe_hessian, mixed_jacobian

    model, th0 = im.foe_inpainting(16, seed=0)
    d = model.data
    params = FoEParams.unflatten(th0 + 0.1, 3, 5)
    prob = InpaintingProblem(d.mask_rows, d.y, d.ridge, d.shape, ImageVector(d.x_true, d.shape))
    rng = np.random.default_rng(9)
    x = ImageVector(rng.standard_normal(256), (16, 16))
    v = rng.standard_normal(256)
    H = foe_hessian(params, prob)
    J = mixed_jacobian(params, x, prob)
    theta = params.flatten()
    assert rel(to_np(H(torch.as_tensor(v, device=cuda))), im.hessian(model, theta)(v)) <= 1e-12
    assert rel(to_np(J.apply_adjoint(torch.as_tensor(v, device=cuda))),
               im.jacobian(model, theta, x.data).apply_adjoint(v)) <= 1e-12
    assert abs(foe_cost(x, params, prob) - im.lower_cost(model, theta, x.data)) <= 1e-12 * abs(
        im.lower_cost(model, theta, x.data))
    assert rel(to_np(foe_gradient(x, params, prob)), im.lower_grad(model, theta, x.data)) <= 1e-12


def test_ordered_sum_kernel_is_left_to_right(cuda):
    """kr_ordered_sum (the sample-ordered hypergradient sum after the all-gather) is
    bitwise the sequential row-by-row accumulation."""
    from paper_2412_08264_b200.distributed import ordered_sum

    g = torch.Generator(device="cpu").manual_seed(5)
    rows = torch.randn(64, 1200, generator=g, dtype=torch.float64) * torch.logspace(-8, 8, 64, dtype=torch.float64)[:, None]
    ref = rows[0].clone()
    for k in range(1, rows.shape[0]):
        ref += rows[k]
    got = ordered_sum(rows.to(cuda)).cpu()
    assert torch.equal(got, ref)
