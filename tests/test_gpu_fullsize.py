"""Size-independent properties at BASELINE.json's FULL sizes (configs[2] = 64 x 256^2 with
J = 8 5x5 filters and the 15x15 blur; configs[3]'s operators at 512^2 with J = 24 7x7 filters
and the 21x21 blur), where the CPU oracle is too slow to run.

The properties are the ones the reference's algorithm guarantees (file:line of the reference):
  * H is symmetric positive definite and linear (operators.py:363-383),
  * J w is linear in w, and the many-column path (materialised Jacobian + fp64 tensor-core
    product) agrees with the few-column kernel (operators.py:386-444),
  * the recycle space handed to a solve has C = H U and C^T C = I (recycling.py:362-383),
  * a recycled MINRES iterate's residual g - H w is orthogonal to C and its norm is the
    solver's |zeta_k| (krylov.py:205-381),
  * the NSC stop rule stopped exactly where its recorded value first fell below delta
    (stopping.py:93-118), never past max_iter,
  * the upper gradient is the sample-ordered sum of the per-sample J w (bilevel.py:340-351).
Tolerances are stated at each assertion; fp64 throughout.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rand(*shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, dtype=torch.float64, device="cuda", generator=g)


def _rel(a, b):
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def _operator_properties(model, theta, X, nsamples):
    from paper_2412_08264_b200.operators import new_columns

    H, J = model.at(theta, X)
    B, n = model.batch, model.n
    u, v = _rand(B, n, seed=1), _rand(B, n, seed=2)
    Hu, Hv = H(u), H(v)
    # symmetry <u, H v> = <H u, v> and positive definiteness, per sample
    lhs, rhs = (u * Hv).sum(1), (Hu * v).sum(1)
    scale = u.norm(dim=1) * Hv.norm(dim=1)
    assert float(((lhs - rhs).abs() / scale).max()) <= 1e-12
    assert float((u * Hu).sum(1).min()) > 0.0
    # linearity
    assert _rel(H(2.0 * u - 3.0 * v), 2.0 * Hu - 3.0 * Hv) <= 1e-13
    # the column-block path applies the same stencil as the vector path (bitwise)
    M = new_columns(B, n, 2, device=u.device)
    M[:, :, 0] = u
    M[:, :, 1] = v
    HM = H.apply_matrix(M)
    assert torch.equal(HM[:, :, 0], Hu) and torch.equal(HM[:, :, 1], Hv)
    # J: linear, and the many-column path (t >= 4) equals the few-column kernel (t < 4)
    ju, jv = J.apply_adjoint(u), J.apply_adjoint(v)
    assert _rel(J.apply_adjoint(2.0 * u - 3.0 * v), 2.0 * ju - 3.0 * jv) <= 1e-12
    idx = list(range(0, B, max(1, B // nsamples)))[:nsamples]
    Js = J.select(idx, H.select(idx)) if len(idx) < B else J
    W = new_columns(len(idx), n, 5, device=u.device)
    cols = [u[idx], v[idx], u[idx] + v[idx], u[idx] - 2.0 * v[idx], 0.5 * v[idx]]
    for c, w in enumerate(cols):
        W[:, :, c] = w
    JW = Js.apply_adjoint_matrix(W)
    for c, w in enumerate(cols):
        assert _rel(JW[:, :, c], Js.apply_adjoint(w.contiguous())) <= 1e-12


def test_c3_full_size_operator_properties(cuda):
    from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

    cfg = CONFIGS["C3"]
    model = make_batch(cfg)
    assert model.batch == 64 and model.n == 256 * 256
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 1)
    _operator_properties(model, th[0], torch.as_tensor(xh[0], device=cuda), nsamples=4)


def test_c4_full_size_operator_properties(cuda):
    """configs[3]'s operators (512^2, J = 24 7x7 filters, 21x21 blur, p = 1200) on two samples."""
    import dataclasses

    from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

    cfg = dataclasses.replace(CONFIGS["C4"], batch=2)
    model = make_batch(cfg)
    assert model.n == 512 * 512 and model.num_params == 1200
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 1)
    _operator_properties(model, th[0], torch.as_tensor(xh[0], device=cuda), nsamples=2)


def test_c3_full_size_recycled_solve_properties(cuda):
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import CONFIGS, make_batch, synthetic_sequence

    cfg = CONFIGS["C3"]
    delta = 1e-6
    model = make_batch(cfg)
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 2)
    X = [torch.as_tensor(x, device=cuda) for x in xh]
    seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=cfg.recycle_dim, delta=delta,
                                                          max_iter=cfg.max_iter))
    hypergradients(model, th[0], X[0], seq)
    hg, res, recs = hypergradients(model, th[1], X[1], seq)
    H, J = model.at(th[1], X[1])
    G = X[1].reshape(model.batch, -1) - model.x_true
    Wsol = torch.stack([r.solution for r in res])
    R = G - H(Wsol)  # true residuals of every sample
    for b in (0, 17, 41, 63):
        r = res[b]
        rec = recs[b]
        assert rec.dim == cfg.recycle_dim
        U, C = rec.U, rec.C  # (n, s)
        s = C.shape[1]
        # C^T C = I and C = H U for the system's own operator
        eye = torch.eye(s, dtype=torch.float64, device=cuda)
        assert float((C.T @ C - eye).abs().max()) <= 1e-10
        assert _rel(H.sample(b).apply_matrix(U.contiguous()), C) <= 1e-9
        # recycled MINRES: residual orthogonal to C, its norm the solver's |zeta_k|
        rb = R[b]
        assert float((C.T @ rb).norm() / rb.norm()) <= 1e-8
        assert abs(float(rb.norm()) - r.residual_norms[r.iterations]) <= 1e-6 * float(rb.norm())
        # the NSC rule stopped at the first value below delta, or at max_iter
        assert 1 <= r.iterations <= cfg.max_iter
        vals = np.asarray(r.stop_values[: r.iterations + 1])
        if r.stop_reason == "tolerance":
            assert vals[r.iterations] < delta and np.all(vals[1 : r.iterations] >= delta)
        else:
            assert r.stop_reason == "max_iter" and r.iterations == cfg.max_iter and np.all(vals[1:] >= delta)
    # hypergradients: J w per sample, and the upper gradient their left-to-right sum
    assert _rel(hg, J.apply_adjoint(Wsol).reshape(model.batch, -1)) <= 1e-13
    from paper_2412_08264_b200.distributed import ordered_sum

    total = ordered_sum(hg)
    acc = torch.zeros_like(hg[0])
    for b in range(model.batch):
        acc = acc + hg[b]
    assert torch.equal(total.reshape(-1), acc)
