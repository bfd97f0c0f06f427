"""CPU tests: the oracle pinned against the reference's golden vectors and fixtures,
plus the operator contracts of the deblurring / TV / phi_eps operators (which
the reference does not have: their values are pinned only by these contracts).

Golden sources: pkg/plots/sample_data/{replay,sweep}.csv (embedded below as
integer columns; floats from tests/golden/*.npz made by make_golden.py) and the
reference's own solves of random SPD systems (spd_solves.npz).
"""

import numpy as np
import pytest

from oracle import cpu_bilevel as ob
from oracle import cpu_imaging as im
from oracle import cpu_krylov as ok
from oracle import cpu_recycle as orc
from tests.conftest import golden

# pkg/plots/sample_data/replay.csv: iterations and flops per system (integer columns)
REPLAY_GOLDEN = {
    "None": ([11, 9, 15, 13, 15, 13], [551232, 459072, 735552, 643392, 735552, 643392]),
    "Ritz-S": ([11, 8, 13, 11, 11, 7], [551232, 496432, 773582, 662722, 662722, 441002]),
    "RGen-L(R)": ([11, 7, 13, 11, 11, 8], [551232, 441002, 773582, 662722, 662722, 496432]),
    "RGen-L(R)-NSC": ([11, 2, 6, 8, 8, 11], None),
}
# pkg/plots/sample_data/sweep.csv: Ritz-S totals for recycle dims 0,2,4,8,12
SWEEP_GOLDEN = {0: (76, 3768192), 2: (72, 3741718), 4: (66, 3554132), 8: (63, 3600160), 12: (60, 3618571)}


@pytest.fixture(scope="module")
def foe12():
    model, th0 = im.foe_inpainting(12, seed=3)
    seq = ob.record_sequence(th0, ob.Batch([model], [model.data.x_true]), max_upper=6)
    ob.compute_references(seq)
    return seq


def test_record_sequence_matches_reference_fixture(foe12):
    d = golden("foe12_seq.npz")
    assert len(foe12.systems) == d["theta"].shape[0]
    for i, s in enumerate(foe12.systems):
        assert np.allclose(s.theta, d["theta"][i], rtol=1e-10, atol=1e-13)
        assert np.allclose(s.x_hats[0], d["x_hat"][i], rtol=1e-10, atol=1e-13)
        assert np.allclose(s.ref_hgs[0], d["ref_hg"][i], rtol=1e-9, atol=1e-13)


@pytest.mark.parametrize("strategy", list(REPLAY_GOLDEN))
def test_replay_csv_golden(foe12, strategy):
    rows = ob.replay(foe12, strategy, recycle_dim=10)
    its, flops = REPLAY_GOLDEN[strategy]
    assert [r.iterations for r in rows] == its
    if flops is not None:
        assert [r.flops for r in rows] == flops
    d = golden("foe12_seq.npz")
    key = strategy.replace("(", "_").replace(")", "_").replace("-", "_")
    for r, hg in zip(rows, d[f"{key}__hg"]):
        assert np.linalg.norm(r.hg - hg) <= 1e-9 * np.linalg.norm(hg)


def test_sweep_csv_golden(foe12):
    for s, (tot_it, tot_fl) in SWEEP_GOLDEN.items():
        strat = "Ritz-S" if s > 0 else "None"
        rows = ob.replay(foe12, strat, recycle_dim=s)
        assert sum(r.iterations for r in rows) == tot_it
        assert sum(r.flops for r in rows) == tot_fl


def test_desk_fixture_totals():
    """Acceptance criterion 8 numbers (test_acceptance.py:261-298) from the reference's desk sequence."""
    d = golden("foe16_seq.npz")
    shape = tuple(int(v) for v in d["shape"])
    data = im.DataTerm("mask", shape, d["y"], scale=1.0, ridge=float(d["ridge"]), mask_rows=d["mask_rows"],
                       x_true=d["x_true"])
    model = im.Model(data, im.Regularizer("filters", int(d["num_filters"]), int(d["kernel_size"]), "quadratic"))
    systems = [ob.FrozenSystem(i, d["theta"][i], [d["x_hat"][i]], [d["g"][i]]) for i in range(d["theta"].shape[0])]
    seq = ob.FrozenSequence(ob.Batch([model], [d["x_true"]]), systems)
    for strat, total in (("None", 371), ("Ritz-S", 177), ("RGen-L(R)", 179), ("RGen-L(R)-NSC", 163)):
        rows = ob.replay(seq, strat, recycle_dim=30)
        assert sum(r.iterations for r in rows) == total, strat


def test_spd_fixtures_match_reference():
    d = golden("spd_solves.npz")
    for trial in range(6):
        M, g, U, C = (d[f"{trial}_{k}"] for k in ("M", "g", "U", "C"))
        H = im.dense_op(M)
        opts = ok.Options(stop_rule=ok.ResidualRule(1e-9), max_iter=400, track_basis=True)
        res = {"minres": ok.minres(H, g, opts), "rminres": ok.rminres(H, g, orc.Recycle(U, C), opts),
               "cg": ok.cg(H, g, ok.Options(stop_rule=ok.ResidualRule(1e-9), max_iter=400))}
        for tag, r in res.items():
            assert r.iterations == int(d[f"{trial}_{tag}_iters"])
            assert r.flops == int(d[f"{trial}_{tag}_flops"])
            assert np.allclose(r.solution, d[f"{trial}_{tag}_solution"], rtol=1e-12, atol=1e-13)


def test_flop_known_answers():
    """test_krylov.py:335-342"""
    assert ok.flops_minres(0, 10, 190) == 230
    assert ok.flops_minres(5, 10, 190) == 1980
    assert ok.flops_minres(1, 1, 1) == 22
    assert ok.flops_rminres(5, 10, 2, 190) == 2940


def test_gsvd_invariants():
    """Acceptance criterion 5 (test_acceptance.py:170-206)."""
    rng = np.random.default_rng(505)
    for _ in range(50):
        p = int(rng.integers(3, 9))
        t = int(rng.integers(2, p + 1))
        Jt = rng.standard_normal((p, t))
        Ht = rng.standard_normal((t, t)) + t * np.eye(t)
        f = orc.gsvd_pair(Jt, Ht)
        scale = max(np.linalg.norm(Jt), np.linalg.norm(Ht))
        assert np.all(np.diff(f.alpha) >= -1e-10)
        assert np.max(np.abs(f.alpha**2 + f.beta**2 - 1)) <= 1e-10
        assert np.max(np.abs(f.v_j.T @ Jt @ f.x - f.d_j())) <= 1e-8 * scale
        assert np.max(np.abs(f.v_h.T @ Ht @ f.x - f.d_h())) <= 1e-8 * scale


def test_nsc_exactness():
    """Acceptance criterion 6: square orthogonal W + full GSVD gives NSC = ||J H^-1 r||."""
    rng = np.random.default_rng(606)
    for _ in range(5):
        n, p = int(rng.integers(8, 16)), int(rng.integers(3, 9))
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        M = Q @ np.diag(np.geomspace(1, 20, n)) @ Q.T
        W = np.linalg.qr(rng.standard_normal((n, n)))[0]
        Jm = rng.standard_normal((p, n))
        jac = im.JacOp(p, n, lambda w, _J=Jm: _J @ w)
        _, nsc = orc.rgen(W, im.dense_op(M), jac, n, "L", "R")
        r = rng.standard_normal(n)
        exact = np.linalg.norm(Jm @ np.linalg.solve(M, r))
        assert abs(orc.nsc_value(nsc, r) - exact) <= 1e-8 * exact


# --------------------------------------------------------------------------
# contracts of the configs' operators (not in the reference)

KINDS = [("filters", dict(blur=9, J=2, q=5)), ("filters", dict(blur=15, sigma=2.5, J=2, q=3)),
         ("tv", dict(blur=9)), ("foe", dict(J=2, q=3))]


def _model(kind, kw, rows=9, cols=11, seed=0):
    from tests.helpers import oracle_models

    models, theta, xh, xt = oracle_models(kind, rows, cols, 1, seed=seed, eps=0.2, **kw)
    return models[0], theta, xh[0], xt[0]


@pytest.mark.parametrize("kind,kw", KINDS)
def test_hessian_symmetric_pd(kind, kw):
    m, th, xh, _ = _model(kind, kw)
    D = im.hessian(m, th, xh).to_dense()
    assert np.max(np.abs(D - D.T)) <= 1e-12 * np.max(np.abs(D))
    assert np.linalg.eigvalsh(0.5 * (D + D.T)).min() > 0


@pytest.mark.parametrize("kind,kw", KINDS)
def test_gradient_and_hessian_finite_differences(kind, kw):
    m, th, xh, _ = _model(kind, kw)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(xh.size)
    h = 1e-6
    fd_g = (im.lower_cost(m, th, xh + h * v) - im.lower_cost(m, th, xh - h * v)) / (2 * h)
    assert abs(fd_g - im.lower_grad(m, th, xh) @ v) <= 1e-6 * max(1.0, abs(fd_g))
    fd_h = (im.lower_grad(m, th, xh + h * v) - im.lower_grad(m, th, xh - h * v)) / (2 * h)
    hv = im.hessian(m, th, xh)(v)
    assert np.linalg.norm(fd_h - hv) <= 1e-5 * np.linalg.norm(hv)


@pytest.mark.parametrize("kind,kw", KINDS)
def test_mixed_jacobian_finite_differences(kind, kw):
    """J w = -d/dtheta <grad_x L(x, theta), w> (operators.py:277-282 convention)."""
    m, th, xh, _ = _model(kind, kw)
    rng = np.random.default_rng(2)
    w = rng.standard_normal(xh.size)
    Jw = im.jacobian(m, th, xh).apply_adjoint(w)
    h = 1e-6
    fd = np.zeros(th.size)
    for i in range(th.size):
        e = np.zeros(th.size)
        e[i] = h
        fd[i] = -(im.lower_grad(m, th + e, xh) @ w - im.lower_grad(m, th - e, xh) @ w) / (2 * h)
    assert np.linalg.norm(fd - Jw) <= 1e-5 * np.linalg.norm(Jw)


def test_hypergradient_vs_finite_differences():
    """Acceptance criterion 7 style (test_acceptance.py:225-258) on the deblur + phi_eps model."""
    cfg = im.DeblurConfig(7, 1, 3, 1.0, 0.01, "filters", 2, 3, eps=0.3, alpha0=-1.0)
    model, xt = im.deblur_sample(cfg, 0)
    th = im.deblur_theta0(cfg)

    def upper(theta):
        x, _ = ob.lower_solve(model, theta, gtol=1e-11, max_iter=20000)
        return 0.5 * float((x - xt) @ (x - xt)), x

    _, xh = upper(th)
    d, _ = ob.hypergradient(model, th, xh, xt, opts=ok.Options(stop_rule=ok.ResidualRule(1e-12), max_iter=5000))
    h = 1e-5
    fd = np.zeros(th.size)
    for i in range(th.size):
        e = np.zeros(th.size)
        e[i] = h
        fd[i] = (upper(th + e)[0] - upper(th - e)[0]) / (2 * h)
    assert np.linalg.norm(d - fd) <= 1e-4 * np.linalg.norm(fd)


def test_conv_matches_loop_oracle():
    """test_operators.py:20-37 quadruple loop (true convolution, zero boundary)."""
    rng = np.random.default_rng(3)
    k = rng.standard_normal((3, 3))
    x = rng.standard_normal((4, 5))
    out = np.zeros_like(x)
    for i in range(4):
        for j in range(5):
            for u in range(3):
                for v in range(3):
                    ii, jj = i - u + 1, j - v + 1
                    if 0 <= ii < 4 and 0 <= jj < 5:
                        out[i, j] += k[u, v] * x[ii, jj]
    assert np.allclose(im.conv_same(x, k), out, atol=1e-13)


def test_tv_adjoint_pairs():
    rng = np.random.default_rng(4)
    x, p = rng.standard_normal((6, 7)), rng.standard_normal((6, 7))
    assert abs(np.sum(im.diff_h(x) * p) - np.sum(x * im.diff_h_adj(p))) <= 1e-12
    assert abs(np.sum(im.diff_v(x) * p) - np.sum(x * im.diff_v_adj(p))) <= 1e-12


def test_product_generator_matches_oracle():
    from paper_2412_08264_b200 import problems as pr

    for name in ("C1", "C2"):
        c = pr.CONFIGS[name]
        oc = im.DeblurConfig(c.size, c.batch, c.blur_size, c.blur_sigma, c.noise, c.reg, c.num_filters,
                             c.kernel_size, c.eps, c.alpha0, c.filter_std, c.seed)
        for k in range(2):
            xt, y = pr.sample_arrays(c, k)
            m, xo = im.deblur_sample(oc, k)
            assert np.array_equal(xt, xo)
            assert np.array_equal(y, m.data.y)
        assert np.array_equal(pr.theta0(c), im.deblur_theta0(oc))


def _spd(rng, n, lo=1e-3, hi=1.0):
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (Q * np.geomspace(lo, hi, n)) @ Q.T, Q


def test_rcg_deflated_cg_properties():
    """Recycled (deflated) CG restatement: exact solve, U^T r = 0 throughout,
    mutually orthogonal residuals, empty space == plain cg, deflating the low end
    of the spectrum cuts iterations, FLOP count."""
    from oracle.cpu_imaging import dense_op

    rng = np.random.default_rng(4)
    n = 80
    M, Q = _spd(rng, n)
    g = rng.standard_normal(n)
    H = dense_op(M)
    Ut = Q[:, :6] + 1e-3 * rng.standard_normal((n, 6))  # near the 6 smallest eigenvectors
    C, R = np.linalg.qr(M @ Ut)
    U = Ut @ np.linalg.inv(R)
    rec = orc.Recycle(U, C)
    opts = ok.Options(stop_rule=ok.ResidualRule(1e-10), max_iter=500, track_basis=True)
    r = ok.rcg(H, g, rec, opts)
    assert r.stop_reason == "tolerance"
    assert np.linalg.norm(r.solution - np.linalg.solve(M, g)) <= 1e-6 * np.linalg.norm(np.linalg.solve(M, g))
    assert np.linalg.norm(U.T @ r.residual_vector) <= 1e-10 * np.linalg.norm(g) * np.linalg.norm(U)
    V = r.basis[:, :12]  # before finite-precision loss of orthogonality
    assert np.max(np.abs(V.T @ V - np.eye(V.shape[1]))) <= 1e-8
    assert np.abs(U.T @ V).max() <= 1e-8 * np.linalg.norm(U)
    plain = ok.cg(H, g, opts)
    assert r.iterations < plain.iterations
    assert r.flops == ok.flops_rcg(r.iterations, n, 6, H.apply_cost)
    e = ok.rcg(H, g, orc.Recycle.empty(n), opts)
    assert e.iterations == plain.iterations and np.array_equal(e.solution, plain.solution)
    with pytest.raises(ok.NonSPDError):
        ok.rcg(dense_op(-M), g, rec, opts)


def test_rcg_sequence_tv():
    """SequenceSolver with method="cg" (BASELINE config 1's recycled CG) on a small
    smoothed-TV deblurring sequence: recycled solves reach the tolerance and the
    hypergradients match an exact solve."""
    cfg = im.DeblurConfig(16, 1, 5, 1.0, 0.01, "tv", 1, 1)
    model, xt = im.deblur_sample(cfg, 0)
    th0 = im.deblur_theta0(cfg)
    rng = np.random.default_rng(0)
    seq = ob.SequenceSolver(ob.SolveConfig.from_strategy("RGen-L(R)", recycle_dim=4, delta=1e-9, max_iter=300,
                                                         method="cg"))
    for step in range(3):
        th = th0 + 0.05 * step
        xh = xt + 0.02 * rng.standard_normal(xt.size)
        H, J = im.hessian(model, th, xh), im.jacobian(model, th, xh)
        res, rec = seq.solve(H, xh - xt, J)
        assert res.stop_reason == "tolerance"
        if step:
            assert rec.dim == 4
        exact = np.linalg.solve(_dense(H), xh - xt)
        hg, hge = J.apply_adjoint(res.solution), J.apply_adjoint(exact)
        assert np.linalg.norm(hg - hge) <= 1e-6 * np.linalg.norm(hge)


def _dense(H):
    return np.column_stack([H(e) for e in np.eye(H.dim)])


def test_c_stencil_matches_numpy_oracle():
    """oracle/cpu_stencil.c (the fixture generator's fast operators) against cpu_imaging's
    scipy restatement: H v and J w to roundoff on config-shaped small problems."""
    import dataclasses

    from oracle import cpu_fast as cf

    for name, size in (("C2", 24), ("C3", 40), ("C4", 48)):
        cfg = dataclasses.replace(im.CONFIGS[name], size=size)
        m, xt = im.deblur_sample(cfg, 1)
        th = im.deblur_theta0(cfg)
        xh = xt + 0.03 * np.random.default_rng(2).standard_normal(xt.size)
        v = np.random.default_rng(3).standard_normal(m.data.n)
        a, b = cf.hessian(m, th, xh)(v), im.hessian(m, th, xh)(v)
        assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)
        ja, jb = cf.jacobian(m, th, xh).apply_adjoint(v), im.jacobian(m, th, xh).apply_adjoint(v)
        assert np.linalg.norm(ja - jb) <= 1e-12 * np.linalg.norm(jb)
