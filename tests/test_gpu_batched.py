"""Whole-batch recycle update (batched.recycle_update) against the per-sample
path (recycling.next_recycle, itself pinned to the oracle in test_gpu_bilevel /
test_gpu_replay), and batched CholQR2 with padding.

Equal in exact arithmetic; compared through basis-independent quantities:
the spanned projectors of U and C, the selected mu values, and Z = W V_H diag(mu)
(sign-free up to column order: Z's columns carry the eigenvector sign, so the
projector of Z and the mu values are compared)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _proj(M):
    Q, _ = torch.linalg.qr(M)
    return Q @ Q.T


def test_cholqr2_rows_padding():
    from paper_2412_08264_b200.batched import _row_mask, cholqr2_rows

    g = torch.Generator(device="cuda").manual_seed(0)
    B, T, n = 3, 12, 500
    dims = [12, 7, 0]
    A = torch.randn(B, T, n, generator=g, dtype=torch.float64, device="cuda")
    for b, d in enumerate(dims):
        A[b, d:] = 0
    mask = _row_mask(dims, T, "cuda")
    Q, F, ok = cholqr2_rows(A, mask)
    assert ok.tolist() == [True, True, True]
    for b, d in enumerate(dims):
        Qb = Q[b, :d]
        assert torch.allclose(Qb @ Qb.T, torch.eye(d, dtype=torch.float64, device="cuda"), atol=1e-14)
        assert torch.all(Q[b, d:] == 0)
        assert torch.allclose(F[b] @ A[b], Q[b], atol=1e-12)
        # A_col = Q_col R with R = F^{-T} upper triangular (positive diagonal)
        R = torch.linalg.inv(F[b, :d, :d]).T
        assert torch.allclose(torch.triu(R), R, atol=1e-12) and bool((R.diagonal() > 0).all())
    # ill-conditioned and rank-deficient blocks are declined
    A2 = A.clone()
    A2[0, 5] = A2[0, 4] * (1 + 1e-12)
    A2[1, 3] = 0
    _, _, ok2 = cholqr2_rows(A2, mask)
    assert ok2.tolist() == [False, False, True]
    # shifted CholeskyQR3 takes cond ~ 1e8 blocks (which CholQR2 declines) ...
    A3 = A.clone()
    A3[0, 5] = A3[0, 4] + 1e-8 * A3[0, 5]
    _, _, ok3 = cholqr2_rows(A3, mask)
    Q3, F3, ok3r, _, _ = cholqr2_rows(A3, mask, robust=True)
    assert ok3.tolist() == [False, True, True] and ok3r.tolist() == [True, True, True]
    Qb = Q3[0, :12]
    assert torch.allclose(Qb @ Qb.T, torch.eye(12, dtype=torch.float64, device="cuda"), atol=1e-14)
    assert torch.dist(F3[0] @ A3[0], Q3[0]) <= 1e-6 * torch.linalg.norm(Q3[0])  # forward error ~ cond * eps
    # ... and still declines near-dependent ones (the reference's pivoted QR drops a column)
    _, _, ok2r, fr, sk = cholqr2_rows(A2, mask, robust=True)
    # ... the robust path reports the breakdown row (the rank-drop round removes it)
    # (sample 0's near-duplicate row survives the shifted passes; the |R_jj| rule drops it)
    assert sk is None and fr.tolist()[1:] == [3, -1]


def _setup(strategy, s=6, size=32, B=4, steps=2):
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import DeblurConfig, make_batch, synthetic_sequence

    cfg = DeblurConfig(size, B, 5, 1.0, 0.01, "filters", 4, 3)
    model = make_batch(cfg)
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), steps + 1)
    seq = SequenceSolver(HessianSolveConfig.from_strategy(strategy, recycle_dim=s, delta=1e-8, max_iter=40))
    seq.batched_update = False
    for i in range(steps):
        hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    H, J = model.at(th[steps], torch.as_tensor(xh[steps], device="cuda"))
    return model, seq, H, J


def _selection_well_posed(st, Hb, Jb, seq, b):
    """False when the S/L/M cut splits a cluster of equal selection keys (then the
    selected subspace is arbitrary in the reference too, e.g. the mu = 0 null
    cluster when t > p)."""
    from paper_2412_08264_b200.recycling import _select_indices, _sym, build_candidate_basis, gsvd_pair

    W = build_candidate_basis(seq._prev_basis[b], seq._prev_recycle[b].U).W
    t = W.shape[1]
    Ht = _sym(W.T @ Hb.apply_matrix(W))
    if st.vec_type == "Ritz":
        key = torch.linalg.eigvalsh(Ht)
    else:
        Jt = Jb.apply_adjoint_matrix(W)
        if Jt.shape[0] < t:
            Jt = torch.cat([Jt, torch.zeros(t - Jt.shape[0], t, dtype=Jt.dtype, device=Jt.device)])
        key = gsvd_pair(Jt, Ht, symmetric=True).mu
    key = key.sort().values
    s = min(seq.cfg.recycle_dim, t)
    sel = set(_select_indices(t, s, st.size, "cpu").tolist())
    scale = float(key.abs().max())
    for i in range(t - 1):
        if (i in sel) != (i + 1 in sel) and float(key[i + 1] - key[i]) <= 1e-6 * scale:
            return False
    return True


def test_declines_small_mu_selections():
    from paper_2412_08264_b200.batched import supports
    from paper_2412_08264_b200.recycling import StrategyDescriptor as S

    assert supports(S.parse("RGen-L(R)-NSC")) and supports(S.parse("Ritz-S")) and supports(S.parse("RGen-L(M)"))
    assert not supports(S.parse("RGen-S(L)")) and not supports(S.parse("RGen-M(R)"))
    assert not supports(S.parse("inner:RGen-L(R)")) and not supports(S.parse("HRitz-S"))
    # harmonic Ritz and inner placement: the native orchestrator only
    assert supports(S.parse("HRitz-S"), native=True) and supports(S.parse("inner:HRitz-S"), native=True)
    assert supports(S.parse("inner:RGen-L(R)"), native=True) and not supports(S.parse("inner:RGen-S(R)"), native=True)


def _harmonic_keys(W, HW):
    """|theta| of the pencil (HW)^T HW rho = theta (HW)^T W rho, ascending (recycling.py:239-272)."""
    import scipy.linalg as sl

    A = (HW.T @ HW).cpu().numpy()
    Bm = (HW.T @ W).cpu().numpy()
    vals = sl.eigh(0.5 * (A + A.T), 0.5 * (Bm + Bm.T), eigvals_only=True)
    return torch.as_tensor(np.sort(np.abs(vals)))


@pytest.mark.parametrize("strategy", ["HRitz-S", "HRitz-L", "HRitz-M"])
def test_harmonic_ritz_native_matches_per_sample(strategy):
    """Harmonic Ritz in the native orchestrator (Cholesky reduction of the pencil) against
    the per-sample reference-semantics path (recycling.harmonic_ritz_select)."""
    from paper_2412_08264_b200.batched import recycle_update_native
    from paper_2412_08264_b200.recycling import _select_indices, build_candidate_basis, next_recycle

    model, seq, H, J = _setup(strategy)
    st = seq.cfg.strategy
    got_all = recycle_update_native(st, seq.cfg.recycle_dim, H, J, seq._prev_basis, seq._prev_recycle)
    for b in range(model.batch):
        ref = next_recycle(st, h_current=H.sample(b), jac_current=J.sample(b), prev_basis=seq._prev_basis[b],
                           prev_recycle=seq._prev_recycle[b], s=seq.cfg.recycle_dim)
        got = got_all[b]
        assert got is not None and got.dim == ref.dim
        W = build_candidate_basis(seq._prev_basis[b], seq._prev_recycle[b].U).W
        key = _harmonic_keys(W, H.sample(b).apply_matrix(W))
        t, sdim = key.numel(), min(seq.cfg.recycle_dim, key.numel())
        sel = set(_select_indices(t, sdim, st.size, "cpu").tolist())
        posed = all(not ((i in sel) != (i + 1 in sel) and float(key[i + 1] - key[i]) <= 1e-6 * float(key.max()))
                    for i in range(t - 1))
        if posed:
            assert torch.dist(_proj(got.C), _proj(ref.C)) <= 1e-8
            assert torch.dist(_proj(got.U), _proj(ref.U)) <= 1e-8
        assert torch.allclose(got.C.T @ got.C, torch.eye(got.dim, dtype=torch.float64, device="cuda"), atol=1e-13)
        HU = H.sample(b).apply_matrix(got.U)
        assert torch.dist(HU, got.C) <= 1e-10 * torch.linalg.norm(HU)


@pytest.mark.parametrize("impl", ["python", "native"])
@pytest.mark.parametrize("strategy", ["RGen-L(R)-NSC", "RGen-L(L)", "RGen-L(M)", "Ritz-S", "Ritz-L", "Ritz-M"])
def test_recycle_update_matches_per_sample(strategy, impl):
    from paper_2412_08264_b200.batched import recycle_update, recycle_update_native
    from paper_2412_08264_b200.recycling import next_recycle

    model, seq, H, J = _setup(strategy)
    st = seq.cfg.strategy
    fn = recycle_update_native if impl == "native" else recycle_update
    batched = fn(st, seq.cfg.recycle_dim, H, J, seq._prev_basis, seq._prev_recycle)
    for b in range(model.batch):
        ref = next_recycle(st, h_current=H.sample(b), jac_current=J.sample(b), prev_basis=seq._prev_basis[b],
                           prev_recycle=seq._prev_recycle[b], s=seq.cfg.recycle_dim)
        got = batched[b]
        assert got is not None
        assert got.dim == ref.dim
        if _selection_well_posed(st, H.sample(b), J.sample(b), seq, b):
            assert torch.dist(_proj(got.C), _proj(ref.C)) <= 1e-8
            assert torch.dist(_proj(got.U), _proj(ref.U)) <= 1e-8
        assert torch.allclose(got.C.T @ got.C, torch.eye(got.dim, dtype=torch.float64, device="cuda"), atol=1e-13)
        HU = H.sample(b).apply_matrix(got.U)
        assert torch.dist(HU, got.C) <= 1e-10 * torch.linalg.norm(HU)
        if ref.nsc_data is not None:
            a, r = got.nsc_data, ref.nsc_data
            assert torch.allclose(a.values, r.values, rtol=1e-8, atol=1e-12)
            assert torch.dist(_proj(a.z_block()), _proj(r.z_block())) <= 1e-8
            # the NSC value of any residual agrees (sign-free)
            v = torch.randn(model.n, dtype=torch.float64, device="cuda")
            na = torch.linalg.vector_norm(a.z_block().T @ v)
            nr = torch.linalg.vector_norm(r.z_block().T @ v)
            # (mu near zero -- size S -- is only absolutely accurate, as in the reference)
            floor = 1e-12 * float(torch.linalg.vector_norm(v)) * r.values.numel() ** 0.5
            assert abs(float(na - nr)) <= 1e-9 * float(nr) + floor


def test_sequence_batched_equals_per_sample():
    """Whole sequences through SequenceSolver: iteration counts and hypergradients agree."""
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import DeblurConfig, make_batch, synthetic_sequence

    cfg = DeblurConfig(48, 4, 7, 1.2, 0.01, "filters", 4, 5)
    model = make_batch(cfg)
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 4)
    out = {}
    for batched in (False, True):
        seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=8, delta=1e-8,
                                                              max_iter=120))
        seq.batched_update = batched
        rows = []
        for i in range(4):
            hg, res, _ = hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
            rows.append((hg.cpu().numpy(), [r.iterations for r in res]))
        out[batched] = rows
    # the two paths are equal in exact arithmetic; in floating point both carry the
    # solve's roundoff amplification, so compare their distances to a tight solve
    from paper_2412_08264_b200 import ResidualNormRule, SolveOptions, minres

    for i, ((hg0, it0), (hg1, it1)) in enumerate(zip(out[False], out[True])):
        assert max(abs(a - b) for a, b in zip(it0, it1)) <= 2
        H, J = model.at(th[i], torch.as_tensor(xh[i], device="cuda"))
        G = torch.as_tensor(xh[i], device="cuda").reshape(model.batch, -1) - model.x_true
        res = minres(H, G, SolveOptions(stop_rule=ResidualNormRule(1e-13), max_iter=3000))
        exact = J.apply_adjoint(torch.stack([r.solution for r in res])).cpu().numpy()
        e0 = np.abs(hg0 - exact).max()
        e1 = np.abs(hg1 - exact).max()
        assert e1 <= 3 * e0 + 1e-9 * np.abs(exact).max(), (i, e0, e1)


@pytest.mark.parametrize("impl", ["python", "native"])
def test_recycle_update_rank_drop(impl):
    """Exactly dependent candidates are dropped as by the reference's pivoted QR (no fallback)."""
    from paper_2412_08264_b200 import batched
    from paper_2412_08264_b200.recycling import next_recycle

    model, seq, H, J = _setup("RGen-L(R)-NSC")
    st = seq.cfg.strategy
    bases = list(seq._prev_basis)
    V0 = bases[0]
    bases[0] = torch.cat([V0, V0[:, :2], 3.0 * V0[:, 5:6]], dim=1)  # three dependent columns
    batched.STATS = {}
    fn = batched.recycle_update_native if impl == "native" else batched.recycle_update
    try:
        got = fn(st, seq.cfg.recycle_dim, H, J, bases, seq._prev_recycle)
        assert batched.STATS["declined"] == 0, batched.STATS
    finally:
        batched.STATS = None
    ref = next_recycle(st, h_current=H.sample(0), jac_current=J.sample(0), prev_basis=bases[0],
                       prev_recycle=seq._prev_recycle[0], s=seq.cfg.recycle_dim)
    assert got[0].nsc_data.w.shape[1] == ref.nsc_data.w.shape[1] == V0.shape[1] + seq._prev_recycle[0].dim
    assert torch.dist(_proj(got[0].C), _proj(ref.C)) <= 1e-8
    assert torch.allclose(got[0].nsc_data.values, ref.nsc_data.values, rtol=1e-8)


@pytest.mark.parametrize("T", [1, 7, 64, 228, 229, 330, 580])
def test_chol_inv_kernel_matches_torch(T, monkeypatch):
    """kr_chol_inv (one CTA per matrix) against the torch.linalg formulation."""
    from paper_2412_08264_b200 import batched

    g = torch.Generator(device="cuda").manual_seed(T)
    B = 5
    dims = torch.tensor([T, max(T - 3, 0), T, 1, T], dtype=torch.int32)
    X = torch.randn(B, T, 3 * T + 4, generator=g, dtype=torch.float64, device="cuda")
    X = X * torch.logspace(0, -3, T, dtype=torch.float64, device="cuda").reshape(1, -1, 1)
    G = X @ X.transpose(1, 2)
    if T > 2:
        G[2, 1, :] = G[2, 0, :]  # breakdown at row 1 of sample 2 (rows 0, 1 equal)
        G[2, :, 1] = G[2, :, 0]
    shift = torch.tensor([0.0, 1e-3, 0.0, 0.0, 2e-6], dtype=torch.float64, device="cuda")
    for scale in (True, False):
        for sh in (None, shift):
            F, info, st = batched._chol_inv(G, dims, scale, sh)
            monkeypatch.setattr(batched, "CHOL_TMAX", -1)
            Ft, infot, stt = batched._chol_inv(G, dims, scale, sh)
            monkeypatch.setattr(batched, "CHOL_TMAX", 640)
            assert info.tolist() == infot.tolist()
            good = info < 0
            assert torch.allclose(st[good, :3], stt[good, :3], rtol=1e-12, atol=0)
            assert torch.allclose(F[good], Ft[good], rtol=1e-9, atol=1e-12 * float(Ft[good].abs().max()))


@pytest.mark.parametrize("cluster,wide", [(True, ()), (False, ()), (True, (330,)), (True, (330, 580))])
def test_qrcp_small_matches_scipy_pivoted_qr(cluster, wide, monkeypatch):
    """kr_qrcp_small on R against scipy.linalg.qr(A, pivoting=True), the reference's
    candidate-basis QR (recycling.py:187-199): same pivots, |R_kk|, rank under the
    1e-10 rule, and the same kept span."""
    import scipy.linalg as sl

    from paper_2412_08264_b200 import batched
    from paper_2412_08264_b200.batched import qrcp_small

    monkeypatch.setattr(batched, "QRCP_CLUSTER", cluster)
    rng = np.random.default_rng(17)
    mats = []
    for t in (1, 5, 40, 120, 220) + wide:
        A = rng.standard_normal((1200, t)) * np.logspace(0, -6, t)
        if t >= 40:
            A[:, 7] = A[:, 3] * (1 + 1e-13)       # numerically dependent
            A[:, 20] = 2.5 * A[:, 11]              # exactly dependent
        mats.append(A)
    T = max(A.shape[1] for A in mats)
    M = np.zeros((len(mats), T, T))
    for b, A in enumerate(mats):
        _, R = np.linalg.qr(A)
        M[b, : A.shape[1], : A.shape[1]] = R.T  # column-major storage of R
    dims = torch.tensor([A.shape[1] for A in mats], dtype=torch.int32)
    Q, Rp, rank, perm = qrcp_small(torch.as_tensor(M, device="cuda"), dims, 1e-10)
    Q, Rp, rank, perm = Q.cpu().numpy(), Rp.cpu().numpy(), rank.cpu().numpy(), perm.cpu().numpy()
    for b, A in enumerate(mats):
        t = A.shape[1]
        Qs, Rs, Ps = sl.qr(A, mode="economic", pivoting=True)
        d = np.abs(np.diag(Rs))
        r_ref = int(np.sum(d > 1e-10 * d[0]))
        assert rank[b] == r_ref, (t, rank[b], r_ref)
        r = r_ref
        assert list(perm[b, :r]) == list(Ps[:r]), t
        assert np.allclose(np.abs(np.diag(Rp[b][:r, :r])), d[:r], rtol=1e-8, atol=1e-14 * d[0])
        _, R = np.linalg.qr(A)
        Qa = np.linalg.qr(A)[0] @ Q[b, :r, :t].T  # kept basis Q_A Q_R[:, :r]
        Pk = Qa @ Qa.T
        Pr = Qs[:, :r] @ Qs[:, :r].T
        assert np.linalg.norm(Pk - Pr) <= 1e-7


@pytest.mark.parametrize("B,T,n", [(1, 7, 5000), (4, 220, 16384), (3, 33, 12288 + 7)])
def test_gram_split_k(B, T, n):
    from paper_2412_08264_b200.batched import gram

    g = torch.Generator(device="cuda").manual_seed(B + T)
    A = torch.randn(B, T, n, generator=g, dtype=torch.float64, device="cuda")
    Bm = torch.randn(B, T, n, generator=g, dtype=torch.float64, device="cuda")
    ref = A @ Bm.transpose(1, 2)
    got = gram(A, Bm)
    assert torch.allclose(got, ref, rtol=0, atol=1e-11 * float(ref.abs().max()))
    assert torch.equal(gram(A, Bm), got)  # deterministic


def _span_dist(A, B):
    """|| (I - P_A) Q_B ||_F for the orthonormal bases of two equal-width column blocks
    (no n x n projector: n = 16384 here)."""
    Qa, _ = torch.linalg.qr(A)
    Qb, _ = torch.linalg.qr(B)
    return float(torch.linalg.matrix_norm(Qb - Qa @ (Qa.T @ Qb)))


def test_recycle_update_rank_drop_block_householder():
    """Exactly dependent candidates in a block large enough (n t >= 2^21) for the
    native orchestrator's block-Householder branch: shifted CholeskyQR3 breaks down at
    the first dependent row, the leading rows are reused, only the remainder goes
    through a Householder QR -- the candidate span, the drop count and the recycle
    space agree with the per-sample reference-semantics path."""
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import DeblurConfig, make_batch, synthetic_sequence
    from paper_2412_08264_b200.recycling import next_recycle

    cfg = DeblurConfig(128, 2, 5, 1.0, 0.01, "filters", 4, 3)
    model = make_batch(cfg)
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 3)
    seq = SequenceSolver(HessianSolveConfig.from_strategy("RGen-L(R)-NSC", recycle_dim=10, delta=1e-14,
                                                          max_iter=150))
    seq.batched_update = False
    for i in range(2):
        hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    H, J = model.at(th[2], torch.as_tensor(xh[2], device="cuda"))
    st = seq.cfg.strategy
    bases = list(seq._prev_basis)
    V0 = bases[0]
    assert V0.shape[1] >= 128
    bases[0] = torch.cat([V0, V0[:, :2] - V0[:, 7:9], 3.0 * V0[:, 5:6]], dim=1)  # three dependent columns, last
    assert model.n * (bases[0].shape[1] + seq._prev_recycle[0].dim) >= 1 << 21
    batched.STATS = {}
    try:
        got = batched.recycle_update_native(st, seq.cfg.recycle_dim, H, J, bases, seq._prev_recycle)
        assert batched.STATS["declined"] == 0, batched.STATS
    finally:
        batched.STATS = None
    ref = next_recycle(st, h_current=H.sample(0), jac_current=J.sample(0), prev_basis=bases[0],
                       prev_recycle=seq._prev_recycle[0], s=seq.cfg.recycle_dim)
    t_kept = V0.shape[1] + seq._prev_recycle[0].dim
    assert got[0].nsc_data.w.shape[1] == ref.nsc_data.w.shape[1] == t_kept
    # candidate spans: the same subspace
    assert _span_dist(got[0].nsc_data.w, ref.nsc_data.w) <= 1e-8
    C = got[0].C
    assert torch.allclose(C.T @ C, torch.eye(C.shape[1], dtype=torch.float64, device="cuda"), atol=1e-13)
    HU = H.sample(0).apply_matrix(got[0].U)
    assert torch.dist(HU, C) <= 1e-10 * torch.linalg.norm(HU)
    if _selection_well_posed(st, H.sample(0), J.sample(0), type("S", (), {"_prev_basis": bases, "_prev_recycle":
                             seq._prev_recycle, "cfg": seq.cfg})(), 0):
        assert _span_dist(C, ref.C) <= 1e-8
        assert torch.allclose(got[0].nsc_data.values, ref.nsc_data.values, rtol=1e-8)


@pytest.mark.parametrize("strategy,dual", [("RGen-L(R)-NSC", "1"), ("RGen-L(R)-NSC", "0"), ("Ritz-L", "1")])
def test_recycle_update_wide_candidates(strategy, dual, monkeypatch):
    """Candidate widths beyond the shared-memory kernels (t ~ 330, the C3 regime): the
    native orchestrator (global-workspace Cholesky / eigen-select, 8-CTA cluster QRCP)
    against the per-sample reference-semantics path.  RGen runs both forms of the GSVD's
    eigen step: the t x t problem Q1^T Q1 (KR_GSVD_DUAL=0) and, since t > p = 208 here, the
    p x p dual Q1 Q1^T (default)."""
    monkeypatch.setenv("KR_GSVD_DUAL", dual)
    from paper_2412_08264_b200 import HessianSolveConfig, SequenceSolver, batched
    from paper_2412_08264_b200.bilevel import hypergradients
    from paper_2412_08264_b200.problems import DeblurConfig, make_batch, synthetic_sequence
    from paper_2412_08264_b200.recycling import next_recycle

    cfg = DeblurConfig(64, 2, 9, 1.5, 0.01, "filters", 8, 5)
    model = make_batch(cfg)
    th, xh = synthetic_sequence(cfg, model.x_true.cpu().numpy(), 3)
    seq = SequenceSolver(HessianSolveConfig.from_strategy(strategy, recycle_dim=30, delta=1e-14, max_iter=290))
    seq.batched_update = False
    for i in range(2):
        hypergradients(model, th[i], torch.as_tensor(xh[i], device="cuda"), seq)
    H, J = model.at(th[2], torch.as_tensor(xh[2], device="cuda"))
    st = seq.cfg.strategy
    T = max(int(V.shape[1]) + r.dim for V, r in zip(seq._prev_basis, seq._prev_recycle))
    assert T > 228, T
    batched.STATS = {}
    try:
        got = batched.recycle_update_native(st, 30, H, J, list(seq._prev_basis), seq._prev_recycle)
        assert batched.STATS["declined"] == 0, batched.STATS
    finally:
        batched.STATS = None
    for b in range(2):
        ref = next_recycle(st, h_current=H.sample(b), jac_current=J.sample(b), prev_basis=seq._prev_basis[b],
                           prev_recycle=seq._prev_recycle[b], s=30)
        C = got[b].C
        assert torch.allclose(C.T @ C, torch.eye(C.shape[1], dtype=torch.float64, device="cuda"), atol=1e-12)
        HU = H.sample(b).apply_matrix(got[b].U)
        assert torch.dist(HU, C) <= 1e-9 * torch.linalg.norm(HU)
        if st.vec_type == "RGen":
            assert got[b].nsc_data.w.shape[1] == ref.nsc_data.w.shape[1]
            assert _span_dist(got[b].nsc_data.w, ref.nsc_data.w) <= 1e-8
        if _selection_well_posed(st, H.sample(b), J.sample(b), seq, b):
            assert _span_dist(C, ref.C) <= 1e-7
            if st.vec_type == "RGen":
                assert torch.allclose(got[b].nsc_data.values, ref.nsc_data.values, rtol=1e-8)


@pytest.mark.parametrize("strategy", ["inner:RGen-L(R)-NSC", "inner:Ritz-S", "inner:HRitz-L"])
def test_inner_placement_native_matches_per_sample(strategy):
    """Inner placement (recycling.py:409-415): the candidates are projected with the
    PREVIOUS system's H (and J), then normalised against the upcoming H -- the native
    orchestrator with op_proj against the per-sample reference-semantics path."""
    from paper_2412_08264_b200.batched import recycle_update_native
    from paper_2412_08264_b200.recycling import _select_indices, build_candidate_basis, next_recycle

    model, seq, H, J = _setup(strategy)
    st = seq.cfg.strategy
    Hp, Jp = seq._prev_h, seq._prev_jac
    got_all = recycle_update_native(st, seq.cfg.recycle_dim, H, J, seq._prev_basis, seq._prev_recycle, H_proj=Hp)
    for b in range(model.batch):
        ref = next_recycle(st, h_current=H.sample(b), h_previous=Hp.sample(b), jac_current=J.sample(b),
                           jac_previous=Jp.sample(b), prev_basis=seq._prev_basis[b],
                           prev_recycle=seq._prev_recycle[b], s=seq.cfg.recycle_dim)
        got = got_all[b]
        assert got is not None and got.dim == ref.dim
        if st.vec_type == "HRitz":
            W = build_candidate_basis(seq._prev_basis[b], seq._prev_recycle[b].U).W
            key = _harmonic_keys(W, Hp.sample(b).apply_matrix(W))
            t, sdim = key.numel(), min(seq.cfg.recycle_dim, key.numel())
            sel = set(_select_indices(t, sdim, st.size, "cpu").tolist())
            posed = all(not ((i in sel) != (i + 1 in sel) and float(key[i + 1] - key[i]) <= 1e-6 * float(key.max()))
                        for i in range(t - 1))
        else:
            posed = _selection_well_posed(st, Hp.sample(b), Jp.sample(b), seq, b)
        if posed:
            assert torch.dist(_proj(got.C), _proj(ref.C)) <= 1e-8
            assert torch.dist(_proj(got.U), _proj(ref.U)) <= 1e-8
        assert torch.allclose(got.C.T @ got.C, torch.eye(got.dim, dtype=torch.float64, device="cuda"), atol=1e-13)
        HU = H.sample(b).apply_matrix(got.U)  # C = H_current U, whatever H projected
        assert torch.dist(HU, got.C) <= 1e-10 * torch.linalg.norm(HU)
        if ref.nsc_data is not None:
            assert torch.allclose(got.nsc_data.values, ref.nsc_data.values, rtol=1e-8, atol=1e-12)
