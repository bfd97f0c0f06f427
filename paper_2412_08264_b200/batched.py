"""Recycle update batched over samples (the B200 layout of ``next_recycle``).

The reference updates one sample at a time through numpy/LAPACK
(recycling.py:386-465).  Here every step of the update runs once for the whole
batch: sample b's t_b candidate vectors are the rows [0, t_b) of a (B, T, n)
block (T = max t_b, zero rows beyond), the n x t products are strided-batched
GEMMs, the t x t factorizations are batched Cholesky (cuSOLVER) and the
selected-eigenpair kernel ``kr_syev_select`` (one CTA per sample).  Padding is
exact: pad rows are zero and the pad block of every Gram matrix is the identity,
so the leading t_b block of each factor is the per-sample factor.

Vectors are stored as ROWS here ((B, t, n): sample b, vector j, n entries), i.e.
the column-major n x t blocks of the reference with one contiguous vector per
row; the per-sample views handed back are the reference's n x t column blocks.
"""

from __future__ import annotations

import ctypes

import numpy as np

import torch

from . import _lib

SIZE_CODES = {"S": 0, "L": 1, "M": 2}
EIG_TMAX = 640  # KR_TMAX


def syev_select(M: torch.Tensor, dims: torch.Tensor, size: str, s: int):
    """Selected eigenpairs of the leading dims[b] x dims[b] blocks of M (B, T, T).

    Returns (lam (B, s), Z (B, s, T), nsel (B,) int32), all on the device:
    eigenvector q of sample b is Z[b, q] (zero beyond dims[b]); see kr_syev_select."""
    B, T, T2 = M.shape
    if T != T2:
        raise ValueError(f"expected square blocks, got {tuple(M.shape)}")
    if M.stride(2) != 1 and M.stride(1) != 1:
        M = M.contiguous()
    M = M.contiguous()
    dims = dims.to(device=M.device, dtype=torch.int32).contiguous()
    lam = torch.zeros(B, max(s, 1), dtype=torch.float64, device=M.device)
    Z = torch.empty(B, max(s, 1), T, dtype=torch.float64, device=M.device)
    nsel = torch.zeros(B, dtype=torch.int32, device=M.device)
    L = _lib.lib()
    wl = int(L.kr_syev_select_workspace(B, T))
    ws = torch.empty(max(wl, 1), dtype=torch.float64, device=M.device)
    # M is symmetrised inside, so row- or column-major reading gives the same matrix
    _lib.check(L.kr_syev_select(M.data_ptr(), T, T * T, dims.data_ptr(), B, T, SIZE_CODES[size], s,
                                lam.data_ptr(), lam.stride(0), Z.data_ptr(), T, Z.stride(0), nsel.data_ptr(),
                                ws.data_ptr(), wl, _lib.stream_ptr()), "kr_syev_select")
    _lib.note_launch("kr_syev_select")
    return lam[:, :s], Z[:, :s], nsel


STATS: dict | None = None  # set to {} to count declined samples per check

QRCP_CLUSTER = True  # kr_qrcp_small_cluster (4 CTAs per matrix, columns in shared memory)


def qrcp_small(M: torch.Tensor, dims: torch.Tensor, rtol: float):
    """QR with column pivoting of the leading dims[b] blocks (kr_qrcp_small).

    M (B, T, T) holds each matrix column-major (M[b, j] = column j).  Returns
    (Q, R, rank, perm): Q[b, j] = column j of Q_R (j < rank, else zero), R[b, j]
    = column j of R_piv (upper triangle, gathered from the kernel's physical
    columns), perm (B, T) the pivot order."""
    B, T, _ = M.shape
    Mw = M.to(torch.float64).contiguous().clone()
    Q = torch.empty_like(Mw)
    rank = torch.empty(B, dtype=torch.int32, device=M.device)
    perm = torch.empty(B, T, dtype=torch.int32, device=M.device)
    work = torch.empty(max(B * T, 1), dtype=torch.float64, device=M.device)
    dims = dims.to(device=M.device, dtype=torch.int32).contiguous()
    fn = _lib.lib().kr_qrcp_small_cluster if QRCP_CLUSTER else _lib.lib().kr_qrcp_small
    _lib.check(fn(Mw.data_ptr(), dims.data_ptr(), B, T, float(rtol), Q.data_ptr(), rank.data_ptr(), perm.data_ptr(),
                  work.data_ptr(), work.numel(), _lib.stream_ptr()), "kr_qrcp_small")
    _lib.note_launch("kr_qrcp_small")
    idx = perm.clamp_min(0).long()
    R = torch.gather(Mw, 1, idx.unsqueeze(2).expand(B, T, T))
    return Q, R, rank, perm


def gram(A: torch.Tensor, Bm: torch.Tensor | None = None) -> torch.Tensor:
    """(B, T, T) with G[b, i, j] = A[b, i] . Bm[b, j] for row blocks (B, T, n):
    kr_gram (split-K over n, fixed-order partial sums) for long rows, bmm else."""
    Bm = A if Bm is None else Bm
    B, T, n = A.shape
    if n < 4096 or B == 0 or T == 0:
        return A @ Bm.transpose(1, 2)
    A = A.contiguous()
    Bm = Bm.contiguous()
    G = torch.empty(B, T, T, dtype=torch.float64, device=A.device)
    L = _lib.lib()
    wl = int(L.kr_gram_workspace(B, T, n))
    ws = torch.empty(max(wl, 1), dtype=torch.float64, device=A.device)
    _lib.check(L.kr_gram(A.data_ptr(), Bm.data_ptr(), n, T * n, B, T, n, G.data_ptr(), T, T * T, ws.data_ptr(), wl,
                         _lib.stream_ptr()), "kr_gram")
    _lib.note_launch("kr_gram", 2)
    return G


QRCP_TMAX = 640  # KR_TMAX (kr_qrcp_small_cluster)
PIVOT_COND = 1e9   # below this cond(A) bound pivoted QR keeps every column (|R_kk| ~ sigma_k > 1e-10 |R_00|)

CHOLQR_TOL = 1e-7   # recycling.CHOLQR_TOL
COND_SCREEN = 1e6   # recycling.COND_SCREEN
COND_LIMIT = 1e12   # recycling.COND_LIMIT


def _row_mask(dims, T: int, device) -> torch.Tensor:
    d = torch.as_tensor(dims, device=device).reshape(-1, 1)
    return (torch.arange(T, device=device).reshape(1, -1) < d).to(torch.float64)


def _identity_pad(G: torch.Tensor, mask: torch.Tensor) -> torch.Tensor:
    """G with the pad rows/columns replaced by those of the identity."""
    return G * (mask.unsqueeze(2) * mask.unsqueeze(1)) + torch.diag_embed(1.0 - mask)


def _masked_extrema(d: torch.Tensor, mask: torch.Tensor):
    live = mask > 0
    big = torch.finfo(d.dtype).max
    return torch.where(live, d, -big).amax(1), torch.where(live, d, big).amin(1)


CHOL_TMAX = 640          # KR_TMAX: kr_chol_inv (shared memory to 228, an L2-resident workspace above)
SKIP_DEPENDENT = False   # remove dependent rows inside the Cholesky passes (kr_chol_inv skip mode)
SHIFTED_COND_MAX = 1e14  # shifted CholeskyQR3 is backward stable below ~1/u; keep a margin


def _chol_inv(G: torch.Tensor, dims: torch.Tensor, scale: bool, shift: torch.Tensor | None = None,
              inverse: bool = True, skip: bool = False):
    """Per sample: D = sqrt(diag G) (scale) or 1, G_s = D^-1 G D^-1 + shift I on the
    leading dims[b] block, G_s = L L^T.  Returns (F, info, stats): F = L^-1 D^-1
    (row-major, identity pad; None unless inverse), info[b] = first failing row or
    -1, stats[b] = (min L_jj, max L_jj, min D).  kr_chol_inv (one CTA per matrix)
    for T <= KR_TMAX (640), torch.linalg otherwise.  skip=True (kernel only): dependent rows
    are removed instead of failing; returns a 4th value, the (B, T) removed mask
    (None on the torch path, which reports the first failing row instead)."""
    B, T, _ = G.shape
    dev = G.device
    dims = dims.to(device=dev, dtype=torch.int32).contiguous()
    if T <= CHOL_TMAX:
        G = G.contiguous()
        F = torch.empty_like(G) if inverse else None
        stats = torch.empty(B, 4, dtype=torch.float64, device=dev)
        info = torch.empty(B, dtype=torch.int32, device=dev)
        skipped = torch.empty(B, T, dtype=torch.uint8, device=dev) if skip else None
        sh = None if shift is None else shift.to(torch.float64).contiguous()
        flags = int(scale) | (2 if inverse else 0) | (4 if skip else 0)
        L = _lib.lib()
        wl = int(L.kr_chol_inv_workspace(B, T))
        ws = torch.empty(max(wl, 1), dtype=torch.float64, device=dev)
        _lib.check(L.kr_chol_inv(G.data_ptr(), T, T * T, dims.data_ptr(), B, T, flags,
                                 0 if sh is None else sh.data_ptr(), 0 if F is None else F.data_ptr(),
                                 T, T * T, stats.data_ptr(), info.data_ptr(),
                                 0 if skipped is None else skipped.data_ptr(), ws.data_ptr(), wl,
                                 _lib.stream_ptr()), "kr_chol_inv")
        _lib.note_launch("kr_chol_inv")
        if skip:
            return F, info, stats, skipped.bool()
        return F, info, stats
    mask = _row_mask(dims, T, dev)
    live = mask > 0
    g = G.diagonal(dim1=1, dim2=2)
    D = torch.where(live & (g > 0), g.clamp_min(0.0).sqrt(), torch.ones_like(g)) if scale else torch.ones_like(g)
    Gs = _identity_pad(0.5 * (G + G.transpose(1, 2)) / (D.unsqueeze(2) * D.unsqueeze(1)), mask)
    if shift is not None:
        Gs = Gs + shift.reshape(-1, 1, 1) * torch.diag_embed(mask)
    L, inf = torch.linalg.cholesky_ex(Gs)
    info = torch.where(inf > 0, inf - 1, torch.full_like(inf, -1)).to(torch.int32)
    # kr_chol_inv's breakdown rule: a pivot L_jj^2 <= 4 t eps Gs_jj is a dependent row
    piv_rtol = 4.0 * dims.to(torch.float64).reshape(-1, 1) * torch.finfo(torch.float64).eps
    tiny = (L.diagonal(dim1=1, dim2=2) ** 2 <= piv_rtol * Gs.diagonal(dim1=1, dim2=2)) & live
    first_tiny = torch.where(tiny, torch.arange(T, device=dev).reshape(1, -1), T).amin(1).to(torch.int32)
    info = torch.where((first_tiny < T) & ((info < 0) | (first_tiny < info)), first_tiny, info)
    hi, lo = _masked_extrema(L.diagonal(dim1=1, dim2=2), mask)
    dmin = torch.where(live, g.clamp_min(0.0).sqrt(), torch.full_like(g, 1e308)).amin(1) if scale \
        else torch.ones_like(lo)
    stats = torch.stack([lo, hi, dmin, torch.zeros_like(lo)], dim=1)
    stats[:, :3] = torch.where((dims > 0).reshape(-1, 1), stats[:, :3], torch.ones_like(stats[:, :3]))
    F = None
    if inverse:
        eye = torch.eye(T, dtype=G.dtype, device=dev).expand(B, T, T)
        F = torch.linalg.solve_triangular(L, eye, upper=False) / D.unsqueeze(1)
    if skip:
        return F, info, stats, None
    return F, info, stats


def cholqr2_rows(A: torch.Tensor, mask: torch.Tensor, robust: bool = False, want_f: bool = True):
    """Orthonormalise rows [0, t_b) of A (B, T, n) (pad rows zero) by two
    Cholesky-QR passes, the first on the row-scaled block (recycling._cholqr2).

    Returns (Q, F, ok): Q = F @ A with orthonormal live rows and zero pad rows;
    F = R^{-T} for the column form A_col = Q_col R (so |R_jj| = 1 / |F_jj|); ok[b]
    is False where the block is too ill-conditioned or rank deficient.  With
    want_f=False, F is replaced by its diagonal (B, T).

    robust=True: samples CholQR2 declines are redone as shifted CholeskyQR3
    (Fukaya, Kannan, Nakatsukasa, Zhang, Yamamoto, SIAM J. Sci. Comput. 2020: a
    first pass on G + sigma I, sigma = 11 (n t + t(t+1)) u ||A_s||^2, then CholQR2),
    backward stable up to cond ~ 1/u; declined only when the bound
    cond(A) <= ||A||_F ||R^{-1}||_F exceeds SHIFTED_COND_MAX.  Also returns the
    first row where a Cholesky broke down (-1 if none)."""
    B, T, n = A.shape
    dims = mask.sum(1).to(torch.int32)
    G = gram(A)
    F1, i1, st = _chol_inv(G, dims, scale=True)
    ok1 = (i1 < 0) & (st[:, 0] > CHOLQR_TOL * st[:, 1]) & (st[:, 2] > 0)
    shifted = robust and not bool(ok1.all())
    if shifted and STATS is not None:
        STATS["shifted"] = STATS.get("shifted", 0) + 1
    if shifted:
        tb = dims.to(torch.float64)  # ||A_s||_2^2 <= ||A_s||_F^2 = t_b after row scaling
        sigma = 11.0 * (n * tb + tb * (tb + 1)) * torch.finfo(A.dtype).eps * tb
        F1, i1, _ = _chol_inv(G, dims, scale=True, shift=torch.where(ok1, torch.zeros_like(sigma), sigma))
    Q = F1 @ A
    ok = i1 < 0
    fail_row = i1.clone()
    Fs = [F1]
    skipped = None
    for _ in range(2 if shifted else 1):
        # (skip mode stays off: the breakdown test of a pass behind a shifted pass
        # fires ~30x above the reference's pivoted-QR drop threshold)
        out = _chol_inv(gram(Q), dims, scale=False, skip=robust and SKIP_DEPENDENT)
        Fk, ik = out[0], out[1]
        if len(out) > 3 and out[3] is not None:
            skipped = out[3] if skipped is None else skipped | out[3]
        Q = Fk @ Q
        Fs.append(Fk)
        fail_row = torch.where((fail_row < 0) & (ik >= 0), ik, fail_row)
        ok = ok & (ik < 0)
    if want_f or shifted:
        F = Fs[0]
        for Fk in Fs[1:]:
            F = Fk @ F
    if shifted:
        cond_bound = torch.linalg.vector_norm(A, dim=(1, 2)) * torch.linalg.matrix_norm(F)
        ok = ok & (ok1 | (cond_bound <= SHIFTED_COND_MAX))
    else:
        ok = ok & ok1
    if not want_f:
        F = Fs[0].diagonal(dim1=1, dim2=2)
        for Fk in Fs[1:]:
            F = F * Fk.diagonal(dim1=1, dim2=2)
    if robust:
        return Q, F, ok, fail_row, skipped
    return Q, F, ok


def _compact_rows(A: torch.Tensor, keep: torch.Tensor):
    """Move the kept rows of every sample to the front (order preserved), zero the rest."""
    B, T, n = A.shape
    ar = torch.arange(T, device=A.device).expand(B, T)
    order = torch.argsort(torch.where(keep, ar, ar + T), dim=1, stable=True)
    out = torch.gather(A, 1, order.unsqueeze(2).expand(B, T, n))
    cnt = keep.sum(1)
    out = out * (ar < cnt.unsqueeze(1)).unsqueeze(2).to(A.dtype)
    return out, cnt


def orth_rows_drop(A: torch.Tensor, dims: list[int], rounds: int = 8):
    """Candidate basis with the reference's rank drop, batched: (W, dims_after, ok).

    recycling._orth_drop removes the rows (columns of the n x t block) whose
    unpivoted |R_jj| <= RANK_TOL max |R_ii| and redoes the QR.  Here one (shifted)
    Cholesky-QR removes the numerically dependent rows inside its second and third
    passes (kr_chol_inv's skip mode: the factor of the Gram without those rows), and
    rows with |R_jj| <= RANK_TOL max |R_ii| in the result are removed too; the kept
    rows of W are compacted to the front.  A removed row's own direction in W is
    below RANK_TOL relative, so no re-factorization is needed.  (On the torch path,
    T > 228, a breakdown row is removed and the QR redone, up to `rounds` times.)"""
    from .recycling import RANK_TOL

    B, T, _ = A.shape
    mask = _row_mask(dims, T, A.device)
    ar = torch.arange(T, device=A.device).reshape(1, -1)
    for _ in range(rounds):
        W, Fd, ok, fail_row, skipped = cholqr2_rows(A, mask, robust=True, want_f=False)
        live = mask > 0
        keep_live = live if skipped is None else live & ~skipped
        rd = 1.0 / Fd.abs()
        rmax, _ = _masked_extrema(rd, keep_live.to(rd.dtype))
        factored = (fail_row < 0) & torch.isfinite(rmax)
        drop = keep_live & (rd <= RANK_TOL * rmax.unsqueeze(1)) & factored.unsqueeze(1)
        if skipped is not None:
            drop = drop | (live & skipped)
        refactor = live & (ar == fail_row.unsqueeze(1))
        if not bool((drop | refactor).any()):
            return W, dims, ok
        if STATS is not None:
            STATS["drop_rounds"] = STATS.get("drop_rounds", 0) + 1
            STATS["dropped_rows"] = STATS.get("dropped_rows", 0) + int((drop | refactor).sum())
        if skipped is not None and not bool(refactor.any()):
            # skip-mode drops only: compact W itself (dropped directions are negligible)
            W, cnt = _compact_rows(W, live & ~drop)
            return W, cnt.cpu().tolist(), ok
        A, cnt = _compact_rows(A, live & ~(drop | refactor))
        dims = cnt.cpu().tolist()
        mask = _row_mask(dims, T, A.device)
    W, _, ok, _, _ = cholqr2_rows(A, mask, robust=True, want_f=False)
    return W, dims, ok


def orth_rows(A: torch.Tensor, dims: list[int]):
    """Candidate basis W = orth(A rows) with the reference's pivoted-QR rank drop
    (recycling.py:187-199), batched: (W, dims_after, ok).

    Every sample first goes through (shifted) Cholesky QR.  Where the block may be
    numerically rank deficient -- cond(A) <= ||A||_F ||R^{-1}||_F above PIVOT_COND,
    or Cholesky QR not applicable -- the pivoted QR of the reference is reproduced:
    pivoted QR of A is Q_A times pivoted QR of the small R factor, so
    kr_qrcp_small runs on R (from the Cholesky QR, or from a Householder QR of the
    sample when shifted CholeskyQR3 cannot be trusted) and the kept basis is
    Q_A Q_R[:, :r] with the reference's |R_kk| > 1e-10 |R_00| rule."""
    from .recycling import RANK_TOL

    B, T, n = A.shape
    if T > QRCP_TMAX:
        return orth_rows_drop(A, dims)
    dev = A.device
    mask = _row_mask(dims, T, dev)
    W, F, ok, _, _ = cholqr2_rows(A, mask, robust=True)
    cond_bound = torch.linalg.vector_norm(A, dim=(1, 2)) * torch.linalg.matrix_norm(F)
    ill = ~ok | (cond_bound > PIVOT_COND)
    ill_h, ok_h = ill.cpu().tolist(), ok.cpu().tolist()
    idx = [b for b in range(B) if ill_h[b] and dims[b] > 0]
    if not idx:
        return W, dims, torch.ones_like(ok)
    if STATS is not None:
        STATS["pivoted"] = STATS.get("pivoted", 0) + len(idx)
    ii = torch.tensor(idx, device=dev)
    Wsub = W[ii].clone()
    M = gram(A[ii], Wsub)  # M[j][i] = a_j . q_i = R[i][j]: R column-major
    for s_, b in enumerate(idx):
        if not ok_h[b]:  # Householder QR where shifted CholeskyQR3 is not trustworthy
            Qh, Rh = torch.linalg.qr(A[b, : dims[b]].T)
            Wsub[s_] = 0.0
            Wsub[s_, : dims[b]] = Qh.T
            M[s_] = 0.0
            M[s_, : dims[b], : dims[b]] = Rh.T
            if STATS is not None:
                STATS["householder"] = STATS.get("householder", 0) + 1
    Qr, _, rank, _ = qrcp_small(M, torch.tensor([dims[b] for b in idx], dtype=torch.int32), RANK_TOL)
    W[ii] = Qr @ Wsub  # rows j < rank: Q_A Q_R[:, j]; the rest zero
    dims = list(dims)
    for s_, r in zip(idx, rank.cpu().tolist()):
        if STATS is not None and r < dims[s_]:
            STATS["dropped_rows"] = STATS.get("dropped_rows", 0) + dims[s_] - r
        dims[s_] = r
    return W, dims, torch.ones_like(ok)


def supports(strategy, native: bool = False) -> bool:
    """Strategies the whole-batch update computes to the reference's accuracy.

    RGen takes its vectors from the eigenpairs of Q1^T Q1 (alpha^2), which are as
    accurate as the reference's SVD of Q1 for alpha near 1 -- the largest mu,
    size L -- but square the gaps between small alpha (sizes S, M); those stay on
    the per-sample SVD path.  Ritz uses eigh(W^T H W) exactly as the reference.
    Harmonic Ritz (harmonic_ritz_select, recycling.py:239-272) and inner placement
    (:409-415) run in the native orchestrator only (Cholesky reduction of the pencil;
    the previous system's operator as op_proj, kr_recycle_update)."""
    if strategy.placement != "outer" and not native:
        return False  # inner placement (recycling.py:409-415): the native orchestrator only
    if strategy.vec_type == "HRitz":
        return native
    return strategy.vec_type == "Ritz" or (strategy.vec_type == "RGen" and strategy.size == "L")


def recycle_update(strategy, s: int, H, J, bases, recycles, reuse_products: bool = True):
    """``next_recycle`` (recycling.py:386-465) for every sample of a batch at once.

    Outer placement, vector types RGen (``rgen_select`` :316-359 + ``gsvd_pair``
    :275-313) and Ritz (``ritz_select`` :226-236); H, J are the batched operators of
    the upcoming system; bases[b] is the previous Lanczos basis (n x k_b) and
    recycles[b] the previous RecycleSpace of sample b.  Returns one RecycleSpace per
    sample, or None where the batched path declines -- CholQR2 conditioning, the
    Hessian-condition screen (recycling._hessian_condition), t_b > EIG_TMAX -- and
    the caller runs the per-sample path of ``recycling.next_recycle`` instead.

    Candidate order is the reference's [V_prev, U_prev]; every downstream quantity
    depends on the candidate span only (exact arithmetic)."""
    import warnings

    from .recycling import RecycleSpace
    from .stopping import NscData

    if not supports(strategy, native=True):
        raise ValueError(f"the batched recycle update covers outer RGen-L / Ritz / HRitz, not {strategy}")
    B = len(bases)
    n = H.dim
    k = [0 if V is None else int(V.shape[1]) for V in bases]
    sp = [0 if r is None else int(r.dim) for r in recycles]
    t = [a + c for a, c in zip(k, sp)]
    T = max(t) if t else 0
    if T == 0 or s == 0:
        return [RecycleSpace.empty(n) for _ in range(B)]
    if T > EIG_TMAX:
        return [None] * B
    if any(s > tb > 0 for tb in t):
        warnings.warn(f"requested {s} recycle vectors but only {min(tb for tb in t if tb > 0)} candidates; "
                      "clamping", stacklevel=3)
    dev = H.model.y.device if getattr(H, "model", None) is not None else bases[0].device
    A = torch.zeros(B, T, n, dtype=torch.float64, device=dev)
    for b in range(B):
        if k[b]:
            A[b, : k[b]] = bases[b].T
        if sp[b]:
            A[b, k[b]: t[b]] = recycles[b].U.T
    # candidate basis W = orth([V_prev, U_prev]) with the rank drop (recycling.py:187-199)
    W, t, ok = orth_rows(A, t)
    mask = _row_mask(t, T, dev)
    tt = torch.tensor(t, dtype=torch.int32, device=dev)
    checks = {"candidates": ok}
    HW = H.apply_matrix(W.transpose(1, 2)).transpose(1, 2)          # (B, T, n)
    Ht = gram(W, HW)
    Ht = 0.5 * (Ht + Ht.transpose(1, 2))                            # _sym(W^T H W)
    mu = VH = None
    if strategy.vec_type == "Ritz":
        _, Z, nsel = syev_select(Ht, tt, strategy.size, s)
        coeffs = Z
    else:
        Jt = J.apply_adjoint_matrix(W.transpose(1, 2)).transpose(1, 2)  # (B, T, p): row j = J w_j
        p = Jt.shape[2]
        # _hessian_condition: Cholesky-pivot screen, exact extreme eigenvalues where it fails
        # Ht = L L^T: (max L_jj / min L_jj)^2 <= cond(Ht) <= ||Ht||_F ||L^-1||_F^2 brackets the
        # condition number; the exact extreme eigenvalues are needed only when the
        # reference's limit falls inside the bracket
        Fh, ih, hst = _chol_inv(Ht, tt, scale=False, inverse=True)
        cond_ub = torch.linalg.matrix_norm(Ht) * torch.linalg.matrix_norm(Fh) ** 2
        screen = (ih < 0) & (hst[:, 0] > 0) & (cond_ub < COND_LIMIT)
        if not bool(screen.all()):
            ext, _, _ = syev_select(Ht, tt, "M", 2)
            lo_, hi_ = ext[:, 0], ext[:, -1]
            # all eigenvalues are in [lo_, hi_]; |.| extremes as in the reference
            smax = torch.maximum(lo_.abs(), hi_.abs())
            exact_ok = (lo_ > 0) & (lo_ >= COND_LIMIT ** -1 * smax)
            screen = screen | exact_ok
        checks["cond_screen"] = screen
        ok = ok & screen
        # gsvd_pair: [Jt; Ht] = Q R, Z from Q1^T Q1, alpha/beta as column norms
        QS, FS, okS = cholqr2_rows(torch.cat([Jt, Ht], dim=2), mask)
        checks["gsvd_qr"] = okS
        ok = ok & okS
        Q1 = QS[:, :, :p]
        _, Z, nsel = syev_select(Q1 @ Q1.transpose(1, 2), tt, strategy.size, s)
        Y = Z @ QS                                                  # (B, s, p + T)
        alpha = torch.linalg.vector_norm(Y[..., :p], dim=2).clamp(0.0, 1.0)
        beta = torch.linalg.vector_norm(Y[..., p:], dim=2)
        ok = ok & ((beta > 0) | (torch.arange(s, device=dev).reshape(1, -1) >= nsel.reshape(-1, 1))).all(1)
        beta_safe = torch.where(beta > 0, beta, torch.ones_like(beta))
        mu = alpha / beta_safe
        VH = Y[..., p:] / beta_safe.unsqueeze(2)                    # rows = V_H columns
        X = Z @ FS                                                  # rows = R^{-1} z
        coeffs = {"R": X, "L": VH, "M": None}[strategy.side]
    if coeffs is None:  # side M: normalised mean of both candidate sets, H applied explicitly
        cand = 0.5 * (VH @ W + X @ W)
        nr = torch.linalg.vector_norm(cand, dim=2, keepdim=True)
        cand = cand / torch.where(nr > 0, nr, torch.ones_like(nr))
        HU = H.apply_matrix(cand.transpose(1, 2)).transpose(1, 2)
    else:
        cand = coeffs @ W
        HU = coeffs @ HW if reuse_products else H.apply_matrix(cand.transpose(1, 2)).transpose(1, 2)
    # prepare_recycle (recycling.py:362-383): H U~ = C R, U = U~ R^{-1}
    smask = _row_mask(nsel, s, dev)
    C, Fu, okU = cholqr2_rows(HU, smask)
    U = Fu @ cand
    checks["prepare_qr"] = okU
    ok = ok & okU
    Znsc = None if mu is None else (mu.unsqueeze(2) * VH) @ W        # rows of W V_H diag(mu)
    ok_h = ok.cpu().tolist()
    if STATS is not None:
        for name, flag in checks.items():
            STATS[name] = STATS.get(name, 0) + int((~flag).sum())
        STATS["declined"] = STATS.get("declined", 0) + sum(1 for b in range(B) if not ok_h[b])
        STATS["samples"] = STATS.get("samples", 0) + B
    nsel_h = nsel.cpu().tolist()
    out = []
    for b in range(B):
        sb = nsel_h[b]
        if t[b] == 0 or sb == 0:
            out.append(RecycleSpace.empty(n))
            continue
        if not ok_h[b]:
            out.append(None)
            continue
        nsc = None
        if mu is not None:
            nsc = NscData(values=mu[b, :sb], v_h=VH[b, :sb, : t[b]].T, w=W[b, : t[b]].T, z=Znsc[b, :sb].T)
        out.append(RecycleSpace(U=U[b, :sb].T, C=C[b, :sb].T, nsc_data=nsc, orthonormal=True))
    return out


NATIVE_TMAX = 640  # KR_TMAX


def _uniform_rows(mats, n, dev):
    """(ptr, ld, bs, keep) describing the n x k_b column blocks `mats` as one strided
    batch when they already are one (views of the same solver buffer), else a copy."""
    live = [(b, m) for b, m in enumerate(mats) if m is not None and m.shape[1] > 0]
    if not live:
        return 0, n, 0, None
    ok = all(m.stride(0) == 1 and (m.shape[1] <= 1 or m.stride(1) == n) for _, m in live)
    if ok and len(live) > 1:
        (b0, m0), (b1, m1) = live[0], live[1]
        bs = (m1.data_ptr() - m0.data_ptr()) // 8 // max(b1 - b0, 1)
        ok = bs > 0 and all(m.data_ptr() == m0.data_ptr() + (b - b0) * bs * 8 for b, m in live)
        if ok:
            return m0.data_ptr() - b0 * bs * 8, n, bs, None
    if ok and len(live) == 1:
        b0, m0 = live[0]
        return m0.data_ptr() - b0 * n * 8 * max(m0.shape[1], 1), n, n * max(m0.shape[1], 1), None
    kmax = max(m.shape[1] for _, m in live)
    buf = torch.zeros(len(mats), kmax, n, dtype=torch.float64, device=dev)
    for b, m in live:
        buf[b, : m.shape[1]] = m.T
    return buf.data_ptr(), n, kmax * n, buf


def _scratch(cache, key, numel, dev):
    """Grow-only device scratch kept in `cache` (per sample group: always used on the
    group's stream, ordered across steps by the caller's stream joins)."""
    if cache is None:
        return torch.empty(max(numel, 1), dtype=torch.float64, device=dev)
    buf = cache.get(key)
    if buf is None or buf.numel() < numel:
        cache[key] = None
        buf = cache[key] = torch.empty(max(numel, 1), dtype=torch.float64, device=dev)
    return buf


def recycle_update_native(strategy, s: int, H, J, bases, recycles, reuse_products: bool = True,
                          scratch: dict | None = None, out: tuple | None = None, out_src: tuple | None = None,
                          H_proj=None, J_proj=None):
    """``recycle_update`` through the native orchestrator ``kr_recycle_update`` (one
    C-ABI call per batch: no Python per-op overhead, no GIL); same contract and
    results.  Falls back to ``recycle_update`` beyond the kernels' t <= KR_TMAX (640).
    ``scratch`` (optional, one dict per stream) keeps the temporaries -- H W and the
    orchestrator's workspace -- across calls instead of reallocating them.  ``out``
    (optional): (U, C, Z) row blocks (B, s, n) to write into -- slices of whole-batch
    buffers, so the solve reads every sample's recycle space in place."""
    from .recycling import RecycleSpace
    from .stopping import NscData

    if not supports(strategy, native=True):
        raise ValueError(f"the batched recycle update covers outer RGen-L / Ritz / HRitz, not {strategy}")
    B = len(bases)
    n = H.dim
    k = [0 if V is None else int(V.shape[1]) for V in bases]
    sp = [0 if r is None else int(r.dim) for r in recycles]
    t = [a + c for a, c in zip(k, sp)]
    T = max(t) if t else 0
    if T == 0 or s == 0:
        return [RecycleSpace.empty(n) for _ in range(B)]
    inner = strategy.placement != "outer"
    if inner and H_proj is None:
        raise ValueError("inner placement needs the previous system's operator (H_proj)")
    if T > NATIVE_TMAX or s > T:
        if strategy.vec_type == "HRitz" or inner:  # not in the torch batched path: per-sample path
            return [None] * B
        return recycle_update(strategy, s, H, J, bases, recycles, reuse_products)
    dev = H.model.y.device if getattr(H, "model", None) is not None else bases[0].device
    vptr, ldv, bsv, vkeep = _uniform_rows(list(bases), n, dev)
    uptr, ldu, bsu, ukeep = _uniform_rows([None if r is None else r.U for r in recycles], n, dev)
    a = _lib.KrRecycleArgs()
    a.batch, a.T, a.s = B, T, s
    a.vec_type = {"Ritz": 0, "RGen": 1, "HRitz": 2}[strategy.vec_type]
    a.size_code = SIZE_CODES[strategy.size]
    a.side = {"R": 0, "L": 1, "M": 2}.get(strategy.side or "R", 0)
    a.reuse_products = int(reuse_products)
    a.V, a.ld_v, a.bs_v = vptr, ldv, bsv
    a.Uprev, a.ld_u, a.bs_u = uptr, ldu, bsu
    if inner:
        # J W of the GSVD uses the previous Jacobian: same kr_op as H_proj (one prepare serves both)
        a.op_proj = ctypes.addressof(H_proj.op)
    kd = np.asarray(k, dtype=np.int32)
    sd = np.asarray(sp, dtype=np.int32)
    td = np.zeros(B, dtype=np.int32)
    ns = np.zeros(B, dtype=np.int32)
    stt = np.zeros(B, dtype=np.int32)
    a.kdims, a.sdims = kd.ctypes.data, sd.ctypes.data
    a.tdims, a.nsel, a.status = td.ctypes.data, ns.ctypes.data, stt.ctypes.data
    f64 = dict(dtype=torch.float64, device=dev)
    # buffers sized for the largest candidate width the caller expects (scratch["tcap"]),
    # so growing T never reaches the device allocator inside a step
    tcap = min(max(T, int(scratch.get("tcap", 0)) if scratch is not None else 0), NATIVE_TMAX)
    W = torch.empty(B * tcap * n, **f64)[: B * T * n].view(B, T, n)
    HW = _scratch(scratch, "hw", B * tcap * n, dev)
    if out is not None:
        U, C, Z = out
        if Z is None:
            Z = torch.empty(B, s, n, **f64)
    else:
        U = torch.empty(B, s, n, **f64)
        C = torch.empty(B, s, n, **f64)
        Z = torch.empty(B, s, n, **f64)
    mu = torch.zeros(B, s, **f64)
    VH = torch.zeros(B, s, T, **f64)
    a.W, a.HW, a.U, a.C = W.data_ptr(), HW.data_ptr(), U.data_ptr(), C.data_ptr()
    a.mu, a.VH, a.Z = mu.data_ptr(), VH.data_ptr(), Z.data_ptr()
    L = _lib.lib()
    a.T = tcap
    wcap = int(L.kr_recycle_workspace(ctypes.byref(H.op), ctypes.byref(a)))
    a.T = T
    wl = int(L.kr_recycle_workspace(ctypes.byref(H.op), ctypes.byref(a)))
    if wl < 0 or wcap < 0:
        _lib.check(-1, "kr_recycle_workspace")
    ws = _scratch(scratch, "ws", max(wl, wcap), dev)
    _lib.check(L.kr_recycle_update(ctypes.byref(H.op), ctypes.byref(a), ws.data_ptr(), ws.numel(),
                                   _lib.stream_ptr()), "kr_recycle_update")
    _lib.note_launch("kr_recycle_update", 40)
    del vkeep, ukeep
    if STATS is not None:
        STATS["declined"] = STATS.get("declined", 0) + int((stt == 1).sum())
        STATS["samples"] = STATS.get("samples", 0) + B
    res = []
    for b in range(B):
        tb, sb = int(td[b]), int(ns[b])
        if stt[b] == 2 or tb == 0 or sb == 0:
            res.append(RecycleSpace.empty(n))
        elif stt[b] == 1:
            res.append(None)
        else:
            nsc = None
            if strategy.vec_type == "RGen":
                nsc = NscData(values=mu[b, :sb], v_h=VH[b, :sb, :tb].T, w=W[b, :tb].T, z=Z[b, :sb].T)
            src = None if out_src is None else (out_src[0], out_src[1], out_src[2], out_src[3] + b) + tuple(out_src[4:])
            res.append(RecycleSpace(U=U[b, :sb].T, C=C[b, :sb].T, nsc_data=nsc, orthonormal=True, batch_src=src))
    return res
