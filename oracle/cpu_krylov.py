"""CPU restatement of MINRES / RMINRES / CG (TEST ORACLE ONLY).

Follows ``/root/reference/pkg/src/krecycle/krylov.py``:
* RMINRES = Alg. 3 with the corrected sign ``w += c_k zeta_{k-1} (vt - bt)``
  (krylov.py:11-15, 326-338);
* breakdown tolerance 1e-13 ||g|| (krylov.py:50, 237); stop test before the
  breakdown test (krylov.py:369-374); r0 = g - H w0 even for w0 = 0 (:224);
* the 5-vector residual recurrence (krylov.py:154-181), enabled whenever the
  stop rule needs the residual vector (:214-215);
* the closed-form FLOP model (krylov.py:119-135), charged at the same sites.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

BREAKDOWN_RTOL = 1e-13


class NonSPDError(RuntimeError):
    """krylov.py:53-54"""


class ResidualRule:
    """||r_k|| < delta, strict (stopping.py:93-99)."""

    kind = "res"
    needs_residual_vector = False

    def __init__(self, delta: float):
        if not delta > 0:
            raise ValueError(f"tolerance must be positive, got {delta}")
        self.delta = float(delta)

    def value(self, res_norm, r):
        return float(res_norm)

    def done(self, v) -> bool:
        return v < self.delta


@dataclass
class Options:
    """krylov.py:57-82"""

    max_iter: int = 500
    initial_guess: np.ndarray | None = None
    stop_rule: object = None
    track_basis: bool = False
    track_residual_vector: bool = False
    reorthogonalize: bool = False
    collect_states: bool = False
    collect_iterates: bool = False
    collect_residual_history: bool = False

    def __post_init__(self):
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")

    def rule(self):
        return self.stop_rule if self.stop_rule is not None else ResidualRule(1e-2)


@dataclass
class Result:
    """krylov.py:102-116"""

    solution: np.ndarray
    iterations: int
    residual_norms: np.ndarray
    flops: int
    stop_reason: str
    stop_values: np.ndarray
    basis: np.ndarray | None = None
    residual_vector: np.ndarray | None = None
    states: list | None = None
    iterates: list | None = None
    residual_history: list | None = None


def flops_minres(k: int, n: int, h: int) -> int:
    _nonneg(k=k, n=n, h=h)
    return h + 4 * n + k * (h + 16 * n)


def flops_rminres(k: int, n: int, s: int, h: int) -> int:
    _nonneg(k=k, n=n, s=s, h=h)
    return h + 4 * n + 6 * n * s + k * (h + 21 * n + 6 * n * s - s)


def flops_cg(k: int, n: int, h: int) -> int:
    _nonneg(k=k, n=n, h=h)
    return h + 3 * n + k * (h + 10 * n)


def _nonneg(**kw):
    for name, val in kw.items():
        if val < 0:
            raise ValueError(f"{name} must be nonnegative, got {val}")


def rminres_core(H, g, U, C, opts: Options) -> Result:
    """krylov.py:205-383."""
    n = H.dim
    g = np.asarray(g, dtype=float)
    if g.shape != (n,):
        raise ValueError(f"right-hand side of shape {g.shape}, operator dim {n}")
    if not np.all(np.isfinite(g)):
        raise ValueError("right-hand side contains non-finite entries")
    s = 0 if U is None else U.shape[1]
    rule = opts.rule()
    track = opts.track_residual_vector or rule.needs_residual_vector
    hc = H.apply_cost
    flops = 0

    w = np.zeros(n) if opts.initial_guess is None else np.array(opts.initial_guess, dtype=float)
    r = g - H(w)
    flops += hc + n
    if s:
        proj = C.T @ r
        w = w + U @ proj
        r = r - C @ proj
        flops += 6 * n * s

    beta = float(np.linalg.norm(r))
    flops += 2 * n
    tol_bd = BREAKDOWN_RTOL * max(float(np.linalg.norm(g)), 1e-300)

    # residual recurrence state (krylov.py:163-181)
    r_vec = r.copy() if track else None
    hvt = [np.zeros(n), np.zeros(n)] if track else None  # (k-1, k-2)
    hbt = [np.zeros(n), np.zeros(n)] if track else None

    norms = [beta]
    svals = [rule.value(beta, r_vec if track else r)]
    basis = [] if opts.track_basis else None
    states = [] if opts.collect_states else None
    iterates = [w.copy()] if opts.collect_iterates else None
    hist = [r.copy()] if opts.collect_residual_history else None

    def finish(k, why):
        return Result(
            solution=w,
            iterations=k,
            residual_norms=np.asarray(norms),
            flops=flops,
            stop_reason=why,
            stop_values=np.asarray(svals),
            basis=None if basis is None else (np.column_stack(basis) if basis else np.zeros((n, 0))),
            residual_vector=None if r_vec is None else r_vec.copy(),
            states=states,
            iterates=iterates,
            residual_history=hist,
        )

    if rule.done(svals[0]):
        return finish(0, "tolerance")
    if beta <= tol_bd:
        return finish(0, "breakdown")

    v = r / beta
    flops += n
    v_old = np.zeros(n)
    zeta = beta
    c1, s1 = 1.0, 0.0  # rotation k-1
    c2, s2 = 0.0, 0.0  # rotation k-2
    vt1, vt2 = np.zeros(n), np.zeros(n)
    bt1, bt2 = (np.zeros(n), np.zeros(n)) if s else (None, None)
    why = "max_iter"
    k = 0
    for k in range(1, opts.max_iter + 1):
        hv = H(v)
        flops += hc
        if s:
            chv = C.T @ hv
            b = U @ chv
            cchv = C @ chv
            u = hv - cchv
            flops += (2 * n * s - s) + (2 * n * s - n) + (2 * n * s - n) + n
        else:
            b = cchv = None
            u = hv.copy()
        alpha = float(v @ u)
        u = u - alpha * v
        u = u - beta * v_old
        flops += 6 * n
        if opts.reorthogonalize and basis is not None:
            for q in basis:
                u -= (q @ u) * q
            if s:
                u -= C @ (C.T @ u)
        if basis is not None:
            basis.append(v)
        beta_new = float(np.linalg.norm(u))
        flops += 3 * n  # norm (2n) + the uniformly booked normalisation (n)
        broke = beta_new <= tol_bd
        if not broke:
            u = u / beta_new

        gamma = s2 * beta
        delta = c1 * c2 * beta + s1 * alpha
        eps = -s1 * c2 * beta + c1 * alpha
        eps_r = float(np.hypot(eps, beta_new))
        if eps_r == 0.0:
            if basis is not None:
                basis.pop()
            k -= 1
            why = "breakdown"
            break
        s_new = beta_new / eps_r
        c_new = eps / eps_r
        zeta_old = zeta
        zeta = -s_new * zeta_old

        vt = (v - gamma * vt2 - delta * vt1) / eps_r
        flops += 5 * n
        if s:
            bt = (b - gamma * bt2 - delta * bt1) / eps_r
            upd = vt - bt
            flops += 6 * n
        else:
            bt = None
            upd = vt
        step = c_new * zeta_old
        w = w + step * upd
        flops += 2 * n

        if track:
            hv_t = (hv - delta * hvt[0] - gamma * hvt[1]) / eps_r
            if cchv is None:
                diff = hv_t
                hbt = [hbt[1], hbt[0]]
            else:
                hb_t = (cchv - delta * hbt[0] - gamma * hbt[1]) / eps_r
                diff = hv_t - hb_t
                hbt = [hb_t, hbt[0]]
            hvt = [hv_t, hvt[0]]
            r_vec -= step * diff
        if states is not None:
            states.append(
                dict(alpha=alpha, beta=beta, beta_next=beta_new, gamma=gamma, delta=delta,
                     epsilon=eps, epsilon_rot=eps_r, givens=(c_new, s_new),
                     givens_prev=(c1, s1), givens_prev2=(c2, s2), zeta=zeta)
            )
        if iterates is not None:
            iterates.append(w.copy())
        if hist is not None:
            hist.append((r_vec if track else g - H(w)).copy())

        norms.append(abs(zeta))
        svals.append(rule.value(abs(zeta), r_vec if track else None))
        if rule.done(svals[-1]):
            why = "tolerance"
            break
        if broke:
            why = "breakdown"
            break
        v_old, v = v, u
        beta = beta_new
        c2, s2, c1, s1 = c1, s1, c_new, s_new
        vt2, vt1 = vt1, vt
        if s:
            bt2, bt1 = bt1, bt
    return finish(k, why)


def minres(H, g, opts: Options | None = None) -> Result:
    """krylov.py:386-388"""
    return rminres_core(H, g, None, None, opts or Options())


def rminres(H, g, recycle, opts: Options | None = None) -> Result:
    """krylov.py:391-405: empty space -> MINRES path; C^T C = I within 1e-8."""
    opts = opts or Options()
    if recycle is None or recycle.dim == 0:
        return rminres_core(H, g, None, None, opts)
    U, C = recycle.U, recycle.C
    if U.shape != C.shape or U.shape[0] != H.dim:
        raise ValueError(f"recycle space shapes U{U.shape} / C{C.shape} do not match operator dim {H.dim}")
    if np.max(np.abs(C.T @ C - np.eye(C.shape[1]))) > 1e-8:
        raise ValueError("recycle space violates C^T C = I beyond 1e-8")
    return rminres_core(H, g, U, C, opts)


def cg(H, g, opts: Options | None = None) -> Result:
    """krylov.py:408-483 (plain CG, NonSPDError on p^T H p <= 0)."""
    opts = opts or Options()
    n = H.dim
    g = np.asarray(g, dtype=float)
    rule = opts.rule()
    hc = H.apply_cost
    w = np.zeros(n) if opts.initial_guess is None else np.array(opts.initial_guess, dtype=float)
    r = g - H(w)
    rr = float(r @ r)
    flops = hc + 3 * n
    rn = float(np.sqrt(rr))
    norms, svals = [rn], [rule.value(rn, r)]
    basis = [] if opts.track_basis else None
    iterates = [w.copy()] if opts.collect_iterates else None
    why, k = "max_iter", 0
    if rule.done(svals[0]):
        why = "tolerance"
    else:
        p = r.copy()
        for k in range(1, opts.max_iter + 1):
            if basis is not None and rn > 0:
                basis.append(r / rn)
            hp = H(p)
            php = float(p @ hp)
            flops += hc + 2 * n
            if php <= 0:
                raise NonSPDError(f"curvature p^T H p = {php:g} <= 0 at iteration {k}; operator is not SPD")
            a = rr / php
            w = w + a * p
            r = r - a * hp
            rr_new = float(r @ r)
            flops += 8 * n
            rn = float(np.sqrt(rr_new))
            norms.append(rn)
            svals.append(rule.value(rn, r))
            if iterates is not None:
                iterates.append(w.copy())
            if rule.done(svals[-1]):
                why = "tolerance"
                break
            p = r + (rr_new / rr) * p
            rr = rr_new
    return Result(
        solution=w, iterations=k, residual_norms=np.asarray(norms), flops=flops,
        stop_reason=why, stop_values=np.asarray(svals),
        basis=None if basis is None else (np.column_stack(basis) if basis else np.zeros((n, 0))),
        residual_vector=r.copy(), iterates=iterates,
    )


def flops_rcg(k: int, n: int, s: int, h: int) -> int:
    """Deflated CG: cg's count (krylov.py:119-135 style) plus the deflation work,
    U^T r, C y, U y once (6ns) and C^T r, U mu per iteration (4ns); the s x s
    Cholesky solves are not counted (O(s^2), like the reference's omissions)."""
    _nonneg(k=k, n=n, s=s, h=h)
    return h + 3 * n + 6 * n * s + k * (h + 10 * n + 4 * n * s)


def rcg(H, g, recycle, opts: Options | None = None) -> Result:
    """Recycled (deflated) CG -- the "recycled CG" of BASELINE config 1; the
    reference ships only plain cg (krylov.py:408-483), so this restates the
    published algorithm: Saad, Yeung, Erhel & Guyomarc'h, "A deflated version of
    the conjugate gradient algorithm", SIAM J. Sci. Comput. 21 (2000), Alg. 2.2,
    with deflation space W = U of a RecycleSpace (C = H U, so W^T H W = U^T C and
    H W = C):

        x0 = x + U M^-1 U^T r,  r0 = r - C M^-1 U^T r   (M = U^T C; U^T r0 = 0)
        p0 = r0 - U M^-1 C^T r0
        a = r.r / p.Hp,  x += a p,  r -= a Hp
        p = r + (r_new.r_new / r.r) p - U M^-1 C^T r_new

    Conventions follow cg exactly (r = g - H w even for w = 0, the stop test on
    the new residual before the direction update, NonSPDError on p^T H p <= 0,
    basis = normalised residuals, which stay mutually orthogonal and orthogonal
    to U).  An empty recycle space is plain cg."""
    if recycle is None or recycle.dim == 0:
        return cg(H, g, opts)
    opts = opts or Options()
    n = H.dim
    g = np.asarray(g, dtype=float)
    U, C = np.asarray(recycle.U, dtype=float), np.asarray(recycle.C, dtype=float)
    s = U.shape[1]
    M = U.T @ C
    Lm = np.linalg.cholesky(0.5 * (M + M.T))

    def msolve(y):
        return np.linalg.solve(Lm.T, np.linalg.solve(Lm, y))

    rule = opts.rule()
    hc = H.apply_cost
    w = np.zeros(n) if opts.initial_guess is None else np.array(opts.initial_guess, dtype=float)
    r = g - H(w)
    y = msolve(U.T @ r)
    w = w + U @ y
    r = r - C @ y
    rr = float(r @ r)
    flops = hc + 3 * n + 6 * n * s
    rn = float(np.sqrt(rr))
    norms, svals = [rn], [rule.value(rn, r)]
    basis = [] if opts.track_basis else None
    iterates = [w.copy()] if opts.collect_iterates else None
    why, k = "max_iter", 0
    if rule.done(svals[0]):
        why = "tolerance"
    else:
        p = r - U @ msolve(C.T @ r)
        for k in range(1, opts.max_iter + 1):
            if basis is not None and rn > 0:
                basis.append(r / rn)
            hp = H(p)
            php = float(p @ hp)
            flops += hc + 2 * n
            if php <= 0:
                raise NonSPDError(f"curvature p^T H p = {php:g} <= 0 at iteration {k}; operator is not SPD")
            a = rr / php
            w = w + a * p
            r = r - a * hp
            rr_new = float(r @ r)
            flops += 8 * n + 4 * n * s
            rn = float(np.sqrt(rr_new))
            norms.append(rn)
            svals.append(rule.value(rn, r))
            if iterates is not None:
                iterates.append(w.copy())
            if rule.done(svals[-1]):
                why = "tolerance"
                break
            p = r + (rr_new / rr) * p - U @ msolve(C.T @ r)
            rr = rr_new
    return Result(
        solution=w, iterations=k, residual_norms=np.asarray(norms), flops=flops,
        stop_reason=why, stop_values=np.asarray(svals),
        basis=None if basis is None else (np.column_stack(basis) if basis else np.zeros((n, 0))),
        residual_vector=r.copy(), iterates=iterates,
    )
