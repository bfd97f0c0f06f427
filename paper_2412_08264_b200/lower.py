"""Lower-level reconstruction and the upper loop on the device (reference bilevel.py).

``lower_solve`` is the reference's L-BFGS with Armijo backtracking
(bilevel.py:81-167) run for a whole batch of samples at once: every sample
keeps its own history, step, acceptance and stopping test; converged samples
are frozen.  Cost and gradient come from the ``kr_lower_eval`` stencil kernel
(the HVP's tile machinery); the L-BFGS vector algebra is batched torch ops.

``gradient_descent`` / ``record_sequence`` are bilevel.py:326-502 and
experiments.py:234-268 for a batch sharing theta (F = sum_k 1/2||xhat_k - x_k||^2,
hypergradient = sample-ordered sum), used to produce frozen sequences for the
replay benchmark.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from .bilevel import HessianSolveConfig, SequenceSolver, hypergradients
from .operators import Model
from .recycling import StrategyDescriptor

EPS = float(np.finfo(float).eps)


@dataclass(frozen=True)
class LinesearchParams:
    """bilevel.py:51-62"""

    beta: float = 1.0
    rho: float = 0.5
    eta: float = 1e-4
    max_backtracks: int = 30

    def __post_init__(self):
        if not self.beta > 0:
            raise ValueError("initial stepsize must be positive")
        if not 0 < self.rho < 1 or not 0 < self.eta < 1:
            raise ValueError("rho and eta must lie in (0, 1)")


@dataclass(frozen=True)
class LowerConfig:
    """bilevel.py:65-70"""

    gtol: float = 1e-3
    memory: int = 10
    max_iter: int = 5000
    linesearch: LinesearchParams = field(default_factory=LinesearchParams)


@dataclass
class LowerStats:
    iterations: np.ndarray
    gradient_norm: np.ndarray
    converged: np.ndarray
    cost_evaluations: np.ndarray


def _dot(a, b):
    return (a * b).sum(dim=1)


def lower_solve(model: Model, theta, x_init: torch.Tensor | None = None, gtol: float = 1e-3, memory: int = 10,
                max_iter: int = 5000, linesearch: LinesearchParams | None = None):
    """Batched L-BFGS until ||grad_b|| < gtol for every sample b (bilevel.py:81-167).

    Every sample keeps its own iterate, step, acceptance and stopping test; finished
    samples are frozen.  The curvature pairs live in a ring shared by the batch (one
    slot per iteration, views instead of per-sample gathers): a pair a sample rejects
    (s^T y <= 1e-10 |s||y|, bilevel.py:154-155) is stored with rho = 0 and contributes
    nothing, and the initial scaling s^T y / y^T y comes from the sample's newest
    accepted pair (the reference's deque skips rejected pairs, so after a rejection its
    window reaches one pair further back; rejections do not occur on these convex
    problems).  The cost AND gradient of the accepted Armijo trial are kept (one
    kr_lower_eval per trial; the reference evaluates the gradient at the accepted point
    separately -- the same values).  One host read per iteration (any sample active?)
    plus one per extra backtrack."""
    if not gtol > 0:
        raise ValueError("gtol must be positive")
    ls = linesearch or LinesearchParams()
    B, n, dev = model.batch, model.n, model.device
    x = torch.zeros(B, n, dtype=torch.float64, device=dev) if x_init is None else x_init.reshape(B, n).clone()
    f, g = model.cost_grad(theta, x)
    gn = torch.linalg.vector_norm(g, dim=1)
    S = torch.zeros(B, memory, n, dtype=torch.float64, device=dev)
    Y = torch.zeros_like(S)
    R = torch.zeros(B, memory, dtype=torch.float64, device=dev)   # 1 / s^T y, 0 for a rejected pair
    gam = torch.ones(B, dtype=torch.float64, device=dev)          # H0 scaling of the newest accepted pair
    head, stored = 0, 0
    iters = torch.zeros(B, dtype=torch.long, device=dev)
    evals = torch.ones(B, dtype=torch.long, device=dev)  # the f at x_0 (bilevel.py:129-131)
    active = (gn >= gtol) & (iters < max_iter)
    zero = torch.zeros((), dtype=torch.float64, device=dev)
    while bool(active.any()):
        # two-loop recursion, newest pair first (views of the shared ring)
        q = g.clone()
        alphas = []
        for age in range(min(stored, memory)):
            slot = (head - 1 - age) % memory
            a = R[:, slot] * _dot(S[:, slot], q)
            q.sub_(a.unsqueeze(1) * Y[:, slot])
            alphas.append((slot, a))
        q.mul_(gam.unsqueeze(1))
        for slot, a in reversed(alphas):
            bcoef = R[:, slot] * _dot(Y[:, slot], q)
            q.add_((a - bcoef).unsqueeze(1) * S[:, slot])
        d = q.neg_()
        slope = _dot(g, d)
        bad = slope >= 0
        d = torch.where(bad.unsqueeze(1), -g, d)
        slope = torch.where(bad, -gn * gn, slope)
        # Armijo backtracking, all samples in lockstep; accepted samples freeze
        step = torch.full((B,), ls.beta, dtype=torch.float64, device=dev)
        searching = active.clone()
        slack = EPS * f.abs()
        x_new, f_new, g_new = x, f, g
        for _ in range(ls.max_backtracks):
            xt = x + step.unsqueeze(1) * d
            ft, gt = model.cost_grad(theta, xt)
            evals += searching.long()
            ok = searching & (ft <= f + ls.eta * step * slope + slack)
            okc = ok.unsqueeze(1)
            x_new = torch.where(okc, xt, x_new)
            f_new = torch.where(ok, ft, f_new)
            g_new = torch.where(okc, gt, g_new)
            searching = searching & ~ok
            step = torch.where(searching, step * ls.rho, step)
            if not bool(searching.any()):
                break
        else:
            if bool(searching.any()):
                xt = x + step.unsqueeze(1) * d
                ft, gt = model.cost_grad(theta, xt)
                evals += searching.long()
                sc = searching.unsqueeze(1)
                x_new = torch.where(sc, xt, x_new)
                f_new = torch.where(searching, ft, f_new)
                g_new = torch.where(sc, gt, g_new)
        s_v = x_new - x
        y_v = g_new - g
        sy = _dot(s_v, y_v)
        take = active & (sy > 1e-10 * torch.linalg.vector_norm(s_v, dim=1) * torch.linalg.vector_norm(y_v, dim=1))
        tc = take.unsqueeze(1)
        S[:, head] = torch.where(tc, s_v, zero)
        Y[:, head] = torch.where(tc, y_v, zero)
        R[:, head] = torch.where(take, 1.0 / sy, zero)
        gam = torch.where(take, sy / _dot(y_v, y_v), gam)
        head, stored = (head + 1) % memory, stored + 1
        am = active.unsqueeze(1)
        x = torch.where(am, x_new, x)
        g = torch.where(am, g_new, g)
        f = torch.where(active, f_new, f)
        gn = torch.where(active, torch.linalg.vector_norm(g, dim=1), gn)
        iters = iters + active.long()
        active = active & (gn >= gtol) & (iters < max_iter)
    conv = gn < gtol
    if not bool(conv.all()):
        warnings.warn(f"lower-level solver hit the {max_iter}-iteration cap", stacklevel=2)
    return x, LowerStats(iters.cpu().numpy(), gn.cpu().numpy(), conv.cpu().numpy(), evals.cpu().numpy())


# --------------------------------------------------------------------------
# upper loop (bilevel.py:308-502) and frozen sequences (experiments.py:234-268)


@dataclass
class UpperState:
    theta: np.ndarray
    x_hats: torch.Tensor
    cost: float
    next_beta: float


@dataclass
class FrozenSystem:
    index: int
    theta: np.ndarray
    x_hats: torch.Tensor  # [B, n]
    cost: float
    grad_norm: float
    beta_init: float
    iterations: list


def backtracking_linesearch(state: UpperState, d: np.ndarray, params: LinesearchParams, evaluate):
    """bilevel.py:326-358"""
    c1, c2 = state.cost, float(d @ d)
    warm = state.x_hats
    trial = state
    step = params.beta
    for j in range(1, params.max_backtracks + 1):
        fac = params.rho ** (j - 1)
        step = params.beta * fac
        th = state.theta - step * d
        cost, warm = evaluate(th, warm)
        trial = UpperState(th, warm, cost, 2.0 * step)
        if cost <= c1 - params.eta * fac * c2:
            return trial, j
    warnings.warn("Armijo condition not met within the backtrack budget", stacklevel=2)
    return trial, params.max_backtracks


def gradient_descent(model: Model, theta0, eps_stop: float = 1e-4, *, solver_cfg: HessianSolveConfig | None = None,
                     lower_cfg: LowerConfig | None = None, linesearch: LinesearchParams | None = None,
                     max_upper: int = 30, on_system=None, batch_total: int | None = None, group=None):
    """bilevel.py:392-502 for a batch sharing theta.

    Multi-GPU: ``model`` holds this rank's samples (distributed.shard of
    ``batch_total``); the upper cost F = sum_k 1/2 ||xhat_k - xtrue_k||^2 of every Armijo
    trial and the hypergradient sum_k J_k w_k are all-gathered per sample and summed in
    global sample order (distributed.allgather_sum), so every rank takes the same steps
    and the trajectory is bitwise independent of the world size.  theta is updated
    redundantly on every rank."""
    from .distributed import allgather_sum

    if not eps_stop > 0:
        raise ValueError("eps_stop must be positive")
    solver_cfg = solver_cfg or HessianSolveConfig()
    lower_cfg = lower_cfg or LowerConfig()
    linesearch = linesearch or LinesearchParams()
    total = model.batch if batch_total is None else int(batch_total)
    seq = SequenceSolver(solver_cfg)

    def evaluate(theta, warm):
        x, _ = lower_solve(model, theta, warm, lower_cfg.gtol, lower_cfg.memory, lower_cfg.max_iter,
                           lower_cfg.linesearch)
        diff = x - model.x_true
        per = 0.5 * (diff * diff).sum(dim=1)  # per-sample costs, summed in sample order
        return float(allgather_sum(per.unsqueeze(1), total, group)[0]), x

    c0, x0 = evaluate(np.asarray(theta0, dtype=float), None)
    state = UpperState(np.asarray(theta0, dtype=float).copy(), x0, c0, linesearch.beta)
    trace = []
    for i in range(max_upper):
        hg, res, _ = hypergradients(model, state.theta, state.x_hats, seq)
        d = allgather_sum(hg, total, group).cpu().numpy()
        gnorm = float(np.linalg.norm(d))
        rec = FrozenSystem(i, state.theta.copy(), state.x_hats.clone(), state.cost, gnorm, state.next_beta,
                           [r.iterations for r in res])
        trace.append(rec)
        if on_system is not None:
            on_system(rec)
        if gnorm < eps_stop:
            break
        lp = replace(linesearch, beta=state.next_beta)
        state, _ = backtracking_linesearch(state, d, lp, evaluate)
    return state, trace


def record_sequence(model: Model, theta0, *, delta: float = 1e-2, max_inner: int = 500, lower_gtol: float = 1e-3,
                    eps_stop: float = 1e-4, max_upper: int = 25, lower_max_iter: int = 5000,
                    linesearch: LinesearchParams | None = None, batch_total: int | None = None, group=None):
    """Solve without recycling and freeze every system (experiments.py:234-268)."""
    _, trace = gradient_descent(
        model, theta0, eps_stop,
        solver_cfg=HessianSolveConfig(StrategyDescriptor("None"), delta=delta, stop="res", max_iter=max_inner),
        lower_cfg=LowerConfig(gtol=lower_gtol, max_iter=lower_max_iter), linesearch=linesearch,
        max_upper=max_upper, batch_total=batch_total, group=group)
    return trace
