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
    """Batched L-BFGS until ||grad_b|| < gtol for every sample b (bilevel.py:81-167)."""
    if not gtol > 0:
        raise ValueError("gtol must be positive")
    ls = linesearch or LinesearchParams()
    B, n, dev = model.batch, model.n, model.device
    x = torch.zeros(B, n, dtype=torch.float64, device=dev) if x_init is None else x_init.reshape(B, n).clone()
    f, g = model.cost_grad(theta, x)
    gn = torch.linalg.vector_norm(g, dim=1)
    S = torch.zeros(B, memory, n, dtype=torch.float64, device=dev)
    Y = torch.zeros_like(S)
    R = torch.zeros(B, memory, dtype=torch.float64, device=dev)
    head = torch.zeros(B, dtype=torch.long, device=dev)   # next slot
    count = torch.zeros(B, dtype=torch.long, device=dev)
    iters = torch.zeros(B, dtype=torch.long, device=dev)
    evals = torch.ones(B, dtype=torch.long, device=dev)  # the f at x_0 (bilevel.py:129-131)
    ar = torch.arange(B, device=dev)
    while True:
        active = (gn >= gtol) & (iters < max_iter)
        if not bool(active.any()):
            break
        # two-loop recursion over each sample's own history, newest first
        q = g.clone()
        alphas = []
        for age in range(memory):
            slot = (head - 1 - age) % memory
            valid = (age < count).to(torch.float64)
            s_a, y_a, r_a = S[ar, slot], Y[ar, slot], R[ar, slot] * valid
            a = r_a * _dot(s_a, q)
            q = q - a.unsqueeze(1) * y_a
            alphas.append((slot, a, valid))
        has = count > 0
        slot0 = (head - 1) % memory
        s0, y0 = S[ar, slot0], Y[ar, slot0]
        gam = torch.where(has, _dot(s0, y0) / torch.where(has, _dot(y0, y0), torch.ones_like(gn)), torch.ones_like(gn))
        q = q * gam.unsqueeze(1)
        for slot, a, valid in reversed(alphas):
            s_a, y_a, r_a = S[ar, slot], Y[ar, slot], R[ar, slot] * valid
            bcoef = r_a * _dot(y_a, q)
            q = q + ((a - bcoef) * valid).unsqueeze(1) * s_a
        d = -q
        slope = _dot(g, d)
        bad = slope >= 0
        d = torch.where(bad.unsqueeze(1), -g, d)
        slope = torch.where(bad, -gn * gn, slope)
        # Armijo backtracking, all samples in lockstep; accepted samples freeze
        step = torch.full((B,), ls.beta, dtype=torch.float64, device=dev)
        searching = active.clone()
        slack = EPS * f.abs()
        x_new, f_new = x.clone(), f.clone()
        for _ in range(ls.max_backtracks):
            xt = x + step.unsqueeze(1) * d
            ft, _ = model.cost_grad(theta, xt)
            evals += searching.long()
            ok = searching & (ft <= f + ls.eta * step * slope + slack)
            x_new = torch.where(ok.unsqueeze(1), xt, x_new)
            f_new = torch.where(ok, ft, f_new)
            searching = searching & ~ok
            step = torch.where(searching, step * ls.rho, step)
            if not bool(searching.any()):
                break
        if bool(searching.any()):
            xt = x + step.unsqueeze(1) * d
            ft, _ = model.cost_grad(theta, xt)
            evals += searching.long()
            x_new = torch.where(searching.unsqueeze(1), xt, x_new)
            f_new = torch.where(searching, ft, f_new)
        _, g_new = model.cost_grad(theta, x_new)
        s_v = x_new - x
        y_v = g_new - g
        sy = _dot(s_v, y_v)
        take = active & (sy > 1e-10 * torch.linalg.vector_norm(s_v, dim=1) * torch.linalg.vector_norm(y_v, dim=1))
        hs = head.clone()
        S[ar[take], hs[take]] = s_v[take]
        Y[ar[take], hs[take]] = y_v[take]
        R[ar[take], hs[take]] = 1.0 / sy[take]
        head = torch.where(take, (head + 1) % memory, head)
        count = torch.where(take, torch.clamp(count + 1, max=memory), count)
        am = active.unsqueeze(1)
        x = torch.where(am, x_new, x)
        g = torch.where(am, g_new, g)
        f = torch.where(active, f_new, f)
        gn = torch.where(active, torch.linalg.vector_norm(g, dim=1), gn)
        iters = iters + active.long()
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
                     max_upper: int = 30, on_system=None):
    """bilevel.py:392-502 for a batch sharing theta."""
    if not eps_stop > 0:
        raise ValueError("eps_stop must be positive")
    solver_cfg = solver_cfg or HessianSolveConfig()
    lower_cfg = lower_cfg or LowerConfig()
    linesearch = linesearch or LinesearchParams()
    seq = SequenceSolver(solver_cfg)

    def evaluate(theta, warm):
        x, _ = lower_solve(model, theta, warm, lower_cfg.gtol, lower_cfg.memory, lower_cfg.max_iter,
                           lower_cfg.linesearch)
        diff = x - model.x_true
        per = 0.5 * (diff * diff).sum(dim=1)
        return float(sum(float(v) for v in per.cpu().numpy())), x

    c0, x0 = evaluate(np.asarray(theta0, dtype=float), None)
    state = UpperState(np.asarray(theta0, dtype=float).copy(), x0, c0, linesearch.beta)
    trace = []
    for i in range(max_upper):
        hg, res, _ = hypergradients(model, state.theta, state.x_hats, seq)
        hg_np = hg.cpu().numpy()
        d = hg_np[0].copy()
        for k in range(1, hg_np.shape[0]):
            d = d + hg_np[k]
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
                    eps_stop: float = 1e-4, max_upper: int = 25, lower_max_iter: int = 5000):
    """Solve without recycling and freeze every system (experiments.py:234-268)."""
    _, trace = gradient_descent(
        model, theta0, eps_stop,
        solver_cfg=HessianSolveConfig(StrategyDescriptor("None"), delta=delta, stop="res", max_iter=max_inner),
        lower_cfg=LowerConfig(gtol=lower_gtol, max_iter=lower_max_iter), max_upper=max_upper)
    return trace
