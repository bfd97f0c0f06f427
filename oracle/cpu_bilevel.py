"""CPU restatement of the bilevel driver (TEST ORACLE ONLY).

Follows ``/root/reference/pkg/src/krecycle/bilevel.py`` (L-BFGS lower solve
:81-167, Armijo upper linesearch :326-358, gradient descent :392-502,
SequenceSolver :225-288, hypergradient :291-305) and
``experiments.py`` (record_sequence :234-268, compute_references :271-311,
replay :390-463), generalised from one sample to a batch of samples that
share theta: F(theta) = sum_k 1/2 ||xhat_k - xtrue_k||^2 and the
hypergradient is the sample-ordered sum of the per-sample J_k w_k.  With one
sample every function reduces to the reference's.
"""

from __future__ import annotations

import warnings
from collections import deque
from dataclasses import dataclass, field, replace

import numpy as np
from scipy.linalg import cho_factor, cho_solve

from . import cpu_imaging as im
from .cpu_krylov import Options, ResidualRule, minres, rcg, rminres
from .cpu_recycle import (ConfigurationError, NscRule, Recycle, Strategy, TrueHgRule,
                          next_recycle)


@dataclass(frozen=True)
class Linesearch:
    """bilevel.py:51-62"""

    beta: float = 1.0
    rho: float = 0.5
    eta: float = 1e-4
    max_backtracks: int = 30


@dataclass(frozen=True)
class LowerStats:
    iterations: int
    gradient_norm: float
    converged: bool
    cost_evaluations: int


def lower_solve(model: im.Model, theta, x_init=None, gtol=1e-3, memory=10, max_iter=5000,
                ls: Linesearch | None = None):
    """L-BFGS with Armijo backtracking until ||grad|| < gtol (bilevel.py:81-167)."""
    if not gtol > 0:
        raise ValueError("gtol must be positive")
    ls = ls or Linesearch()
    x = np.zeros(model.n) if x_init is None else np.array(x_init, dtype=float)
    fcost = lambda v: im.lower_cost(model, theta, v)
    fgrad = lambda v: im.lower_grad(model, theta, v)
    g = fgrad(x)
    gn = float(np.linalg.norm(g))
    mem: deque = deque(maxlen=memory)
    evals, f, it = 0, None, 0
    while gn >= gtol and it < max_iter:
        q = g.copy()
        coef = []
        for sv, yv, rho in reversed(mem):
            a = rho * (sv @ q)
            coef.append(a)
            q -= a * yv
        if mem:
            sv, yv, _ = mem[-1]
            q *= (sv @ yv) / (yv @ yv)
        for (sv, yv, rho), a in zip(mem, reversed(coef)):
            q += (a - rho * (yv @ q)) * sv
        d = -q
        slope = float(g @ d)
        if slope >= 0:
            d = -g
            slope = -gn**2
        if f is None:
            f = fcost(x)
            evals += 1
        step = ls.beta
        ok = False
        slack = np.finfo(float).eps * abs(f)
        for _ in range(ls.max_backtracks):
            xn = x + step * d
            fn = fcost(xn)
            evals += 1
            if fn <= f + ls.eta * step * slope + slack:
                ok = True
                break
            step *= ls.rho
        if not ok:
            xn = x + step * d
            fn = fcost(xn)
            evals += 1
        gnew = fgrad(xn)
        sv = xn - x
        yv = gnew - g
        sy = float(sv @ yv)
        if sy > 1e-10 * np.linalg.norm(sv) * np.linalg.norm(yv):
            mem.append((sv, yv, 1.0 / sy))
        x, g, f = xn, gnew, fn
        gn = float(np.linalg.norm(g))
        it += 1
    if gn >= gtol:
        warnings.warn(f"lower-level solver hit the {max_iter}-iteration cap with gradient norm {gn:.3e}",
                      stacklevel=2)
    return x, LowerStats(it, gn, gn < gtol, evals)


@dataclass(frozen=True)
class SolveConfig:
    """bilevel.py:194-222"""

    strategy: Strategy = field(default_factory=lambda: Strategy("None"))
    recycle_dim: int = 30
    delta: float = 1e-2
    stop: str = "res"
    max_iter: int = 500
    warm_start: bool = False
    inner_tol: float = 1e-13
    dense_limit: int = 2000
    method: str = "minres"  # "minres" (reference) or "cg" (recycled CG, BASELINE config 1)

    def __post_init__(self):
        if self.stop not in ("res", "nsc", "true-hg"):
            raise ValueError(f"unknown stop rule {self.stop!r}")
        if self.method not in ("minres", "cg"):
            raise ValueError(f"unknown Krylov method {self.method!r}")
        if self.stop == "nsc" and self.strategy.vec_type not in ("GSVD", "RGen"):
            raise ConfigurationError("the projected stopping criterion needs a GSVD-based strategy")

    @classmethod
    def from_strategy(cls, strategy, **kw):
        if isinstance(strategy, str):
            strategy = Strategy.parse(strategy)
        if strategy.nsc:
            kw.setdefault("stop", "nsc")
        return cls(strategy=strategy, **kw)


class SequenceSolver:
    """Carries (V_prev, recycle_prev, H_prev, J_prev, w_prev) between systems (bilevel.py:225-288)."""

    def __init__(self, cfg: SolveConfig):
        self.cfg = cfg
        self.first = True
        self.prev_basis = None
        self.prev_recycle = None
        self.prev_h = None
        self.prev_jac = None
        self.prev_solution = None

    def solve(self, H, g, jac):
        cfg = self.cfg
        if cfg.strategy.is_none or self.first:
            rec = Recycle.empty(H.dim)
        else:
            rec = next_recycle(cfg.strategy, h_current=H, h_previous=self.prev_h, jac_current=jac,
                               jac_previous=self.prev_jac, prev_basis=self.prev_basis,
                               prev_recycle=self.prev_recycle, s=cfg.recycle_dim,
                               dense_limit=cfg.dense_limit)
        self.first = False
        if cfg.stop == "res":
            rule = ResidualRule(cfg.delta)
        elif cfg.stop == "true-hg":
            rule = TrueHgRule(cfg.delta, jac, H, cfg.inner_tol, cfg.dense_limit)
        else:
            rule = NscRule(cfg.delta, rec.nsc_data) if rec.nsc_data is not None else ResidualRule(cfg.delta)
        opts = Options(max_iter=cfg.max_iter, stop_rule=rule, track_basis=not cfg.strategy.is_none,
                       initial_guess=self.prev_solution if cfg.warm_start else None)
        res = (rminres if cfg.method == "minres" else rcg)(H, g, rec, opts)
        self.prev_basis, self.prev_recycle = res.basis, rec
        self.prev_h, self.prev_jac, self.prev_solution = H, jac, res.solution
        return res, rec


def hypergradient(model: im.Model, theta, x_hat, x_true, recycle=None, opts=None):
    """bilevel.py:291-305"""
    H = im.hessian(model, theta, x_hat)
    J = im.jacobian(model, theta, x_hat)
    res = rminres(H, np.asarray(x_hat) - np.asarray(x_true), recycle, opts)
    return J.apply_adjoint(res.solution), res


# --------------------------------------------------------------------------
# multi-sample gradient descent (bilevel.py:308-502)


@dataclass(frozen=True)
class UpperState:
    theta: np.ndarray
    x_hats: tuple
    cost: float
    next_beta: float


@dataclass
class UpperRecord:
    index: int
    theta: np.ndarray
    x_hats: list
    cost: float
    grad_norm: float
    theta_next: np.ndarray | None
    iterations: list
    flops: list
    stop_reasons: list
    recycle_dims: list
    linesearch_trials: int
    w_hats: list
    hg: np.ndarray
    beta_init: float


def backtracking(state: UpperState, d, params: Linesearch, evaluate):
    """Smallest j with F(theta - beta rho^{j-1} d) <= F(theta) - eta rho^{j-1} d^T d,
    trial lower solves warm started from the previous trial (bilevel.py:326-358)."""
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
    warnings.warn("Armijo condition not met; returning the smallest-step trial", stacklevel=2)
    return trial, params.max_backtracks


@dataclass
class Batch:
    """A batch of samples sharing theta: models[k] carries y_k (and x_true_k)."""

    models: list
    x_trues: list

    @property
    def size(self):
        return len(self.models)


def gradient_descent(theta0, batch: Batch, eps_stop=1e-4, *, solver_cfg: SolveConfig | None = None,
                     lower_gtol=1e-3, lower_memory=10, lower_max_iter=5000,
                     linesearch: Linesearch | None = None, max_upper=30):
    """bilevel.py:392-502 with F summed over the batch."""
    if not eps_stop > 0:
        raise ValueError("eps_stop must be positive")
    solver_cfg = solver_cfg or SolveConfig()
    linesearch = linesearch or Linesearch()
    solvers = [SequenceSolver(solver_cfg) for _ in range(batch.size)]

    def evaluate(theta, warm):
        xs, cost = [], 0.0
        for k, model in enumerate(batch.models):
            x, _ = lower_solve(model, theta, None if warm is None else warm[k], lower_gtol,
                               lower_memory, lower_max_iter)
            diff = x - batch.x_trues[k]
            cost += 0.5 * float(diff @ diff)
            xs.append(x)
        return cost, tuple(xs)

    c0, xs = evaluate(np.asarray(theta0, dtype=float), None)
    state = UpperState(np.asarray(theta0, dtype=float).copy(), xs, c0, linesearch.beta)
    trace = []
    reason = "max_upper"
    for i in range(max_upper):
        d = None
        its, fl, why, dims, ws = [], [], [], [], []
        for k, model in enumerate(batch.models):
            H = im.hessian(model, state.theta, state.x_hats[k])
            J = im.jacobian(model, state.theta, state.x_hats[k])
            res, rec = solvers[k].solve(H, state.x_hats[k] - batch.x_trues[k], J)
            hg = J.apply_adjoint(res.solution)
            d = hg if d is None else d + hg
            its.append(res.iterations)
            fl.append(res.flops)
            why.append(res.stop_reason)
            dims.append(rec.dim)
            ws.append(res.solution.copy())
        gnorm = float(np.linalg.norm(d))
        if gnorm < eps_stop:
            trace.append(UpperRecord(i, state.theta.copy(), list(state.x_hats), state.cost, gnorm, None,
                                     its, fl, why, dims, 0, ws, d, state.next_beta))
            reason = "gradient_norm"
            break
        lp = replace(linesearch, beta=state.next_beta)
        new_state, trials = backtracking(state, d, lp, evaluate)
        trace.append(UpperRecord(i, state.theta.copy(), list(state.x_hats), state.cost, gnorm,
                                 new_state.theta.copy(), its, fl, why, dims, trials, ws, d, lp.beta))
        state = new_state
    return state, trace, reason


# --------------------------------------------------------------------------
# frozen sequences and replay (experiments.py:234-463)


@dataclass
class FrozenSystem:
    index: int
    theta: np.ndarray
    x_hats: list
    gs: list
    cost: float = 0.0
    beta_init: float = 1.0
    w_stars: list | None = None
    ref_hgs: list | None = None


@dataclass
class FrozenSequence:
    batch: Batch
    systems: list

    def hessian(self, i, k):
        return im.hessian(self.batch.models[k], self.systems[i].theta, self.systems[i].x_hats[k])

    def jacobian(self, i, k):
        return im.jacobian(self.batch.models[k], self.systems[i].theta, self.systems[i].x_hats[k])


def record_sequence(theta0, batch: Batch, *, delta=1e-2, max_inner=500, lower_gtol=1e-3,
                    eps_stop=1e-4, max_upper=25) -> FrozenSequence:
    """Run GD without recycling and freeze every system (experiments.py:234-268)."""
    _, trace, _ = gradient_descent(
        theta0, batch, eps_stop,
        solver_cfg=SolveConfig(Strategy("None"), delta=delta, stop="res", max_iter=max_inner),
        lower_gtol=lower_gtol, max_upper=max_upper)
    systems = [FrozenSystem(r.index, r.theta, [x.copy() for x in r.x_hats],
                            [r.x_hats[k] - batch.x_trues[k] for k in range(batch.size)],
                            r.cost, r.beta_init) for r in trace]
    return FrozenSequence(batch, systems)


def compute_references(seq: FrozenSequence, delta_ref=1e-13, dense_limit=2000):
    """w* by dense Cholesky + refinement, else reorthogonalised MINRES (experiments.py:271-311)."""
    for i, sysm in enumerate(seq.systems):
        sysm.w_stars, sysm.ref_hgs = [], []
        for k in range(seq.batch.size):
            H = seq.hessian(i, k)
            g = sysm.gs[k]
            tol = delta_ref * (1 + np.linalg.norm(g))
            if H.dim <= dense_limit:
                fac = cho_factor(H.to_dense())
                w = cho_solve(fac, g)
                for _ in range(40):
                    r = g - H(w)
                    if np.linalg.norm(r) <= tol:
                        break
                    w = w + cho_solve(fac, r)
            else:
                w = minres(H, g, Options(max_iter=4 * H.dim, stop_rule=ResidualRule(tol),
                                         reorthogonalize=True, track_basis=True)).solution
            sysm.w_stars.append(w)
            sysm.ref_hgs.append(seq.jacobian(i, k).apply_adjoint(w))
    return seq


@dataclass
class ReplayRow:
    system: int
    sample: int
    iterations: int
    flops: int
    effective_recycle_dim: int
    stop_reason: str
    final_stop_value: float
    final_residual: float
    hg: np.ndarray
    hg_rel_error: float | None


def replay(seq: FrozenSequence, strategy, stop=None, recycle_dim=30, delta=1e-2, max_inner=500,
           systems=None):
    """Per-sample SequenceSolver over the frozen systems (experiments.py:390-463, one-step cost omitted)."""
    if isinstance(strategy, str):
        strategy = Strategy.parse(strategy)
    if stop is None:
        stop = "nsc" if strategy.nsc else "res"
    cfg = SolveConfig.from_strategy(strategy, recycle_dim=recycle_dim, delta=delta, stop=stop,
                                    max_iter=max_inner)
    solvers = [SequenceSolver(cfg) for _ in range(seq.batch.size)]
    rows = []
    idx = range(len(seq.systems)) if systems is None else systems
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        for i in idx:
            sysm = seq.systems[i]
            for k in range(seq.batch.size):
                H, J = seq.hessian(i, k), seq.jacobian(i, k)
                res, rec = solvers[k].solve(H, sysm.gs[k], J)
                hg = J.apply_adjoint(res.solution)
                err = None
                if sysm.ref_hgs is not None:
                    ref = sysm.ref_hgs[k]
                    err = float(np.linalg.norm(ref - hg) / np.linalg.norm(ref))
                rows.append(ReplayRow(i, k, res.iterations, res.flops, rec.dim, res.stop_reason,
                                      float(res.stop_values[-1]), float(res.residual_norms[-1]), hg, err))
    return rows


def one_step_cost(seq: FrozenSequence, i: int, direction, lower_gtol=1e-3):
    """experiments.py:364-387 (batch form)."""
    sysm = seq.systems[i]
    b = seq.batch

    def evaluate(theta, warm):
        xs, cost = [], 0.0
        for k, model in enumerate(b.models):
            x, _ = lower_solve(model, theta, warm[k], lower_gtol)
            diff = x - b.x_trues[k]
            cost += 0.5 * float(diff @ diff)
            xs.append(x)
        return cost, tuple(xs)

    state = UpperState(sysm.theta, tuple(sysm.x_hats), sysm.cost, sysm.beta_init)
    new_state, _ = backtracking(state, direction, Linesearch(beta=sysm.beta_init), evaluate)
    return new_state.cost
