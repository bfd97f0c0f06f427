"""Replay experiments over frozen sequences on the device (reference experiments.py).

``replay`` re-solves a frozen sequence under one recycle strategy and collects the
per-system metrics of the reference's ``ReplayRow`` (experiments.py:390-463) for every
sample of the batch; ``compute_references`` forms high-accuracy hypergradients
(:271-311); ``dimension_sweep`` (:505-535) and ``cg_vs_minres`` (:538-579) are the
reference's sweeps -- the BASELINE config-5 recycling-stress study runs them
(scripts/sweep_c5.py).  Everything runs batched through the device SequenceSolver /
persistent solvers; only the per-system scalars come back to the host.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from .bilevel import HessianSolveConfig, SequenceSolver, hypergradients
from .krylov import SolveOptions, cg, minres
from .recycling import StrategyDescriptor
from .stopping import ResidualNormRule

__all__ = ["ReplayMetrics", "ReplayRow", "cg_vs_minres", "compute_references", "dimension_sweep", "replay"]


@dataclass(frozen=True)
class ReplayRow:
    """experiments.py:314-330 (plus the sample index of a batch)."""

    strategy: str
    stop: str
    delta: float
    recycle_dim: int
    system: int
    sample: int
    iterations: int
    cum_iterations: int
    flops: int
    cum_flops: int
    effective_recycle_dim: int
    stop_reason: str
    final_stop_value: float
    final_residual: float
    hg_rel_error: float | None


@dataclass
class ReplayMetrics:
    rows: list = field(default_factory=list)
    total_iterations: int = 0
    total_flops: int = 0
    max_hg_rel_error: float | None = None
    mean_hg_rel_error: float | None = None


def compute_references(model, thetas, xhats, delta_ref: float = 1e-13, max_iter: int = 20000):
    """High-accuracy hypergradients J w* per system and sample (experiments.py:271-311): MINRES
    without recycling to a residual below delta_ref (1 + ||g||) (the reference uses dense
    Cholesky for n <= 2000 and reorthogonalised MINRES beyond; here MINRES to the same
    residual target).  Returns a list of (B, p) tensors."""
    refs = []
    for th, X in zip(thetas, xhats):
        X = torch.as_tensor(X, device=model.device).reshape(model.batch, -1)
        H, J = model.at(th, X)
        G = X - model.x_true
        tol = delta_ref * (1.0 + float(torch.linalg.vector_norm(G, dim=1).max()))
        res = minres(H, G if model.batch > 1 else G[0], SolveOptions(max_iter=max_iter,
                                                                      stop_rule=ResidualNormRule(tol)))
        res = res if isinstance(res, list) else [res]
        W = torch.stack([r.solution for r in res])
        refs.append(J.apply_adjoint(W if model.batch > 1 else W[0]).reshape(model.batch, -1))
    return refs


def replay(model, thetas, xhats, strategy, stop: str | None = None, recycle_dim: int = 30, delta: float = 1e-2,
           max_inner: int = 500, refs=None, method: str = "minres") -> ReplayMetrics:
    """experiments.py:390-463 over a batch: re-solve every system under ``strategy``."""
    if isinstance(strategy, str):
        strategy = StrategyDescriptor.parse(strategy)
    if stop is None:
        stop = "nsc" if strategy.nsc else "res"
    solver = SequenceSolver(HessianSolveConfig.from_strategy(strategy, recycle_dim=recycle_dim, delta=delta,
                                                             stop=stop, max_iter=max_inner, method=method))
    out = ReplayMetrics()
    errors = []
    cum_it = [0] * model.batch
    cum_fl = [0] * model.batch
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # dimension clamps are routine
        for i, (th, X) in enumerate(zip(thetas, xhats)):
            X = torch.as_tensor(X, device=model.device).reshape(model.batch, -1)
            hg, res, recs = hypergradients(model, th, X, solver)
            for b, (r, rec) in enumerate(zip(res, recs)):
                cum_it[b] += r.iterations
                cum_fl[b] += r.flops
                err = None
                if refs is not None:
                    ref = refs[i][b]
                    err = float(torch.linalg.vector_norm(ref - hg[b]) / torch.linalg.vector_norm(ref))
                    errors.append(err)
                out.rows.append(ReplayRow(str(strategy), stop, delta, recycle_dim, i, b, r.iterations, cum_it[b],
                                          r.flops, cum_fl[b], rec.dim, r.stop_reason, float(r.stop_values[-1]),
                                          float(r.residual_norms[-1]), err))
    out.total_iterations = sum(cum_it)
    out.total_flops = sum(cum_fl)
    if errors:
        out.max_hg_rel_error = max(errors)
        out.mean_hg_rel_error = float(np.mean(errors))
    return out


def dimension_sweep(model, thetas, xhats, strategy, dims, stop: str | None = None, delta: float = 1e-2,
                    max_inner: int = 500, refs=None) -> list:
    """experiments.py:505-535: totals per recycle dimension (s = 0 -> no recycling, and the
    residual rule, since there is no GSVD data without a recycle space)."""
    if isinstance(strategy, str):
        strategy = StrategyDescriptor.parse(strategy)
    rows = []
    for s in dims:
        use = strategy if s > 0 else StrategyDescriptor(vec_type="None")
        use_stop = stop
        if s == 0 and (stop == "nsc" or (stop is None and strategy.nsc)):
            use_stop = "res"
        m = replay(model, thetas, xhats, use, stop=use_stop, recycle_dim=s, delta=delta, max_inner=max_inner,
                   refs=refs)
        rows.append([str(strategy), s, m.total_iterations, m.total_flops, m.max_hg_rel_error, m.mean_hg_rel_error])
    return rows


def cg_vs_minres(model, thetas, xhats, delta: float = 1e-2, max_inner: int = 500, refs=None) -> list:
    """experiments.py:538-579: cold- and warm-started CG and MINRES, no recycling."""
    rows = []
    for name, solve in (("minres", minres), ("cg", cg)):
        for start in ("cold", "warm"):
            cum = [0] * model.batch
            prev = None
            for i, (th, X) in enumerate(zip(thetas, xhats)):
                X = torch.as_tensor(X, device=model.device).reshape(model.batch, -1)
                H, J = model.at(th, X)
                G = X - model.x_true
                guess = prev if start == "warm" else None
                res = solve(H, G if model.batch > 1 else G[0],
                            SolveOptions(max_iter=max_inner, stop_rule=ResidualNormRule(delta), initial_guess=guess))
                res = res if isinstance(res, list) else [res]
                W = torch.stack([r.solution for r in res])
                prev = W if model.batch > 1 else W[0]
                hg = J.apply_adjoint(prev).reshape(model.batch, -1)
                for b, r in enumerate(res):
                    cum[b] += r.iterations
                    err = None
                    if refs is not None:
                        ref = refs[i][b]
                        err = float(torch.linalg.vector_norm(ref - hg[b]) / torch.linalg.vector_norm(ref))
                    rows.append([name, start, i, b, r.iterations, cum[b], r.flops, float(r.residual_norms[-1]), err])
    return rows
