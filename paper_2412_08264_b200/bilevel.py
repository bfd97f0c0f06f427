"""Sequence solver and hypergradient on the device (reference bilevel.py).

``SequenceSolver`` keeps, per training sample, the previous Krylov basis,
recycle space, operator and Jacobian (bilevel.py:225-288) -- all device
resident -- and solves a whole batch of samples with ONE persistent RMINRES
launch per upper step.  ``hypergradient`` is bilevel.py:291-305.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field

import torch

from .krylov import SolveOptions, SolveResult, rminres
from .operators import FoEParams, ImageVector, InpaintingProblem, Model, as_device, _foe_model
from .recycling import RecycleSpace, StrategyDescriptor, next_recycle
from .stopping import ConfigurationError, NscRule, ResidualNormRule

__all__ = ["HessianSolveConfig", "SequenceSolver", "hypergradient", "hypergradients"]


@dataclass(frozen=True)
class HessianSolveConfig:
    """bilevel.py:194-222 (+ ``reuse_products``: form H U~ from H W, see recycling.py)."""

    strategy: StrategyDescriptor = field(default_factory=lambda: StrategyDescriptor(vec_type="None"))
    recycle_dim: int = 30
    delta: float = 1e-2
    stop: str = "res"
    max_iter: int = 500
    warm_start: bool = False
    inner_tol: float = 1e-13
    dense_limit: int = 2000
    reuse_products: bool = True

    def __post_init__(self):
        if self.stop not in ("res", "nsc", "true-hg"):
            raise ValueError(f"unknown stop rule {self.stop!r}")
        if self.stop == "nsc" and self.strategy.vec_type not in ("GSVD", "RGen"):
            raise ConfigurationError("the projected stopping criterion needs a GSVD-based strategy; "
                                     f"got {self.strategy}")

    @classmethod
    def from_strategy(cls, strategy, **kwargs) -> "HessianSolveConfig":
        if isinstance(strategy, str):
            strategy = StrategyDescriptor.parse(strategy)
        if strategy.nsc:
            kwargs.setdefault("stop", "nsc")
        return cls(strategy=strategy, **kwargs)


class SequenceSolver:
    """Solves consecutive Hessian systems of a batch of samples, carrying the
    recycling state of each sample (bilevel.py:225-288).

    ``solve(H, g, J)`` with a single-sample operator and g of shape (n,)
    returns ``(SolveResult, RecycleSpace)`` like the reference; with a batched
    operator and g of shape (B, n) it returns two lists.
    """

    def __init__(self, cfg: HessianSolveConfig):
        if cfg.stop == "true-hg":
            raise NotImplementedError("the true-hypergradient rule is an oracle; use the CPU oracle for it")
        self.cfg = cfg
        self._first = True
        self._prev_basis: list | None = None
        self._prev_recycle: list | None = None
        self._prev_h = None
        self._prev_jac = None
        self._prev_solution = None

    def _needs_basis(self) -> bool:
        return not self.cfg.strategy.is_none

    def solve(self, hessian, g, jac):
        cfg = self.cfg
        g = as_device(g)
        single = g.dim() == 1
        B = 1 if single else g.shape[0]
        n = hessian.dim
        if cfg.strategy.is_none or self._first:
            recycles = [RecycleSpace.empty(n) for _ in range(B)]
        else:
            recycles = []
            for b in range(B):
                hb = hessian if B == 1 else hessian.sample(b)
                jb = jac if (B == 1 or jac is None) else jac.sample(b)
                hp = None if self._prev_h is None else (self._prev_h if B == 1 else self._prev_h.sample(b))
                jp = None if self._prev_jac is None else (self._prev_jac if B == 1 else self._prev_jac.sample(b))
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", UserWarning)
                    recycles.append(next_recycle(
                        cfg.strategy, h_current=hb, h_previous=hp, jac_current=jb, jac_previous=jp,
                        prev_basis=self._prev_basis[b], prev_recycle=self._prev_recycle[b],
                        s=cfg.recycle_dim, dense_limit=cfg.dense_limit, reuse_products=cfg.reuse_products))
        self._first = False
        rules = []
        for rec in recycles:
            if cfg.stop == "nsc" and rec.nsc_data is not None:
                rules.append(NscRule(cfg.delta, rec.nsc_data))
            else:  # res, or nsc on the first system (bilevel.py:269-273)
                rules.append(ResidualNormRule(cfg.delta))
        init = self._prev_solution if cfg.warm_start else None
        opts = SolveOptions(max_iter=cfg.max_iter, stop_rule=rules if B > 1 else rules[0],
                            track_basis=self._needs_basis(), initial_guess=init)
        results = rminres(hessian, g, recycles if B > 1 else recycles[0], opts)
        res_list = [results] if single else results
        self._prev_basis = [r.basis for r in res_list]
        self._prev_recycle = recycles
        self._prev_h = hessian
        self._prev_jac = jac
        self._prev_solution = torch.stack([r.solution for r in res_list]) if not single else res_list[0].solution
        if single:
            return res_list[0], recycles[0]
        return res_list, recycles


def hypergradient(params: FoEParams, x_hat: ImageVector, prob: InpaintingProblem,
                  recycle: RecycleSpace | None = None, opts: SolveOptions | None = None):
    """Solve H w = xhat - xtrue and return (J w, result) (bilevel.py:291-305)."""
    if prob.x_true is None:
        raise ValueError("problem has no ground-truth image")
    model = _foe_model(params, prob)
    H, J = model.at(params.flatten(), x_hat.data)
    g = as_device(x_hat.data) - as_device(prob.x_true.data)
    result = rminres(H, g, recycle, opts)
    return J.apply_adjoint(result.solution), result


def hypergradients(model: Model, theta, x_hats: torch.Tensor, solver: SequenceSolver):
    """Per-sample hypergradients J_k w_k of a batch at (theta, xhat_k) with recycling;
    returns (hg [B, p], results, recycles).  The sample-ordered sum is the upper gradient."""
    H, J = model.at(theta, x_hats)
    G = x_hats.reshape(model.batch, -1) - model.x_true
    results, recycles = solver.solve(H, G if model.batch > 1 else G[0], J)
    if model.batch == 1:
        results, recycles = [results], [recycles]
    W = torch.stack([r.solution for r in results])
    hg = J.apply_adjoint(W if model.batch > 1 else W[0])
    return hg.reshape(model.batch, -1), results, recycles
