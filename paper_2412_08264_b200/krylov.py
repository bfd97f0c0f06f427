"""MINRES / RMINRES / CG mirroring ``krecycle.krylov`` (reference krylov.py).

Each call is ONE persistent cooperative kernel (``kr_rminres`` / ``kr_cg``)
that runs every iteration of every sample of a batch on the device; the host
sees the result once.  Semantics follow krylov.py:205-483: Alg. 3 with the
corrected sign, breakdown at 1e-13 ||g||, stop test before breakdown test,
the 5-vector residual recurrence when the rule needs r, and the closed-form
FLOP model (krylov.py:119-135) in ``SolveResult.flops``.

Batching: ``g`` of shape (B, n) with a batched operator solves B independent
systems in one launch and returns a list of results; ``recycle`` and the
stop rule may then be per-sample lists.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import KrSolveArgs, NonSPDError
from .operators import as_device, columns, new_columns
from .stopping import NscRule, ResidualNormRule, StopRule

__all__ = ["BREAKDOWN_RTOL", "NonSPDError", "SolveOptions", "SolveResult", "TridiagState", "cg", "flops_cg",
           "flops_minres", "flops_rcg", "flops_rminres", "minres", "rcg", "rminres"]

BREAKDOWN_RTOL = 1e-13


@dataclass
class SolveOptions:
    """krylov.py:57-82.  The per-iteration diagnostics (reorthogonalize,
    collect_*) are host-loop test hooks of the reference; the persistent
    kernel does not produce them and raises if they are requested."""

    max_iter: int = 500
    initial_guess: object = None
    stop_rule: StopRule | None = None
    track_basis: bool = False
    track_residual_vector: bool = False
    reorthogonalize: bool = False
    collect_states: bool = False
    collect_iterates: bool = False
    collect_residual_history: bool = False
    # not in the reference: None = the reference's behaviour (the residual vector is
    # tracked and returned when the stop rule needs it, krylov.py:214-215); False = do not
    # materialise it (the device solver evaluates NSC in s-space and, with the basis kept,
    # needs no residual vector at all -- SequenceSolver uses this)
    residual_vector: bool | None = None

    def __post_init__(self):
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")

    def rule(self) -> StopRule:
        return self.stop_rule if self.stop_rule is not None else ResidualNormRule(1e-2)


@dataclass(frozen=True)
class TridiagState:
    """krylov.py:85-99 (kept for API compatibility)."""

    alpha: float
    beta: float
    beta_next: float
    gamma: float
    delta: float
    epsilon: float
    epsilon_rot: float
    givens: tuple
    givens_prev: tuple
    givens_prev2: tuple
    zeta: float


@dataclass
class SolveResult:
    """krylov.py:102-116; solution / basis / residual_vector are device tensors."""

    solution: torch.Tensor
    iterations: int
    residual_norms: np.ndarray
    flops: int
    stop_reason: str
    stop_values: np.ndarray
    basis: torch.Tensor | None = None
    residual_vector: torch.Tensor | None = None
    states: list | None = None
    iterates: list | None = None
    residual_history: list | None = None


def _check_counts(**kw):
    for name, v in kw.items():
        if v < 0:
            raise ValueError(f"{name} must be nonnegative, got {v}")


def flops_minres(k_total: int, n: int, h_cost: int) -> int:
    """krylov.py:119-122"""
    _check_counts(k_total=k_total, n=n, h_cost=h_cost)
    return h_cost + 4 * n + k_total * (h_cost + 16 * n)


def flops_rminres(k_total: int, n: int, s: int, h_cost: int) -> int:
    """krylov.py:125-128"""
    _check_counts(k_total=k_total, n=n, s=s, h_cost=h_cost)
    return h_cost + 4 * n + 6 * n * s + k_total * (h_cost + 21 * n + 6 * n * s - s)


def flops_rcg(k_total: int, n: int, s: int, h_cost: int) -> int:
    """Deflated CG: flops_cg plus U^T r, C y, U y once and C^T r, U mu per iteration
    (oracle cpu_krylov.flops_rcg)."""
    _check_counts(k_total=k_total, n=n, s=s, h_cost=h_cost)
    return h_cost + 3 * n + 6 * n * s + k_total * (h_cost + 10 * n + 4 * n * s)


def flops_cg(k_total: int, n: int, h_cost: int) -> int:
    """krylov.py:131-135"""
    _check_counts(k_total=k_total, n=n, h_cost=h_cost)
    return h_cost + 3 * n + k_total * (h_cost + 10 * n)


def _unsupported(opts: SolveOptions):
    for flag in ("reorthogonalize", "collect_states", "collect_iterates", "collect_residual_history"):
        if getattr(opts, flag):
            raise NotImplementedError(f"SolveOptions.{flag} is a host-loop diagnostic; the device solver "
                                      "runs the whole iteration in one kernel and does not record it")


def _as_batch(H, g):
    g = as_device(g)
    single = g.dim() == 1
    G = g.reshape(1, -1) if single else g
    if G.shape[1] != H.dim:
        raise ValueError(f"right-hand side of shape {tuple(g.shape)}, operator dim {H.dim}")
    if G.shape[0] != H.batch:
        raise ValueError(f"{G.shape[0]} right-hand sides for an operator batch of {H.batch}")
    # checked with the solve's results (one device -> host transfer per launch, no sync here)
    return G.contiguous(), single


def _batched_gram(A, Bm):
    from .batched import gram

    return gram(A, Bm)


def _per_sample(x, B):
    if isinstance(x, (list, tuple)):
        if len(x) != B:
            raise ValueError(f"expected {B} per-sample entries, got {len(x)}")
        return list(x)
    return [x] * B


def _rule_kind(rule) -> int:
    from .stopping import TrueHgErrorRule

    if isinstance(rule, NscRule):
        return 1
    if isinstance(rule, ResidualNormRule):
        return 0
    if isinstance(rule, TrueHgErrorRule):
        return 2
    raise NotImplementedError(f"the device solver evaluates residual and NSC rules only, got {type(rule).__name__}")


import os as _os

_PAD = int(_os.environ.get("KR_PAD", "0"))  # debug: guard-pad solver buffers (doubles each side)
_PAD_ONLY = set(filter(None, _os.environ.get("KR_PAD_ONLY", "").split(",")))


def _buf(tag, *shape, zero=False, dev=None):
    if _PAD and (not _PAD_ONLY or tag in _PAD_ONLY):
        numel = 1
        for d in shape:
            numel *= d
        flat = torch.full((numel + 2 * _PAD,), float("nan"), dtype=torch.float64, device=dev)
        t = flat[_PAD: _PAD + numel].view(*shape)
        if zero:
            t.zero_()
        return t
    f = torch.zeros if zero else torch.empty
    return f(*shape, dtype=torch.float64, device=dev)


class _Launch:
    """Device buffers + kr_solve_args for one batched solve."""

    def __init__(self, H, G, recycles, rules, opts, want_basis, deflate=False, plain_cg=False):
        B, n = G.shape
        dev = G.device
        self.B, self.n = B, n
        self.max_iter = opts.max_iter
        a = KrSolveArgs()
        a.max_iter = opts.max_iter
        a.g = G.data_ptr()
        self.keep = [G]
        w0 = opts.initial_guess
        if w0 is not None:
            w0 = as_device(w0).reshape(B, n).contiguous()
            self.keep.append(w0)
            a.w0 = w0.data_ptr()
        # (r)minres contract: non-finite g -> ValueError; the reference's cg has no such
        # check (krylov.py:408-483) and runs the NaNs through to max_iter
        self.finite = torch.ones((), dtype=torch.bool, device=dev) if plain_cg else torch.isfinite(G).all()
        dims = [0 if r is None else r.dim for r in recycles]
        s = max(dims) if dims else 0
        self.dims = dims
        a.s = s
        # recycle spaces written by the batched update into whole-batch (B, s, n) rows
        # are read in place; anything else is stacked (zero-padded to s columns)
        src = [getattr(r, "batch_src", None) for r in recycles]
        off = src[0][3] if src and src[0] is not None else 0
        self.inplace = (s > 0 and not _PAD and all(x is not None for x in src)
                        and all(x[0] is src[0][0] and x[3] == off + b for b, x in enumerate(src))
                        and src[0][0].shape[0] >= off + B and tuple(src[0][0].shape[1:]) == (s, n)
                        and all(d == s for d in dims))
        if s:
            if self.inplace:
                U, C = src[0][0][off: off + B], src[0][1][off: off + B]
            else:
                U = _buf("U", B, s, n, zero=True, dev=dev)
                C = _buf("C", B, s, n, zero=True, dev=dev)
                for b, r in enumerate(recycles):
                    if r is not None and r.dim:
                        U[b, : r.dim] = r.U.T
                        C[b, : r.dim] = r.C.T
            self.U, self.C = U, C
            self.keep += [U, C]
            a.U, a.C, a.ld_uc, a.bs_uc = U.data_ptr(), C.data_ptr(), n, s * n
            if deflate:  # recycled CG: Minv = (U^T C)^{-1}, identity on padded columns
                # one Cholesky+inverse launch (kr_chol_inv on the leading dims[b] block, identity
                # pad), Minv = F^T F with F = L^{-1}; a failed factorization (U^T H U not SPD) is
                # reported with the results (no host sync before the solve launch)
                from .batched import _chol_inv

                M = U @ C.transpose(1, 2)
                M = 0.5 * (M + M.transpose(1, 2))
                d = torch.tensor(dims, dtype=torch.int32)
                F, info, _ = _chol_inv(M, d, scale=False)
                Minv = (F.transpose(1, 2) @ F).contiguous()
                self.spd_info = info
                self.keep += [Minv, F]
                a.Minv = Minv.data_ptr()
        kinds = {_rule_kind(r) for r in rules}
        if len(kinds) != 1:
            raise ValueError("one launch needs one rule kind; split the batch")
        kind = kinds.pop()
        deltas = {float(r.delta) for r in rules}
        if len(deltas) != 1:
            raise ValueError("one launch needs one tolerance")
        a.stop_kind = kind
        a.delta = deltas.pop()
        # cg always returns its final residual (krylov.py:482: residual_vector=r.copy());
        # (r)minres tracks it when asked or when NSC needs it (krylov.py:214-215) -- unless the
        # caller waived it and the basis is kept (then the kernel keeps Z^T r in s-space)
        want_r = opts.track_residual_vector or (kind >= 1 and opts.residual_vector is not False)
        track = want_r or plain_cg or (kind == 1 and not want_basis)
        a.track_residual = int(track)
        if kind == 2:
            # true hypergradient error: Z = J's rows, Z^T C -> J U, nsc_r0 = J w* - J w0
            data = [r.device_data(G[b]) for b, r in enumerate(rules)]
            p = data[0][0].shape[0]
            Z = torch.stack([d[0] for d in data]).contiguous()            # (B, p, n)
            r0 = torch.stack([d[1] for d in data])                        # (B, p)
            if w0 is not None:
                r0 = r0 - torch.bmm(Z, w0.unsqueeze(2)).squeeze(2)
            r0 = r0.contiguous()
            a.nsc_s, a.Z, a.ld_z, a.bs_z = p, Z.data_ptr(), n, p * n
            a.nsc_r0 = r0.data_ptr()
            self.keep += [Z, r0]
            if s:
                ZtC = torch.bmm(Z, self.U.transpose(1, 2)).contiguous()   # J U (B, p, s)
                a.ZtC = ZtC.data_ptr()
                self.keep.append(ZtC)
        if kind == 1:
            zs = [r.data.z_block() for r in rules]
            ns = max(z.shape[1] for z in zs)
            zsrc = src[0][2][off: off + B] if s and self.inplace and src[0][2] is not None else None
            if (zsrc is not None and ns == s
                    and all(z.data_ptr() == zsrc[b].data_ptr() and z.shape[1] == s for b, z in enumerate(zs))):
                Z = zsrc
            else:
                Z = _buf("Z", B, ns, n, zero=True, dev=dev)
                for b, z in enumerate(zs):
                    Z[b, : z.shape[1]] = z.T
            a.nsc_s, a.Z, a.ld_z, a.bs_z = ns, Z.data_ptr(), n, ns * n
            self.keep.append(Z)
            if s:
                # (B, ns, s) Z^T C: formed by the batched update on the group streams when Z and C
                # are its in-place rows, else a split-K Gram over the pixels here
                pre = src[0][4] if (Z is zsrc and zsrc is not None and len(src[0]) > 4) else None
                if pre is not None:
                    ZtC = pre[off: off + B]
                else:
                    ZtC = (_batched_gram(Z, self.C) if ns == s else torch.bmm(Z, self.C.transpose(1, 2))).contiguous()
                a.ZtC = ZtC.data_ptr()
                self.keep.append(ZtC)
        self.w = _buf("w", B, n, dev=dev)
        a.w = self.w.data_ptr()
        self.r = _buf("r", B, n, dev=dev) if track else None
        if track:
            a.r = self.r.data_ptr()
        self.basis = None
        self.want_basis = want_basis
        if want_basis or kind == 2:  # the true-hg rule runs in the shared-block kernel (basis kept)
            self.basis = _buf("basis", B, opts.max_iter, n, dev=dev)
            a.basis, a.ld_basis, a.bs_basis = self.basis.data_ptr(), n, opts.max_iter * n
        self.res = _buf("res", B, opts.max_iter + 1, dev=dev)
        self.vals = _buf("vals", B, opts.max_iter + 1, dev=dev)
        self.iters = torch.zeros(B, dtype=torch.int32, device=dev)
        self.reasons = torch.zeros(B, dtype=torch.int32, device=dev)
        a.res_norms, a.stop_vals = self.res.data_ptr(), self.vals.data_ptr()
        a.iters, a.reasons = self.iters.data_ptr(), self.reasons.data_ptr()
        self.args = a
        self.track = track

    def run(self, H, fn_ws, fn):
        L = _lib.lib()
        wl = fn_ws(ctypes.byref(H.op), ctypes.byref(self.args))
        if wl < 0:
            _lib.check(-1, "workspace query")
        ws = _buf("ws", max(int(wl), 1), dev=self.w.device)
        ev = None
        if _lib.PROFILE is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        _lib.check(fn(ctypes.byref(H.op), ctypes.byref(self.args), ws.data_ptr(), int(wl), _lib.stream_ptr()),
                   "solver")
        _lib.note_launch(fn.__name__, 1)
        if ev is not None:
            ev[1].record()
            _lib.PROFILE.append((ev[0], ev[1], {"kernel": fn.__name__, "B": self.B, "n": self.n,
                                                "s": int(self.args.s), "nsc": int(self.args.nsc_s),
                                                "iters": self.iters}))
        self.ws = ws

    def results(self, H, flop_fn):
        # one device -> host transfer for all the per-sample scalars and histories
        m = self.max_iter + 1
        spd = getattr(self, "spd_info", None)
        spd_ok = torch.ones(1, dtype=torch.float64, device=self.iters.device) if spd is None else \
            (spd < 0).all().to(torch.float64).reshape(1)
        host = torch.cat([self.iters.to(torch.float64), self.reasons.to(torch.float64), self.res.reshape(-1),
                          self.vals.reshape(-1), self.finite.to(torch.float64).reshape(1), spd_ok]).cpu().numpy()
        if host[-2] != 1.0:
            raise ValueError("right-hand side contains non-finite entries")
        if host[-1] != 1.0:
            raise ValueError("U^T H U is not positive definite; the recycle space does not fit H")
        host = host[:-2]
        iters = host[: self.B].astype(np.int64)
        reasons = host[self.B: 2 * self.B].astype(np.int64)
        res = host[2 * self.B: 2 * self.B + self.B * m].reshape(self.B, m)
        vals = host[2 * self.B + self.B * m:].reshape(self.B, m)
        out = []
        for b in range(self.B):
            k = int(iters[b])
            why = _lib.REASONS[int(reasons[b])]
            if why == "nonspd":
                raise NonSPDError(f"curvature p^T H p <= 0 at iteration {k}; operator is not SPD")
            basis = None
            if self.basis is not None and self.want_basis:
                basis = self.basis[b, :k].T  # (n, k), contiguous columns
            out.append(SolveResult(
                solution=self.w[b], iterations=k, residual_norms=res[b, : k + 1].copy(),
                flops=flop_fn(k, self.dims[b] if hasattr(self, "dims") else 0),
                stop_reason=why, stop_values=vals[b, : k + 1].copy(), basis=basis,
                residual_vector=None if self.r is None else self.r[b]))
        return out


def _split_by_rule(rules):
    """Contiguous runs of samples sharing (rule kind, tolerance): one launch per run."""
    runs: list = []
    key_prev = None
    for b, r in enumerate(rules):
        key = (_rule_kind(r), float(r.delta))
        if key != key_prev:
            runs.append([])
            key_prev = key
        runs[-1].append(b)
    return runs


def _solve(H, g, recycle, opts, kind):
    opts = opts or SolveOptions()
    _unsupported(opts)
    G, single = _as_batch(H, g)
    B, n = G.shape
    recycles = _per_sample(recycle, B)
    rule = opts.stop_rule if isinstance(opts.stop_rule, (list, tuple)) else opts.rule()
    rules = _per_sample(rule, B)
    check = []
    for r in recycles:
        if r is None or r.dim == 0:
            continue
        if r.U.shape != r.C.shape or r.U.shape[0] != H.dim:
            raise ValueError(f"recycle space shapes U{tuple(r.U.shape)} / C{tuple(r.C.shape)} "
                             f"do not match operator dim {H.dim}")
        if not getattr(r, "orthonormal", False):  # krylov.py:402-404 for caller-built spaces
            ctc = r.C.T @ r.C
            check.append((ctc - torch.eye(r.dim, dtype=ctc.dtype, device=ctc.device)).abs().max())
    if check and float(torch.stack(check).max()) > 1e-8:
        raise ValueError("recycle space violates C^T C = I beyond 1e-8")
    groups = _split_by_rule(rules)
    results: list = [None] * B
    L = _lib.lib()
    for idx in groups:
        if len(groups) == 1:
            Hs, Gs, rs, rec = H, G, [rules[b] for b in idx], [recycles[b] for b in idx]
        else:
            Hs = _subbatch(H, idx)
            Gs = G[idx].contiguous()
            rs, rec = [rules[b] for b in idx], [recycles[b] for b in idx]
        sub_opts = opts
        if opts.initial_guess is not None:
            w0 = as_device(opts.initial_guess).reshape(B, n)
            sub_opts = SolveOptions(**{**opts.__dict__, "initial_guess": w0[idx].contiguous(), "stop_rule": None})
        if kind == "cg":
            if any(r is not None and r.dim for r in rec):
                raise ValueError("plain CG takes no recycle space; use rcg")
            launch = _Launch(Hs, Gs, [None] * len(idx), rs, sub_opts, opts.track_basis, plain_cg=True)
            launch.run(Hs, L.kr_cg_workspace, L.kr_cg)
            res = launch.results(Hs, lambda k, s: flops_cg(k, n, H.apply_cost))
        elif kind == "rcg":
            launch = _Launch(Hs, Gs, rec, rs, sub_opts, opts.track_basis, deflate=True)
            launch.run(Hs, L.kr_cg_workspace, L.kr_cg)
            res = launch.results(
                Hs, lambda k, s: flops_rcg(k, n, s, H.apply_cost) if s else flops_cg(k, n, H.apply_cost))
        else:
            launch = _Launch(Hs, Gs, rec, rs, sub_opts, opts.track_basis)
            launch.run(Hs, L.kr_rminres_workspace, L.kr_rminres)
            res = launch.results(
                Hs, lambda k, s: flops_rminres(k, n, s, H.apply_cost) if s else flops_minres(k, n, H.apply_cost))
        for b, r in zip(idx, res):
            results[b] = r
    return results[0] if single else results


def _subbatch(H, idx):
    """Operator restricted to the contiguous sample run idx."""
    if len(idx) == 1:
        return H.sample(idx[0])
    return H.slice(idx[0], idx[0] + len(idx))


def minres(H, g, opts: SolveOptions | None = None):
    """krylov.py:386-388"""
    return _solve(H, g, None, opts, "rminres")


def rminres(H, g, recycle, opts: SolveOptions | None = None):
    """krylov.py:391-405: empty recycle space -> the MINRES path of the same kernel."""
    return _solve(H, g, recycle, opts, "rminres")


def cg(H, g, opts: SolveOptions | None = None):
    """krylov.py:408-483"""
    return _solve(H, g, None, opts, "cg")


def rcg(H, g, recycle, opts: SolveOptions | None = None):
    """Recycled (deflated) CG with the recycle space (U, C = H U) as deflation
    space -- BASELINE config 1's "recycled CG"; the reference has plain cg only
    (krylov.py:408-483), so this follows the published deflated CG (Saad, Yeung,
    Erhel & Guyomarc'h, SIAM J. Sci. Comput. 21 (2000)), restated in the oracle as
    cpu_krylov.rcg.  Same options, results and NonSPDError as cg; an empty
    recycle space is plain cg."""
    return _solve(H, g, recycle, opts, "rcg")
