"""Sequence solver and hypergradient on the device (reference bilevel.py).

``SequenceSolver`` keeps, per training sample, the previous Krylov basis,
recycle space, operator and Jacobian (bilevel.py:225-288) -- all device
resident -- and solves a whole batch of samples with ONE persistent RMINRES
launch per upper step.  ``hypergradient`` is bilevel.py:291-305.
"""

from __future__ import annotations

import os
import threading
import warnings
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import torch

from .batched import gram as batched_gram, recycle_update, recycle_update_native, supports as batched_supports
from .krylov import SolveOptions, SolveResult, rcg, rminres
from .operators import (DenseOperator, FoEParams, HessianOperator, ImageVector, InpaintingProblem, Model,
                        StencilJacobian, as_device, _foe_model)
from .recycling import RecycleSpace, StrategyDescriptor, next_recycle
from .stopping import ConfigurationError, NscRule, ResidualNormRule, TrueHgErrorRule

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
    method: str = "minres"  # "minres" (reference RMINRES) or "cg" (recycled CG, BASELINE config 1)

    def __post_init__(self):
        if self.stop not in ("res", "nsc", "true-hg"):
            raise ValueError(f"unknown stop rule {self.stop!r}")
        if self.method not in ("minres", "cg"):
            raise ValueError(f"unknown Krylov method {self.method!r}")
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


_LINALG_WARM = False


def _warm_linalg():
    """torch initialises its cuSOLVER / linalg backends lazily and not thread-safely;
    touch every routine next_recycle uses once on the calling thread first."""
    global _LINALG_WARM
    if _LINALG_WARM:
        return
    a = torch.eye(4, dtype=torch.float64, device="cuda") * 2.0
    torch.linalg.cholesky_ex(a)
    torch.linalg.qr(a)
    # the tall Householder QR of the rank-drop path uses other cuSOLVER kernels than a
    # 4 x 4 one; load them now rather than inside a timed step
    torch.linalg.qr(torch.randn(4096, 64, dtype=torch.float64, device="cuda"))
    torch.linalg.eigh(torch.randn(64, 64, dtype=torch.float64, device="cuda"))
    torch.linalg.eigh(a)
    torch.linalg.eigvalsh(a)
    torch.linalg.svdvals(a)
    torch.linalg.solve_triangular(a, a, upper=True)
    torch.linalg.cholesky(a)
    torch.argsort(a[0], stable=True)
    torch.cuda.synchronize()
    _LINALG_WARM = True


def _warm_thread(shape=None):
    """The library routines of the recycle update, once on the calling thread at the
    shapes they run at (handle creation and kernel selection are per thread)."""
    a = torch.randn(64, 64, dtype=torch.float64, device="cuda")
    g = a @ a.T + 64 * torch.eye(64, dtype=torch.float64, device="cuda")
    torch.linalg.cholesky_ex(g)
    torch.linalg.solve_triangular(torch.linalg.cholesky(g), g, upper=False)
    torch.linalg.qr(torch.randn(4096, 64, dtype=torch.float64, device="cuda"))
    torch.linalg.eigh(g)
    torch.linalg.eigvalsh(g)
    torch.bmm(a.unsqueeze(0), a.unsqueeze(0))
    # the library's own cuSOLVER handle (rank-deficient Householder branch) is per host thread as well
    from . import _lib
    from .batched import gram
    gram(torch.zeros(1, 2, 4096, dtype=torch.float64, device="cuda"))
    _lib.check(_lib.lib().kr_thread_warmup(), "kr_thread_warmup")
    torch.cuda.current_stream().synchronize()


_PHASE_DEBUG = os.environ.get("KR_SOLVE_DEBUG") is not None
# sample-group streams at high priority: the orchestrator's H W (thousands of blocks) runs
# on a lowest-priority side stream, so the other group's latency-bound kernels are not
# queued behind it (KR_GROUP_PRIORITY=0 restores default priorities)
_GROUP_PRIORITY = int(os.environ.get("KR_GROUP_PRIORITY", "-1"))


def _phase_clock():
    """Synchronised wall clock for KR_SOLVE_DEBUG phase timing (None when off)."""
    if not _PHASE_DEBUG:
        return None
    import time
    torch.cuda.synchronize()
    return time.perf_counter()


class SequenceSolver:
    """Solves consecutive Hessian systems of a batch of samples, carrying the
    recycling state of each sample (bilevel.py:225-288).

    ``solve(H, g, J)`` with a single-sample operator and g of shape (n,)
    returns ``(SolveResult, RecycleSpace)`` like the reference; with a batched
    operator and g of shape (B, n) it returns two lists.
    """

    def __init__(self, cfg: HessianSolveConfig):
        self.cfg = cfg
        self._first = True
        self._prev_basis: list | None = None
        self._prev_recycle: list | None = None
        self._prev_h = None
        self._prev_jac = None
        self._prev_solution = None
        self.max_workers = 8
        self.batched_update = True
        self.groups = int(os.environ.get("KR_RECYCLE_GROUPS", "4"))
        # the update orchestrated in C++ (kr_recycle_update); 0 = the torch orchestration
        self.native_update = os.environ.get("KR_NATIVE_RECYCLE", "1") != "0"
        # per-group solves overlapping the other groups' recycle updates (KR_PIPELINE=1).  Off by
        # default: a persistent solve launched while another group's full-GPU kernels are still
        # dispatching gets only part of its blocks resident, the resident ones spin at the
        # per-sample barriers and hold SMs, and the step got slower (C2: 23 -> 28 ms)
        self.pipelined = os.environ.get("KR_PIPELINE", "0") == "1"
        self._gstreams = None
        self._gpool = None
        self._scratch = {}  # per sample group: the native update's temporaries
        self.sort_groups = os.environ.get("KR_SORT_GROUPS", "1") != "0"
        self._streams = None
        self._pool = None

    def _needs_basis(self) -> bool:
        return not self.cfg.strategy.is_none

    def reserve(self, batch: int, nbytes: int, shape: tuple[int, int] | None = None) -> None:
        """Pre-size the caching-allocator pools of the per-sample worker streams (each
        stream has its own pool) so steady-state steps never call cudaMalloc."""
        # the allocator's small-block pool (blocks <= 1 MB, 2 MB segments) on the caller's
        # stream: the per-solve vectors (w, r, histories) come from it
        small = [torch.empty(1 << 17, dtype=torch.float64, device="cuda") for _ in range(24)]
        del small
        if batch <= 1 or self.max_workers <= 1:
            return
        _warm_linalg()
        ng = max(1, min(self.groups, batch))
        if self.batched_update and ng > 1:
            if self._gstreams is None or len(self._gstreams) < ng:
                self._gstreams = [torch.cuda.Stream(priority=_GROUP_PRIORITY) for _ in range(ng)]
                self._gpool = ThreadPoolExecutor(max_workers=ng)
            # only the lanes that will run (see _recycle_batched) get a pool
            per_group = -(-batch // ng) * nbytes
            budget = int(0.45 * torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)
            nl = max(1, min(ng, budget // max(per_group, 1)))
            for st in self._gstreams[:nl]:
                with torch.cuda.stream(st):
                    torch.empty(min(per_group, budget // nl) // 8, dtype=torch.float64, device="cuda")
            # torch creates cuBLAS / cuSOLVER handles per host thread on first use (tens of
            # ms): touch them on every worker thread now, not inside a step
            gate = threading.Barrier(ng)

            def warm(g):
                gate.wait()
                with torch.cuda.stream(self._gstreams[g]):
                    _warm_thread(shape)
                return g

            list(self._gpool.map(warm, range(ng)))
            # group 0 runs on the calling thread (_recycle_batched): warm its handles too
            with torch.cuda.stream(self._gstreams[0]):
                _warm_thread(shape)
            torch.cuda.synchronize()
            return
        if self._streams is None or len(self._streams) < batch:
            self._streams = [torch.cuda.Stream() for _ in range(batch)]
            self._pool = ThreadPoolExecutor(max_workers=min(batch, self.max_workers))
        for st in self._streams:
            with torch.cuda.stream(st):
                torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()

    def _batched(self, hessian, jac) -> bool:
        """Whether the whole-batch recycle update (batched.recycle_update) applies."""
        st = self.cfg.strategy
        if not self.batched_update or not batched_supports(st, native=self.native_update):
            return False
        if not isinstance(hessian, HessianOperator) or isinstance(hessian, DenseOperator):
            return False
        if st.placement != "outer" and not isinstance(self._prev_h, HessianOperator):
            return False
        return st.vec_type in ("Ritz", "HRitz") or isinstance(jac, StencilJacobian)

    def _group_members(self, B: int, ng: int):
        """Sample groups of the batched update.  Sorted by candidate width t_b (default):
        each group's update is padded to its widest sample, so grouping similar widths cuts
        the padded H W columns and n x T^2 GEMM work (C3: ~26 % / ~40 % less than contiguous
        groups).  KR_SORT_GROUPS=0: contiguous sample ranges."""
        if not self.sort_groups or self.pipelined or self._prev_basis is None:
            return [list(range(g * B // ng, (g + 1) * B // ng)) for g in range(ng)]
        t = [(0 if V is None else int(V.shape[1])) + (0 if r is None else int(r.dim))
             for V, r in zip(self._prev_basis, self._prev_recycle)]
        order = sorted(range(B), key=lambda b: (t[b], b))
        return [order[g * B // ng: (g + 1) * B // ng] for g in range(ng)]

    def _recycle_batched(self, hessian, jac, B, then=None):
        """Whole-batch recycle update in ``groups`` sample groups, each on its own host
        thread and CUDA stream: a group's latency-bound t x t kernels (one CTA per
        sample) overlap the other groups' GEMMs and stencils."""
        cfg = self.cfg
        ng = max(1, min(self.groups, B))
        members = self._group_members(B, ng)
        shared = None
        if self.native_update:
            # whole-batch (B, s, n) outputs, each group writing its rows: the solve then
            # reads U, C, Z in place (no per-sample restacking)
            s, n = cfg.recycle_dim, hessian.dim
            dev = (hessian.model.device if getattr(hessian, "model", None) is not None
                   else torch.device("cuda", torch.cuda.current_device()))
            f64 = dict(dtype=torch.float64, device=dev)
            shared = (torch.empty(B, s, n, **f64), torch.empty(B, s, n, **f64),
                      torch.empty(B, s, n, **f64) if cfg.strategy.vec_type == "RGen" else None)
            # Z^T C of every group's rows, formed on the group's stream right after its update
            # (off the path between the last update and the solve launch)
            ztc = torch.empty(B, s, s, **f64) if shared[2] is not None else None

        # concurrent lanes: each lane runs its groups one after another on its own stream with
        # one set of scratch buffers (H W, W, candidates, QR workspaces: ~48 n t bytes per
        # sample); as many lanes as the memory budget holds (C2/C3: one per group; C4 -- 16
        # samples x 512^2 x t 540 -- two)
        tcap = cfg.max_iter + cfg.recycle_dim + 1
        per_group = 48 * hessian.dim * tcap * max(len(m) for m in members)
        budget = int(0.45 * torch.cuda.get_device_properties(torch.cuda.current_device()).total_memory)
        nl = max(1, min(ng, budget // max(per_group, 1)))

        def run(g, idx):
            lo, hi = idx[0], idx[-1] + 1
            contiguous = idx == list(range(lo, hi))
            inner = cfg.strategy.placement != "outer"
            hp = None
            if contiguous:
                hs = hessian if (lo, hi) == (0, B) else hessian.slice(lo, hi)
                js = jac if (lo, hi) == (0, B) or jac is None else jac.slice(lo, hi)
                if inner:  # inner placement projects with the previous system's operator
                    hp = self._prev_h if (lo, hi) == (0, B) else self._prev_h.slice(lo, hi)
            else:  # the group's per-sample tables gathered (a few hundred MB at C3: ~0.1 ms)
                hs = hessian.select(idx)
                js = None if jac is None else jac.select(idx, hs)
                if inner:
                    hp = self._prev_h.select(idx)
            bases = [self._prev_basis[i] for i in idx]
            prevs = [self._prev_recycle[i] for i in idx]
            if self.native_update:
                sc = self._scratch.setdefault(g % nl, {"tcap": tcap})
                if contiguous:
                    out = tuple(None if x is None else x[lo:hi] for x in shared)
                    recs = recycle_update_native(cfg.strategy, cfg.recycle_dim, hs, js, bases, prevs,
                                                 cfg.reuse_products, scratch=sc, out=out, out_src=shared + (lo, ztc),
                                                 H_proj=hp)
                    full = all(r is not None and r.dim == cfg.recycle_dim for r in recs)
                    if ztc is not None and full:
                        ztc[lo:hi] = batched_gram(shared[2][lo:hi], shared[1][lo:hi])
                else:
                    # group-local outputs, then scattered into the whole-batch rows the solve reads
                    nb = len(idx)
                    loc = sc.get("out")
                    if loc is None or loc[0].shape[0] != nb:
                        loc = tuple(None if x is None else torch.empty(nb, *x.shape[1:], dtype=x.dtype, device=x.device)
                                    for x in shared)
                        sc["out"] = loc
                    recs = recycle_update_native(cfg.strategy, cfg.recycle_dim, hs, js, bases, prevs,
                                                 cfg.reuse_products, scratch=sc, out=loc, out_src=None, H_proj=hp)
                    it = torch.as_tensor(idx, dtype=torch.long, device=shared[0].device)
                    for x, y in zip(shared, loc):
                        if x is not None:
                            x.index_copy_(0, it, y)
                    full = all(r is not None and r.dim == cfg.recycle_dim for r in recs)
                    if ztc is not None and full:
                        ztc.index_copy_(0, it, batched_gram(loc[2], loc[1]))
                    recs = [self._rebase(r, shared, idx[i], ztc) for i, r in enumerate(recs)]
            else:
                recs = recycle_update(cfg.strategy, cfg.recycle_dim, hs, js, bases, prevs, cfg.reuse_products)
            # samples the batched path declined take the per-sample reference path
            return [r if r is not None else self._recycle_one(hessian, jac, B, idx[i]) for i, r in enumerate(recs)]

        def assemble(parts):
            out = [None] * B
            for idx, recs in zip(members, parts):
                for i, r in zip(idx, recs):
                    out[i] = r
            return out

        if ng == 1:
            recs = run(0, members[0])
            return recs if then is None else (recs, then(0, B, recs))
        main = torch.cuda.current_stream()
        if self._gstreams is None or len(self._gstreams) < ng:
            _warm_linalg()
            self._gstreams = [torch.cuda.Stream(priority=_GROUP_PRIORITY) for _ in range(ng)]
            self._gpool = ThreadPoolExecutor(max_workers=ng)

        def work(g):
            st = self._gstreams[g % nl]
            st.wait_stream(main)
            extra = None
            idx = members[g]
            with torch.cuda.stream(st):
                recs = run(g, idx)
                if then is not None:  # the group's own solve, overlapping the other groups' updates
                    if idx != list(range(idx[0], idx[-1] + 1)):
                        raise RuntimeError("pipelined solves need contiguous sample groups (KR_SORT_GROUPS=0)")
                    extra = then(idx[0], idx[-1] + 1, recs)
            for rec in recs:
                for t in (rec.U, rec.C) + ((rec.nsc_data.values, rec.nsc_data.v_h, rec.nsc_data.w,
                                           rec.nsc_data.z_block()) if rec.nsc_data is not None else ()):
                    if t is not None:
                        t.record_stream(main)
            for r in extra or ():
                for t in (r.solution, r.basis, r.residual_vector):
                    if t is not None:
                        t.record_stream(main)
            return recs, extra

        def lane(l):
            return [work(g) for g in range(l, ng, nl)]

        # lanes 1.. on the pool, lane 0 on this thread (one thread hand-off fewer)
        futs = [self._gpool.submit(lane, l) for l in range(1, nl)]
        done = [lane(0)] + [f.result() for f in futs]
        parts = [None] * ng
        for l, res in enumerate(done):
            for j, r in enumerate(res):
                parts[l + j * nl] = r
        for l in range(nl):
            main.wait_stream(self._gstreams[l])
        out = assemble([recs for recs, _ in parts])
        if then is None:
            return out
        return out, [r for _, extra in parts for r in extra]

    @staticmethod
    def _rebase(rec, shared, b, ztc):
        """The recycle space ``rec`` (group-local rows) re-pointed at row b of the whole-batch
        buffers it was copied into, so the solve reads it in place."""
        from .stopping import NscData

        if rec is None or rec.dim == 0:
            return rec
        d = rec.dim
        nd = rec.nsc_data
        if nd is not None and shared[2] is not None:
            nd = NscData(values=nd.values, v_h=nd.v_h, w=nd.w, z=shared[2][b, :d].T)
        return RecycleSpace(U=shared[0][b, :d].T, C=shared[1][b, :d].T, nsc_data=nd, orthonormal=True,
                            batch_src=(shared[0], shared[1], shared[2], b, ztc))

    def _recycle_one(self, hessian, jac, B, b):
        cfg = self.cfg
        hb = hessian if B == 1 else hessian.sample(b)
        jb = jac if (B == 1 or jac is None) else jac.sample(b)
        hp = None if self._prev_h is None else (self._prev_h if B == 1 else self._prev_h.sample(b))
        jp = None if self._prev_jac is None else (self._prev_jac if B == 1 else self._prev_jac.sample(b))
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            return next_recycle(cfg.strategy, h_current=hb, h_previous=hp, jac_current=jb, jac_previous=jp,
                                prev_basis=self._prev_basis[b], prev_recycle=self._prev_recycle[b],
                                s=cfg.recycle_dim, dense_limit=cfg.dense_limit, reuse_products=cfg.reuse_products)

    def _recycle_all(self, hessian, jac, B):
        """next_recycle for every sample.  The per-sample updates are independent and
        dominated by latency-bound t x t decompositions, so with B > 1 each sample runs
        on its own host thread and CUDA stream (torch releases the GIL inside ops);
        the caller's stream waits for all of them."""
        if self._batched(hessian, jac):
            return self._recycle_batched(hessian, jac, B)
        if B == 1 or self.max_workers <= 1:
            return [self._recycle_one(hessian, jac, B, b) for b in range(B)]
        main = torch.cuda.current_stream()
        if self._streams is None or len(self._streams) < B:
            _warm_linalg()
            self._streams = [torch.cuda.Stream() for _ in range(B)]
            self._pool = ThreadPoolExecutor(max_workers=min(B, self.max_workers))

        def work(b):
            st = self._streams[b]
            st.wait_stream(main)
            with torch.cuda.stream(st):
                rec = self._recycle_one(hessian, jac, B, b)
            for t in (rec.U, rec.C) + ((rec.nsc_data.values, rec.nsc_data.v_h, rec.nsc_data.w)
                                       if rec.nsc_data is not None and rec.nsc_data.w is not None else ()):
                t.record_stream(main)
            return rec

        recs = list(self._pool.map(work, range(B)))
        for b in range(B):
            main.wait_stream(self._streams[b])
        return recs

    def _options(self, recycles, init, hessian=None, jac=None):
        """Stop rules per sample (bilevel.py:264-276) and the solve options."""
        cfg = self.cfg
        rules = []
        B = len(recycles)
        for b, rec in enumerate(recycles):
            if cfg.stop == "true-hg":  # bilevel.py:267-268 (an experiment oracle)
                hb = hessian if B == 1 else hessian.sample(b)
                jb = jac if B == 1 else jac.sample(b)
                rules.append(TrueHgErrorRule(cfg.delta, jb, hb, cfg.inner_tol, cfg.dense_limit))
            elif cfg.stop == "nsc" and rec.nsc_data is not None:
                rules.append(NscRule(cfg.delta, rec.nsc_data))
            else:  # res, or nsc on the first system (bilevel.py:269-273)
                rules.append(ResidualNormRule(cfg.delta))
        # the residual vector is not materialised (the reference's SequenceSolver never reads
        # it; NSC runs in s-space on the device)
        return SolveOptions(max_iter=cfg.max_iter, stop_rule=rules if len(rules) > 1 else rules[0],
                            track_basis=self._needs_basis(), initial_guess=init, residual_vector=False)

    def solve(self, hessian, g, jac):
        cfg = self.cfg
        g = as_device(g)
        single = g.dim() == 1
        B = 1 if single else g.shape[0]
        n = hessian.dim
        # one batched solve for all samples: the persistent kernel is latency bound per
        # iteration, so a launch over 8 samples costs what one over 4 does
        t0 = _phase_clock()
        init = self._prev_solution if cfg.warm_start else None
        if isinstance(init, list):
            init = torch.stack(init)
        solve = rminres if cfg.method == "minres" else rcg
        results = None
        if cfg.strategy.is_none or self._first:
            recycles = [RecycleSpace.empty(n) for _ in range(B)]
        elif self.pipelined and B > 1 and self._batched(hessian, jac) and min(self.groups, B) > 1:
            # each sample group solves right after its own recycle update, on its own
            # stream: group A's solve overlaps group B's (latency-bound) update kernels.
            # Per-sample results are bitwise those of one batched launch (same blocks per sample).
            def then(lo, hi, recs):
                hs = hessian.slice(lo, hi)
                w0 = None if init is None else init[lo:hi].contiguous()
                return solve(hs, g[lo:hi], recs, self._options(recs, w0, hs, jac.slice(lo, hi)))

            recycles, results = self._recycle_batched(hessian, jac, B, then=then)
        else:
            recycles = self._recycle_all(hessian, jac, B)
        t1 = _phase_clock()
        self._first = False
        if results is None:
            results = solve(hessian, g, recycles if B > 1 else recycles[0],
                            self._options(recycles, init, hessian, jac))
        if t0 is not None:
            t2 = _phase_clock()
            import sys
            print(f"solve phases: recycle {1e3 * (t1 - t0):.1f} ms, krylov {1e3 * (t2 - t1):.1f} ms", file=sys.stderr)
        res_list = [results] if single else results
        self._prev_basis = [r.basis for r in res_list]
        self._prev_recycle = recycles
        self._prev_h = hessian
        self._prev_jac = jac
        # kept as views; stacked only when a warm start asks for it (no per-step allocation)
        self._prev_solution = [r.solution for r in res_list] if not single else res_list[0].solution
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
