"""Frozen sequences of Hessian systems: recording and the ``krecycle-sequence-v1`` layout.

The reference freezes every upper-level system of a recycling-free bilevel run
(``record_sequence``, experiments.py:234-268) and stores it as a directory
(``save_sequence`` / ``load_sequence``, experiments.py:673-775): ``manifest.json``
plus flat little-endian float64 arrays under ``arrays/``.  Here the same layout is
kept for a BATCH of deblurring samples sharing theta (the BASELINE configs):

    manifest.json            format "krecycle-sequence-v1", problem "deblur-batch",
                             config (problems.DeblurConfig fields), first sample,
                             batch, shape, n, p, num_systems, per-system metadata
    arrays/xtrue.f64         [batch][n]
    arrays/y.f64             [batch][n]
    arrays/theta_XXX.f64     [p]
    arrays/xhat_XXX.f64      [batch][n]      (the system's lower-level solutions)
    arrays/theta_next_XXX.f64

g = xhat - xtrue is not stored (the reference stores it and checks it against
xhat - xtrue to 1e-12, experiments.py:221-231; it is recomputed here).
``record`` runs the device upper loop (lower.gradient_descent: batched L-BFGS to
``lower_gtol``, Armijo backtracking, recycling-free hypergradient solves) and
freezes every system it visits.
"""

from __future__ import annotations

import json
from dataclasses import asdict, dataclass, field
from pathlib import Path

import numpy as np
import torch

from .operators import Model, as_device
from .problems import DeblurConfig, gaussian_taps, make_batch

__all__ = ["FORMAT_NAME", "FrozenSequence", "FrozenSystem", "load_sequence", "record", "save_sequence",
           "solve_path"]

FORMAT_NAME = "krecycle-sequence-v1"


@dataclass
class FrozenSystem:
    """One frozen upper-level system (experiments.py:180-196 SystemRecord)."""

    index: int
    theta: np.ndarray
    x_hats: np.ndarray            # [batch, n]
    iterations: list = field(default_factory=list)
    cost: float = float("nan")
    grad_norm: float = float("nan")
    beta_init: float = float("nan")
    theta_next: np.ndarray | None = None


@dataclass
class FrozenSequence:
    """A batch problem plus its frozen systems (experiments.py:198-231 SequenceRecord)."""

    config: DeblurConfig
    first: int
    x_true: np.ndarray            # [batch, n]
    y: np.ndarray                 # [batch, n]
    systems: list
    notes: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return int(self.x_true.shape[0])

    def __len__(self) -> int:
        return len(self.systems)

    def model(self, device=None) -> Model:
        """Device model of the sequence's samples (the stored data, not regenerated)."""
        c = self.config
        return Model(shape=(c.size, c.size), batch=self.batch, data_kind="blur", data_scale=2.0, ridge=0.0,
                     y=as_device(self.y, device), x_true=as_device(self.x_true, device),
                     taps=gaussian_taps(c.blur_size, c.blur_sigma), reg_kind=c.reg, potential="smooth_abs",
                     eps=c.eps, num_filters=c.num_filters, ksize=c.kernel_size)

    def validate(self):
        n = self.x_true.shape[1]
        for rec in self.systems:
            if rec.x_hats.shape != (self.batch, n):
                raise ValueError(f"system {rec.index}: x_hat of shape {rec.x_hats.shape}, expected {(self.batch, n)}")
            if not np.all(np.isfinite(rec.x_hats)) or not np.all(np.isfinite(rec.theta)):
                raise ValueError(f"system {rec.index}: non-finite entries")


def _write(path: Path, a) -> None:
    path.write_bytes(np.asarray(a, dtype="<f8").ravel().tobytes())


def _read(path: Path) -> np.ndarray:
    return np.frombuffer(path.read_bytes(), dtype="<f8").copy()


def save_sequence(seq: FrozenSequence, out_dir) -> Path:
    """experiments.py:680-723 for a batch."""
    out = Path(out_dir)
    arrays = out / "arrays"
    arrays.mkdir(parents=True, exist_ok=True)
    _write(arrays / "xtrue.f64", seq.x_true)
    _write(arrays / "y.f64", seq.y)
    meta = []
    for rec in seq.systems:
        tag = f"{rec.index:03d}"
        _write(arrays / f"theta_{tag}.f64", rec.theta)
        _write(arrays / f"xhat_{tag}.f64", rec.x_hats)
        if rec.theta_next is not None:
            _write(arrays / f"theta_next_{tag}.f64", rec.theta_next)
        meta.append({"index": rec.index, "iterations": [int(v) for v in rec.iterations], "cost": float(rec.cost),
                     "grad_norm": float(rec.grad_norm), "beta_init": float(rec.beta_init),
                     "has_theta_next": rec.theta_next is not None})
    c = seq.config
    manifest = {
        "format": FORMAT_NAME,
        "problem": "deblur-batch",
        "config": asdict(c),
        "first_sample": seq.first,
        "batch": seq.batch,
        "shape": [c.size, c.size],
        "n": int(seq.x_true.shape[1]),
        "p": int(seq.systems[0].theta.size) if seq.systems else 0,
        "num_systems": len(seq.systems),
        "systems": meta,
        "notes": {"array_format": "flat little-endian float64, sample-major", **seq.notes},
    }
    (out / "manifest.json").write_text(json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return out


def load_sequence(in_dir) -> FrozenSequence:
    """experiments.py:726-775 for a batch; raises ValueError on a foreign directory."""
    root = Path(in_dir)
    manifest = json.loads((root / "manifest.json").read_text())
    if manifest.get("format") != FORMAT_NAME:
        raise ValueError(f"{root}: not a {FORMAT_NAME} directory")
    if manifest.get("problem") != "deblur-batch":
        raise ValueError(f"{root}: problem {manifest.get('problem')!r} is not a deblurring batch "
                         "(the reference's FoE-inpainting sequences load with krecycle.experiments.load_sequence)")
    cfg = DeblurConfig(**manifest["config"])
    B, n = int(manifest["batch"]), int(manifest["n"])
    arrays = root / "arrays"
    systems = []
    for m in manifest["systems"]:
        tag = f"{m['index']:03d}"
        systems.append(FrozenSystem(
            index=int(m["index"]), theta=_read(arrays / f"theta_{tag}.f64"),
            x_hats=_read(arrays / f"xhat_{tag}.f64").reshape(B, n), iterations=list(m["iterations"]),
            cost=m["cost"], grad_norm=m["grad_norm"], beta_init=m["beta_init"],
            theta_next=_read(arrays / f"theta_next_{tag}.f64") if m["has_theta_next"] else None))
    seq = FrozenSequence(cfg, int(manifest["first_sample"]), _read(arrays / "xtrue.f64").reshape(B, n),
                         _read(arrays / "y.f64").reshape(B, n), systems, manifest.get("notes", {}))
    seq.validate()
    return seq


def record(cfg: DeblurConfig, systems: int, *, first: int = 0, count: int | None = None, lower_gtol: float = 1e-8,
           delta: float = 1e-2, max_inner: int | None = None, lower_max_iter: int = 20000, device=None,
           theta0=None, eps_stop: float = 0.0, linesearch=None) -> FrozenSequence:
    """Record ``systems`` upper-level systems of the recycling-free bilevel run
    (experiments.py:234-268): device L-BFGS to ``lower_gtol``, Armijo upper steps,
    hypergradients with RMINRES (no recycling, residual rule ``delta``)."""
    from .lower import record_sequence
    from .problems import theta0 as default_theta0

    model = make_batch(cfg, first, count, device=device)
    th0 = default_theta0(cfg) if theta0 is None else np.asarray(theta0, dtype=float)
    trace = record_sequence(model, th0, delta=delta, max_inner=max_inner or cfg.max_iter, lower_gtol=lower_gtol,
                            eps_stop=max(eps_stop, 1e-300), max_upper=systems, lower_max_iter=lower_max_iter,
                            linesearch=linesearch)
    recs = []
    for i, r in enumerate(trace):
        nxt = trace[i + 1].theta if i + 1 < len(trace) else None
        recs.append(FrozenSystem(r.index, np.asarray(r.theta, dtype=float).copy(),
                                 r.x_hats.detach().cpu().numpy().copy(), list(r.iterations), r.cost, r.grad_norm,
                                 r.beta_init, None if nxt is None else np.asarray(nxt, dtype=float).copy()))
    seq = FrozenSequence(cfg, first, model.x_true.cpu().numpy().copy(), model.y.cpu().numpy().copy(), recs,
                         {"recorder": "paper_2412_08264_b200.lower.record_sequence (device L-BFGS + Armijo GD)",
                          "lower_gtol": lower_gtol, "delta": delta,
                          "beta0": None if linesearch is None else linesearch.beta})
    seq.validate()
    return seq


def solve_path(cfg: DeblurConfig, thetas, *, first: int = 0, count: int | None = None, lower_gtol: float = 1e-6,
               lower_max_iter: int = 5000, device=None) -> FrozenSequence:
    """Frozen systems at a prescribed theta path: x_hat_i = the device L-BFGS minimiser of
    the lower problem at theta_i (bilevel.py:81-167, to gradient norm ``lower_gtol``),
    warm-started from x_hat_{i-1}.  The systems are real lower-level solutions (H and
    g = x_hat - x_true as a bilevel run produces them); only the upper-level path is
    prescribed instead of taken by gradient descent (one lower solve per system instead
    of a line search of them)."""
    from .lower import lower_solve

    model = make_batch(cfg, first, count, device=device)
    recs, x = [], None
    for i, th in enumerate(thetas):
        th = np.asarray(th, dtype=float)
        x, st = lower_solve(model, th, x, gtol=lower_gtol, max_iter=lower_max_iter)
        diff = x - model.x_true
        cost = float((0.5 * (diff * diff).sum(dim=1)).sum())
        recs.append(FrozenSystem(i, th.copy(), x.detach().cpu().numpy().copy(), [int(v) for v in st.iterations],
                                 cost, float("nan"), float("nan"),
                                 np.asarray(thetas[i + 1], dtype=float).copy() if i + 1 < len(thetas) else None))
    seq = FrozenSequence(cfg, first, model.x_true.cpu().numpy().copy(), model.y.cpu().numpy().copy(), recs,
                         {"recorder": "sequence.solve_path (device L-BFGS minimiser at each theta of a prescribed "
                                      "path; iterations = L-BFGS iterations)", "lower_gtol": lower_gtol})
    seq.validate()
    return seq
