"""Shared test helpers: matching oracle (CPU) and device models on the same seeded inputs."""

from __future__ import annotations

import numpy as np

from oracle import cpu_imaging as im


def oracle_models(kind: str, rows: int, cols: int, batch: int, seed: int = 0, *, blur: int = 9, sigma: float = 1.5,
                  J: int = 3, q: int = 5, eps: float = 1e-2):
    """Seeded oracle models (one per sample) sharing theta, and theta, x_hats, x_trues."""
    rng = np.random.default_rng(seed)
    n = rows * cols
    shape = (rows, cols)
    models, x_trues = [], []
    taps = im.gaussian_taps(blur, sigma)
    for b in range(batch):
        xt = np.clip(im.piecewise_constant(max(rows, cols), rng)[:rows, :cols], 0, 1).ravel()
        if kind == "foe":
            m = int(np.ceil(0.4 * n))
            mask = np.sort(rng.permutation(n)[:m])
            y = xt[mask] + 0.05 * rng.standard_normal(m)
            data = im.DataTerm("mask", shape, y, scale=1.0, ridge=1e-3, mask_rows=mask, x_true=xt)
            reg = im.Regularizer("filters", J, q, "quadratic")
        else:
            ax = im.conv_same(xt.reshape(shape), np.outer(taps, taps)).ravel()
            y = ax + 0.01 * rng.standard_normal(n)
            data = im.DataTerm("blur", shape, y, scale=2.0, ridge=0.0, taps=taps, x_true=xt)
            if kind == "tv":
                reg = im.Regularizer("tv", eps=eps)
            else:
                reg = im.Regularizer("filters", J, q, "smooth_abs", eps)
        models.append(im.Model(data, reg))
        x_trues.append(xt)
    reg = models[0].reg
    if reg.kind == "tv":
        theta = np.array([-3.0 + 0.2 * rng.standard_normal()])
    else:
        ks = [0.3 * rng.standard_normal((q, q)) for _ in range(J)]
        theta = im.pack_theta(-1.0 + 0.3 * rng.standard_normal(J), ks)
    x_hats = [xt + 0.05 * rng.standard_normal(n) for xt in x_trues]
    return models, theta, np.stack(x_hats), np.stack(x_trues)


def device_model(models):
    """paper_2412_08264_b200.Model equivalent of a list of oracle models."""
    from paper_2412_08264_b200.operators import Model, as_device

    d0, reg = models[0].data, models[0].reg
    B, n = len(models), d0.n
    ys, masks = [], []
    for m in models:
        d = m.data
        if d.kind == "mask":
            ysc = np.zeros(n)
            ysc[d.mask_rows] = d.y
            ys.append(ysc)
            masks.append(d.mask_diag())
        else:
            ys.append(d.y)
    return Model(shape=tuple(d0.shape), batch=B, data_kind=d0.kind, data_scale=d0.scale, ridge=d0.ridge,
                 y=as_device(np.stack(ys)), x_true=as_device(np.stack([m.data.x_true for m in models])),
                 mask=as_device(np.stack(masks)) if masks else None, taps=d0.taps, reg_kind=reg.kind,
                 potential=reg.potential, eps=reg.eps, num_filters=reg.num_filters, ksize=reg.ksize)


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    den = max(np.linalg.norm(b), 1e-300)
    return float(np.linalg.norm(a - b) / den)


def to_np(t):
    return t.detach().cpu().numpy()
