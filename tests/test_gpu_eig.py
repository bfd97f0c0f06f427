"""kr_syev_select (one-CTA selected eigenpairs) against numpy's LAPACK eigh.

Oracle: numpy.linalg.eigh (dsyevd), the eigensolver the reference's
ritz_select uses (recycling.py:233); selection = _select_indices
(recycling.py:202-213) after _clamp_dim.  Eigenvectors are compared as
|cos| = 1 (sign is arbitrary in LAPACK too) when the eigenvalue is separated
from the rest of the spectrum, and through the spanned projector for clusters.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _select(t, s, size):
    s = min(s, t)
    if size == "S":
        return np.arange(s)
    if size == "L":
        return np.arange(t - s, t)
    lo = s // 2
    return np.concatenate([np.arange(lo), np.arange(t - (s - lo), t)])


def _check(M_list, size, s, tol_val=1e-12, tol_vec=1e-9):
    from paper_2412_08264_b200.batched import syev_select

    B = len(M_list)
    T = max(m.shape[0] for m in M_list)
    Mp = np.zeros((B, T, T))
    for b, m in enumerate(M_list):
        Mp[b, : m.shape[0], : m.shape[0]] = m
        Mp[b, m.shape[0]:, :] = np.nan  # pad content must not matter
        Mp[b, :, m.shape[0]:] = np.nan
    dims = torch.tensor([m.shape[0] for m in M_list], dtype=torch.int32)
    lam, Z, nsel = syev_select(torch.as_tensor(Mp, device="cuda"), dims, size, s)
    lam, Z, nsel = lam.cpu().numpy(), Z.cpu().numpy(), nsel.cpu().numpy()
    for b, m in enumerate(M_list):
        t = m.shape[0]
        w, V = np.linalg.eigh(0.5 * (m + m.T))
        idx = _select(t, s, size)
        assert nsel[b] == len(idx)
        scale = max(np.abs(w).max(), 1e-300)
        assert np.max(np.abs(lam[b, : len(idx)] - w[idx])) <= tol_val * scale, (b, lam[b, : len(idx)], w[idx])
        Zb = Z[b, : len(idx), :t].T  # t x s
        assert np.all(Z[b, : len(idx), t:] == 0) and np.all(Z[b, len(idx):] == 0)
        assert np.max(np.abs(Zb.T @ Zb - np.eye(len(idx)))) <= 1e-12
        # residual ||M z - lambda z|| small for every selected pair
        res = np.linalg.norm(m @ Zb - Zb * w[idx], axis=0)
        assert np.max(res) <= 1e-11 * scale * np.sqrt(t), res
        # vectors of isolated eigenvalues match LAPACK up to sign
        gaps = np.array([np.min(np.abs(np.delete(w, i) - w[i])) if t > 1 else np.inf for i in idx])
        for q, i in enumerate(idx):
            if gaps[q] > 1e-6 * scale:
                c = abs(Zb[:, q] @ V[:, i])
                assert abs(1 - c) <= tol_vec * (scale / gaps[q]) ** 2 + 1e-12, (b, q, c, gaps[q])
                k = np.argmax(np.abs(Zb[:, q]))
                assert Zb[k, q] > 0


def _rand_sym(rng, t, eigs=None):
    Q, _ = np.linalg.qr(rng.standard_normal((t, t)))
    if eigs is None:
        eigs = rng.standard_normal(t)
    return (Q * eigs) @ Q.T


@pytest.mark.parametrize("size", ["S", "L", "M"])
def test_random_batches_mixed_sizes(size):
    rng = np.random.default_rng(3)
    mats = [_rand_sym(rng, t) for t in (1, 2, 3, 17, 64, 150, 220, 228)]
    _check(mats, size, 20)


def test_gram_like_spectra():
    """Q1^T Q1 of an orthonormal (p + t) x t block with p < t: eigenvalues in [0, 1],
    a zero cluster of size t - p, strongly graded top end (the GSVD input)."""
    rng = np.random.default_rng(5)
    mats = []
    for t, p in ((220, 208), (150, 40), (60, 80)):
        Q, _ = np.linalg.qr(rng.standard_normal((p + t, t)) * np.logspace(0, -6, t))
        Q1 = Q[:p]
        mats.append(Q1.T @ Q1)
    _check(mats, "L", 20)
    _check(mats, "S", 20, tol_vec=1.0)  # the zero cluster: only the projector/residual are defined


def test_clusters_and_multiplicity():
    rng = np.random.default_rng(7)
    t = 120
    eigs = np.sort(rng.uniform(1, 2, t))
    eigs[-8:] = 3.0 + 1e-13 * np.arange(8)          # tight cluster at the top
    eigs[-14:-8] = 2.5 + 1e-5 * np.arange(6)        # loose cluster below it
    eigs[:5] = 0.5                                   # exact multiplicity at the bottom
    mats = [_rand_sym(rng, t, eigs), _rand_sym(rng, t, eigs[::-1].copy())]
    _check(mats, "L", 20)
    _check(mats, "S", 10)
    _check(mats, "M", 30)


def test_graded_and_scaled():
    rng = np.random.default_rng(11)
    t = 200
    mats = [_rand_sym(rng, t, np.logspace(-8, 4, t)), 1e-6 * _rand_sym(rng, t), 1e6 * _rand_sym(rng, t)]
    _check(mats, "L", 16)
    _check(mats, "S", 16, tol_vec=1e3)


def test_diagonal_and_tridiagonal_inputs():
    rng = np.random.default_rng(13)
    t = 50
    D = np.diag(rng.standard_normal(t))
    Tm = np.diag(rng.standard_normal(t)) + np.diag(rng.standard_normal(t - 1), 1)
    Tm = Tm + np.triu(Tm, 1).T
    _check([D, Tm, np.eye(t)], "M", 12)


@pytest.mark.parametrize("size", ["S", "L", "M"])
def test_wide_candidates_global_variant(size):
    """t > 228 (C3-C5 candidate widths): the full matrix lives in the global workspace."""
    rng = np.random.default_rng(23)
    mats = [_rand_sym(rng, t) for t in (229, 330, 401, 580, 640)]
    _check(mats, size, 40)


def test_wide_gram_like_spectra():
    """C3-like GSVD input: p = 208 < t = 330 (zero cluster of 122) and C4-like p = 1200 > t = 540."""
    rng = np.random.default_rng(29)
    mats = []
    for t, p in ((330, 208), (540, 600)):
        Q, _ = np.linalg.qr(rng.standard_normal((p + t, t)) * np.logspace(0, -6, t))
        Q1 = Q[:p]
        mats.append(Q1.T @ Q1)
    _check(mats, "L", 40)


def test_rejects_too_large_t():
    from paper_2412_08264_b200.batched import syev_select

    with pytest.raises(ValueError):
        syev_select(torch.zeros(1, 641, 641, dtype=torch.float64, device="cuda"), torch.tensor([641]), "L", 4)
