"""Dense point-mass filter with FFT time update, restated.

TEST INFRASTRUCTURE ONLY (the CUDA path in paper_2501_07942_b200/dense.py is
checked against it).  Follows ``ttpmf.filters.dense_fft_pmf_step``
(filters.py:888-934) with its pieces:

* initial_pmd_dense          filters.py:487-494
* measurement_update (dense) filters.py:564-572
* _finalize_dense            filters.py:439-451
* moments_from_pmd (dense)   filters.py:323-333
* kalman_predict             filters.py:366-375
* RegularGridInterpolator(linear, fill 0) at grid_pred @ F^-T   filters.py:911-916
  (scipy's find_indices + hypercube sum, restated below)
* kernel N(disp; 0, Q) * cell_volume / |det F|                  filters.py:920-927
* _circular_convolve (numpy fftn / ifftn)                       filters.py:732-736

A dense state is ``(axes, weights)`` with weights of shape ``grid.shape``.
"""

from __future__ import annotations

import itertools

import numpy as np

from oracle.pmf import MASS_FLOOR, Degenerate, Gauss, design_grid, likelihood, steps_of


def all_points(axes):
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.stack([m.reshape(-1) for m in mesh], axis=1)


def cell_volume(axes):
    return float(np.prod(steps_of(axes)))


def finalize(w, axes, diag):
    """_finalize_dense (filters.py:439-451)."""
    if not np.isfinite(w).all():
        raise Degenerate("dense weights contain non-finite values")
    neg = w[w < 0.0]
    diag["clipped_mass"] += float(-neg.sum()) * cell_volume(axes) if neg.size else 0.0
    w = np.maximum(w, 0.0)
    mass = float(w.sum()) * cell_volume(axes)
    diag["mass_before_norm"] = mass
    if mass <= MASS_FLOOR:
        raise Degenerate("dense weights carry no probability mass")
    return w / mass


def initial(mean, cov, cfg):
    """initial_pmd_dense (filters.py:487-494)."""
    axes = design_grid(mean, cov, cfg["n_per_axis"], cfg["sigma_mult"])
    shape = tuple(a.size for a in axes)
    vals = Gauss(cov).pdf(all_points(axes) - np.asarray(mean, dtype=float)).reshape(shape)
    diag = {"clipped_mass": 0.0, "mass_before_norm": float("nan")}
    return axes, finalize(vals, axes, diag), diag


def moments(axes, w):
    """moments_from_pmd, dense branch (filters.py:323-333) + _spd_repair."""
    wv = w.reshape(-1) * cell_volume(axes)
    mass = float(wv.sum())
    if not np.isfinite(mass) or mass <= 0.0:
        raise Degenerate("PMD has non-positive total mass")
    pts = all_points(axes)
    mean = pts.T @ wv / mass
    centered = pts - mean
    cov = centered.T @ (centered * wv[:, None]) / mass
    cov = 0.5 * (cov + cov.T)
    lo = float(np.linalg.eigvalsh(cov)[0])
    fixed = False
    if not lo > 0.0:
        scale = max(float(np.trace(cov)) / cov.shape[0], 1.0)
        cov = cov + (1e-9 * scale - min(lo, 0.0)) * np.eye(cov.shape[0])
        fixed = True
    return mean, cov, fixed


def find_indices(grid, x):
    """scipy RegularGridInterpolator find_indices: interval i with
    grid[i] <= x < grid[i+1] (clipped to [0, n-2]) and (x - g[i]) / (g[i+1] - g[i])."""
    n = grid.size
    i = np.searchsorted(grid, x, side="right") - 1
    i = np.clip(i, 0, n - 2)
    return i, (x - grid[i]) / (grid[i + 1] - grid[i])


def interp_linear(axes, w, pts):
    """RegularGridInterpolator(axes, w, 'linear', bounds_error=False, fill_value=0)(pts)."""
    d = len(axes)
    idx, dist = zip(*(find_indices(axes[k], pts[:, k]) for k in range(d)))
    out = np.zeros(pts.shape[0])
    for corner in itertools.product((0, 1), repeat=d):
        weight = np.ones(pts.shape[0])
        ii = []
        for k, b in enumerate(corner):
            weight = weight * (dist[k] if b else 1.0 - dist[k])
            ii.append(idx[k] + b)
        out = out + w[tuple(ii)] * weight
    oob = np.zeros(pts.shape[0], dtype=bool)
    for k in range(d):
        oob |= (pts[:, k] < axes[k][0]) | (pts[:, k] > axes[k][-1])
    out[oob] = 0.0
    return out


def kernel(axes_pred, spec):
    """N(disp; 0, Q) * cell_volume / |det F| on ifftshift displacements (filters.py:920-927)."""
    shape = tuple(a.size for a in axes_pred)
    idx = np.indices(shape).reshape(len(shape), -1).T
    st = steps_of(axes_pred)
    disp = np.empty(idx.shape)
    for k, n in enumerate(shape):
        half = (n - 1) // 2
        disp[:, k] = np.where(idx[:, k] <= half, idx[:, k], idx[:, k] - n) * st[k]
    F = np.asarray(spec["F"], dtype=float)
    return Gauss(spec["Q"]).pdf(disp).reshape(shape) * cell_volume(axes_pred) / abs(np.linalg.det(F))


def step(axes, w, spec, z, cfg):
    """dense_fft_pmf_step (filters.py:888-934); returns (axes_pred, w_pred, diag)."""
    diag = {"clipped_mass": 0.0, "mass_before_norm": float("nan"), "outlier": False}
    F = np.asarray(spec["F"], dtype=float)
    Q = np.asarray(spec["Q"], dtype=float)
    if z is not None:
        lik = likelihood(spec, z, all_points(axes)).reshape(w.shape)
        prod = w * lik
        mass = float(prod.sum()) * cell_volume(axes)
        if not np.isfinite(mass) or mass <= MASS_FLOOR:
            diag["outlier"] = True
        else:
            w = finalize(prod, axes, diag)
    mean, cov, fixed = moments(axes, w)
    diag["filt_mean"], diag["filt_cov"], diag["spd_fixed"] = mean, cov, fixed
    pm = F @ mean
    pc = F @ cov @ F.T + Q
    pc = 0.5 * (pc + pc.T)
    axes_pred = design_grid(pm, pc, cfg["n_per_axis"], cfg["sigma_mult"])
    shape = tuple(a.size for a in axes_pred)
    sheared = interp_linear(axes, w, all_points(axes_pred) @ np.linalg.inv(F).T).reshape(shape)
    ker = kernel(axes_pred, spec)
    raw = np.fft.ifftn(np.fft.fftn(ker) * np.fft.fftn(sheared)).real
    return axes_pred, finalize(raw, axes_pred, diag), diag
