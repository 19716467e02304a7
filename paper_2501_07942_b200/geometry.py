"""Host-side grid geometry of the TT-FFT step (tiny O(d^3) numpy work).

These are the reference's own small dense steps between the device stages:
moment post-processing and SPD repair (filters.py:275-333), Kalman predict
(filters.py:366-375), moment-designed grids (grids.py:148-167), corner
pull-back and the circumscribing grid (filters.py:769-786, grids.py:72-83).
Grids travel to the device as (base, step, off) triples, from which the
kernels rebuild every coordinate with the same two roundings numpy uses.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

from paper_2501_07942_b200 import _abi


class Axes:
    """Equidistant per-axis coordinates of one grid, plus the device form."""

    def __init__(self, base, step, off, n):
        self.base = np.asarray(base, dtype=float).reshape(-1)
        self.step = np.asarray(step, dtype=float).reshape(-1)
        self.off = np.asarray(off, dtype=np.int64).reshape(-1)
        self.n = np.asarray(n, dtype=np.int64).reshape(-1)

    @property
    def dim(self) -> int:
        return self.base.size

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(v) for v in self.n)

    def axes(self) -> tuple[np.ndarray, ...]:
        return tuple(b + s * (np.arange(int(n)) - int(o))
                     for b, s, o, n in zip(self.base, self.step, self.off, self.n))

    def steps(self) -> np.ndarray:
        return np.array([(a[-1] - a[0]) / (a.size - 1) for a in self.axes()])

    def cell_volume(self) -> float:
        return float(np.prod(self.steps()))

    def device(self) -> np.ndarray:
        rec = np.zeros(_abi.MAXD, dtype=_abi.AXIS)
        d = self.dim
        rec["base"][:d] = self.base
        rec["step"][:d] = self.step
        rec["off"][:d] = self.off
        rec["n"][:d] = self.n
        return rec

    def corners(self) -> np.ndarray:
        ax = self.axes()
        return np.array(list(itertools.product(*[(a[0], a[-1]) for a in ax])))


def counts(n_per_axis, d):
    if np.isscalar(n_per_axis):
        return [int(n_per_axis)] * d
    return [int(v) for v in n_per_axis]


def design_grid(mean, cov, n_per_axis, sigma_mult) -> Axes:
    """grids.py:148-167."""
    mean = np.asarray(mean, dtype=float).reshape(-1)
    var = np.diag(np.atleast_2d(cov))
    cnt = counts(n_per_axis, mean.size)
    if any(c % 2 == 0 for c in cnt):
        raise ValueError(f"point counts must be odd, got {tuple(cnt)}")
    if sigma_mult <= 0:
        raise ValueError("sigma_mult must be positive")
    if np.any(var <= 0):
        raise ValueError("covariance diagonal must be positive to span a grid")
    steps = [2.0 * (sigma_mult * math.sqrt(v)) / (c - 1) for v, c in zip(var, cnt)]
    return Axes(mean, steps, [(c - 1) // 2 for c in cnt], cnt)


def grid_from_bounds(lows, highs, n_per_axis) -> Axes:
    """grids.py:72-83."""
    lows = np.atleast_1d(np.asarray(lows, dtype=float))
    highs = np.atleast_1d(np.asarray(highs, dtype=float))
    cnt = counts(n_per_axis, lows.size)
    if np.any(highs <= lows):
        raise ValueError("each upper bound must exceed its lower bound")
    return Axes(lows, [(h - l) / (c - 1) for l, h, c in zip(lows, highs, cnt)], [0] * len(cnt), cnt)


def spd_repair(cov):
    """filters.py:275-284."""
    cov = 0.5 * (cov + cov.T)
    lo = float(np.linalg.eigvalsh(cov)[0])
    if lo > 0.0:
        return cov, False
    scale = max(float(np.trace(cov)) / cov.shape[0], 1.0)
    return cov + (1e-9 * scale - min(lo, 0.0)) * np.eye(cov.shape[0]), True


def moments_from_raw(raw, d, cell_volume):
    """filters.py:297-333 from the device's un-normalised dots.

    Returns (mass, mean, cov, spd_fixed); mass may be non-positive (caller
    raises DegenerateDensityError).
    """
    mass = float(raw[0]) * cell_volume
    if not math.isfinite(mass) or mass <= 0.0:
        return mass, None, None, False
    mean = np.empty(d)
    for i in range(d):
        mean[i] = float(raw[1 + i]) * cell_volume / mass
    second = np.empty((d, d))
    q = 1 + d
    for i in range(d):
        for j in range(i, d):
            second[i, j] = second[j, i] = float(raw[q]) * cell_volume / mass
            q += 1
    cov, fixed = spd_repair(second - np.outer(mean, mean))
    return mass, mean, cov, fixed


def kalman_predict(mean, cov, F, Q):
    """filters.py:366-375 (linear dynamics)."""
    m = (np.atleast_2d(mean) @ F.T).reshape(-1)
    c = F @ cov @ F.T + Q
    return m, 0.5 * (c + c.T)


def redesign(mean, cov, F, Q, Finv, n_per_axis, sigma_mult):
    """filters.py:769-786 -> (filtering-grid Axes, predictive-grid Axes)."""
    pm, pc = kalman_predict(mean, cov, F, Q)
    pred = design_grid(pm, pc, n_per_axis, sigma_mult)
    mapped = pred.corners() @ Finv.T
    filt = grid_from_bounds(mapped.min(axis=0), mapped.max(axis=0), n_per_axis)
    return filt, pred


def seed_lattice(shape, budget=4096) -> np.ndarray:
    """filters.py:106-117."""
    s = 1
    while math.prod(len(range(0, n, s)) for n in shape) > budget:
        s += 1
    mesh = np.meshgrid(*[np.arange(0, n, s, dtype=np.int64) for n in shape], indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1).astype(np.int32)


def probe_cells(shape, count=4096) -> np.ndarray:
    """filters.py:433-434: default_rng(0) probe cells for the negative mass."""
    rng = np.random.default_rng(0)
    return np.stack([rng.integers(0, n, count) for n in shape], axis=1).astype(np.int32)


def gauss_consts(cov):
    """(lower Cholesky, log normaliser) as GaussianDensity (models.py:30-52)."""
    cov = np.atleast_2d(np.asarray(cov, dtype=float))
    if cov.shape[0] != cov.shape[1]:
        raise ValueError("covariance must be square")
    if not np.allclose(cov, cov.T, rtol=1e-10, atol=1e-14):
        raise ValueError("covariance must be symmetric")
    try:
        chol = np.linalg.cholesky(cov)
    except np.linalg.LinAlgError as exc:
        raise ValueError("covariance must be positive definite") from exc
    log_det = 2.0 * float(np.sum(np.log(np.diag(chol))))
    return chol, -0.5 * (cov.shape[0] * math.log(2.0 * math.pi) + log_det)


def solve_factors(chol):
    """The factors numpy.linalg.solve(chol, b) works with inside
    GaussianDensity.logpdf (models.py:60-63): LAPACK dgetrf of the Cholesky
    factor (row-major LU), 0-based sequential row swaps and the reciprocal
    pivots the trsm kernels multiply by."""
    from scipy.linalg import lu_factor
    lu, piv = lu_factor(np.atleast_2d(np.asarray(chol, dtype=float)), check_finite=False)
    return np.ascontiguousarray(lu), piv.astype(np.int32), 1.0 / np.diag(lu)


def pcg64_state(seed: int) -> list[int]:
    """numpy default_rng(seed) PCG64 state as the six words of ttgbf_cross_cfg."""
    st = np.random.PCG64(seed).state
    s, inc = st["state"]["state"], st["state"]["inc"]
    m = (1 << 64) - 1
    return [s & m, s >> 64, inc & m, inc >> 64, int(st["has_uint32"]), int(st["uinteger"])]
