"""Grids, measurement models and the TT-FFT filter step, restated.

TEST INFRASTRUCTURE ONLY.  Follows ``ttpmf.filters`` (Algorithm 3,
filters.py:937-985), ``ttpmf.grids`` and ``ttpmf.models`` for the TT path.

A *model spec* is a plain dict shared with the tests and the product:
``{"F", "Q", "R", "h", "H" (linear only), "angle_components"}`` where ``h``
names one of the measurement kinds in :data:`H_KINDS`.  A filter state is
``(axes, cores)``; per-step diagnostics are returned as a dict.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

from oracle import ttcore as T
from oracle.cross import greedy_cross

MASS_FLOOR = 1e-300   # filters.py:100
N_PROBES = 4096       # filters.py:101
SEED_BUDGET = 4096    # filters.py:103


class Degenerate(RuntimeError):
    """Mirror of ``DegenerateDensityError`` (filters.py:120)."""


# -- measurement kinds --------------------------------------------------------

def _h_linear(x, spec):
    return x @ np.asarray(spec["H"], dtype=float).T


def _h_range_bearing(x, spec):
    return np.column_stack([np.hypot(x[:, 0], x[:, 1]), np.arctan2(x[:, 1], x[:, 0])])


def _h_range_bearing_deg(x, spec):      # models.py:201-206 (radar)
    return np.column_stack([np.hypot(x[:, 0], x[:, 1]),
                            np.degrees(np.arctan2(x[:, 1], x[:, 0]))])


def _h_norm_bearing_deg(x, spec):       # models.py:281-285 (scaling_model, dim>=2)
    return np.column_stack([np.linalg.norm(x, axis=1),
                            np.degrees(np.arctan2(x[:, 1], x[:, 0]))])


def _h_abs_first(x, spec):              # models.py:268-270 (scaling_model(1))
    return np.abs(x[:, :1])


def _h_range_az_el(x, spec):            # BASELINE config 3
    return np.column_stack([np.linalg.norm(x[:, :3], axis=1),
                            np.arctan2(x[:, 1], x[:, 0]),
                            np.arctan2(x[:, 2], np.hypot(x[:, 0], x[:, 1]))])


def _h_chain_quadratic(x, spec):        # BASELINE config 4
    return np.column_stack([x[:, :-1] ** 2 + x[:, 1:] ** 2, x[:, -1:]])


H_KINDS = {
    "linear": _h_linear,
    "range_bearing": _h_range_bearing,
    "range_bearing_deg": _h_range_bearing_deg,
    "norm_bearing_deg": _h_norm_bearing_deg,
    "abs_first": _h_abs_first,
    "range_az_el": _h_range_az_el,
    "chain_quadratic": _h_chain_quadratic,
}


class Gauss:
    """Zero-mean normal pdf via Cholesky + solve.  models.py:30-69."""

    def __init__(self, cov):
        self.cov = np.atleast_2d(np.asarray(cov, dtype=float))
        self.chol = np.linalg.cholesky(self.cov)
        logdet = 2.0 * float(np.sum(np.log(np.diag(self.chol))))
        self.log_norm = -0.5 * (self.cov.shape[0] * math.log(2.0 * math.pi) + logdet)

    def pdf(self, diff):
        diff = np.atleast_2d(np.asarray(diff, dtype=float))
        y = np.linalg.solve(self.chol, diff.T)
        return np.exp(self.log_norm - 0.5 * np.sum(y * y, axis=0))


def wrap_deg(res, comps):
    """Angle residual wrap to (-180, 180].  models.py:72-82."""
    res = np.atleast_2d(np.array(res, dtype=float))
    for c in comps:
        res[:, c] = 180.0 - np.mod(180.0 - res[:, c], 360.0)
    return res


def likelihood(spec, z, x):
    """p(z | x).  models.py:150-153."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    hz = np.atleast_2d(H_KINDS[spec["h"]](x, spec))
    res = wrap_deg(hz - np.asarray(z, dtype=float), spec.get("angle_components", ()))
    return Gauss(spec["R"]).pdf(res)


# -- grids --------------------------------------------------------------------

def design_grid(mean, cov, n, sigma_mult):
    """grids.py:148-167 (odd n, centre on the mean)."""
    mean = np.asarray(mean, dtype=float).reshape(-1)
    var = np.diag(np.atleast_2d(cov))
    counts = [int(n)] * mean.size if np.isscalar(n) else [int(v) for v in n]
    if any(c % 2 == 0 for c in counts):
        raise ValueError("point counts must be odd")
    if np.any(var <= 0):
        raise ValueError("covariance diagonal must be positive")
    axes = []
    for mu, v, c in zip(mean, var, counts):
        half = sigma_mult * math.sqrt(v)
        axes.append(mu + (2.0 * half / (c - 1)) * (np.arange(c) - (c - 1) // 2))
    return axes


def grid_from_bounds(lo, hi, n):
    """grids.py:72-83."""
    lo = np.atleast_1d(np.asarray(lo, dtype=float))
    hi = np.atleast_1d(np.asarray(hi, dtype=float))
    counts = [int(n)] * lo.size if np.isscalar(n) else [int(v) for v in n]
    return [a + ((b - a) / (c - 1)) * np.arange(c) for a, b, c in zip(lo, hi, counts)]


def steps_of(axes):
    return np.array([(a[-1] - a[0]) / (a.size - 1) for a in axes])


def cell_volume(axes) -> float:
    return float(np.prod(steps_of(axes)))


def points_for(axes, idx):
    idx = np.asarray(idx, dtype=np.intp)
    return np.column_stack([a[idx[:, k]] for k, a in enumerate(axes)])


def corners(axes):
    return np.array(list(itertools.product(*[(a[0], a[-1]) for a in axes])))


def seed_lattice(shape, budget=SEED_BUDGET):
    """filters.py:106-117."""
    s = 1
    while math.prod(len(range(0, n, s)) for n in shape) > budget:
        s += 1
    mesh = np.meshgrid(*[np.arange(0, n, s, dtype=np.intp) for n in shape], indexing="ij")
    return np.stack([m.ravel() for m in mesh], axis=1)


def probe_indices(shape):
    """Negative-mass probe cells drawn from default_rng(0).  filters.py:433-434."""
    rng = np.random.default_rng(0)
    return np.stack([rng.integers(0, n, N_PROBES) for n in shape], axis=1)


# -- filter pieces -------------------------------------------------------------

def negative_mass(cores, axes, guard):
    """filters.py:427-436."""
    shape = tuple(a.size for a in axes)
    total = math.prod(shape)
    if total <= guard:
        dense = T.to_full(cores, limit=guard)
        neg = dense[dense < 0.0]
        return float(-neg.sum()) * cell_volume(axes) if neg.size else 0.0
    vals = T.at_indices(cores, probe_indices(shape))
    return float(np.maximum(-vals, 0.0).mean()) * total * cell_volume(axes)


def finalize(cores, axes, cfg, diag):
    """Round, renormalise, clipped-mass diagnostic.  filters.py:454-479."""
    dv = cell_volume(axes)
    if cfg.get("normalize_before_round", False):
        mass = T.total(cores) * dv
        diag["mass_before_norm"] = mass
        if not math.isfinite(mass) or mass <= MASS_FLOOR:
            raise Degenerate("TT weights carry no probability mass")
        out = T.round_tt(T.scaled(cores, 1.0 / mass), cfg["round_tol"], cfg.get("round_max_rank"))
    else:
        out = T.round_tt(cores, cfg["round_tol"], cfg.get("round_max_rank"))
        mass = T.total(out) * dv
        diag["mass_before_norm"] = mass
        if not math.isfinite(mass) or mass <= MASS_FLOOR:
            raise Degenerate("TT weights carry no probability mass")
        out = T.scaled(out, 1.0 / mass)
    diag["clipped_mass"] = diag.get("clipped_mass", 0.0) + negative_mass(
        out, axes, cfg.get("densify_guard", 2 ** 22))
    return out


def _cross(shape, fn, cc, seeds=None):
    return greedy_cross(shape, fn, tol=cc["tol"], max_rank=cc["max_rank"],
                        max_sweeps=cc.get("max_sweeps", 60), rng_seed=cc.get("rng_seed", 0),
                        validation_count=cc.get("validation_count", 100), seed_indices=seeds)


def _record(diag, name, res):
    diag.setdefault("cross", {})[name] = (res.achieved_error, res.evaluator_calls,
                                         res.sweeps, res.converged)


def initial(mean, cov, cfg, cc):
    """filters.py:497-513."""
    axes = design_grid(mean, cov, cfg["n_per_axis"], cfg["sigma_mult"])
    g = Gauss(cov)
    mean = np.asarray(mean, dtype=float)
    res = _cross(tuple(a.size for a in axes), lambda idx: g.pdf(points_for(axes, idx) - mean), cc)
    diag = {}
    _record(diag, "initial_pmd", res)
    return axes, finalize(res.cores, axes, cfg, diag), diag


def measurement_update(axes, cores, spec, z, cfg, cc, diag):
    """TT branch of filters.py:521-563.  Returns (cores, outlier)."""
    shape = tuple(a.size for a in axes)
    res = _cross(shape, lambda idx: likelihood(spec, z, points_for(axes, idx)), cc,
                 seeds=seed_lattice(shape))
    _record(diag, "likelihood", res)
    diag.setdefault("stage_lik", res.cores)
    prod = T.kron_cores(cores, res.cores)
    mass = T.total(prod) * cell_volume(axes)
    if not math.isfinite(mass) or mass <= MASS_FLOOR:
        diag["outlier"] = True
        return cores, True
    return finalize(prod, axes, cfg, diag), False


def spd_repair(cov):
    """filters.py:275-284."""
    cov = 0.5 * (cov + cov.T)
    lo = float(np.linalg.eigvalsh(cov)[0])
    if lo > 0.0:
        return cov, False
    scale = max(float(np.trace(cov)) / cov.shape[0], 1.0)
    return cov + (1e-9 * scale - min(lo, 0.0)) * np.eye(cov.shape[0]), True


def raw_moments(axes, cores):
    """mass, first and raw second moments (TT branch of filters.py:297-322)."""
    d = len(axes)
    dv = cell_volume(axes)
    mass = T.total(cores) * dv
    if not math.isfinite(mass) or mass <= 0.0:
        raise Degenerate("PMD has non-positive total mass")
    ones = [np.ones(a.size) for a in axes]

    def cdot(vecs):
        return T.inner(cores, T.rank1(vecs)) * dv

    mean = np.empty(d)
    for i in range(d):
        v = list(ones)
        v[i] = axes[i]
        mean[i] = cdot(v) / mass
    m2 = np.empty((d, d))
    for i in range(d):
        for j in range(i, d):
            v = list(ones)
            if i == j:
                v[i] = axes[i] ** 2
            else:
                v[i], v[j] = axes[i], axes[j]
            m2[i, j] = m2[j, i] = cdot(v) / mass
    return mass, mean, m2


def moments(axes, cores):
    """filters.py:287-333 -> (mean, cov, spd_fixed)."""
    _, mean, m2 = raw_moments(axes, cores)
    cov, fixed = spd_repair(m2 - np.outer(mean, mean))
    return mean, cov, fixed


def kalman_predict(mean, cov, spec):
    """filters.py:366-375 (linear dynamics)."""
    F = np.asarray(spec["F"], dtype=float)
    m = (np.atleast_2d(mean) @ F.T).reshape(-1)
    c = F @ cov @ F.T + np.asarray(spec["Q"], dtype=float)
    return m, 0.5 * (c + c.T)


def redesign_geometry(mean, cov, spec, cfg):
    """filters.py:769-786 -> (filtering-grid axes, predictive-grid axes)."""
    pm, pc = kalman_predict(mean, cov, spec)
    pred = design_grid(pm, pc, cfg["n_per_axis"], cfg["sigma_mult"])
    fin = np.linalg.inv(np.asarray(spec["F"], dtype=float))
    mapped = corners(pred) @ fin.T
    filt = grid_from_bounds(mapped.min(axis=0), mapped.max(axis=0), cfg["n_per_axis"])
    return filt, pred


def kernel_values(spec, axes, idx):
    """filters.py:682-706: N(disp F^T; 0, Q) * cell volume, ifftshift layout."""
    idx = np.asarray(idx)
    st = steps_of(axes)
    disp = np.empty(idx.shape, dtype=float)
    for k, a in enumerate(axes):
        n = a.size
        disp[:, k] = np.where(idx[:, k] <= (n - 1) // 2, idx[:, k], idx[:, k] - n) * st[k]
    return Gauss(spec["Q"]).pdf(disp @ np.asarray(spec["F"], dtype=float).T) * cell_volume(axes)


def step(axes, cores, spec, z, cfg, cc):
    """One Algorithm-3 step.  filters.py:937-985.

    Returns (pred_axes, pred_cores, diag) where diag carries the filtering
    moments and the reference's diagnostic fields.
    """
    diag = {"clipped_mass": 0.0, "outlier": False}
    if z is None:
        fcores = cores
    else:
        fcores, _ = measurement_update(axes, cores, spec, z, cfg, cc, diag)
    mean, cov, fixed = moments(axes, fcores)
    diag["filt_mean"], diag["filt_cov"], diag["spd_fixed"] = mean, cov, fixed
    diag["pred_mean"], diag["pred_cov"] = kalman_predict(mean, cov, spec)
    faxes, paxes = redesign_geometry(mean, cov, spec, cfg)
    shifted = finalize(T.regrid(fcores, axes, faxes), faxes, cfg, diag)
    shape = tuple(a.size for a in faxes)
    kres = _cross(shape, lambda idx: kernel_values(spec, faxes, idx), cc)
    _record(diag, "kernel", kres)
    conv = T.fft_conv(kres.cores, shifted, cfg["round_tol"], cfg.get("round_max_rank"))
    finv = np.linalg.inv(np.asarray(spec["F"], dtype=float))
    pshape = tuple(a.size for a in paxes)

    def realign(idx):
        return T.at_points(conv, faxes, points_for(paxes, idx) @ finv.T)

    rres = _cross(pshape, realign, cc, seeds=seed_lattice(pshape))
    _record(diag, "realign", rres)
    out = finalize(rres.cores, paxes, cfg, diag)
    diag["stages"] = {"kernel": kres.cores, "conv": conv, "shifted": shifted,
                      "filt_cores": fcores, "realign": rres.cores, "faxes": faxes,
                      "lik": diag.get("stage_lik"), "paxes": paxes}
    return paxes, out, diag


# -- Algorithm 2: TT standard point-mass filter (filters.py:855-885) -------------

def transition_values(spec, new_axes, old_axes, idx):
    """transition_blackbox (filters.py:653-679) via _transition_values
    (filters.py:580-588): N(x_new - F x_old; 0, Q) * cell_volume(old)."""
    idx = np.asarray(idx)
    d = len(new_axes)
    xn = points_for(new_axes, idx[:, :d])
    xo = points_for(old_axes, idx[:, d:])
    F = np.asarray(spec["F"], dtype=float)
    return Gauss(spec["Q"]).pdf(xn - xo @ F.T) * cell_volume(old_axes)


def step_std(axes, cores, spec, z, cfg, cc):
    """tt_pmf_step (filters.py:855-885): measurement update, moments, Kalman
    prediction, new grid, transition cross over (new, old) modes, backward
    contraction, scale by the old cell volume, finalize."""
    diag = {"clipped_mass": 0.0, "outlier": False}
    fcores = cores if z is None else measurement_update(axes, cores, spec, z, cfg, cc, diag)[0]
    mean, cov, fixed = moments(axes, fcores)
    diag["filt_mean"], diag["filt_cov"], diag["spd_fixed"] = mean, cov, fixed
    pm, pc = kalman_predict(mean, cov, spec)
    diag["pred_mean"], diag["pred_cov"] = pm, pc
    new_axes = design_grid(pm, pc, cfg["n_per_axis"], cfg["sigma_mult"])
    shape = tuple(a.size for a in new_axes) + tuple(a.size for a in axes)
    tres = _cross(shape, lambda idx: transition_values(spec, new_axes, axes, idx), cc)
    _record(diag, "transition", tres)
    raw = T.scaled(T.einsum_tpm(tres.cores, fcores), cell_volume(axes))
    out = finalize(raw, new_axes, cfg, diag)
    diag["stages"] = {"transition": tres.cores, "filt_cores": fcores}
    return new_axes, out, diag
