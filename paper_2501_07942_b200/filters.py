"""Reference-compatible filter API on the B200 engine (drop-in for ``ttpmf.filters``).

Same names, argument meaning and error behaviour as the reference's TT path:

=========================  ===========================================
this module                reference (pkg/src/ttpmf)
=========================  ===========================================
GridConfig                 filters.py:129-161
StepDiagnostics            filters.py:164-188
PmdEstimate                filters.py:191-230
DegenerateDensityError     filters.py:120
initial_pmd_tt             filters.py:497-513
measurement_update         filters.py:521-563 (TT branch)
moments_from_pmd           filters.py:287-333 (TT branch)
grid_redesign              filters.py:799-824 (TT branch)
kalman_predict             filters.py:366-375
tt_fft_pmf_step            filters.py:937-985
tt_pmf_step                filters.py:855-885 (Algorithm 2)
=========================  ===========================================

Every density operation runs in ``libttgbf.so`` on the GPU; weights stay
device-resident between calls (:class:`~paper_2501_07942_b200.tensor_train.TensorTrain`).
Models are :class:`~paper_2501_07942_b200.models.StateSpaceModel` descriptors
whose measurement function is one of the enumerated kinds the device
evaluates; an arbitrary Python callable is rejected (no CPU fallback).
"""

from __future__ import annotations

from collections import OrderedDict

import math
from dataclasses import dataclass, field, replace

import numpy as np

from paper_2501_07942_b200 import _abi
from paper_2501_07942_b200 import geometry as geo
from paper_2501_07942_b200.bank import BankConfig, FilterBank
from paper_2501_07942_b200.grids import Grid, MomentEstimate
from paper_2501_07942_b200.models import StateSpaceModel
from paper_2501_07942_b200.tensor_train import TensorTrain

__all__ = ["CrossConfig", "DegenerateDensityError", "GridConfig", "PmdEstimate", "StepDiagnostics",
           "grid_redesign", "initial_pmd_tt", "kalman_predict", "measurement_update",
           "moments_from_pmd", "tt_fft_pmf_step", "tt_pmf_step"]


class DegenerateDensityError(RuntimeError):
    """Raised when a density collapses to zero or non-finite mass."""


@dataclass(frozen=True)
class GridConfig:
    n_per_axis: int = 33
    sigma_mult: float = 4.0
    round_tol: float = 1e-8
    round_max_rank: int | None = None
    normalize_before_round: bool = False
    densify_guard: int = 2 ** 22

    def __post_init__(self) -> None:
        if self.n_per_axis < 3 or self.n_per_axis % 2 == 0:
            raise ValueError("n_per_axis must be an odd integer >= 3")
        if not self.sigma_mult > 0:
            raise ValueError("sigma_mult must be positive")
        if self.round_tol < 0:
            raise ValueError("round_tol must be nonnegative")
        if self.round_max_rank is not None and self.round_max_rank < 1:
            raise ValueError("round_max_rank must be a positive integer")
        if self.densify_guard < 1:
            raise ValueError("densify_guard must be positive")


@dataclass
class CrossConfig:
    """tt_algorithms.py:93-115 (+ device resource knobs with defaults)."""

    tol: float = 1e-6
    max_rank: int = 40
    max_sweeps: int = 60
    rng_seed: int = 0
    validation_count: int = 100
    seed_indices: np.ndarray | None = None
    cache_cap: int = 1 << 20

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ValueError("tol must be positive")
        if self.max_rank < 1 or self.max_sweeps < 1 or self.validation_count < 1:
            raise ValueError("max_rank, max_sweeps and validation_count must be >= 1")


@dataclass
class StepDiagnostics:
    filt_moments: MomentEstimate | None = None
    pred_moments: MomentEstimate | None = None
    mass_before_norm: float = float("nan")
    clipped_mass: float = 0.0
    outlier: bool = False
    spd_fixed: bool = False
    tpm_bytes: int = 0
    pmd_bytes: int = 0
    interp_seconds: float = 0.0
    cross_info: dict = field(default_factory=dict)
    warnings: list = field(default_factory=list)

    def record_cross(self, name, info):
        self.cross_info[name] = info
        if not info[3]:
            self.warnings.append(f"cross '{name}' did not converge")


@dataclass(frozen=True)
class PmdEstimate:
    grid: Grid
    weights: TensorTrain
    kind: str
    diag: StepDiagnostics | None = None

    def __post_init__(self) -> None:
        if self.kind not in ("predictive", "filtering"):
            raise ValueError("kind must be 'predictive' or 'filtering'")
        if not isinstance(self.weights, TensorTrain):
            raise TypeError("weights must be a device TensorTrain (dense weights are not on this path)")
        if self.weights.shape != self.grid.shape:
            raise ValueError("TT weights shape does not match grid shape")

    @property
    def is_tt(self) -> bool:
        return True

    def storage_bytes(self) -> int:
        return self.weights.storage_bytes()

    def mass(self) -> float:
        from paper_2501_07942_b200.tensor_train import tt_sum
        return tt_sum(self.weights) * self.grid.cell_volume


# ---------------------------------------------------------------------------
# engine access: one cached single-filter bank per (model, configs)
# ---------------------------------------------------------------------------
_BANK_LIMIT = 4                       # banks kept alive (LRU); each owns device workspaces
_BANKS: "OrderedDict[tuple, FilterBank]" = OrderedDict()
_PLACEHOLDERS: dict = {}


def _spec_key(spec) -> tuple:
    """Content key of a model spec: two StateSpaceModel objects with the same
    F, Q, R, h, H and angle components share one engine bank."""
    out = []
    for name in sorted(spec):
        v = spec[name]
        if isinstance(v, np.ndarray):
            out.append((name, v.shape, v.dtype.str, v.tobytes()))
        elif isinstance(v, (list, tuple)):
            out.append((name, tuple(v)))
        else:
            out.append((name, v))
    return tuple(out)


def _bank(model: StateSpaceModel, cfg: GridConfig, cross: CrossConfig) -> FilterBank:
    key = (_spec_key(model.spec), cfg, cross.tol, cross.max_rank, cross.max_sweeps, cross.rng_seed,
           cross.validation_count, cross.cache_cap)
    b = _BANKS.get(key)
    if b is not None:
        _BANKS.move_to_end(key)
        return b
    bc = BankConfig(n_per_axis=cfg.n_per_axis, sigma_mult=cfg.sigma_mult, round_tol=cfg.round_tol,
                    round_max_rank=cfg.round_max_rank, normalize_before_round=cfg.normalize_before_round,
                    densify_guard=cfg.densify_guard, tol=cross.tol, max_rank=cross.max_rank,
                    max_sweeps=cross.max_sweeps, rng_seed=cross.rng_seed,
                    validation_count=cross.validation_count, cache_cap=cross.cache_cap)
    while len(_BANKS) >= _BANK_LIMIT:
        _BANKS.popitem(last=False)       # frees the evicted bank's device buffers
    b = FilterBank(model.spec, bc, 1)
    _BANKS[key] = b
    return b


def release_banks() -> None:
    """Drop every cached engine bank (and its device memory)."""
    _BANKS.clear()


def _raise(status: int, where: str):
    if status == _abi.E_DEGENERATE:
        raise DegenerateDensityError(f"{where}: TT weights carry no probability mass")
    if status in (_abi.E_ARG, _abi.E_NONFINITE):
        raise ValueError(f"{where}: {_abi.status_text(status)}")
    raise MemoryError(f"{where}: {_abi.status_text(status)}") if status in (_abi.E_WORKSPACE, _abi.E_CACHE, _abi.E_STATE_CAP) \
        else RuntimeError(f"{where}: {_abi.status_text(status)}")


def _load(bank: FilterBank, pmd: PmdEstimate):
    bank.load_tt(0, pmd.weights, pmd.grid.device_axes)


def _read(bank: FilterBank, grid: Grid) -> TensorTrain:
    return bank.read_tt(0)


def _cross_tuple(row, slot):
    return FilterBank.cross_info(row, slot)


# ---------------------------------------------------------------------------
# API
# ---------------------------------------------------------------------------
def initial_pmd_tt(prior: MomentEstimate, cfg: GridConfig, cross_cfg: CrossConfig,
                   model: StateSpaceModel | None = None) -> PmdEstimate:
    """TT Gaussian prior PMD built with the device greedy cross (filters.py:497-513)."""
    if model is None:
        model = _PLACEHOLDERS.setdefault(prior.dim, StateSpaceModel.placeholder(prior.dim))
    bank = _bank(model, cfg, cross_cfg)
    dg = bank.init_prior(prior.mean, prior.cov)
    if dg["status"][0] != 0:
        _raise(int(dg["status"][0]), "initial_pmd_tt")
    diag = StepDiagnostics()
    diag.record_cross("initial_pmd", _cross_tuple(dg[0], 0))
    diag.mass_before_norm = float(dg["mass_before_norm"][0])
    diag.clipped_mass = float(dg["clipped_mass"][0])
    grid = Grid.from_axes(bank.grids[0])
    return PmdEstimate(grid, _read(bank, grid), "predictive", diag)


def measurement_update(pmd: PmdEstimate, model: StateSpaceModel, z, cfg: GridConfig,
                       cross_cfg: CrossConfig | None = None, diag: StepDiagnostics | None = None) -> PmdEstimate:
    """filters.py:521-563 (TT branch)."""
    if diag is None:
        diag = StepDiagnostics()
    if z is None:
        return PmdEstimate(pmd.grid, pmd.weights, "filtering", diag)
    if cross_cfg is None:
        raise ValueError("TT measurement update requires a CrossConfig")
    bank = _bank(model, cfg, cross_cfg)
    _load(bank, pmd)
    dg = bank.measure(np.asarray(z, dtype=float)[None])
    st = int(dg["status"][0])
    if st != 0:
        _raise(st, "measurement_update")
    diag.record_cross("likelihood", _cross_tuple(dg[0], 0))
    if dg["outlier"][0]:
        diag.outlier = True
        diag.warnings.append("measurement likelihood underflow; kept prior")
        return PmdEstimate(pmd.grid, pmd.weights, "filtering", diag)
    diag.mass_before_norm = float(dg["mass_before_norm"][0])
    diag.clipped_mass += float(dg["clipped_mass"][0])
    return PmdEstimate(pmd.grid, _read(bank, pmd.grid), "filtering", diag)


def moments_from_pmd(pmd: PmdEstimate) -> tuple[MomentEstimate, bool]:
    """filters.py:287-333 (TT branch) on the device moment contractions."""
    from paper_2501_07942_b200.tensor_train import tt_raw_moments
    raw = tt_raw_moments(pmd.weights, pmd.grid.device_axes)
    mass, mean, cov, fixed = geo.moments_from_raw(raw, pmd.grid.dim, pmd.grid.cell_volume)
    if mean is None:
        raise DegenerateDensityError("PMD has non-positive total mass")
    return MomentEstimate(mean=mean, cov=cov), fixed


def kalman_predict(m: MomentEstimate, model: StateSpaceModel) -> MomentEstimate:
    mean, cov = geo.kalman_predict(m.mean, m.cov, model.F, model.Q)
    return MomentEstimate(mean=mean, cov=cov)


def grid_redesign(pmd: PmdEstimate, model: StateSpaceModel, cfg: GridConfig, moments: MomentEstimate | None = None,
                  diag: StepDiagnostics | None = None, cross_cfg: CrossConfig | None = None):
    """filters.py:799-824: interpolate onto the pre-convolution grid + finalize."""
    from paper_2501_07942_b200.tensor_train import tt_interpolate, finalize
    if diag is None:
        diag = StepDiagnostics()
    if moments is None:
        moments, fixed = moments_from_pmd(pmd)
        diag.spd_fixed = diag.spd_fixed or fixed
    faxes, paxes = geo.redesign(moments.mean, moments.cov, model.F, model.Q, model.Finv, cfg.n_per_axis,
                                cfg.sigma_mult)
    gf = Grid.from_axes(faxes)
    shifted = tt_interpolate(pmd.weights, pmd.grid, gf)
    w, mass, clipped = finalize(shifted, gf, cfg)
    diag.mass_before_norm = mass
    diag.clipped_mass += clipped
    return PmdEstimate(gf, w, "filtering", diag), Grid.from_axes(paxes)


def tt_fft_pmf_step(pmd: PmdEstimate, model: StateSpaceModel, z, cfg: GridConfig,
                    cross_cfg: CrossConfig) -> PmdEstimate:
    """One Algorithm-3 step on the GPU (filters.py:937-985)."""
    bank = _bank(model, cfg, cross_cfg)
    _load(bank, pmd)
    zz = np.zeros((1, model.dim_z)) if z is None else np.asarray(z, dtype=float)[None]
    dm = bank.measure(zz, has_z=[0 if z is None else 1])
    st = int(dm["status"][0])
    if st != 0:
        _raise(st, "tt_fft_pmf_step (measurement)")
    diag = StepDiagnostics()
    if z is not None:
        diag.record_cross("likelihood", _cross_tuple(dm[0], 0))
        if dm["outlier"][0]:
            diag.outlier = True
            diag.warnings.append("measurement likelihood underflow; kept prior")
    geom = bank.geometry(dm)
    if geom[0][0] != "ok":
        raise DegenerateDensityError("PMD has non-positive total mass")
    mean, cov, fixed, faxes, paxes = geom[0][1]
    diag.filt_moments = MomentEstimate(mean=mean, cov=cov)
    diag.spd_fixed = fixed
    pm, pc = geo.kalman_predict(mean, cov, model.F, model.Q)
    diag.pred_moments = MomentEstimate(mean=pm, cov=pc)
    dt = bank.time_update(geom)
    st = int(dt["status"][0])
    if st != 0:
        _raise(st, "tt_fft_pmf_step (time update)")
    diag.record_cross("kernel", _cross_tuple(dt[0], 1))
    diag.record_cross("realign", _cross_tuple(dt[0], 2))
    diag.mass_before_norm = float(dt["mass_before_norm"][0])
    diag.clipped_mass = float(dt["clipped_mass"][0])   # device accumulates over both stages
    grid = Grid.from_axes(paxes)
    w = _read(bank, grid)
    diag.pmd_bytes = w.storage_bytes()
    return PmdEstimate(grid, w, "predictive", diag)


def tt_pmf_step(pmd: PmdEstimate, model: StateSpaceModel, z, cfg: GridConfig,
                cross_cfg: CrossConfig) -> PmdEstimate:
    """One Algorithm-2 step on the GPU (filters.py:855-885): measurement update,
    moments, Kalman prediction, new grid, transition cross over the (new, old)
    modes, tt_einsum_tpm contraction, scale by the old cell volume, finalize."""
    if 2 * model.dim_x > _abi.MAXD:
        raise ValueError("the transition tensor has 2d modes; d <= 8 on the device")
    bank = _bank(model, cfg, cross_cfg)
    _load(bank, pmd)
    zz = np.zeros((1, model.dim_z)) if z is None else np.asarray(z, dtype=float)[None]
    dm = bank.measure(zz, has_z=[0 if z is None else 1])
    st = int(dm["status"][0])
    if st != 0:
        _raise(st, "tt_pmf_step (measurement)")
    diag = StepDiagnostics()
    if z is not None:
        diag.record_cross("likelihood", _cross_tuple(dm[0], 0))
        if dm["outlier"][0]:
            diag.outlier = True
            diag.warnings.append("measurement likelihood underflow; kept prior")
    geom = bank.geometry(dm)
    if geom[0][0] != "ok":
        raise DegenerateDensityError("PMD has non-positive total mass")
    mean, cov, fixed, _, paxes = geom[0][1]
    diag.filt_moments = MomentEstimate(mean=mean, cov=cov)
    diag.spd_fixed = fixed
    pm, pc = geo.kalman_predict(mean, cov, model.F, model.Q)
    diag.pred_moments = MomentEstimate(mean=pm, cov=pc)
    dt = bank.time_update_std(geom)
    st = int(dt["status"][0])
    if st != 0:
        _raise(st, "tt_pmf_step (time update)")
    diag.record_cross("transition", _cross_tuple(dt[0], 1))
    diag.mass_before_norm = float(dt["mass_before_norm"][0])
    diag.clipped_mass = float(dt["clipped_mass"][0])
    grid = Grid.from_axes(paxes)
    w = _read(bank, grid)
    diag.pmd_bytes = w.storage_bytes()
    return PmdEstimate(grid, w, "predictive", diag)
