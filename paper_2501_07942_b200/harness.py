"""Benchmark-harness integration: a ``ttfft-gpu`` filter
for the reference's compare/scaling harness.

Mirrors ``ttpmf.bench`` (reference ``pkg/src/ttpmf/bench.py``):

* :class:`RunConfig` keeps the reference's field names, defaults and
  validation (bench.py:83-125) for the fields this filter uses;
* :func:`run_compare` / :func:`run_scaling` (bench.py:495-577) run every
  Monte Carlo run of a scenario as ONE :class:`FilterBank` (one CTA per run,
  stage kernels per step) instead of a Python loop over runs;
* :class:`FilterOutcome` has the reference's fields (bench.py:236-253) and
  is filled exactly as ``_run_grid_filter`` does (bench.py:317-392): RMSE
  over all runs and steps, max clipped mass, max |mass - 1|, cross
  diagnostics, run-0 trace;
* :func:`emit_csv` writes the same ``summary.csv`` (9 columns,
  bench.py:563-565), ``trace_<filter>.csv`` and ``timings.txt`` layout, so a
  GPU row can sit beside the reference's CPU rows.

``ms_per_step`` is the batched device time of one step divided by the runs
in the batch (the GPU advances every run in one launch per stage).  A run
whose step raises DegenerateDensityError is recorded as the outcome's
``failure`` (the reference aborts the filter on the first exception,
bench.py:466-478).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import Sequence

import numpy as np

from .bank import BankConfig, FilterBank
from .configs import SPECS, scaling_spec, simulate

FILTER_NAMES = ("ttfft-gpu", "tt-gpu", "fft-gpu")   # reference rows: ttfft, tt, fft
COMPARE_SCENARIOS = ("radar", "linear1d", "linear2d")


class ConfigError(ValueError):
    """Invalid benchmark configuration (bench.py:75)."""


def _linear2d_spec():
    """radar_identity_model (models.py:225-238)."""
    s = dict(SPECS["radar"])
    s.update({"h": "linear", "H": np.eye(2), "angle_components": (), "name": "linear2d"})
    return s


def _linear1d_spec():
    """linear_gaussian_1d (models.py:241-252)."""
    return {"F": np.array([[0.9]]), "Q": np.array([[1.0]]), "R": np.array([[1.0]]), "h": "linear",
            "H": np.array([[1.0]]), "angle_components": (), "name": "linear1d"}


@dataclass(frozen=True)
class RunConfig:
    """The reference RunConfig fields this filter depends on (bench.py:83-125)."""

    scenario: str
    filters: tuple = FILTER_NAMES
    runs: int = 10
    k_f: int = 10
    master_seed: int = 2024
    n_per_axis: int = 33
    sigma_mult: float = 4.0
    round_tol: float = 1e-8
    round_max_rank: int | None = None
    cross_tol: float = 1e-2
    cross_max_rank: int = 150
    cross_seed: int = 0
    out_dir: str = "results"
    ws_mb: int = 256

    def __post_init__(self):
        object.__setattr__(self, "filters", tuple(self.filters))
        if not self.scenario:
            raise ConfigError("scenario must be a non-empty string")
        if self.runs < 1:
            raise ConfigError("runs must be >= 1")
        if self.k_f < 1:
            raise ConfigError("k_f must be >= 1")
        if self.n_per_axis < 3 or self.n_per_axis % 2 == 0:
            raise ConfigError("n_per_axis must be odd and >= 3")
        for name in ("sigma_mult", "round_tol", "cross_tol"):
            if getattr(self, name) <= 0:
                raise ConfigError(f"{name} must be > 0")
        if self.cross_max_rank < 1:
            raise ConfigError("cross max_rank must be >= 1")
        unknown = [f for f in self.filters if f not in FILTER_NAMES]
        if unknown:
            raise ConfigError(f"unknown filters {unknown}; available: {list(FILTER_NAMES)}")

    def bank_config(self, runs: int) -> BankConfig:
        return BankConfig(n_per_axis=self.n_per_axis, sigma_mult=self.sigma_mult, round_tol=self.round_tol,
                          round_max_rank=self.round_max_rank, tol=self.cross_tol,
                          max_rank=self.cross_max_rank, rng_seed=self.cross_seed, ws_bytes=self.ws_mb << 20,
                          state_doubles=1 << 18, cache_cap=1 << 18)


@dataclass(frozen=True)
class FilterOutcome:
    """Aggregated result of one filter over all Monte Carlo runs (bench.py:236-253)."""

    name: str
    dim: int
    rmse: tuple | None
    rel_diff_pct: float | None
    bytes_tpm: int
    bytes_pmd: int
    storage_estimated: bool
    ms_per_step: float | None
    clipped_mass: float | None
    max_mass_dev: float | None
    failure: str | None
    skipped: str | None
    diagnostics: tuple = ()
    trace: tuple | None = None


@dataclass(frozen=True)
class RunReport:
    scenario: str
    runs: int
    k_f: int
    rows: tuple = field(default_factory=tuple)

    def row(self, name: str, dim: int | None = None) -> FilterOutcome:
        for r in self.rows:
            if r.name == name and (dim is None or r.dim == dim):
                return r
        raise KeyError(f"no outcome for filter {name!r} (dim {dim})")


def scenario_model(scenario: str):
    """(spec, prior mean, prior cov) as _scenario_model (bench.py:291-301)."""
    radar_prior = (np.array([20.0, 20.0]), np.diag([9.0, 9.0]))
    if scenario == "radar":
        return (SPECS["radar"],) + radar_prior
    if scenario == "linear2d":
        return (_linear2d_spec(),) + radar_prior
    if scenario == "linear1d":
        return _linear1d_spec(), np.zeros(1), 2.0 * np.eye(1)
    raise ConfigError(f"unknown compare scenario {scenario!r}; available: {list(COMPARE_SCENARIOS)}")


def trajectories(cfg: RunConfig, spec, mean, cov):
    """_trajectories (bench.py:304-314): SeedSequence((master_seed, run, 0))."""
    st, ms = [], []
    for r in range(cfg.runs):
        s, m = simulate(spec, mean, cov, cfg.k_f, np.random.SeedSequence((cfg.master_seed, r, 0)))
        st.append(s)
        ms.append(m)
    return np.stack(st), np.stack(ms)


def _pmd_bytes(bank: FilterBank) -> int:
    """TensorTrain.storage_bytes of the largest current density (8 * sum core sizes)."""
    best = 0
    for h in bank.headers():
        d = int(h["d"])
        n, r = h["n"][:d], h["r"][: d + 1]
        best = max(best, 8 * int(sum(int(r[k]) * int(n[k]) * int(r[k + 1]) for k in range(d))))
    return best


def run_filter_gpu(name, spec, mean, cov, states, meas, cfg: RunConfig, backend=None) -> FilterOutcome:
    """_run_grid_filter (bench.py:317-392) for every run at once on the device
    (ttfft-gpu: tt_fft_pmf_step; tt-gpu: tt_pmf_step), or run by run for the
    dense fft-gpu filter (dense_fft_pmf_step)."""
    if name not in FILTER_NAMES:
        raise ConfigError(f"unknown filter {name!r}")
    if name == "fft-gpu":
        return _run_dense_gpu(name, spec, mean, cov, states, meas, cfg, backend)
    runs, k_f = meas.shape[0], meas.shape[1]
    d = np.asarray(spec["F"]).shape[0]
    bank = FilterBank(spec, cfg.bank_config(runs), runs, backend=backend)
    dg = bank.init_prior(mean, cov)
    if np.any(dg["status"] != 0):
        bad = int(np.nonzero(dg["status"] != 0)[0][0])
        return _failed(name, d, f"run {bad}: initial density status {int(dg['status'][bad])}")
    times, errors = [], []
    clipped = mass_dev = before_dev = cross_err = 0.0
    calls = unconv = 0
    bytes_pmd = _pmd_bytes(bank)
    trace = []
    sync = getattr(bank.be, "sync", None)
    for k in range(k_f):
        if sync:
            sync()
        t0 = time.perf_counter()
        res = bank.step(meas[:, k], standard=(name == "tt-gpu"))
        if sync:
            sync()
        times.append((time.perf_counter() - t0) / runs)
        st = res["status"]
        if np.any(st != 0):
            bad = int(np.nonzero(st != 0)[0][0])
            return _failed(name, d, f"run {bad} step {k}: status {int(st[bad])} "
                                    f"({bank.lib.ttgbf_status_string(int(st[bad])).decode()})")
        err = res["mean"] - states[:, k]
        errors.append(err)
        rec = res["time"]   # the step's StepDiagnostics (one diag record per filter across the stages)
        clipped = max(clipped, float(np.max(rec["clipped_mass"])))
        mb = rec["mass_before_norm"]
        mb = mb[np.isfinite(mb)]
        if mb.size:
            before_dev = max(before_dev, float(np.max(np.abs(mb - 1.0))))
        for q in range(3):
            ci = rec["cross"][:, q]
            used = ci["calls"] > 0
            if used.any():
                cross_err = max(cross_err, float(np.max(ci["achieved"][used])))
                calls += int(ci["calls"][used].sum())
                unconv += int((ci["converged"][used] == 0).sum())
        bytes_pmd = max(bytes_pmd, _pmd_bytes(bank))
        for i in range(runs):   # PmdEstimate.mass (filters.py:227): tt_sum * cell volume
            m = _tt_sum(bank.cores(i)) * bank.grids[i].cell_volume()
            mass_dev = max(mass_dev, abs(m - 1.0))
        trace.append((float(k), *states[0, k], *res["mean"][0], *err[0]))
    rmse = tuple(float(v) for v in np.sqrt(np.mean(np.square(np.concatenate(errors)), axis=0)))
    diagnostics = (("cross_achieved_max", cross_err), ("cross_calls_total", float(calls)),
                   ("cross_unconverged_steps", float(unconv)), ("max_mass_before_norm_dev", before_dev))
    return FilterOutcome(name=name, dim=d, rmse=rmse, rel_diff_pct=None, bytes_tpm=0, bytes_pmd=bytes_pmd,
                         storage_estimated=False, ms_per_step=1000.0 * float(np.median(times)),
                         clipped_mass=clipped, max_mass_dev=mass_dev, failure=None, skipped=None,
                         diagnostics=diagnostics, trace=tuple(trace))


def _run_dense_gpu(name, spec, mean, cov, states, meas, cfg: RunConfig, backend=None) -> FilterOutcome:
    """The reference's dense 'fft' row (bench.py:321-327 with dense_fft_pmf_step)."""
    from .dense import DegenerateDensityError, DenseFFTFilter
    runs, k_f = meas.shape[0], meas.shape[1]
    d = np.asarray(spec["F"]).shape[0]
    f = DenseFFTFilter(spec, cfg.n_per_axis, cfg.sigma_mult, backend)
    times, errors, trace = [], [], []
    clipped = mass_dev = before_dev = 0.0
    for r in range(runs):
        f.initial(mean, cov)
        for k in range(k_f):
            f.be.sync()
            t0 = time.perf_counter()
            try:
                dg = f.step(meas[r, k])
            except DegenerateDensityError as exc:
                return _failed(name, d, f"run {r} step {k}: {exc}")
            f.be.sync()
            times.append(time.perf_counter() - t0)
            err = dg.filt_mean - states[r, k]
            errors.append(err)
            clipped = max(clipped, dg.clipped_mass)
            if math.isfinite(dg.mass_before_norm):
                before_dev = max(before_dev, abs(dg.mass_before_norm - 1.0))
            pos, neg = f._reduce(f.w, f._axes_host(f.grid), 0)
            mass_dev = max(mass_dev, abs((pos + neg) * f.grid.cell_volume() - 1.0))
            if r == 0:
                trace.append((float(k), *states[0, k], *dg.filt_mean, *err))
    rmse = tuple(float(v) for v in np.sqrt(np.mean(np.square(np.array(errors)), axis=0)))
    return FilterOutcome(name=name, dim=d, rmse=rmse, rel_diff_pct=None, bytes_tpm=f.total * 8,
                         bytes_pmd=f.total * 8, storage_estimated=False,
                         ms_per_step=1000.0 * float(np.median(times)), clipped_mass=clipped, max_mass_dev=mass_dev,
                         failure=None, skipped=None,
                         diagnostics=(("max_mass_before_norm_dev", before_dev),), trace=tuple(trace))


def _tt_sum(cores) -> float:
    v = np.ones(1)
    for c in cores:
        v = v @ c.sum(axis=1)
    return float(v[0])


def _failed(name, d, msg):
    return FilterOutcome(name=name, dim=d, rmse=None, rel_diff_pct=None, bytes_tpm=0, bytes_pmd=0,
                         storage_estimated=False, ms_per_step=None, clipped_mass=None, max_mass_dev=None,
                         failure=msg, skipped=None)


def with_rel_diffs(rows, reference_rmse=None):
    """rel_diff_pct against a dense-filter RMSE when one is supplied (bench.py:481-492)."""
    if reference_rmse is None:
        return tuple(rows)
    out = []
    for r in rows:
        if r.rmse is None:
            out.append(r)
        else:
            rel = 100.0 * max(abs(a - b) / b for a, b in zip(r.rmse, reference_rmse))
            out.append(replace(r, rel_diff_pct=rel))
    return tuple(out)


def run_compare(cfg: RunConfig, backend=None, reference_rmse=None) -> RunReport:
    """run_compare (bench.py:495-504) for the GPU filters."""
    spec, mean, cov = scenario_model(cfg.scenario)
    states, meas = trajectories(cfg, spec, mean, cov)
    rows = [run_filter_gpu(n, spec, mean, cov, states, meas, cfg, backend) for n in cfg.filters]
    return RunReport(cfg.scenario, cfg.runs, cfg.k_f, with_rel_diffs(rows, reference_rmse))


def run_scaling(cfg: RunConfig, dims: Sequence[int], backend=None) -> list:
    """run_scaling (bench.py:507-560): scaling_model(dim), prior N(20*1, 9 I)."""
    reports = []
    for dim in dims:
        if dim < 2:
            raise ConfigError(f"scaling dimensions must be >= 2, got {dim}")
        spec = scaling_spec(dim)
        mean, cov = 20.0 * np.ones(dim), 9.0 * np.eye(dim)
        states, meas = trajectories(cfg, spec, mean, cov)
        rows = tuple(run_filter_gpu(n, spec, mean, cov, states, meas, cfg, backend) for n in cfg.filters)
        reports.append(RunReport(f"scaling-{dim}", cfg.runs, cfg.k_f, rows))
    return reports


# ---------------------------------------------------------------------------
# CSV output (bench.py:563-650)
# ---------------------------------------------------------------------------
SUMMARY_HEADER = "filter,d,rmse_x,rmse_y,rel_diff_pct,bytes_tpm,bytes_pmd,ms_per_step,clipped_mass"


def _axis_label(i: int) -> str:
    return ("x", "y")[i] if i < 2 else f"x{i + 1}"


def _fmt(value, spec: str) -> str:
    return "" if value is None else format(value, spec)


def _bytes_field(value: int, estimated: bool) -> str:
    return f"estimated:{value}" if estimated else str(value)


def summary_lines(report: RunReport) -> list:
    lines = [SUMMARY_HEADER]
    for r in report.rows:
        rmse_x = _fmt(r.rmse[0] if r.rmse else None, ".6f")
        rmse_y = _fmt(r.rmse[1] if r.rmse is not None and len(r.rmse) > 1 else None, ".6f")
        lines.append(",".join([r.name, str(r.dim), rmse_x, rmse_y, _fmt(r.rel_diff_pct, ".4f"),
                               _bytes_field(r.bytes_tpm, r.storage_estimated),
                               _bytes_field(r.bytes_pmd, r.storage_estimated), "",
                               _fmt(r.clipped_mass, ".3e")]))
    return lines


def emit_csv(report: RunReport, out_dir) -> list:
    """summary.csv (wall-clock left empty, as the reference), per-filter
    trace CSVs and timings.txt."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    written = []
    p = out / "summary.csv"
    p.write_text("\n".join(summary_lines(report)) + "\n", encoding="utf-8")
    written.append(p)
    for r in report.rows:
        if not r.trace:
            continue
        d = r.dim
        head = (["k"] + [f"true_{_axis_label(i)}" for i in range(d)] + [f"est_{_axis_label(i)}" for i in range(d)]
                + [f"err_{_axis_label(i)}" for i in range(d)])
        lines = [",".join(head)] + [",".join([str(int(row[0]))] + [format(v, ".9g") for v in row[1:]])
                                    for row in r.trace]
        tp = out / f"trace_{r.name}.csv"
        tp.write_text("\n".join(lines) + "\n", encoding="utf-8")
        written.append(tp)
    tl = ["# median per-step wall clock in milliseconds (filter steps only);",
          "# batched device step time divided by the runs in the batch;",
          "# measured anew each execution, not part of the deterministic CSV outputs"]
    for r in report.rows:
        value = "skipped" if r.skipped else _fmt(r.ms_per_step, ".3f") or "failed"
        tl.append(f"{r.name} d={r.dim} {value}")
    tpath = out / "timings.txt"
    tpath.write_text("\n".join(tl) + "\n", encoding="utf-8")
    written.append(tpath)
    return written


def failures(report: RunReport):
    return tuple(r for r in report.rows if r.failure is not None)


def finite(x) -> bool:
    return x is not None and math.isfinite(x)
