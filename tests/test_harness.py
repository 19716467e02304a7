"""Harness integration: the ttfft-gpu filter row in the
reference's compare harness layout (ttpmf/bench.py:83-125, 563-650)."""

import numpy as np
import pytest

from paper_2501_07942_b200 import harness as H


def test_runconfig_validation():
    with pytest.raises(H.ConfigError):
        H.RunConfig(scenario="radar", n_per_axis=32)
    with pytest.raises(H.ConfigError):
        H.RunConfig(scenario="radar", filters=("dense",))
    with pytest.raises(H.ConfigError):
        H.RunConfig(scenario="")
    with pytest.raises(H.ConfigError):
        H.scenario_model("nope")
    cfg = H.RunConfig(scenario="radar")
    assert (cfg.runs, cfg.k_f, cfg.master_seed, cfg.n_per_axis, cfg.sigma_mult) == (10, 10, 2024, 33, 4.0)


def test_trajectories_match_reference_seeding():
    """_trajectories (bench.py:304-314): run r uses SeedSequence((master_seed, r, 0))."""
    from paper_2501_07942_b200.configs import simulate
    cfg = H.RunConfig(scenario="radar", runs=3, k_f=4)
    spec, m, c = H.scenario_model("radar")
    st, ms = H.trajectories(cfg, spec, m, c)
    s2, m2 = simulate(spec, m, c, 4, np.random.SeedSequence((2024, 2, 0)))
    assert np.array_equal(st[2], s2) and np.array_equal(ms[2], m2)


def test_emit_csv_layout(tmp_path):
    row = H.FilterOutcome(name="ttfft-gpu", dim=2, rmse=(1.25, 0.5), rel_diff_pct=None, bytes_tpm=0,
                          bytes_pmd=4096, storage_estimated=False, ms_per_step=1.5, clipped_mass=1e-3,
                          max_mass_dev=1e-15, failure=None, skipped=None,
                          trace=((0.0, 1.0, 2.0, 1.1, 2.2, 0.1, 0.2),))
    rep = H.RunReport("radar", 2, 1, (row,))
    paths = H.emit_csv(rep, tmp_path)
    assert [p.name for p in paths] == ["summary.csv", "trace_ttfft-gpu.csv", "timings.txt"]
    lines = (tmp_path / "summary.csv").read_text().splitlines()
    assert lines[0] == "filter,d,rmse_x,rmse_y,rel_diff_pct,bytes_tpm,bytes_pmd,ms_per_step,clipped_mass"
    assert lines[1] == "ttfft-gpu,2,1.250000,0.500000,,0,4096,,1.000e-03"
    tr = (tmp_path / "trace_ttfft-gpu.csv").read_text().splitlines()
    assert tr[0] == "k,true_x,true_y,est_x,est_y,err_x,err_y"
    assert tr[1] == "0,1,2,1.1,2.2,0.1,0.2"
    assert (tmp_path / "timings.txt").read_text().splitlines()[-1] == "ttfft-gpu d=2 1.500"


def _compare_with_oracle(backend, runs, k_f):
    """run_compare('radar') against the oracle run by run: run 0's trace means
    within 1e-8 (tier-3 tolerance) and the RMSE row within 1e-7.  Cross tol
    1e-10 makes every cross exact (pivot-independent, SURVEY 8(c) tier 3);
    at the harness default 1e-2 single runs are ulp-chaotic."""
    from oracle import pmf
    cfg = H.RunConfig(scenario="radar", filters=("ttfft-gpu",), runs=runs, k_f=k_f, cross_tol=1e-10)
    rep = H.run_compare(cfg, backend=backend)
    row = rep.row("ttfft-gpu")
    assert row.failure is None, row.failure
    spec, m, c = H.scenario_model("radar")
    states, meas = H.trajectories(cfg, spec, m, c)
    g = {"n_per_axis": 33, "sigma_mult": 4.0, "round_tol": 1e-8}
    x = {"tol": 1e-10, "max_rank": 150, "rng_seed": 0}
    errs = []
    for r in range(cfg.runs):
        axes, cores, _ = pmf.initial(m, c, g, x)
        for k in range(cfg.k_f):
            axes, cores, diag = pmf.step(axes, cores, spec, meas[r, k], g, x)
            errs.append(diag["filt_mean"] - states[r, k])
            if r == 0:
                got = np.array(row.trace[k][3:5])
                assert row.trace[k][0] == k and np.array_equal(row.trace[k][1:3], states[0, k])
                assert np.max(np.abs(got - diag["filt_mean"])) <= 1e-8 * np.max(np.abs(diag["filt_mean"]))
    rmse = np.sqrt(np.mean(np.square(np.array(errs)), axis=0))
    assert np.allclose(row.rmse, rmse, rtol=1e-7, atol=0)
    assert row.max_mass_dev < 1e-10
    assert row.ms_per_step > 0
    assert dict(row.diagnostics)["cross_calls_total"] > 0


def test_compare_radar_hostsim_matches_oracle():
    from hostsim import HostBackend
    _compare_with_oracle(HostBackend(), runs=2, k_f=2)


@pytest.mark.gpu
def test_compare_radar_gpu_matches_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    _compare_with_oracle(None, runs=4, k_f=4)


def _compare_standard(backend):
    """tt-gpu row (tt_pmf_step) on the linear1d scenario with an exact
    transition cross, against the oracle run by run."""
    from oracle import pmf
    cfg = H.RunConfig(scenario="linear1d", filters=("tt-gpu",), runs=2, k_f=3, cross_tol=1e-12,
                      cross_max_rank=40)
    row = H.run_compare(cfg, backend=backend).row("tt-gpu")
    assert row.failure is None, row.failure
    spec, m, c = H.scenario_model("linear1d")
    states, meas = H.trajectories(cfg, spec, m, c)
    g = {"n_per_axis": 33, "sigma_mult": 4.0, "round_tol": 1e-8}
    x = {"tol": 1e-12, "max_rank": 40, "rng_seed": 0}
    errs = []
    for r in range(cfg.runs):
        axes, cores, _ = pmf.initial(m, c, g, x)
        for k in range(cfg.k_f):
            axes, cores, dg = pmf.step_std(axes, cores, spec, meas[r, k], g, x)
            errs.append(dg["filt_mean"] - states[r, k])
    rmse = np.sqrt(np.mean(np.square(np.array(errs)), axis=0))
    assert np.allclose(row.rmse, rmse, rtol=1e-7, atol=0)


def test_compare_standard_hostsim():
    from hostsim import HostBackend
    _compare_standard(HostBackend())


@pytest.mark.gpu
def test_compare_standard_and_dense_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    _compare_standard(None)
    from oracle import dense as D
    cfg = H.RunConfig(scenario="radar", filters=("fft-gpu",), runs=2, k_f=3)
    row = H.run_compare(cfg).row("fft-gpu")
    assert row.failure is None, row.failure
    spec, m, c = H.scenario_model("radar")
    states, meas = H.trajectories(cfg, spec, m, c)
    errs = []
    for r in range(cfg.runs):
        axes, w, _ = D.initial(m, c, {"n_per_axis": 33, "sigma_mult": 4.0})
        for k in range(cfg.k_f):
            axes, w, dg = D.step(axes, w, spec, meas[r, k], {"n_per_axis": 33, "sigma_mult": 4.0})
            errs.append(dg["filt_mean"] - states[r, k])
    rmse = np.sqrt(np.mean(np.square(np.array(errs)), axis=0))
    assert np.allclose(row.rmse, rmse, rtol=1e-8, atol=0)
    assert row.max_mass_dev <= 1e-12
