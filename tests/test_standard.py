"""Algorithm 2 -- the TT standard point-mass filter tt_pmf_step
(filters.py:855-885): transition cross over the
concatenated (new grid, old grid) modes + tt_einsum_tpm contraction.

CPU: the oracle against the reference's golden trajectories
(tests/golden/standard.npz) and the host emulation of the device engine
against the same goldens.  GPU: the sm_100a engine through the C-ABI.
Tolerances: means 1e-8, covariances / densities 1e-7, equal ranks.
"""

import numpy as np
import pytest

from conftest import load_tt
from oracle import pmf
from oracle import ttcore as T
from paper_2501_07942_b200.configs import SPECS

LIN1 = {"F": np.array([[0.9]]), "Q": np.array([[1.0]]), "R": np.array([[1.0]]), "h": "linear",
        "H": np.array([[1.0]]), "angle_components": ()}
CASES = {"linear1d": (LIN1, np.zeros(1), 2.0 * np.eye(1), {"tol": 1e-8, "max_rank": 20, "rng_seed": 0}),
         "linear1d_exact": (LIN1, np.zeros(1), 2.0 * np.eye(1), {"tol": 1e-12, "max_rank": 40, "rng_seed": 0}),
         "scaling2": (SPECS["scaling2"], np.array([20.0, 20.0]), np.diag([9.0, 9.0]),
                      {"tol": 1e-10, "max_rank": 150, "rng_seed": 0})}
GRID = {"n_per_axis": 33, "sigma_mult": 4.0, "round_tol": 1e-8}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def test_einsum_tpm_dense():
    """tt_einsum_tpm against the dense contraction (test_tt_algorithms.py:160-190)."""
    rng = np.random.default_rng(0)
    t = [rng.standard_normal(s) for s in [(1, 4, 3), (3, 5, 2), (2, 4, 3), (3, 5, 1)]]
    w = [rng.standard_normal(s) for s in [(1, 4, 2), (2, 5, 1)]]
    full_t = T.to_full(t)
    full_w = T.to_full(w)
    ref = np.einsum("abcd,cd->ab", full_t, full_w)
    assert rel(T.to_full(T.einsum_tpm(t, w)), ref) <= 1e-13


# steps compared: all where the reference's transition cross decisions are
# reproducible; scaling2's cross stops at the rank cap unconverged (error
# ~1), so from step 2 on its pivots follow ulp-level differences
STEPS = {"linear1d": 5, "linear1d_exact": 5, "scaling2": 2}


@pytest.mark.parametrize("name", ["linear1d", "linear1d_exact", "scaling2"])
def test_oracle_standard_pinned(golden, name):
    z = golden("standard")
    spec, mean, cov, cc = CASES[name]
    axes, cores, _ = pmf.initial(mean, cov, GRID, cc)
    assert rel(T.to_full(cores), T.to_full(load_tt(z, f"{name}/init"))) <= 1e-13
    for k in range(STEPS[name]):
        axes, cores, dg = pmf.step_std(axes, cores, spec, z[f"{name}/z"][k], GRID, cc)
        assert rel(dg["filt_mean"], z[f"{name}/{k}/filt_mean"]) <= 1e-12
        assert rel(dg["filt_cov"], z[f"{name}/{k}/filt_cov"]) <= 1e-11
        ref = load_tt(z, f"{name}/{k}/pred")
        assert T.ranks_of(cores) == T.ranks_of(ref)
        assert rel(T.to_full(cores), T.to_full(ref)) <= 1e-9   # einsum contraction order
        c = z[f"{name}/{k}/cross"]
        assert dg["cross"]["transition"][1] == int(c[1][1])      # evaluator calls, bit-identical cross


def bank_standard(backend, golden, name):
    """The device engine's Algorithm-2 stages (FilterBank.measure / geometry /
    time_update_std) against the golden trajectory; returns per-step errors."""
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    z = golden("standard")
    spec, mean, cov, cc = CASES[name]
    cfg = BankConfig(n_per_axis=33, sigma_mult=4.0, round_tol=1e-8, tol=cc["tol"], max_rank=cc["max_rank"],
                     rng_seed=0, ws_bytes=512 << 20, state_doubles=1 << 18, cache_cap=1 << 20)
    bank = FilterBank(spec, cfg, 1, backend=backend)
    assert int(bank.init_prior(mean, cov)["status"][0]) == 0
    assert rel(T.to_full(bank.cores(0)), T.to_full(load_tt(z, f"{name}/init"))) <= 1e-12
    rows = []
    for k in range(STEPS[name]):
        dm = bank.measure(z[f"{name}/z"][k][None])
        assert int(dm["status"][0]) == 0
        geom = bank.geometry(dm)
        dt = bank.time_update_std(geom)
        assert int(dt["status"][0]) == 0, dt["status"]
        ref = load_tt(z, f"{name}/{k}/pred")
        got = bank.cores(0)
        rows.append({"mean": rel(geom[0][1][0], z[f"{name}/{k}/filt_mean"]),
                     "cov": rel(geom[0][1][1], z[f"{name}/{k}/filt_cov"]),
                     "dens": rel(T.to_full(got), T.to_full(ref)),
                     "ranks": (T.ranks_of(got), T.ranks_of(ref)),
                     "calls": (int(dt["cross"][0][1]["calls"]), int(z[f"{name}/{k}/cross"][1][1]))})
    return rows


def check_rows(rows):
    for r in rows:
        assert r["mean"] <= 1e-8 and r["cov"] <= 1e-7 and r["dens"] <= 1e-7, r
        assert r["ranks"][0] == r["ranks"][1], r


def test_standard_hostsim(golden):
    from hostsim import HostBackend
    check_rows(bank_standard(HostBackend(), golden, "linear1d_exact"))


def test_tracks_kalman_hostsim():
    """The reference's own Algorithm-2 test (test_filters.py:307-321): on the 1-D
    linear-Gaussian model the filtered moments track the Kalman filter."""
    from hostsim import HostBackend
    _tracks_kalman(HostBackend())


def _tracks_kalman(backend):
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    from paper_2501_07942_b200.configs import simulate
    mean, cov = np.zeros(1), np.array([[2.0]])
    states, zs = simulate(LIN1, mean, cov, 10, np.random.SeedSequence(11))
    cfg = BankConfig(n_per_axis=33, sigma_mult=4.0, round_tol=1e-8, tol=1e-8, max_rank=20, rng_seed=0,
                     ws_bytes=256 << 20, state_doubles=1 << 16, cache_cap=1 << 18)
    bank = FilterBank(LIN1, cfg, 1, backend=backend)
    bank.init_prior(mean, cov)
    m, P = mean.copy(), cov.copy()
    F, Q, R = 0.9, 1.0, 1.0
    for k in range(10):
        # Kalman update then predict (kalman_reference, filters.py:393-419)
        K = P[0, 0] / (P[0, 0] + R)
        mf, Pf = m[0] + K * (zs[k][0] - m[0]), (1 - K) * P[0, 0]
        dm = bank.measure(zs[k][None])
        geom = bank.geometry(dm)
        gm, gc = geom[0][1][0], geom[0][1][1]
        assert abs(gm[0] - mf) <= 0.01 * np.sqrt(Pf)
        assert abs(gc[0, 0] - Pf) <= 0.01 * Pf
        assert int(bank.time_update_std(geom)["status"][0]) == 0
        m, P = np.array([F * mf]), np.array([[F * F * Pf + Q]])


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    return CudaBackend()


@pytest.mark.gpu
def test_standard_gpu(golden, cuda):
    check_rows(bank_standard(cuda, golden, "linear1d_exact"))


@pytest.mark.gpu
def test_standard_unconverged_cross_gpu(golden, cuda):
    """scaling2 with the reference's settings: the transition cross stops at the
    rank cap with error ~1, so its pivots (and the predicted density) follow
    ulp-level differences.  Compared: the measurement stage (filtered means of
    step 0) and the time update's invariants (completes, unit mass)."""
    rows = bank_standard_loose(cuda, golden, "scaling2")
    assert rows[0]["mean"] <= 1e-8 and rows[0]["cov"] <= 1e-7
    for r in rows:
        assert abs(r["mass"] - 1.0) <= 1e-10


def bank_standard_loose(backend, golden, name):
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    z = golden("standard")
    spec, mean, cov, cc = CASES[name]
    cfg = BankConfig(n_per_axis=33, sigma_mult=4.0, round_tol=1e-8, tol=cc["tol"], max_rank=cc["max_rank"],
                     rng_seed=0, ws_bytes=512 << 20, state_doubles=1 << 18, cache_cap=1 << 20)
    bank = FilterBank(spec, cfg, 1, backend=backend)
    bank.init_prior(mean, cov)
    rows = []
    for k in range(STEPS[name]):
        dm = bank.measure(z[f"{name}/z"][k][None])
        geom = bank.geometry(dm)
        dt = bank.time_update_std(geom)
        assert int(dt["status"][0]) == 0, dt["status"]
        got = bank.cores(0)
        rows.append({"mean": rel(geom[0][1][0], z[f"{name}/{k}/filt_mean"]),
                     "cov": rel(geom[0][1][1], z[f"{name}/{k}/filt_cov"]),
                     "mass": T.total(got) * bank.grids[0].cell_volume()})
    return rows


@pytest.mark.gpu
def test_tracks_kalman_gpu(cuda):
    _tracks_kalman(cuda)


@pytest.mark.gpu
def test_tt_pmf_step_api_gpu(golden, cuda):
    """filters.tt_pmf_step (reference name and signature) on linear1d_exact."""
    from paper_2501_07942_b200 import filters as Fl
    from paper_2501_07942_b200.grids import MomentEstimate
    from paper_2501_07942_b200.models import StateSpaceModel
    z = golden("standard")
    model = StateSpaceModel.from_spec(LIN1)
    cfg = Fl.GridConfig(n_per_axis=33, sigma_mult=4.0)
    cc = Fl.CrossConfig(tol=1e-12, max_rank=40, rng_seed=0)
    pmd = Fl.initial_pmd_tt(MomentEstimate(np.zeros(1), 2.0 * np.eye(1)), cfg, cc, model=model)
    for k in range(3):
        pmd = Fl.tt_pmf_step(pmd, model, z[f"linear1d_exact/z"][k], cfg, cc)
        assert rel(pmd.diag.filt_moments.mean, z[f"linear1d_exact/{k}/filt_mean"]) <= 1e-8
        ref = load_tt(z, f"linear1d_exact/{k}/pred")
        assert rel(T.to_full(pmd.weights.numpy_cores()), T.to_full(ref)) <= 1e-7
        assert "transition" in pmd.diag.cross_info
