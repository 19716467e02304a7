"""The cross black boxes (ttgbf_eval_blackbox) against values produced by the
REAL reference (tests/golden/models.npz): StateSpaceModel.likelihood
(models.py:150-153) at 300 random points and _kernel_values (filters.py:697-706)
at 200 grid indices, for all 8 model specs -- including cv6 (range_az_el with
the correlated-Q kernel, BASELINE C3/C5) and chain10 (chain_quadratic, C4) --
plus the prior pdf and the realign evaluator against the oracle.  Relative
tolerance 1e-13.  Runs on the GPU (-m gpu) and, for the CPU suite, on the
engine's host emulation."""

import numpy as np
import pytest

from oracle import ttcore as T
from paper_2501_07942_b200 import evaluators as ev
from paper_2501_07942_b200 import geometry as geo
from paper_2501_07942_b200.configs import SPECS
from scenario_util import rel, use_backend

TOL = 1e-13
# likelihood / kernel values are exp(log-density): one ulp of the log-density
# (the solve and the transcendental functions round differently from numpy's
# LAPACK / SVML code) moves the value by 2**-52 |log v|, up to ~1e-13 here
TOL_EXP = 1e-12


def kernel_grid(z, name, d):
    axes = np.split(z[f"{name}/kaxes"], d)
    return geo.grid_from_bounds([a[0] for a in axes], [a[-1] for a in axes], [a.size for a in axes])


def check_models(golden):
    z = golden("models")
    for name, spec in SPECS.items():
        d = spec["F"].shape[0]
        lik = ev.likelihood_at_points(spec, z[f"{name}/z"], z[f"{name}/x"])
        assert rel(lik, z[f"{name}/lik"]) <= TOL_EXP, (name, "likelihood", rel(lik, z[f"{name}/lik"]))
        kern = ev.kernel_values(spec, kernel_grid(z, name, d), z[f"{name}/kidx"])
        assert rel(kern, z[f"{name}/kern"]) <= TOL_EXP, (name, "kernel", rel(kern, z[f"{name}/kern"]))


def check_prior_realign():
    rng = np.random.default_rng(3)
    spec = SPECS["cv6"]
    d = 6
    mean = np.array([10.0, 10.0, 10.0, 1.0, 1.0, 1.0])
    cov = np.diag([1.0, 1.0, 1.0, 0.1, 0.1, 0.1])
    cov[0, 1] = cov[1, 0] = 0.2
    grid = geo.design_grid(mean, cov, 17, 6.0)
    idx = np.stack([rng.integers(0, 17, 500) for _ in range(d)], axis=1)
    got = ev.prior_values(mean, cov, grid, idx)
    x = np.stack([grid.axes()[k][idx[:, k]] for k in range(d)], axis=1) - mean
    L = np.linalg.cholesky(cov)
    sol = np.linalg.solve(L, x.T)
    ref = np.exp(-0.5 * np.sum(sol * sol, axis=0)) / np.sqrt((2 * np.pi) ** d * np.linalg.det(cov))
    assert rel(got, ref) <= 1e-12
    # realign: a random TT on the filtering grid at F^-1 y, y on the predictive grid
    from paper_2501_07942_b200.tensor_train import TensorTrain
    ranks = (1, 3, 5, 4, 6, 2, 1)
    cores = [rng.standard_normal((ranks[k], 17, ranks[k + 1])) for k in range(d)]
    fgrid = geo.design_grid(mean, 2.0 * cov, 17, 6.0)
    F = np.asarray(spec["F"])
    pgrid = geo.design_grid(F @ mean, F @ cov @ F.T + np.asarray(spec["Q"]), 17, 6.0)
    got = ev.realign_values(spec, TensorTrain.from_cores(cores), fgrid, pgrid, idx)
    y = np.stack([pgrid.axes()[k][idx[:, k]] for k in range(d)], axis=1)
    pts = y @ np.linalg.inv(F).T
    ref = T.at_points(cores, fgrid.axes(), pts)
    assert rel(got, ref) <= TOL


def test_evaluators_hostsim(golden):
    from hostsim import HostBackend
    use_backend(HostBackend())
    check_models(golden)
    check_prior_realign()


@pytest.mark.gpu
def test_evaluators_gpu(golden):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    use_backend(CudaBackend())
    check_models(golden)
    check_prior_realign()
