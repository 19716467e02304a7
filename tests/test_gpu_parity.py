"""GPU parity: the sm_100a library through the C-ABI against the oracle and
the reference's golden vectors (tolerances from BASELINE.json north_star:
means 1e-8, covariances/densities 1e-7 relative, equal ranks)."""

import numpy as np
import pytest

from conftest import load_tt
from oracle import ttcore as T
from scenario_util import check, compare_scenario, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    return CudaBackend()


@pytest.mark.parametrize("name", ["scaling2_tight", "radar_deg", "identity2", "cv4_step0"])
def test_golden_trajectory_gpu(golden, cuda, name):
    check(compare_scenario(golden, name, cuda))


@pytest.mark.parametrize("case", ["s3", "s4", "s6"])
def test_primitives_gpu(golden, cuda, case):
    from scenario_util import check_primitives, use_backend
    use_backend(cuda)
    check_primitives(golden, case)


def test_round_rank_deficient_gpu(golden, cuda):
    from paper_2501_07942_b200 import tensor_train as G
    from scenario_util import use_backend
    use_backend(cuda)
    z = golden("primitives")
    a = G.TensorTrain.from_cores(load_tt(z, "sq/a"))
    got = G.tt_round(G.tt_hadamard(a, a), 1e-10)
    ref = load_tt(z, "sq/round")
    assert got.ranks == T.ranks_of(ref)
    assert rel(T.to_full(got.numpy_cores()), T.to_full(ref)) <= 1e-12


@pytest.mark.parametrize("case", ["s3", "s4", "s6"])
def test_large_eval_gpu(golden, cuda, case):
    from scenario_util import check_large_eval, use_backend
    use_backend(cuda)
    check_large_eval(golden, case)


@pytest.mark.parametrize("ranks,tol", [((1, 60, 60, 1), 1e-6), ((1, 40, 90, 40, 1), 1e-8), ((1, 130, 70, 1), 1e-10)])
def test_round_tall_cores_gpu(cuda, ranks, tol):
    """Tall unfoldings (m = n*r' > 2048): two-level panels, Gram-built T, DMMA
    trailing updates and the in-place triangular R multiply, against the
    oracle's numpy rounding (tensor_train.py:327)."""
    from paper_2501_07942_b200 import tensor_train as G
    from scenario_util import use_backend
    use_backend(cuda)
    rs = np.random.RandomState(sum(ranks))
    n = 65 if len(ranks) == 4 else 21
    cores = []
    for k in range(len(ranks) - 1):
        core = rs.randn(ranks[k], n, ranks[k + 1])
        core *= (0.7 ** np.arange(ranks[k + 1]))[None, None, :]   # decaying spectrum -> real truncation
        cores.append(core)
    ref = T.round_tt(cores, tol)
    got = G.tt_round(G.TensorTrain.from_cores(cores), tol)
    assert got.ranks == T.ranks_of(ref)
    assert rel(T.to_full(got.numpy_cores()), T.to_full(ref)) <= 1e-11


def test_squeeze_ranks_gpu(golden, cuda):
    """Exact-rank squeeze of the cross outputs on BASELINE C3 (correlated-Q
    kernel: its cross output is rank deficient): the ranks the products use
    are below the cross's on some bond, never above."""
    import numpy as np
    from scenario_util import baseline_bank, check_squeeze_ranks
    z = golden("baseline")
    cfg, bank = baseline_bank("C3", 4, cuda)
    Z = np.stack([z[f"C3/{r}/z"] for r in range(4)])
    recs = bank.run(Z, 1, cfg["x0_mean"], cfg["x0_cov"])
    d = cfg["spec"]["F"].shape[0]
    assert (recs["status"][:, 0] == 0).any()
    dropped = check_squeeze_ranks(recs[:, 0], d, expect_drop=True)
    print({"squeezed_bond_directions": dropped})


@pytest.mark.parametrize("name", ["scaling2_tight", "radar_deg", "identity2", "cv4_step0"])
def test_persistent_run_gpu(golden, cuda, name):
    """The benchmarked path -- ttgbf_filter_run, one persistent launch with
    device geometry (geom.cuh) -- against the reference's tier-3 trajectories:
    filtered mean and full covariance every step, mass_before_norm,
    clipped_mass, cross call counts, final density and ranks."""
    from scenario_util import check_run, compare_scenario_run
    check_run(compare_scenario_run(golden, name, cuda))


@pytest.mark.parametrize("name,ws_mb", [("radar_deg", 64), ("cv4_step0", 160)])
def test_persistent_run_overflow_gpu(golden, cuda, name, ws_mb):
    """Force the overflow workspaces: a slot too small for the FFT product /
    Hadamard rounding makes the step redo that stage in a borrowed buffer
    (spin-locked pool, both classes); the result must be the in-slot result."""
    from scenario_util import check_run, compare_scenario_run
    rows_small = compare_scenario_run(golden, name, cuda, ws_bytes=ws_mb << 20, big_slots=1, big_bytes=256 << 20,
                                      big2_slots=1, big2_bytes=1 << 30)
    check_run(rows_small)
    rows = compare_scenario_run(golden, name, cuda)
    for a, b in zip(rows, rows_small):
        assert a == b, (a, b)


@pytest.mark.parametrize("ranks,n,cap", [((1, 90, 700, 120, 1), 21, 20), ((1, 200, 640, 300, 1), 17, None)])
def test_round_wide_gpu(cuda, ranks, n, cap):
    """Product-width rounding (the bench's FFT products reach rank ~700): the
    truncated rank-revealing SVD (pivoted QR stopped at 1e-3 delta) against
    the oracle's full numpy SVD rounding (tensor_train.py:327-360), with the
    rank cap binding and with the tolerance deciding."""
    from paper_2501_07942_b200 import tensor_train as G
    from scenario_util import use_backend
    use_backend(cuda)
    rs = np.random.RandomState(sum(ranks))
    cores = []
    for k in range(len(ranks) - 1):
        core = rs.randn(ranks[k], n, ranks[k + 1])
        core *= (0.93 ** np.arange(ranks[k + 1]))[None, None, :]
        cores.append(core)
    ref = T.round_tt(cores, 1e-8, cap)
    got = G.tt_round(G.TensorTrain.from_cores(cores), 1e-8, cap)
    assert got.ranks == T.ranks_of(ref)
    rng = np.random.default_rng(3)
    idx = np.stack([rng.integers(0, n, 10_000) for _ in range(len(ranks) - 1)], axis=1)
    a, b = T.at_indices(got.numpy_cores(), idx), T.at_indices(ref, idx)
    assert np.max(np.abs(a - b)) <= 1e-9 * np.max(np.abs(b))
