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
