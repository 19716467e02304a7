"""GPU parity on the BASELINE configs against full-step goldens of the REAL
reference (tests/golden/baseline.npz, make_golden.baseline): runs 0-7 of
C1/C2/C3 (metric cross, steps 0-1 or 0-2) and C4 (int64-key workaround only,
see make_golden._BigKeyEvaluator), through both engine paths:

* the stage API (FilterBank.step: measure launch, host numpy geometry,
  time-update launch), and
* the persistent kernel ttgbf_filter_run with device geometry -- the path
  bench.py times.

Per (run, step): the reference's failure step is reproduced (status), and for
completed steps the filtered mean (1e-8) and full covariance (1e-7), the
density at 10^4 seeded indices (1e-7), the output ranks, the grid axes,
mass_before_norm, clipped_mass and the three cross call counts match."""

import pytest

from scenario_util import check_baseline, compare_baseline

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    return CudaBackend()


@pytest.mark.parametrize("name", ["C1", "C3", "C2", "C4"])
def test_baseline_stage_api_gpu(golden, cuda, name):
    check_baseline(compare_baseline(golden, name, cuda))


@pytest.mark.parametrize("name", ["C1", "C3", "C2", "C4"])
def test_baseline_persistent_gpu(golden, cuda, name):
    check_baseline(compare_baseline(golden, name, cuda, persistent=True))
