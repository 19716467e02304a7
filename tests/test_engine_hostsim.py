"""CPU: the CUDA engine source, compiled for a one-thread emulated CTA,
against the reference's golden trajectories (tier-3 parity: converging crosses)."""

import pytest

from hostsim import HostBackend
from scenario_util import check, compare_scenario


@pytest.fixture(scope="module")
def backend():
    return HostBackend()


@pytest.mark.parametrize("name", ["scaling2_tight", "radar_deg", "identity2", "cv4_step0"])
def test_golden_trajectory_hostsim(golden, backend, name):
    check(compare_scenario(golden, name, backend))


@pytest.mark.parametrize("case", ["s3", "s4", "s6"])
def test_primitives_hostsim(golden, backend, case):
    from scenario_util import check_primitives, use_backend
    use_backend(backend)
    check_primitives(golden, case)


@pytest.mark.parametrize("name", ["scaling2_tight", "radar_deg", "identity2", "cv4_step0"])
def test_persistent_run_hostsim(golden, backend, name):
    from scenario_util import check_run, compare_scenario_run
    check_run(compare_scenario_run(golden, name, backend))


@pytest.mark.parametrize("case", ["s3", "s4", "s6"])
def test_large_eval_hostsim(golden, backend, case):
    from scenario_util import check_large_eval, use_backend
    use_backend(backend)
    check_large_eval(golden, case)
