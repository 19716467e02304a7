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


def test_squeeze_ranks_hostsim(golden, backend):
    """Rank log of the exact-rank squeeze on a golden scenario (full-rank cross
    outputs there: nothing may grow; the drop itself is asserted on C3, GPU)."""
    from scenario_util import SCENARIOS, FilterBank, bank_config, check_squeeze_ranks
    name = "radar_deg"
    z = golden("trajectories")
    sc = SCENARIOS[name]
    bank = FilterBank(sc["spec"], bank_config(sc), 1, backend=backend)
    done = int(z[f"{name}/done"])
    recs = bank.run(z[f"{name}/z"][None, :, :], done, sc["x0_mean"], sc["x0_cov"])[0]
    check_squeeze_ranks(recs[:done], sc["spec"]["F"].shape[0], expect_drop=False)
