"""The device's numpy-compatible draws (warp-parallel PCG64 + Lemire + Floyd /
tail-shuffle choice), compiled for the host emulation, against numpy itself."""

import ctypes

import numpy as np
import pytest

from hostsim import build
from paper_2501_07942_b200.geometry import pcg64_state


@pytest.fixture(scope="module")
def lib():
    lib = ctypes.CDLL(build())
    lib.ttgbf_test_draws.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    return lib


def state_of(rng):
    st = rng.bit_generator.state
    m = (1 << 64) - 1
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s & m, s >> 64, inc & m, inc >> 64, st["has_uint32"], st["uinteger"]], dtype=np.uint64)


def run(lib, kind, rng, shape=(1,), K=0, pop=0, size=0):
    st = state_of(rng)
    sh = np.asarray(shape, dtype=np.int32)
    n = K * len(shape) if kind == 0 else size
    out = np.zeros(max(n, 1), dtype=np.int64)
    rc = lib.ttgbf_test_draws(kind, st.ctypes.data, sh.ctypes.data, len(shape), K, pop, size, out.ctypes.data)
    assert rc == 0
    return out[:n], st


@pytest.mark.parametrize("seed", range(6))
def test_integers_match_numpy(lib, seed):
    rng = np.random.default_rng(seed)
    for trial in range(8):
        shape = tuple(int(v) for v in np.random.RandomState(trial + 10 * seed).randint(1, 200, size=1 + trial % 7))
        K = 1 + 37 * trial
        got, st = run(lib, 0, rng, shape=shape, K=K)
        ref = rng.integers(0, shape, size=(K, len(shape)))
        assert np.array_equal(got.reshape(K, -1), ref)
        assert np.array_equal(st, state_of(rng))


@pytest.mark.parametrize("pop,size", [(5, 3), (33, 10), (1000, 10), (5000, 1024), (9999, 4096), (10001, 1024),
                                      (20000, 4096), (300000, 4096), (150000, 32768), (12000, 32768 // 4),
                                      (1030, 1024), (2049, 2048), (4097, 4096), (2000000, 32768)])
def test_choice_matches_numpy(lib, pop, size):
    for seed in range(3):
        rng = np.random.default_rng(seed)
        rng.integers(0, 7)            # leave a buffered half-word in the stream
        got, st = run(lib, 1, rng, pop=pop, size=size)
        ref = rng.choice(pop, size=size, replace=False)
        assert np.array_equal(got, ref)
        assert np.array_equal(st, state_of(rng))


# -- the same streams through the C-ABI entry ttgbf_rng_draws: host emulation
# (CPU suite) and the sm_100a kernel itself (-m gpu), where the draws are
# warp-parallel, the tail-shuffle steps are resolved by all threads and only
# the interacting ones replayed in order
CHOICES = [(33, 10), (2600, 1024), (5000, 1024), (9999, 4096), (10001, 1024), (20000, 4096), (60000, 4096),
           (300000, 4096), (150000, 32768), (12000, 8192), (1030, 1024), (4097, 4096), (1000000, 32768), (900, 700)]


def check_abi_draws():
    from paper_2501_07942_b200 import evaluators as ev
    for seed in range(2):
        rng = np.random.default_rng(seed)
        rng.integers(0, 7)
        for shape, K in [((65,) * 6, 56), ((33, 129, 7), 300)]:
            got, st = ev.rng_draws(state_of(rng), shape=shape, K=K)
            ref = rng.integers(0, shape, size=(K, len(shape)))
            assert np.array_equal(got.reshape(K, -1), ref), (shape, K)
            assert np.array_equal(st, state_of(rng))
        for pop, size in CHOICES:
            got, st = ev.rng_draws(state_of(rng), pop=pop, size=size)
            ref = rng.choice(pop, size=size, replace=False)
            assert np.array_equal(got, ref), (pop, size, int((got != ref).sum()))
            assert np.array_equal(st, state_of(rng)), (pop, size)


def test_abi_draws_hostsim():
    from hostsim import HostBackend
    from scenario_util import use_backend
    use_backend(HostBackend())
    check_abi_draws()


@pytest.mark.gpu
def test_abi_draws_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    from scenario_util import use_backend
    use_backend(CudaBackend())
    check_abi_draws()
