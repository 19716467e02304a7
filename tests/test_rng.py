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
