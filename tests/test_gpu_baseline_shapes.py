"""GPU primitive parity at the BASELINE configs' full shapes (SURVEY 8(c) tier 1
at S4b / S6 / S10): C2 (d=4, N=129, cap 20), C3/C5 (d=6, N=65, cap 20) and C4
(d=10, N=129, cap 32) -- the last has no reference trajectory (the reference
overflows int64 in ravel_multi_index), so its pin is the oracle's
restated primitives on seeded TTs of that shape.

Compared through the C-ABI against oracle/ttcore.py: Hadamard (exact),
rounding of the Hadamard product with the config's tol / cap (equal ranks,
values at 10^4 seeded indices 1e-10 relative to the largest), FFT convolution
+ rounding, interpolation onto a shifted grid, raw moments (1e-10).
"""

import numpy as np
import pytest

from oracle import pmf
from oracle import ttcore as T

pytestmark = pytest.mark.gpu

SHAPES = {   # name: (d, n, cap, ranks of a (kernel-like), ranks of b (density-like))
    "C2": (4, 129, 20, 6, 12),
    "C3": (6, 65, 20, 5, 10),
    "C4": (10, 129, 32, 4, 8),
}


@pytest.fixture(scope="module")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2501_07942_b200.backend import CudaBackend
    from scenario_util import use_backend
    be = CudaBackend()
    use_backend(be)
    return be


def gauss_like_tt(rng, d, n, r, width):
    """Positive, smooth, decaying cores (density-like spectra)."""
    x = np.linspace(-1.0, 1.0, n)
    cores = []
    for k in range(d):
        rl = 1 if k == 0 else r
        rr = 1 if k == d - 1 else r
        c = np.empty((rl, n, rr))
        for a in range(rl):
            for b in range(rr):
                mu = rng.uniform(-0.3, 0.3)
                c[a, :, b] = np.exp(-((x - mu) / width) ** 2) * 0.7 ** (a + b) + 1e-3 * rng.standard_normal(n)
        cores.append(c)
    return cores


def sample_rel(got, ref, n=10_000, seed=3):
    shape = T.mode_sizes(ref)
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, s, n) for s in shape], axis=1)
    a, b = T.at_indices(got, idx), T.at_indices(ref, idx)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_primitives_at_baseline_shape(cuda, name):
    from paper_2501_07942_b200 import tensor_train as G
    from paper_2501_07942_b200 import geometry as geo
    from paper_2501_07942_b200.grids import Grid
    d, n, cap, ra, rb = SHAPES[name]
    rng = np.random.default_rng(2024 + d)
    a = gauss_like_tt(rng, d, n, ra, 0.2)
    b = gauss_like_tt(rng, d, n, rb, 0.5)
    ga, gb = G.TensorTrain.from_cores(a), G.TensorTrain.from_cores(b)
    had = G.tt_hadamard(ga, gb)
    ref_had = T.kron_cores(a, b)
    for x, y in zip(had.numpy_cores(), ref_had):
        assert np.array_equal(x, y)
    got = G.tt_round(had, 1e-8, cap)
    ref = T.round_tt(ref_had, 1e-8, cap)
    assert got.ranks == T.ranks_of(ref)
    assert sample_rel(got.numpy_cores(), ref) <= 1e-10
    conv = G.tt_fft_convolve(ga, gb, 1e-8, cap)
    ref_conv = T.fft_conv(a, b, 1e-8, cap)
    assert conv.ranks == T.ranks_of(ref_conv)
    assert sample_rel(conv.numpy_cores(), ref_conv) <= 1e-10
    # interpolation onto a shifted, slightly wider grid
    old = geo.grid_from_bounds([-1.0] * d, [1.0] * d, [n] * d)
    new = geo.grid_from_bounds([-1.1 + 0.03 * k for k in range(d)], [0.9 + 0.02 * k for k in range(d)], [n] * d)
    gi = G.tt_interpolate(gb, Grid(old), Grid(new))
    ref_i = T.regrid(b, old.axes(), new.axes())
    assert sample_rel(gi.numpy_cores(), ref_i) <= 1e-12
    # raw moments (mass, first, second) on the old grid
    raw = G.tt_raw_moments(gb, old)
    mass, mean, m2 = pmf.raw_moments(old.axes(), b)
    dv = old.cell_volume()
    assert abs(raw[0] * dv - mass) <= 1e-11 * abs(mass)
    assert np.max(np.abs(raw[1:1 + d] * dv / mass - mean)) <= 1e-10 * max(1.0, np.max(np.abs(mean)))
