"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures come from ``tests/golden/make_golden.py`` (run where
/root/reference exists).  Agreement here is what lets the GPU tests use the
oracle as the checker on the GPU box.
"""

import numpy as np
import pytest

from conftest import load_tt
from oracle import ttcore as T
from oracle import pmf
from oracle.cross import greedy_cross
from paper_2501_07942_b200.configs import SPECS

CASES = ["s3", "s4", "s6"]


def dense(c):
    return T.to_full(c)


def close(a, b, rtol=1e-13):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(np.max(np.abs(b)), 1e-300)
    assert np.max(np.abs(a - b)) <= rtol * scale, np.max(np.abs(a - b)) / scale


@pytest.mark.parametrize("case", CASES)
def test_primitives_pinned(golden, case):
    z = golden("primitives")
    a, b = load_tt(z, f"{case}/a"), load_tt(z, f"{case}/b")
    had = T.kron_cores(a, b)
    for x, y in zip(had, load_tt(z, f"{case}/had")):
        assert np.array_equal(x, y)
    for tag, tol, cap in [("t0", 0.0, None), ("t8", 1e-8, None), ("t3", 1e-3, None),
                          ("c3", 1e-8, 3), ("t2c5", 1e-2, 5)]:
        got = T.round_tt(had, tol, cap)
        ref = load_tt(z, f"{case}/round_{tag}")
        assert T.ranks_of(got) == T.ranks_of(ref)
        close(dense(got), dense(ref), 1e-12)
    assert T.total(a) == float(z[f"{case}/sum"])
    assert T.inner(a, b) == float(z[f"{case}/dot"])
    assert np.array_equal(T.at_indices(a, z[f"{case}/idx"]), z[f"{case}/eval"])
    shape = T.mode_sizes(a)
    if f"{case}/conv/d" in z.files:
        got = T.fft_conv(b, a, 1e-8, None)
        close(dense(got), dense(load_tt(z, f"{case}/conv")))
        got4 = T.fft_conv(b, a, 1e-8, 4)
        assert T.ranks_of(got4) == T.ranks_of(load_tt(z, f"{case}/conv_c4"))
    cuts = np.cumsum(shape)[:-1]
    old = np.split(z[f"{case}/old_axes"], cuts)
    new = np.split(z[f"{case}/new_axes"], cuts)
    for x, y in zip(T.regrid(a, old, new), load_tt(z, f"{case}/interp")):
        assert np.array_equal(x, y)
    assert np.array_equal(T.at_points(a, old, z[f"{case}/pts"]), z[f"{case}/at_points"])


def test_round_rank_deficient_and_zero(golden):
    z = golden("primitives")
    a = load_tt(z, "sq/a")
    got = T.round_tt(T.kron_cores(a, a), 1e-10)
    ref = load_tt(z, "sq/round")
    assert T.ranks_of(got) == T.ranks_of(ref)
    close(dense(got), dense(ref))
    assert T.ranks_of(load_tt(z, "zero/round")) == (1, 1, 1, 1)


@pytest.mark.parametrize("tag,kw", [
    ("g3_tol6", dict(tol=1e-6, max_rank=40, rng_seed=0)),
    ("g3_tol2", dict(tol=1e-2, max_rank=6, rng_seed=3)),
    ("g3_seeded", dict(tol=1e-8, max_rank=40, rng_seed=1, seeds=True)),
])
def test_cross_pinned(golden, tag, kw):
    z = golden("crosses")
    axes = np.split(z["g3/axes"], [17, 36])
    g = pmf.Gauss(z["g3/cov"])
    mean = z["g3/mean"]
    seeds = pmf.seed_lattice((17, 19, 15), 64) if kw.pop("seeds", False) else None
    res = greedy_cross((17, 19, 15), lambda idx: g.pdf(pmf.points_for(axes, idx) - mean),
                       seed_indices=seeds, **kw)
    ref = load_tt(z, tag)
    info = z[f"{tag}/info"]
    assert T.ranks_of(res.cores) == T.ranks_of(ref)
    for x, y in zip(res.cores, ref):
        assert np.array_equal(x, y)
    assert (res.achieved_error, res.evaluator_calls, res.sweeps, float(res.converged)) == tuple(info)


@pytest.mark.parametrize("name", sorted(SPECS))
def test_models_pinned(golden, name):
    z = golden("models")
    spec = SPECS[name]
    got = pmf.likelihood(spec, z[f"{name}/z"], z[f"{name}/x"])
    close(got, z[f"{name}/lik"], 1e-15)
    d = spec["F"].shape[0]
    n = 9 if d > 4 else 11
    axes = np.split(z[f"{name}/kaxes"], np.arange(1, d) * n)
    close(pmf.kernel_values(spec, axes, z[f"{name}/kidx"]), z[f"{name}/kern"], 1e-15)
