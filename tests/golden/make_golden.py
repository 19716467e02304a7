"""Generate golden vectors from the REAL reference package (build container only).

Run:  PYTHONPATH=/root/reference/pkg/src OMP_NUM_THREADS=1 python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Every array here comes out of ``ttpmf``
itself (the reference at /root/reference/pkg/src); the oracle and the CUDA
path are pinned against these files by the tests, which never read
/root/reference at run time.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = os.environ.get("TTPMF_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from ttpmf import tensor_train as rtt  # noqa: E402
from ttpmf import tt_algorithms as rta  # noqa: E402
from ttpmf import filters as rf  # noqa: E402
from ttpmf import models as rm  # noqa: E402
from ttpmf.grids import Grid, MomentEstimate  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_2501_07942_b200.configs import model_spec, reference_h  # noqa: E402


def rand_tt(rng, shape, ranks, decay=False):
    cores = []
    for k, n in enumerate(shape):
        c = rng.standard_normal((ranks[k], n, ranks[k + 1]))
        if decay:
            c *= np.exp(-0.7 * np.arange(ranks[k + 1]))[None, None, :]
        cores.append(c)
    return rtt.TensorTrain(tuple(cores))


def pack_tt(out, key, tt):
    out[f"{key}/d"] = np.array(len(tt.cores))
    for k, c in enumerate(tt.cores):
        out[f"{key}/{k}"] = np.asarray(c)


def ref_model(spec):
    return rm.StateSpaceModel(dim_x=spec["F"].shape[0], dim_z=spec["R"].shape[0],
                              h=reference_h(spec), Q=spec["Q"], R=spec["R"], F=spec["F"],
                              angle_components=tuple(spec.get("angle_components", ())))


def primitives():
    rng = np.random.default_rng(20250107)
    out = {}
    cases = [
        ("s3", (7, 9, 5), (1, 4, 6, 1)),
        ("s4", (33, 33, 33, 33), (1, 6, 9, 5, 1)),
        ("s6", (15, 13, 11, 9, 13, 15), (1, 5, 8, 12, 7, 4, 1)),
    ]
    for name, shape, ranks in cases:
        a = rand_tt(rng, shape, ranks, decay=True)
        b = rand_tt(rng, shape, tuple(max(1, r // 2) for r in ranks))
        pack_tt(out, f"{name}/a", a)
        pack_tt(out, f"{name}/b", b)
        h = rtt.tt_hadamard(a, b)
        pack_tt(out, f"{name}/had", h)
        for tag, tol, cap in [("t0", 0.0, None), ("t8", 1e-8, None), ("t3", 1e-3, None),
                              ("c3", 1e-8, 3), ("t2c5", 1e-2, 5)]:
            pack_tt(out, f"{name}/round_{tag}", rtt.tt_round(h, tol, cap))
        out[f"{name}/sum"] = np.array(rtt.tt_sum(a))
        out[f"{name}/dot"] = np.array(rtt.tt_dot(a, b))
        idx = np.stack([rng.integers(0, n, 500) for n in shape], axis=1)
        out[f"{name}/idx"] = idx
        out[f"{name}/eval"] = rtt.tt_eval_many(a, idx)
        if all(n % 2 == 1 for n in shape):
            pack_tt(out, f"{name}/conv", rta.tt_fft_convolve(b, a, 1e-8, None))
            pack_tt(out, f"{name}/conv_c4", rta.tt_fft_convolve(b, a, 1e-8, 4))
        old = Grid(tuple(np.linspace(-1.0 - k, 2.0 + k, n) for k, n in enumerate(shape)))
        new = Grid(tuple(np.linspace(-1.5 - k, 1.7 + k, n) for k, n in enumerate(shape)))
        out[f"{name}/old_axes"] = np.concatenate(old.axes)
        out[f"{name}/new_axes"] = np.concatenate(new.axes)
        pack_tt(out, f"{name}/interp", rta.tt_interpolate(a, old, new))
        pts = np.column_stack([rng.uniform(a_[0] - 0.2, a_[-1] + 0.2, 400) for a_ in old.axes])
        out[f"{name}/pts"] = pts
        out[f"{name}/at_points"] = rta.tt_eval_at_points(a, old.axes, pts)
    # rank-deficient Hadamard square (H3)
    a = rand_tt(rng, (9, 9, 9, 9), (1, 3, 4, 3, 1))
    sq = rtt.tt_hadamard(a, a)
    pack_tt(out, "sq/a", a)
    pack_tt(out, "sq/round", rtt.tt_round(sq, 1e-10, None))
    pack_tt(out, "zero/round", rtt.tt_round(rtt.TensorTrain(tuple(np.zeros((1 if k == 0 else 2, 5, 1 if k == 2 else 2)) for k in range(3))), 1e-8))
    np.savez_compressed(os.path.join(HERE, "primitives.npz"), **out)


def crosses():
    out = {}
    # separable-ish correlated Gaussian d=3 and a thin ridge likelihood d=2
    axes3 = [np.linspace(-3, 3, 17), np.linspace(-2, 4, 19), np.linspace(-4, 1, 15)]
    cov = np.array([[1.0, 0.4, 0.1], [0.4, 1.5, -0.3], [0.1, -0.3, 0.8]])
    g = rm.GaussianDensity(cov)
    mean = np.array([0.2, 0.9, -1.4])
    grid = Grid(tuple(axes3))

    def f3(idx):
        return g.pdf(grid.points_for(idx) - mean)

    for tag, cc in [("g3_tol6", rta.CrossConfig(tol=1e-6, max_rank=40, rng_seed=0)),
                    ("g3_tol2", rta.CrossConfig(tol=1e-2, max_rank=6, rng_seed=3)),
                    ("g3_seeded", rta.CrossConfig(tol=1e-8, max_rank=40, rng_seed=1,
                                                  seed_indices=rf._seed_lattice(grid.shape, 64)))]:
        res = rta.greedy_cross(rta.BlackBoxTensor(shape=grid.shape, evaluate_many=f3), cc)
        pack_tt(out, tag, res.tt)
        out[f"{tag}/info"] = np.array([res.achieved_error, res.evaluator_calls, res.sweeps,
                                       float(res.converged)])
    out["g3/axes"] = np.concatenate(axes3)
    out["g3/cov"] = cov
    out["g3/mean"] = mean
    np.savez_compressed(os.path.join(HERE, "crosses.npz"), **out)


def models():
    from paper_2501_07942_b200.configs import SPECS
    rng = np.random.default_rng(7)
    out = {}
    for name, spec in SPECS.items():
        m = ref_model(spec)
        d = spec["F"].shape[0]
        x = rng.normal(5.0, 3.0, size=(300, d))
        z = m.measure(x[:1])[0] + 0.1
        out[f"{name}/x"] = x
        out[f"{name}/z"] = z
        out[f"{name}/lik"] = m.likelihood(z, x)
        axes = [np.linspace(-2.0 - k, 3.0 + k, 9 if d > 4 else 11) for k in range(d)]
        grid = Grid(tuple(axes))
        idx = np.stack([rng.integers(0, a.size, 200) for a in axes], axis=1)
        out[f"{name}/kidx"] = idx
        out[f"{name}/kaxes"] = np.concatenate(axes)
        out[f"{name}/kern"] = rf._kernel_values(m, grid, idx)
    np.savez_compressed(os.path.join(HERE, "models.npz"), **out)


def trajectories():
    """Full Algorithm-3 runs where the reference's crosses converge (tier 3)."""
    from paper_2501_07942_b200.configs import SCENARIOS
    out = {}
    for name in ("scaling2_tight", "radar_deg", "identity2", "cv4_step0"):
        sc = SCENARIOS[name]
        spec = sc["spec"]
        m = ref_model(spec)
        traj = rm.simulate(m, sc["x0_mean"], sc["x0_cov"], sc["steps"],
                           seed=np.random.SeedSequence((2024, 0, 0)))
        gcfg = rf.GridConfig(**sc["grid"])
        ccfg = rta.CrossConfig(**sc["cross"])
        t0 = time.time()
        pmd = rf.initial_pmd_tt(MomentEstimate(sc["x0_mean"], sc["x0_cov"]), gcfg, ccfg)
        pack_tt(out, f"{name}/init", pmd.weights)
        out[f"{name}/init_axes"] = np.stack(pmd.grid.axes)
        out[f"{name}/z"] = traj.measurements
        out[f"{name}/x"] = traj.states
        done = 0
        for k in range(sc["steps"]):
            try:
                pmd = rf.tt_fft_pmf_step(pmd, m, traj.measurements[k], gcfg, ccfg)
            except rf.DegenerateDensityError:
                break
            dg = pmd.diag
            out[f"{name}/{k}/filt_mean"] = dg.filt_moments.mean
            out[f"{name}/{k}/filt_cov"] = dg.filt_moments.cov
            out[f"{name}/{k}/axes"] = np.stack(pmd.grid.axes)
            out[f"{name}/{k}/diag"] = np.array([dg.mass_before_norm, dg.clipped_mass,
                                                float(dg.outlier), float(dg.spd_fixed)])
            out[f"{name}/{k}/cross"] = np.array([list(dg.cross_info[c]) for c in
                                                 ("likelihood", "kernel", "realign")], dtype=float)
            pack_tt(out, f"{name}/{k}/pred", pmd.weights)
            done += 1
        out[f"{name}/done"] = np.array(done)
        print(name, "steps", done, "%.1fs" % (time.time() - t0), flush=True)
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **out)


def standard():
    """tt_pmf_step trajectories (Algorithm 2) where the
    transition cross converges: linear1d (the reference's own test config,
    test_filters.py:307-321) and scaling2 with cross tol 1e-10."""
    from paper_2501_07942_b200.configs import SPECS
    lin1 = {"F": np.array([[0.9]]), "Q": np.array([[1.0]]), "R": np.array([[1.0]]), "h": "linear",
            "H": np.array([[1.0]]), "angle_components": ()}
    cases = [("linear1d", lin1, np.zeros(1), 2.0 * np.eye(1), {"tol": 1e-8, "max_rank": 20, "rng_seed": 0}, 5),
             ("linear1d_exact", lin1, np.zeros(1), 2.0 * np.eye(1), {"tol": 1e-12, "max_rank": 40, "rng_seed": 0}, 5),
             ("scaling2", SPECS["scaling2"], np.array([20.0, 20.0]), np.diag([9.0, 9.0]),
              {"tol": 1e-10, "max_rank": 150, "rng_seed": 0}, 3)]
    out = {}
    for name, spec, mean, cov, cross, steps in cases:
        m = ref_model(spec)
        traj = rm.simulate(m, mean, cov, steps, seed=np.random.SeedSequence((2024, 0, 0)))
        gcfg = rf.GridConfig(n_per_axis=33, sigma_mult=4.0, round_tol=1e-8)
        ccfg = rta.CrossConfig(**cross)
        t0 = time.time()
        pmd = rf.initial_pmd_tt(MomentEstimate(mean, cov), gcfg, ccfg)
        pack_tt(out, f"{name}/init", pmd.weights)
        out[f"{name}/z"] = traj.measurements
        done = 0
        for k in range(steps):
            try:
                pmd = rf.tt_pmf_step(pmd, m, traj.measurements[k], gcfg, ccfg)
            except rf.DegenerateDensityError:
                break
            dg = pmd.diag
            out[f"{name}/{k}/filt_mean"] = dg.filt_moments.mean
            out[f"{name}/{k}/filt_cov"] = dg.filt_moments.cov
            out[f"{name}/{k}/axes"] = np.stack(pmd.grid.axes)
            out[f"{name}/{k}/diag"] = np.array([dg.mass_before_norm, dg.clipped_mass, float(dg.outlier),
                                                float(dg.spd_fixed)])
            out[f"{name}/{k}/cross"] = np.array([list(dg.cross_info[c]) for c in ("likelihood", "transition")],
                                                dtype=float)
            pack_tt(out, f"{name}/{k}/pred", pmd.weights)
            done += 1
        out[f"{name}/done"] = np.array(done)
        print(name, "steps", done, "%.1fs" % (time.time() - t0), flush=True)
    np.savez_compressed(os.path.join(HERE, "standard.npz"), **out)


def dense():
    """dense_fft_pmf_step trajectories: radar (d=2, full
    densities) and the BASELINE config-1 model (d=4, N=33; densities at 10^4
    seeded indices)."""
    from paper_2501_07942_b200.configs import SPECS
    out = {}
    cases = [("radar", SPECS["radar"], np.array([20.0, 20.0]), np.diag([9.0, 9.0]), 33, 4.0, 5),
             ("cv4", SPECS["cv4"], np.array([10.0, 10.0, 1.0, 1.0]), np.diag([1.0, 1.0, 0.1, 0.1]), 33, 6.0, 3)]
    for name, spec, mean, cov, n, sig, steps in cases:
        m = ref_model(spec)
        traj = rm.simulate(m, mean, cov, steps, seed=np.random.SeedSequence((2024, 0, 0)))
        gcfg = rf.GridConfig(n_per_axis=n, sigma_mult=sig, round_tol=1e-8)
        pmd = rf.initial_pmd_dense(MomentEstimate(mean, cov), gcfg)
        shape = pmd.weights.shape
        idx = np.stack([np.random.default_rng(7).integers(0, s, 10000) for s in shape], axis=1)
        out[f"{name}/idx"] = idx
        out[f"{name}/z"] = traj.measurements
        out[f"{name}/init_sample"] = pmd.weights[tuple(idx.T)]
        if len(shape) == 2:
            out[f"{name}/init"] = pmd.weights
        for k in range(steps):
            pmd = rf.dense_fft_pmf_step(pmd, m, traj.measurements[k], gcfg)
            dg = pmd.diag
            out[f"{name}/{k}/filt_mean"] = dg.filt_moments.mean
            out[f"{name}/{k}/filt_cov"] = dg.filt_moments.cov
            out[f"{name}/{k}/axes"] = np.stack(pmd.grid.axes)
            out[f"{name}/{k}/diag"] = np.array([dg.mass_before_norm, dg.clipped_mass, float(dg.outlier),
                                                float(dg.spd_fixed)])
            out[f"{name}/{k}/sample"] = pmd.weights[tuple(idx.T)]
            out[f"{name}/{k}/sum"] = np.array(float(pmd.weights.sum()))
            if len(shape) == 2:
                out[f"{name}/{k}/pred"] = pmd.weights
        out[f"{name}/steps"] = np.array(steps)
    np.savez_compressed(os.path.join(HERE, "dense.npz"), **out)


class _BigKeyEvaluator(rta._CachedEvaluator):
    """The reference's _CachedEvaluator (tt_algorithms.py:137-208) with its
    int64 ``ravel_multi_index`` key replaced by the exact C-order flat index
    as a Python int.  d=10, N=129 (BASELINE config 4) has 129**10 > 2**63
    cells, so the stock class raises in ``initial_pmd_tt``; this is the ONLY
    change (keys still sort ascending in C order, misses are still appended
    sorted-unique, ``sample_cache`` still draws positions with the same rng
    call), so every decision of ``greedy_cross`` is otherwise the reference's.
    Used for config 4 only."""

    def __init__(self, bb):
        super().__init__(bb)
        w = [1] * len(self._shape)
        for k in range(len(self._shape) - 2, -1, -1):
            w[k] = w[k + 1] * int(self._shape[k + 1])
        self._w = w
        self._keys: list[int] = []

    def _flat(self, idx):
        return [sum(int(i) * w for i, w in zip(row, self._w)) for row in idx.tolist()]

    def _unflat(self, keys):
        out = np.empty((len(keys), len(self._shape)), dtype=np.intp)
        for j, key in enumerate(keys):
            for k, w in enumerate(self._w):
                out[j, k], key = divmod(key, w)
        return out

    def __call__(self, idx):
        idx = np.asarray(idx, dtype=np.intp).reshape(-1, len(self._shape))
        keys = self._flat(idx)
        miss = sorted({k for k in keys if k not in self._pos})
        if miss:
            arr = self._unflat(miss)
            vals = np.asarray(self._bb.evaluate_many(arr), dtype=float).reshape(-1)
            if vals.shape != (len(miss),):
                raise ValueError("evaluator returned wrong number of values")
            if not np.all(np.isfinite(vals)):
                raise ValueError("evaluator returned a non-finite value")
            self.calls += len(miss)
            if len(vals):
                self.max_abs = max(self.max_abs, float(np.max(np.abs(vals))))
            need = self._count + len(miss)
            self._grow(need)
            self._val_buf[self._count: need] = vals
            self._pos.update(zip(miss, range(self._count, need)))
            self._keys.extend(miss)
            self._count = need
        return self._val_buf[np.array([self._pos[k] for k in keys], dtype=np.int64)]

    def sample_cache(self, rng, count):
        if self._count > count:
            sel = rng.choice(self._count, size=count, replace=False)
        else:
            sel = np.arange(self._count)
        return self._unflat([self._keys[j] for j in sel]), self._val_buf[sel].copy()


BASELINE_RUNS = {"C3": (8, 2), "C2": (8, 2), "C1": (8, 3), "C4": (8, 2)}
SAMPLE_SEED = 12345
SAMPLE_COUNT = 10_000


def sample_indices(shape):
    """The 10^4 seeded grid indices at which densities are compared (north star)."""
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.stack([rng.integers(0, n, SAMPLE_COUNT) for n in shape], axis=1)


def _perturbed_cross(seed, scaled=False):
    """greedy_cross whose black box returns v * (1 + s * 2**-52), s in {-1, 0, 1}
    a deterministic hash of the multi-index: the
    reference's own sensitivity to one-ulp evaluator differences.  scaled=True
    uses v * (1 + s * 2**-52 * max(1, |log v|)) instead: the values are
    exp(log-density), so a one-ulp difference in the log-density (what any
    independent evaluation of the same formula has) is a relative error of
    ulp(log v) ~ 2**-52 |log v| in v."""
    stock = rta.greedy_cross
    w = np.array([1000003, 10007, 101, 7919, 31, 13, 3, 17, 5, 29, 7, 11, 19, 23, 37, 41], dtype=np.int64)

    def wrapped(bb, cfg):
        inner = bb.evaluate_many

        def ev(idx):
            idx = np.asarray(idx, dtype=np.int64)
            v = np.asarray(inner(idx), dtype=float)
            s = ((idx @ w[: idx.shape[1]] + seed) % 3) - 1
            if scaled:
                with np.errstate(divide="ignore"):
                    amp = np.maximum(1.0, np.abs(np.log(np.abs(v))))
                amp[~np.isfinite(amp)] = 1.0
                return v * (1.0 + s * 2.0 ** -52 * amp)
            return v * (1.0 + s * 2.0 ** -52)

        return stock(rta.BlackBoxTensor(shape=bb.shape, evaluate_many=ev), cfg)
    return wrapped


class _NoisyNumpy:
    """numpy with every einsum result moved by one ulp in a direction hashed
    from its bits: stands in for a different summation order in the cross's
    interpolant dot products (tt_algorithms.py:380-382, tensor_train.py:129-158)."""

    def __init__(self, seed):
        self._seed = seed

    def __getattr__(self, name):
        return getattr(np, name)

    def einsum(self, *a, **k):
        out = np.einsum(*a, **k)
        if not isinstance(out, np.ndarray) or out.dtype != np.float64:
            return out
        bits = out.view(np.uint64)
        s = ((bits * np.uint64(0x9E3779B97F4A7C15) + np.uint64(self._seed)) >> np.uint64(61)) % np.uint64(3)
        s = s.astype(np.int64) - 1
        return np.where(s > 0, np.nextafter(out, np.inf), np.where(s < 0, np.nextafter(out, -np.inf), out))


class _NoisyScipy:
    """scipy with linalg.lstsq solving a copy of A whose entries are moved by
    one ulp in hashed directions: stands in for the roundoff differences of
    any other pivoted-QR implementation of the cross's core solve
    (tt_algorithms.py:305, gelsy)."""

    def __init__(self, seed):
        import scipy
        self._scipy = scipy
        self._seed = seed
        outer = self

        class _Linalg:
            def __getattr__(self, name):
                return getattr(scipy.linalg, name)

            def lstsq(self, a, b, *args, **kw):
                a = np.array(a, dtype=float, copy=True)
                bits = a.view(np.uint64)
                h = ((bits * np.uint64(0x9E3779B97F4A7C15) + np.uint64(outer._seed)) >> np.uint64(61)) % np.uint64(3)
                h = h.astype(np.int64) - 1
                a = np.where(h > 0, np.nextafter(a, np.inf), np.where(h < 0, np.nextafter(a, -np.inf), a))
                return scipy.linalg.lstsq(a, b, *args, **kw)
        self.linalg = _Linalg()

    def __getattr__(self, name):
        return getattr(self._scipy, name)


def baseline_band():
    """The same runs as baseline() with perturbed arithmetic: p1, p2 black-box
    values moved by one ulp (two hash seeds), p3, p4 by one ulp of the
    log-density, p5, p6 the cross's einsum results (interpolant dot products)
    by one ulp, p7, p8 the entries of the cross's core lstsq matrices by one
    ulp: tests/golden/baseline_band.npz.  |perturbed - baseline| per
    (run, step) is the reference's self-disagreement band (Appendix A.3)."""
    stock_f, stock_a = rf.greedy_cross, rta.greedy_cross
    parts = {}
    try:
        for seed, scaled in ((1, False), (2, False), (3, True), (4, True)):
            rf.greedy_cross = _perturbed_cross(seed, scaled)
            part = baseline(write=False)
            parts.update({f"p{seed}/{k}": v for k, v in part.items()})
        rf.greedy_cross = stock_f
        for seed in (5, 6):
            rta.np = _NoisyNumpy(seed)
            try:
                part = baseline(write=False)
            finally:
                rta.np = np
            parts.update({f"p{seed}/{k}": v for k, v in part.items()})
        stock_sp = rta.scipy
        for seed in (7, 8):
            rta.scipy = _NoisyScipy(seed)
            try:
                part = baseline(write=False)
            finally:
                rta.scipy = stock_sp
            parts.update({f"p{seed}/{k}": v for k, v in part.items()})
    finally:
        rf.greedy_cross, rta.greedy_cross = stock_f, stock_a
    np.savez_compressed(os.path.join(HERE, "baseline_band.npz"), **summarize_band(parts))


PERTURBATIONS = (1, 2, 3, 4, 5, 6, 7, 8)


def summarize_band(parts):
    """Compact band file: per config/run the perturbed runs' completed-step
    counts (p1..p4/done) and per (run, step) the max relative difference of
    the filtered mean, covariance and density sample from baseline.npz."""
    z = np.load(os.path.join(HERE, "baseline.npz"))

    def rel(a, b):
        return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))
    out = {}
    for name in BASELINE_RUNS:
        runs, steps = int(z[f"{name}/runs"]), int(z[f"{name}/steps"])
        for r in range(runs):
            for p in PERTURBATIONS:
                out[f"p{p}/{name}/{r}/done"] = parts[f"p{p}/{name}/{r}/done"]
                for k in range(steps):
                    sk, pk = f"{name}/{r}/{k}", f"p{p}/{name}/{r}/{k}"
                    if f"{sk}/sample" in z.files and f"{pk}/sample" in parts:
                        out[f"{pk}/rel"] = np.array([rel(parts[f"{pk}/filt_mean"], z[f"{sk}/filt_mean"]),
                                                     rel(parts[f"{pk}/filt_cov"], z[f"{sk}/filt_cov"]),
                                                     rel(parts[f"{pk}/sample"], z[f"{sk}/sample"])])
    return out


def baseline(write=True):
    """Full tt_fft_pmf_step goldens on the BASELINE configs with
    the metric cross (configs.METRIC_CROSS): per run (trajectory seed
    SeedSequence((2024, run, 0))), per step: filtered moments, grid axes,
    diagnostics, cross info, output ranks and the output density at 10^4
    seeded indices; the step at which DegenerateDensityError fired, if any.
    Config 4 runs with _BigKeyEvaluator (see its docstring)."""
    from paper_2501_07942_b200.configs import BASELINE_CONFIGS
    only = os.environ.get("BASELINE_ONLY")
    path = os.path.join(HERE, "baseline.npz")
    out = dict(np.load(path)) if (write and only and os.path.exists(path)) else {}
    stock = rta._CachedEvaluator
    for name, (runs, steps) in BASELINE_RUNS.items():
        if only and name not in only.split(","):
            continue
        for key in [k for k in out if k.startswith(name + "/")]:
            del out[key]
        cfg = BASELINE_CONFIGS[name]
        spec = cfg["spec"]
        m = ref_model(spec)
        gcfg = rf.GridConfig(**cfg["grid"])
        ccfg = rta.CrossConfig(**cfg["cross"])
        d = spec["F"].shape[0]
        idx = sample_indices((cfg["grid"]["n_per_axis"],) * d)
        out[f"{name}/idx"] = idx
        rta._CachedEvaluator = _BigKeyEvaluator if name == "C4" else stock
        try:
            for run in range(runs):
                traj = rm.simulate(m, cfg["x0_mean"], cfg["x0_cov"], cfg["steps"],
                                   seed=np.random.SeedSequence((2024, run, 0)))
                key = f"{name}/{run}"
                out[f"{key}/z"] = traj.measurements[:steps]
                t0 = time.time()
                try:
                    pmd = rf.initial_pmd_tt(MomentEstimate(cfg["x0_mean"], cfg["x0_cov"]), gcfg, ccfg)
                except rf.DegenerateDensityError:
                    out[f"{key}/done"] = np.array(-1)
                    continue
                out[f"{key}/init/ranks"] = np.array(pmd.weights.ranks)
                out[f"{key}/init/sample"] = rtt.tt_eval_many(pmd.weights, idx)
                out[f"{key}/init/cross"] = np.array(list(pmd.diag.cross_info["initial_pmd"]), dtype=float)
                done = 0
                times = []
                for k in range(steps):
                    ts = time.time()
                    try:
                        pmd = rf.tt_fft_pmf_step(pmd, m, traj.measurements[k], gcfg, ccfg)
                    except rf.DegenerateDensityError:
                        break
                    times.append(time.time() - ts)
                    dg = pmd.diag
                    sk = f"{key}/{k}"
                    out[f"{sk}/filt_mean"] = dg.filt_moments.mean
                    out[f"{sk}/filt_cov"] = dg.filt_moments.cov
                    out[f"{sk}/axes"] = np.stack(pmd.grid.axes)
                    out[f"{sk}/diag"] = np.array([dg.mass_before_norm, dg.clipped_mass, float(dg.outlier),
                                                  float(dg.spd_fixed)])
                    out[f"{sk}/cross"] = np.array([list(dg.cross_info[c]) for c in
                                                   ("likelihood", "kernel", "realign")], dtype=float)
                    out[f"{sk}/ranks"] = np.array(pmd.weights.ranks)
                    out[f"{sk}/sample"] = rtt.tt_eval_many(pmd.weights, idx)
                    out[f"{sk}/sum"] = np.array(float(rtt.tt_sum(pmd.weights)))
                    done += 1
                out[f"{key}/done"] = np.array(done)
                out[f"{key}/seconds"] = np.array(times)
                print(name, run, "steps", done, "fail" if done < steps else "",
                      " ".join("%.1fs" % t for t in times), "total %.1fs" % (time.time() - t0), flush=True)
        finally:
            rta._CachedEvaluator = stock
        out[f"{name}/runs"] = np.array(runs)
        out[f"{name}/steps"] = np.array(steps)
    if write:
        np.savez_compressed(path, **out)
    return out


if __name__ == "__main__":
    which = sys.argv[1:] or ["primitives", "crosses", "models", "trajectories", "dense", "standard"]
    for w in which:
        t = time.time()
        globals()[w]()
        print(w, "done %.1fs" % (time.time() - t), flush=True)
