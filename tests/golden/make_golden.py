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


if __name__ == "__main__":
    which = sys.argv[1:] or ["primitives", "crosses", "models", "trajectories", "dense", "standard"]
    for w in which:
        t = time.time()
        globals()[w]()
        print(w, "done %.1fs" % (time.time() - t), flush=True)
