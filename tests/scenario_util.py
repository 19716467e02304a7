"""Shared helpers: run a golden scenario through the FilterBank on a backend."""

import numpy as np

from conftest import load_tt
from oracle import ttcore as T
from paper_2501_07942_b200.bank import BankConfig, FilterBank
from paper_2501_07942_b200.configs import SCENARIOS


def bank_config(sc, **kw):
    g, x = sc["grid"], sc["cross"]
    base = dict(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                round_max_rank=g.get("round_max_rank"), tol=x["tol"], max_rank=x["max_rank"],
                rng_seed=x["rng_seed"], ws_bytes=512 << 20, state_doubles=1 << 18, cache_cap=1 << 18)
    base.update(kw)
    return BankConfig(**base)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def compare_scenario(golden, name, backend):
    """Run the golden scenario; return a list of per-step error dicts."""
    z = golden("trajectories")
    sc = SCENARIOS[name]
    bank = FilterBank(sc["spec"], bank_config(sc), 1, backend=backend)
    dg = bank.init_prior(sc["x0_mean"], sc["x0_cov"])
    assert int(dg["status"][0]) == 0
    ref0 = load_tt(z, f"{name}/init")
    got0 = bank.cores(0)
    out = [{"step": -1, "dens": rel(T.to_full(got0), T.to_full(ref0)),
            "ranks": (T.ranks_of(got0), T.ranks_of(ref0))}]
    zs = z[f"{name}/z"]
    for k in range(int(z[f"{name}/done"])):
        res = bank.step(zs[k][None])
        assert int(res["status"][0]) == 0, res["status"]
        got = bank.cores(0)
        ref = load_tt(z, f"{name}/{k}/pred")
        out.append({"step": k, "mean": rel(res["mean"][0], z[f"{name}/{k}/filt_mean"]),
                    "cov": rel(res["cov"][0], z[f"{name}/{k}/filt_cov"]),
                    "dens": rel(T.to_full(got), T.to_full(ref)),
                    "ranks": (T.ranks_of(got), T.ranks_of(ref)),
                    "axes": rel(np.stack(bank.grids[0].axes()), z[f"{name}/{k}/axes"])})
    return out


TOL = {"mean": 1e-8, "cov": 1e-7, "dens": 1e-7, "axes": 1e-8}


def check(rows):
    for r in rows:
        for key, tol in TOL.items():
            if key in r:
                assert r[key] <= tol, (r, key)
        assert r["ranks"][0] == r["ranks"][1], r


def use_backend(be):
    from paper_2501_07942_b200 import tensor_train as G
    if G._CTX.get("be") is not be:
        G._CTX.clear()
        G._CTX["be"] = be


def check_primitives(golden, case):
    from paper_2501_07942_b200 import tensor_train as G
    from paper_2501_07942_b200.grids import Grid
    from paper_2501_07942_b200 import geometry as geo
    z = golden("primitives")
    a = G.TensorTrain.from_cores(load_tt(z, f"{case}/a"))
    b = G.TensorTrain.from_cores(load_tt(z, f"{case}/b"))
    had = G.tt_hadamard(a, b)
    for x, y in zip(had.numpy_cores(), load_tt(z, f"{case}/had")):
        assert np.array_equal(x, y)
    for tag, tol, cap in [("t0", 0.0, None), ("t8", 1e-8, None), ("t3", 1e-3, None), ("c3", 1e-8, 3),
                          ("t2c5", 1e-2, 5)]:
        got = G.tt_round(had, tol, cap)
        ref = load_tt(z, f"{case}/round_{tag}")
        assert got.ranks == T.ranks_of(ref), (tag, got.ranks, T.ranks_of(ref))
        assert rel(T.to_full(got.numpy_cores()), T.to_full(ref)) <= 1e-12, tag
    assert abs(G.tt_sum(a) - float(z[f"{case}/sum"])) <= 1e-12 * abs(float(z[f"{case}/sum"]))
    assert rel(G.tt_eval_many(a, z[f"{case}/idx"]), z[f"{case}/eval"]) <= 1e-13
    if f"{case}/conv/d" in z.files:
        got = G.tt_fft_convolve(b, a, 1e-8, None)
        ref = load_tt(z, f"{case}/conv")
        assert got.ranks == T.ranks_of(ref)
        assert rel(T.to_full(got.numpy_cores()), T.to_full(ref)) <= 1e-12
        assert G.tt_fft_convolve(b, a, 1e-8, 4).ranks == T.ranks_of(load_tt(z, f"{case}/conv_c4"))
    shape = a.shape
    cuts = np.cumsum(shape)[:-1]
    old = np.split(z[f"{case}/old_axes"], cuts)
    new = np.split(z[f"{case}/new_axes"], cuts)
    og = Grid(geo.grid_from_bounds([o[0] for o in old], [o[-1] for o in old], list(shape)))
    ng = Grid(geo.grid_from_bounds([o[0] for o in new], [o[-1] for o in new], list(shape)))
    for k in range(len(shape)):   # linspace vs from_bounds agree to rounding only
        assert rel(og.axes[k], old[k]) <= 1e-14 and rel(ng.axes[k], new[k]) <= 1e-14
    ref_i = T.regrid(load_tt(z, f"{case}/a"), og.axes, ng.axes)
    got_i = G.tt_interpolate(a, og, ng)
    assert rel(T.to_full(got_i.numpy_cores()), T.to_full(ref_i)) <= 1e-13
    pts = z[f"{case}/pts"]
    assert rel(G.tt_eval_at_points(a, og, pts), T.at_points(load_tt(z, f"{case}/a"), og.axes, pts)) <= 1e-13




def compare_scenario_run(golden, name, backend):
    """The persistent multi-step kernel (device geometry) on a golden scenario."""
    z = golden("trajectories")
    sc = SCENARIOS[name]
    bank = FilterBank(sc["spec"], bank_config(sc), 1, backend=backend)
    done = int(z[f"{name}/done"])
    zs = z[f"{name}/z"][None, :, :]
    recs = bank.run(zs, done, sc["x0_mean"], sc["x0_cov"])[0]
    rows = []
    for k in range(done):
        r = recs[k]
        assert int(r["status"]) == 0 and int(r["k"]) == k, (k, r["status"], r["k"])
        d = sc["spec"]["F"].shape[0]
        rows.append({"step": k, "mean": rel(r["mean"][:d], z[f"{name}/{k}/filt_mean"]),
                     "cov": rel(r["cov_diag"][:d], np.diag(z[f"{name}/{k}/filt_cov"]))})
    got = bank.cores(0)
    ref = load_tt(z, f"{name}/{done - 1}/pred")
    rows.append({"step": "final", "dens": rel(T.to_full(got), T.to_full(ref)),
                 "ranks": (T.ranks_of(got), T.ranks_of(ref))})
    return rows


def check_large_eval(golden, case):
    """tt_eval_many / tt_eval_at_points on batches large enough for the
    bucketed (SMEM-staged / DMMA) evaluation path."""
    from paper_2501_07942_b200 import tensor_train as G
    from paper_2501_07942_b200.grids import Grid
    from paper_2501_07942_b200 import geometry as geo
    z = golden("primitives")
    cores = load_tt(z, f"{case}/a")
    a = G.TensorTrain.from_cores(cores)
    shape = a.shape
    rng = np.random.default_rng(5)
    idx = np.stack([rng.integers(0, n, 5000) for n in shape], axis=1)
    assert rel(G.tt_eval_many(a, idx), T.at_indices(cores, idx)) <= 1e-13
    cuts = np.cumsum(shape)[:-1]
    old = np.split(z[f"{case}/old_axes"], cuts)
    og = Grid(geo.grid_from_bounds([o[0] for o in old], [o[-1] for o in old], list(shape)))
    pts = np.column_stack([rng.uniform(ax[0] - 0.2, ax[-1] + 0.2, 5000) for ax in og.axes])
    assert rel(G.tt_eval_at_points(a, og, pts), T.at_points(cores, og.axes, pts)) <= 1e-13
