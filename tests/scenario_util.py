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




def compare_scenario_run(golden, name, backend, **bank_kw):
    """The persistent multi-step kernel (device geometry) on a golden scenario:
    per step the filtered mean and full covariance, mass_before_norm,
    clipped_mass and the three cross call counts; the final density and ranks."""
    from paper_2501_07942_b200 import _abi
    z = golden("trajectories")
    sc = SCENARIOS[name]
    bank = FilterBank(sc["spec"], bank_config(sc, **bank_kw), 1, backend=backend)
    done = int(z[f"{name}/done"])
    zs = z[f"{name}/z"][None, :, :]
    recs = bank.run(zs, done, sc["x0_mean"], sc["x0_cov"])[0]
    d = sc["spec"]["F"].shape[0]
    covs = _abi.rec_cov(recs, d)
    rows = []
    for k in range(done):
        r = recs[k]
        assert int(r["status"]) == 0 and int(r["k"]) == k, (k, r["status"], r["k"])
        ref_diag = z[f"{name}/{k}/diag"]
        rows.append({"step": k, "mean": rel(r["mean"][:d], z[f"{name}/{k}/filt_mean"]),
                     "cov": rel(covs[k], z[f"{name}/{k}/filt_cov"]),
                     "mass_before_norm": abs(float(r["mass_before_norm"]) - ref_diag[0]) / abs(ref_diag[0]),
                     "clipped_mass": abs(float(r["clipped_mass"]) - ref_diag[1]) / max(1.0, abs(ref_diag[1])),
                     "calls": (tuple(int(v) for v in r["calls"]),
                               tuple(int(v) for v in z[f"{name}/{k}/cross"][:, 1]))})
    got = bank.cores(0)
    ref = load_tt(z, f"{name}/{done - 1}/pred")
    rows.append({"step": "final", "dens": rel(T.to_full(got), T.to_full(ref)),
                 "ranks": (T.ranks_of(got), T.ranks_of(ref))})
    return rows


RUN_TOL = {"mean": 1e-8, "cov": 1e-7, "dens": 1e-7, "mass_before_norm": 1e-8, "clipped_mass": 1e-9}


def check_run(rows, calls=True):
    for r in rows:
        for key, tol in RUN_TOL.items():
            if key in r:
                assert r[key] <= tol, (r, key)
        if "ranks" in r:
            assert r["ranks"][0] == r["ranks"][1], r
        if calls and "calls" in r:   # counts follow pivot ties at roundoff level: 10 %
            for a, b in zip(*r["calls"]):
                assert abs(a - b) <= 0.1 * b, r


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


# ---------------------------------------------------------------------------
# BASELINE-config goldens (tests/golden/baseline.npz, make_golden.baseline):
# full tt_fft_pmf_step runs of the real reference on configs C1-C4.
# ---------------------------------------------------------------------------
def baseline_bank(cfg_name, count, backend, **kw):
    from paper_2501_07942_b200.configs import BASELINE_CONFIGS
    cfg = BASELINE_CONFIGS[cfg_name]
    g, x = cfg["grid"], cfg["cross"]
    base = dict(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                round_max_rank=g["round_max_rank"], tol=x["tol"], max_rank=x["max_rank"], rng_seed=x["rng_seed"],
                ws_bytes=1 << 30, state_doubles=1 << 20, cache_cap=1 << 21)
    base.update(kw)
    return cfg, FilterBank(cfg["spec"], BankConfig(**base), count, backend=backend)


def compare_baseline(golden, cfg_name, backend, persistent=False, runs=None, **bank_kw):
    """Run the golden runs of one BASELINE config as one filter bank, through
    the stage API (bank.step: measure launch, host geometry, time-update
    launch) or the persistent kernel (bank.run one step per launch, device
    geometry).  Returns one row per (run, step) the reference attempted."""
    from paper_2501_07942_b200 import _abi
    z = golden("baseline")
    nruns, steps = int(z[f"{cfg_name}/runs"]), int(z[f"{cfg_name}/steps"])
    runs = list(range(nruns)) if runs is None else list(runs)
    idx = z[f"{cfg_name}/idx"]
    cfg, bank = baseline_bank(cfg_name, len(runs), backend, **bank_kw)
    d = cfg["spec"]["F"].shape[0]
    Z = np.stack([z[f"{cfg_name}/{r}/z"] for r in runs])
    done = [int(z[f"{cfg_name}/{r}/done"]) for r in runs]
    rows = []
    if not persistent:
        dg = bank.init_prior(cfg["x0_mean"], cfg["x0_cov"])
        for j, r in enumerate(runs):
            key = f"{cfg_name}/{r}/init"
            assert int(dg["status"][j]) == 0, (r, dg["status"][j])
            got = bank.cores(j)
            rows.append({"run": r, "step": -1, "ranks": (T.ranks_of(got), tuple(z[f"{key}/ranks"])),
                         "dens": rel(T.at_indices(got, idx), z[f"{key}/sample"]),
                         "calls": (int(dg["cross"][j][0]["calls"]), int(z[f"{key}/cross"][1]))})
    alive = np.ones(len(runs), dtype=bool)
    for k in range(steps):
        if persistent:
            recs = bank.run(Z, 1, cfg["x0_mean"], cfg["x0_cov"])[:, 0]
            status = recs["status"]
            covs = _abi.rec_cov(recs, d)
        else:
            res = bank.step(Z[:, k])
            status = res["status"]
            dt = res["time"]
        for j, r in enumerate(runs):
            if not alive[j] or k > done[j]:
                continue
            sk = f"{cfg_name}/{r}/{k}"
            failed_ref = k == done[j]
            row = {"run": r, "step": k, "status": (int(status[j]), failed_ref)}
            if not failed_ref and int(status[j]) == 0:
                got = bank.cores(j)
                ref_diag = z[f"{sk}/diag"]
                ref_cross = z[f"{sk}/cross"]
                if persistent:
                    mean, cov = recs["mean"][j][:d], covs[j]
                    mb, cm = float(recs["mass_before_norm"][j]), float(recs["clipped_mass"][j])
                    calls = tuple(int(v) for v in recs["calls"][j])
                else:
                    mean, cov = res["mean"][j], res["cov"][j]
                    mb, cm = float(dt["mass_before_norm"][j]), float(dt["clipped_mass"][j])
                    calls = (int(res["measure"]["cross"][j][0]["calls"]),) + \
                        tuple(int(dt["cross"][j][q]["calls"]) for q in (1, 2))
                row.update({
                    "mean": rel(mean, z[f"{sk}/filt_mean"]), "cov": rel(cov, z[f"{sk}/filt_cov"]),
                    "dens": rel(T.at_indices(got, idx), z[f"{sk}/sample"]),
                    "ranks": (T.ranks_of(got), tuple(z[f"{sk}/ranks"])),
                    "axes": rel(np.stack(bank.grids[j].axes()), z[f"{sk}/axes"]),
                    "mass_before_norm": abs(mb - ref_diag[0]) / abs(ref_diag[0]),
                    "clipped_mass": abs(cm - ref_diag[1]) / max(1.0, abs(ref_diag[1])),
                    "calls": (calls, tuple(int(v) for v in ref_cross[:, 1])),
                })
            rows.append(row)
            if int(status[j]) != 0 or failed_ref:
                alive[j] = False
    return rows


BASELINE_TOL = {"mean": 1e-8, "cov": 1e-7, "dens": 1e-7, "axes": 1e-8, "mass_before_norm": 1e-8,
                "clipped_mass": 1e-9}


def check_baseline(rows):
    bad = []
    for r in rows:
        if "status" in r:
            st, failed_ref = r["status"]
            if (st != 0) != failed_ref:
                bad.append((r["run"], r["step"], "status", st, failed_ref))
                continue
        for key, tol in BASELINE_TOL.items():
            if key in r and not r[key] <= tol:
                bad.append((r["run"], r["step"], key, r[key]))
        for key in ("ranks", "calls"):
            if key in r and r[key][0] != r[key][1]:
                bad.append((r["run"], r["step"], key, r[key]))
    assert not bad, bad


def reference_band(golden, cfg_name):
    """Per (run, step): the reference's own disagreement with itself when its
    black-box values are perturbed by one ulp (p1, p2) or one ulp of the
    log-density (p3, p4), its cross's einsum dot products by one ulp (p5, p6)
    or the entries of its core-solve matrices by one ulp (p7, p8) --
    tests/golden/baseline_band.npz.  inf where a
    perturbed run's failure step differs.  Returns {(run, step): band dict}."""
    z, b = golden("baseline"), golden("baseline_band")
    runs, steps = int(z[f"{cfg_name}/runs"]), int(z[f"{cfg_name}/steps"])
    out = {}
    for r in range(runs):
        done = int(z[f"{cfg_name}/{r}/done"])
        unstable = False
        for k in range(min(steps, done + 1)):
            sk = f"{cfg_name}/{r}/{k}"
            band = {"mean": 0.0, "cov": 0.0, "dens": 0.0}
            for p in (1, 2, 3, 4, 5, 6, 7, 8):
                pd = int(b[f"p{p}/{cfg_name}/{r}/done"])
                if (k < done) != (k < pd) or unstable:
                    band = {key: np.inf for key in band}
                    break
                if k < done:
                    m, c, dd = b[f"p{p}/{sk}/rel"]
                    band["mean"], band["cov"], band["dens"] = (max(band["mean"], m), max(band["cov"], c),
                                                              max(band["dens"], dd))
            stable = band["dens"] <= 1e-9 and band["mean"] <= 1e-10 and band["cov"] <= 1e-9
            out[(r, k)] = dict(band, stable=stable)
            unstable = unstable or not stable
    return out


def check_baseline_band(rows, band, min_stable=1):
    """Rows where the reference is stable under its own perturbations must
    match it at the north-star tolerances (status, mean 1e-8, cov 1e-7,
    density 1e-7, ranks); elsewhere the reference itself is ulp-chaotic
    (SURVEY 8(c) tier 4) and only validity is required.  Returns a summary."""
    bad, n_stable, n_chaotic, n_match_chaotic = [], 0, 0, 0
    for r in rows:
        if r["step"] < 0:
            continue
        key = (r["run"], r["step"])
        if key not in band:
            continue
        st, failed_ref = r["status"]
        if band[key]["stable"]:
            n_stable += 1
            if (st != 0) != failed_ref:
                bad.append((key, "status", st, failed_ref))
                continue
            for k, tol in (("mean", 1e-8), ("cov", 1e-7), ("dens", 1e-7)):
                if k in r and not r[k] <= tol:
                    bad.append((key, k, r[k]))
            if "ranks" in r and r["ranks"][0] != r["ranks"][1]:
                bad.append((key, "ranks", r["ranks"]))
        else:
            n_chaotic += 1
            assert st in (0, 3), (key, st)
            if st == 0 and not failed_ref and all(r.get(k, 1.0) <= tol for k, tol in
                                                   (("mean", 1e-8), ("cov", 1e-7), ("dens", 1e-7))):
                n_match_chaotic += 1
    assert not bad, bad
    assert n_stable >= min_stable, (n_stable, n_chaotic)
    return {"stable": n_stable, "chaotic": n_chaotic, "chaotic_matched": n_match_chaotic}


def check_squeeze_ranks(recs, d, expect_drop):
    """The exact-rank squeeze of the cross outputs (filter.cuh tt_squeeze): a
    step record carries the kernel / likelihood ranks as the cross returned
    them (slots 4 / 1) and as the products used them (slots 9 / 8).  Squeezed
    ranks never exceed the cross's; with expect_drop (BASELINE C3: the
    correlated-Q kernel cross is rank deficient) some bond must shrink.
    Returns the number of bond directions removed."""
    dropped = 0
    for r in recs:
        if int(r["status"]) != 0:
            continue
        ranks = r["ranks"]
        for raw, sq in ((4, 9), (1, 8)):
            a, b = ranks[raw][: d + 1], ranks[sq][: d + 1]
            assert int(b[0]) == 1 and int(b[d]) == 1, (raw, b)
            assert all(int(y) <= int(x) for x, y in zip(a, b)), (raw, a, b)
            dropped += int(sum(int(x) - int(y) for x, y in zip(a, b)))
    if expect_drop:
        assert dropped > 0, "the squeeze removed no direction on a rank-deficient cross output"
    return dropped
