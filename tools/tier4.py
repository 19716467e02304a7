"""Tier-4 report: on the BASELINE configs, the distribution of
the step at which DegenerateDensityError ends a run and the step-0 filtered
means, for the oracle (reference algorithm, host processes) and for the
engine (GPU, persistent kernel), on the same 256 seeded trajectories.

  python tools/tier4.py oracle --out profiles/r02_tier4_oracle.json      # CPU, this container or the box
  python tools/tier4.py gpu --out gpurun_out/r02_tier4_gpu.json          # GPU box
  python tools/tier4.py compare profiles/r02_tier4_oracle.json gpurun_out/r02_tier4_gpu.json
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_07942_b200.configs import BASELINE_CONFIGS, simulate  # noqa: E402

STEPS = {"C1": 3, "C2": 2, "C3": 2}
RUNS_OF = {"C1": 256, "C2": 256, "C3": 64}   # C3 oracle steps take 2-60 s each


def _oracle_run(arg):
    name, run = arg
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import pmf
    cfg = BASELINE_CONFIGS[name]
    g = cfg["grid"]
    occ = {"n_per_axis": g["n_per_axis"], "sigma_mult": g["sigma_mult"], "round_tol": g["round_tol"],
           "round_max_rank": g["round_max_rank"]}
    _, z = simulate(cfg["spec"], cfg["x0_mean"], cfg["x0_cov"], STEPS[name], np.random.SeedSequence((2024, run, 0)))
    axes, cores, _ = pmf.initial(cfg["x0_mean"], cfg["x0_cov"], occ, cfg["cross"])
    mean0 = None
    for k in range(STEPS[name]):
        try:
            axes, cores, dg = pmf.step(axes, cores, cfg["spec"], z[k], occ, cfg["cross"])
        except pmf.Degenerate:
            return run, k, mean0
        if k == 0:
            mean0 = dg["filt_mean"].tolist()
    return run, STEPS[name], mean0


def oracle(out, names=None):
    import multiprocessing as mp
    res = json.load(open(out)) if os.path.exists(out) else {}
    with mp.get_context("spawn").Pool(max(1, len(os.sched_getaffinity(0)) - 1)) as pool:
        for name in (names or STEPS):
            t0 = time.time()
            rows = pool.map(_oracle_run, [(name, r) for r in range(RUNS_OF[name])], chunksize=1)
            res[name] = {"fail_step": [int(r[1]) for r in sorted(rows)], "mean0": [r[2] for r in sorted(rows)]}
            print(name, "%.0fs" % (time.time() - t0), flush=True)
            json.dump(res, open(out, "w"))


def gpu(out):
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    res = {}
    for name in STEPS:
        RUNS = RUNS_OF[name]
        cfg = BASELINE_CONFIGS[name]
        g, x = cfg["grid"], cfg["cross"]
        bc = BankConfig(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                        round_max_rank=g["round_max_rank"], tol=x["tol"], max_rank=x["max_rank"],
                        rng_seed=x["rng_seed"], ws_bytes=320 << 20, state_doubles=1 << 18, cache_cap=1 << 20,
                        ws_slots=148, big_slots=32, big_bytes=1 << 30, big2_slots=8, big2_bytes=3 << 29)
        Z = np.stack([simulate(cfg["spec"], cfg["x0_mean"], cfg["x0_cov"], STEPS[name],
                               np.random.SeedSequence((2024, r, 0)))[1] for r in range(RUNS)])
        bank = FilterBank(cfg["spec"], bc, RUNS)
        fail = np.full(RUNS, STEPS[name])
        alive = np.ones(RUNS, bool)
        mean0 = [None] * RUNS
        t0 = time.time()
        for k in range(STEPS[name]):
            recs = bank.run(Z, 1, cfg["x0_mean"], cfg["x0_cov"])[:, 0]
            for i in range(RUNS):
                if not alive[i]:
                    continue
                if int(recs["status"][i]) != 0:
                    fail[i] = k
                    alive[i] = False
                elif k == 0:
                    mean0[i] = recs["mean"][i][: cfg["spec"]["F"].shape[0]].tolist()
        res[name] = {"fail_step": fail.tolist(), "mean0": mean0}
        print(name, "%.0fs" % (time.time() - t0), flush=True)
        del bank
        import torch
        torch.cuda.empty_cache()
    json.dump(res, open(out, "w"))


def compare(a_path, b_path):
    a, b = json.load(open(a_path)), json.load(open(b_path))
    rep = {}
    for name in STEPS:
        if name not in a or name not in b:
            continue
        RUNS = min(len(a[name]["fail_step"]), len(b[name]["fail_step"]))
        fa, fb = np.array(a[name]["fail_step"][:RUNS]), np.array(b[name]["fail_step"][:RUNS])
        hist = {int(s): [int((fa == s).sum()), int((fb == s).sum())] for s in range(STEPS[name] + 1)}
        both = [i for i in range(RUNS) if a[name]["mean0"][i] is not None and b[name]["mean0"][i] is not None]
        rels = [float(np.max(np.abs(np.array(a[name]["mean0"][i]) - np.array(b[name]["mean0"][i])))
                      / np.max(np.abs(a[name]["mean0"][i]))) for i in both]
        rep[name] = {"runs": RUNS, "fail_step_hist_oracle_gpu": hist, "same_fail_step": float(np.mean(fa == fb)),
                     "step0_both_completed": len(both),
                     "step0_mean_rel_le_1e-8": float(np.mean(np.array(rels) <= 1e-8)) if rels else None,
                     "step0_mean_rel_median": float(np.median(rels)) if rels else None}
    print(json.dumps(rep, indent=1))
    return rep


if __name__ == "__main__":
    if sys.argv[1] == "oracle":
        names = sys.argv[sys.argv.index("--configs") + 1].split(",") if "--configs" in sys.argv else None
        oracle(sys.argv[sys.argv.index("--out") + 1], names)
    elif sys.argv[1] == "gpu":
        gpu(sys.argv[sys.argv.index("--out") + 1])
    else:
        compare(sys.argv[2], sys.argv[3])
