"""Single-filter stage profile for ncu: run one C5 filter through the stage
API for --skip steps (not profiled), then profile one measurement launch and
one time-update launch (kernel cross, FFT conv + rounding, realign cross).

  ncu --profile-from-start off --set full --import-source on -o gpurun_out/st \
      python tools/prof_stage.py --run 0 --skip 2
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--run", type=int, default=0)
    p.add_argument("--skip", type=int, default=2)
    p.add_argument("--filters", type=int, default=1)
    a = p.parse_args()
    import torch
    from bench import PROF_NAMES, trajectories
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    from paper_2501_07942_b200.configs import BASELINE_CONFIGS

    cfg = BASELINE_CONFIGS["C5"]
    g, x = cfg["grid"], cfg["cross"]
    bcfg = BankConfig(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                      round_max_rank=g["round_max_rank"], tol=x["tol"], max_rank=x["max_rank"],
                      rng_seed=x["rng_seed"], ws_bytes=1024 << 20, state_doubles=1 << 17, cache_cap=1 << 20)
    for run in range(a.run, a.run + 64):   # first run that survives --skip steps
        _, meas = trajectories(cfg, range(run, run + a.filters))
        bank = FilterBank(cfg["spec"], bcfg, a.filters)
        bank.init_prior(cfg["x0_mean"], cfg["x0_cov"])
        ok = True
        for k in range(a.skip):
            if np.any(bank.step(meas[:, k])["status"] != 0):
                ok = False
                break
        if ok:
            break
    print("run", run, file=sys.stderr)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    dm = bank.measure(meas[:, a.skip])
    geom = bank.geometry(dm)
    dt = bank.time_update(geom)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    cyc = dt["cycles"].sum(axis=0).astype(float)
    prof = dt["prof"].sum(axis=0).astype(float)
    tot = max(cyc.sum(), 1.0)
    print(json.dumps({"status": dt["status"].tolist(), "stage_ms": (cyc / 1.965e6).round(2).tolist(),
                      "prof_ms": {nm: round(float(prof[q] / 1.965e6), 2) for q, nm in enumerate(PROF_NAMES)},
                      "ranks": dt["ranks"][0].tolist(),
                      "calls": [int(v) for v in dt["cross"][0]["calls"]]}))


if __name__ == "__main__":
    main()
