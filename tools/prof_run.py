"""Profiling driver for ncu: B filters of the bench workload, W warm-up steps
(not profiled), then K steps inside cudaProfilerStart/Stop.

  ncu --profile-from-start off --set full --import-source on -o gpurun_out/x \
      python tools/prof_run.py --batch 296 --warmup 2 --steps 1

Prints the per-stage / engine-profile shares of the profiled launch.
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
    p.add_argument("--batch", type=int, default=296)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--steps", type=int, default=1)
    p.add_argument("--config", default="C5")
    p.add_argument("--ws-mb", type=int, default=256)
    a = p.parse_args()
    import torch
    from bench import PROF_NAMES, trajectories
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    from paper_2501_07942_b200.configs import BASELINE_CONFIGS

    cfg = BASELINE_CONFIGS[a.config]
    g, x = cfg["grid"], cfg["cross"]
    from paper_2501_07942_b200 import _abi
    lib = _abi.load_library()
    slots = torch.cuda.get_device_properties(0).multi_processor_count * int(lib.ttgbf_ctas_per_sm())
    bcfg = BankConfig(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                      round_max_rank=g["round_max_rank"], tol=x["tol"], max_rank=x["max_rank"],
                      rng_seed=x["rng_seed"], ws_bytes=a.ws_mb << 20, state_doubles=1 << 17,
                      cache_cap=1 << 20, ws_slots=min(slots, a.batch), big_slots=16, big_bytes=1280 << 20)
    _, meas = trajectories(cfg, range(a.batch))
    bank = FilterBank(cfg["spec"], bcfg, a.batch)
    if a.warmup:
        bank.run(meas, a.warmup, cfg["x0_mean"], cfg["x0_cov"])
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    recs = bank.run(meas, a.steps, cfg["x0_mean"], cfg["x0_cov"])
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    dg = bank._diag()
    cyc = dg["cycles"].sum(axis=0).astype(float)
    prof = dg["prof"].sum(axis=0).astype(float)
    tot = max(cyc.sum(), 1.0)
    print(json.dumps({
        "completed": int((recs["status"] == 0).sum()), "attempted": int((recs["status"] >= 0).sum()),
        "stage_share": (cyc / tot).round(4).tolist(),
        "prof_share": {nm: round(float(prof[q] / tot), 4) for q, nm in enumerate(PROF_NAMES)},
    }))


if __name__ == "__main__":
    main()
