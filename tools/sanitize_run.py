"""One small persistent launch (ttgbf_filter_run) plus one stage-API step for
compute-sanitizer (memcheck / racecheck / synccheck):

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2501_07942_b200.bank import BankConfig, FilterBank
    from paper_2501_07942_b200.configs import SCENARIOS, simulate
    name = sys.argv[1] if len(sys.argv) > 1 else "cv4_step0"
    sc = SCENARIOS[name]
    g, x = sc["grid"], sc["cross"]
    bc = BankConfig(n_per_axis=g["n_per_axis"], sigma_mult=g["sigma_mult"], round_tol=g["round_tol"],
                    round_max_rank=g.get("round_max_rank"), tol=x["tol"], max_rank=x["max_rank"], rng_seed=x["rng_seed"],
                    ws_bytes=64 << 20, state_doubles=1 << 17, cache_cap=1 << 18, big_slots=1, big_bytes=256 << 20)
    Z = np.stack([simulate(sc["spec"], sc["x0_mean"], sc["x0_cov"], sc["steps"], np.random.SeedSequence((2024, r, 0)))[1]
                  for r in range(2)])
    bank = FilterBank(sc["spec"], bc, 2)
    recs = bank.run(Z, 1, sc["x0_mean"], sc["x0_cov"])
    print("persistent statuses", recs["status"].tolist())
    bank2 = FilterBank(sc["spec"], BankConfig(**{**bc.__dict__, "big_slots": 0}), 1)
    bank2.init_prior(sc["x0_mean"], sc["x0_cov"])
    out = bank2.step(Z[:1, 0])
    print("stage statuses", out["status"].tolist())


if __name__ == "__main__":
    main()
