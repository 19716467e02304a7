"""Per-(run, step) agreement of the engine with the reference's BASELINE-config
goldens (tests/golden/baseline.npz) and, when present, the reference's own
ulp self-disagreement band (tests/golden/baseline_band.npz).

  python tools/baseline_report.py [--backend cuda|hostsim] [--configs C1,C3] [--out file.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="cuda")
    ap.add_argument("--configs", default="C1,C3,C2,C4")
    ap.add_argument("--modes", default="stage,persistent")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    from scenario_util import compare_baseline
    golden = lambda n: np.load(os.path.join(ROOT, "tests", "golden", n + ".npz"))  # noqa: E731
    if a.backend == "cuda":
        from paper_2501_07942_b200.backend import CudaBackend
        be = CudaBackend()
        kw = {}
    else:
        from hostsim import HostBackend
        be = HostBackend()
        kw = dict(ws_bytes=256 << 20, state_doubles=1 << 18, cache_cap=1 << 20)
    report = {}
    for name in a.configs.split(","):
        for mode in a.modes.split(","):
            t0 = time.time()
            rows = compare_baseline(golden, name, be, persistent=(mode == "persistent"), **kw)
            clean = []
            for r in rows:
                c = {}
                for k, v in r.items():
                    if isinstance(v, tuple):
                        c[k] = [list(map(int, x)) if isinstance(x, tuple) else (int(x) if not isinstance(x, bool) else x)
                                for x in v]
                    elif isinstance(v, (np.floating, float)):
                        c[k] = float(v)
                    else:
                        c[k] = v
                clean.append(c)
            report[f"{name}/{mode}"] = {"seconds": time.time() - t0, "rows": clean}
            print(name, mode, "%.1fs" % (time.time() - t0), flush=True)
            for c in clean:
                print("  ", json.dumps(c), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
