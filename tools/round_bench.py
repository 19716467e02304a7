"""Single-CTA TT rounding micro-benchmark (one heavy FFT-product-like TT).

  python tools/round_bench.py [--ranks 1,90,360,500,780,440,1] [--n 65] [--reps 2]

Times ttgbf_tt_round on one TT with the given ranks (random cores with a
decaying spectrum) and prints the algorithmic GFLOP of the right-to-left QR
sweep and the achieved rate.  Used for ncu captures of the rounding alone.
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def qr_flops(ranks, n):
    d = len(ranks) - 1
    r = list(ranks)
    fl = 0.0
    for k in range(d - 1, 0, -1):
        m, rl = n * r[k + 1], r[k]
        kk = min(m, rl)
        fl += 2.0 * m * rl * kk - 2.0 / 3.0 * kk ** 3
        fl += 2.0 * r[k - 1] * n * rl * kk / 2          # triangular R multiply
        r[k] = kk
    return fl


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ranks", default="1,90,360,500,780,440,1")
    p.add_argument("--n", type=int, default=65)
    p.add_argument("--reps", type=int, default=2)
    p.add_argument("--tol", type=float, default=1e-8)
    a = p.parse_args()
    ranks = [int(x) for x in a.ranks.split(",")]
    import torch
    from paper_2501_07942_b200 import tensor_train as G
    from paper_2501_07942_b200.backend import CudaBackend
    be = CudaBackend()
    G._CTX["be"] = be
    G.WS_BYTES = 2 << 30
    rs = np.random.RandomState(0)
    cores = []
    for k in range(len(ranks) - 1):
        c = rs.randn(ranks[k], a.n, ranks[k + 1])
        c *= (0.9 ** np.arange(ranks[k + 1]))[None, None, :]
        cores.append(c)
    tt = G.TensorTrain.from_cores(cores)
    out = G.tt_round(tt, a.tol, 20)     # warm-up (also loads the library)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        out = G.tt_round(tt, a.tol, 20)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    fl = qr_flops(ranks, a.n)
    t = min(ts)
    print(f"ranks {ranks} n {a.n}: {t:.3f} s, QR-sweep {fl / 1e9:.1f} GFLOP -> {fl / t / 1e9:.1f} GFLOP/s (1 CTA); "
          f"out ranks {out.ranks}")


if __name__ == "__main__":
    main()
