"""Dense FFT point-mass filter throughput on one B200.

  python tools/dense_bench.py [--n 129] [--steps 5] [--warmup 3]

Model: BASELINE config 1/2 (d=4 CV, range+bearing, N_pa+1 points per axis).
Reports steps/s, the per-kernel device time (CUDA events on the launch
stream), the DFT kernel's FP64 rate against the measured DGEMM peak and the
whole step's algorithmic HBM bytes against MEASURED_PEAKS.json, plus the
oracle (numpy, reference algorithm) step time on the host for N <= 65.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=129)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--cpu", action="store_true")
    a = p.parse_args()
    import torch
    from paper_2501_07942_b200.configs import SPECS, simulate
    from paper_2501_07942_b200.dense import DenseFFTFilter
    from paper_2501_07942_b200 import roofline as rl
    spec = SPECS["cv4"]
    mean, cov = np.array([10.0, 10.0, 1.0, 1.0]), np.diag([1.0, 1.0, 0.1, 0.1])
    kf = a.warmup + a.steps
    _, zs = simulate(spec, mean, cov, kf, np.random.SeedSequence((2024, 0, 0)))
    f = DenseFFTFilter(spec, a.n, 6.0)
    f.initial(mean, cov)
    for k in range(a.warmup):
        f.step(zs[k])
    torch.cuda.synchronize()
    # DFT kernel alone (one forward axis pass over the complex buffer), events on the launch stream
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for axis in range(f.d):
        f.lib.ttgbf_dense_dft(f.cb.ptr, f.shape_h.ptr, f.d, axis, 0, f.roots.ptr, f.be.stream_ptr)
    e1.record(st)
    torch.cuda.synchronize()
    dft_s = e0.elapsed_time(e1) / 1e3 / f.d
    n1 = next((q for q in range(2, int(a.n ** 0.5) + 1) if a.n % q == 0), 1)
    macs = (n1 + a.n // n1 + 1) if n1 > 1 else a.n   # two-stage Cooley-Tukey in SMEM (csrc/dense.cu)
    dft_flops = 8.0 * macs * f.total           # 8 flops per complex multiply-add
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record(st)
    t0 = time.perf_counter()
    for k in range(a.warmup, kf):
        f.step(zs[k])
    s1.record(st)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    dev = s0.elapsed_time(s1) / 1e3
    # algorithmic HBM bytes per point per step (d=4): likelihood r+w 16, mass reduce 8,
    # finalize reduce 8 + scale 16, moments 2x8, interp 8 + 16, kernel 16,
    # 3 transforms x d axes x (16 + 16), product 48, real 24, final reduce 8 + scale 16
    bpp = 16 + 8 + 8 + 16 + 16 + 24 + 16 + 3 * f.d * 32 + 48 + 24 + 8 + 16
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 7700.0}
    fp64 = rl.measure_fp64_peak(torch, torch.device("cuda", 0))
    out = {"metric": "dense FFT PMF steps/s (d=4 CV, N_pa=%d)" % (a.n - 1), "n": a.n, "points": f.total,
           "value": a.steps / dev, "unit": "steps/s", "ms_per_step": 1e3 * dev / a.steps,
           "wall_ms_per_step": 1e3 * wall / a.steps, "launches_per_step": None,
           "hbm": {"bytes_per_step": bpp * f.total, "achieved_gbs": bpp * f.total * a.steps / dev / 1e9,
                   "peak_gbs": peaks["hbm_gbs"]},
           "dft_kernel": {"ms_per_axis_pass": 1e3 * dft_s, "complex_macs_per_point": macs,
                          "tflops": dft_flops / dft_s / 1e12,
                          "fp64_peak_tflops": fp64, "frac": dft_flops / dft_s / 1e12 / fp64}}
    if a.cpu and a.n <= 65:
        from oracle import dense as D
        cfg = {"n_per_axis": a.n, "sigma_mult": 6.0}
        axes, w, _ = D.initial(mean, cov, cfg)
        t0 = time.perf_counter()
        for k in range(2):
            axes, w, _ = D.step(axes, w, spec, zs[k], cfg)
        out["cpu_baseline"] = {"ms_per_step": 1e3 * (time.perf_counter() - t0) / 2, "kind": "port", "cores": 1}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
