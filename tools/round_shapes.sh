#!/bin/bash
# Rounding micro-benchmark over product-TT shapes seen in the C5 FFT convolution
# (tools/round_bench.py, one CTA, deterministic random cores).
for r in 1,40,80,120,160,60,1 1,100,160,180,280,90,1 1,90,360,500,780,440,1; do
  python tools/round_bench.py --ranks $r --reps 2
done
