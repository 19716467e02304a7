#!/bin/bash
# A/B of library variants on the bench: tools/gpu_ab3.sh "<variant tags, '-' = default>" [bench args...]
set -x
mkdir -p gpurun_out
tags=$1; shift
for v in $tags; do
  lv=$v; [ "$v" = "-" ] && lv=""
  TTGBF_LIB_VARIANT=$lv timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/r02_ab_$v.json 2> gpurun_out/r02_ab_$v.err
  echo "variant=$v rc=$?"; tail -c 600 gpurun_out/r02_ab_$v.err
  python tools/bench_show.py gpurun_out/r02_ab_$v.json | head -8
done
