#!/bin/bash
# Quick evidence run: GPU parity suite + bench line (tag = $1).
set -x
tag=${1:-x}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_pytest_gpu_$tag.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu_$tag.log
tail -3 gpurun_out/r02_pytest_gpu_$tag.log
timeout 1200 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/r02_bench_$tag.json 2> gpurun_out/r02_bench_$tag.err; echo BENCH_RC=$?
tail -c 1500 gpurun_out/r02_bench_$tag.err
