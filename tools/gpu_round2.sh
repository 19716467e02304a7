#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log
tail -3 gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo BENCH_RC=$?
timeout 2400 python tools/tier4.py gpu --out gpurun_out/r02_tier4_gpu.json > gpurun_out/r02_tier4_gpu.log 2>&1; echo TIER4_RC=$?
bash tools/gpu_ncu.sh
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02_sanitizer_$tool.log 2>&1; echo "SAN $tool rc=$?"; tail -3 gpurun_out/r02_sanitizer_$tool.log
done
