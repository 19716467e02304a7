#!/bin/bash
# compute-sanitizer on one small persistent launch + one stage-API step (cv4_step0) and on the device RNG entry.
set -x
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02_sanitizer_$tool.log 2>&1; echo "SAN $tool rc=$?"; tail -4 gpurun_out/r02_sanitizer_$tool.log
done
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_rng.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_sanitizer_racecheck_rng.log 2>&1; echo "SAN rng rc=$?"; tail -4 gpurun_out/r02_sanitizer_racecheck_rng.log
