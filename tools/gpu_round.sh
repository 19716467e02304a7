#!/bin/bash
# One GPU session: tests, baseline report, A/B bench of library variants, tier-4 GPU leg.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log
tail -3 gpurun_out/r02_pytest_gpu.log
timeout 1200 python tools/baseline_report.py --backend cuda --out gpurun_out/r02_baseline_report.json > gpurun_out/r02_baseline_report.log 2>&1; echo REPORT_RC=$?
for v in "" rl; do
  TTGBF_LIB_VARIANT=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab_$v.json 2> gpurun_out/r02_ab_$v.err
  echo "variant=$v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02_ab_$v.json'));print(d['value'], d['roofline']['frac'], d['engine_prof_share'])"
done
timeout 2400 python tools/tier4.py gpu --out gpurun_out/r02_tier4_gpu.json > gpurun_out/r02_tier4_gpu.log 2>&1; echo TIER4_RC=$?
