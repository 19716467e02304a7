#!/bin/bash
# A/B of library variants on the bench + tier-4 GPU leg + compute-sanitizer.
set -x
mkdir -p gpurun_out
for v in "" rl; do
  TTGBF_LIB_VARIANT=$v timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab_$v.json 2> gpurun_out/r02_ab_$v.err
  echo "variant=$v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02_ab_$v.json'));print(d['value'], d['roofline']['frac'], d['engine_prof_share'])"
done
if [ "${TIER4:-0}" = "1" ]; then
timeout 2400 python tools/tier4.py gpu --out gpurun_out/r02_tier4_gpu.json > gpurun_out/r02_tier4_gpu.log 2>&1; echo TIER4_RC=$?
fi
if [ "${SAN:-0}" = "1" ]; then
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02_sanitizer_$tool.log 2>&1; echo "SAN $tool rc=$?"; tail -3 gpurun_out/r02_sanitizer_$tool.log
done
fi
