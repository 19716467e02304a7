#!/bin/bash
# One GPU session: tests, baseline report, bench, ncu launch list + full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log
tail -3 gpurun_out/r02_pytest_gpu.log
if [ "${SKIP_BENCH:-0}" != "1" ]; then
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo BENCH_RC=$?
tail -c 600 gpurun_out/r02_bench.json
fi
if [ "${NCU:-0}" = "1" ]; then
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv --log-file gpurun_out/r02_ncu_launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1; echo NCU1_RC=$?
timeout 1800 ncu --profile-from-start off --set full --import-source on --clock-control none -f -o gpurun_out/r02_full_filter_run python tools/prof_run.py --batch 296 --warmup 2 --steps 1 > gpurun_out/r02_ncu_full.log 2>&1; echo NCU2_RC=$?
fi
