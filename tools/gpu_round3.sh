#!/bin/bash
# Round-2 evidence run: GPU parity suite, bench line, ncu launch list of the bench command, C5 counters.
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log
tail -3 gpurun_out/r02_pytest_gpu.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo BENCH_RC=$?
tail -c 3000 gpurun_out/r02_bench.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_ncu_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1; echo NCU_L_RC=$?
bash tools/gpu_ncu.sh
