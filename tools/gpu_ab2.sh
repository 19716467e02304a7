#!/bin/bash
set -x
mkdir -p gpurun_out
for v in "" qu1 rl ns4 ns16; do
  TTGBF_LIB_VARIANT=$v timeout 600 python tools/round_batch_bench.py --count 296 > gpurun_out/r02_roundab_$v.json 2>&1; echo "variant=$v rc=$?"; cat gpurun_out/r02_roundab_$v.json | tail -1
  TTGBF_LIB_VARIANT=$v timeout 600 python tools/round_batch_bench.py --count 296 --ranks 1,200,320,400,560,200,1 > gpurun_out/r02_roundab2_$v.json 2>&1; tail -1 gpurun_out/r02_roundab2_$v.json
done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo BENCH_RC=$?
python -c "import json;d=json.load(open('gpurun_out/r02_bench.json'));print(d['value'], d['roofline']['frac'], d['engine_prof_share'])"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log; tail -2 gpurun_out/r02_pytest_gpu.log
