set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo PYTEST_RC=$? >> gpurun_out/r02_pytest_gpu.log
timeout 900 python tools/baseline_report.py --backend cuda --out gpurun_out/r02_baseline_report.json > gpurun_out/r02_baseline_report.log 2>&1; echo RC=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo BENCH_RC=$?
tail -2 gpurun_out/r02_bench.json
