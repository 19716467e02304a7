for v in "" c3 c4; do
  TTGBF_LIB_VARIANT=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_var$v.json 2> gpurun_out/r02_bench_var$v.err
  echo "variant=$v rc=$?"; python -c "import json;d=json.load(open('gpurun_out/r02_bench_var$v.json'));print(d['value'], d['config']['workspace_slots'], d['config']['workspace_mb_per_slot'], d['overflow_ws'])"
done
