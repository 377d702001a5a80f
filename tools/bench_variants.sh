for v in wide p64 pnone default; do
  if [ $v = default ]; then unset I4_LIB_OVERRIDE; else export I4_LIB_OVERRIDE=$PWD/build_variants/$v.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-per-linear --no-gate > gpurun_out/bv_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bv_$v.json')); print('$v', round(d['ms_per_step'],3), {k: round(v['us_per_step']) for k,v in d['kernels'].items()})"
done
