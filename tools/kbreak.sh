# per-kernel breakdown (CUPTI, PDL-off capture) of the bench step for several configs
for c in ${CFGS:-cfg2_bert_base_ffn1 cfg3_bert_large_ffn_up}; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c', round(d['ms_per_step']*1e3,1), 'us  bf16', round(d['bf16_cublas_ms_per_step']*1e3,1), {k: round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done
