timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for c in cfg2_bert_base_ffn1 cfg3_bert_large_ffn_up cfg3_bert_large_qkv cfg4_vit_b16_ffn_up; do
  for v in 0 auto; do
    I4_BWD_CONCURRENT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$c conc=$v', round(d['ms_per_step']*1e3,1), 'us  bf16', round(d['bf16_cublas_ms_per_step']*1e3,1))"
  done
done
