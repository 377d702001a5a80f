# concurrent grad_X || grad_W: pairs given to grad_X and grad_W split-K (experiment)
c=${CFG:-cfg2_bert_base_ffn1}
for spec in "auto:" "24:1" "37:1" "48:1" "48:2" "48:3" "40:2" "44:2" "52:2"; do
  px=${spec%%:*}; ws=${spec#*:}
  if [ "$px" = auto ]; then unset I4_BWD_CONCURRENT I4_BWD_WSPLIT; else export I4_BWD_CONCURRENT=$px I4_BWD_WSPLIT=$ws; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --config $c 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); k=d['kernels']; print('$c px=$px wsplit=$ws', round(d['ms_per_step']*1e3,1), 'us; pair', round(k.get('gemm_i8_dgrad||gemm_i8_wgrad',{}).get('avg_us',0),1), 'd', round(k['gemm_i8_dgrad']['avg_us'],1), 'w', round(k['gemm_i8_wgrad']['avg_us'],1))"
done
