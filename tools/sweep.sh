#!/bin/bash
# bench every single-linear BASELINE shape (one GPU) into gpurun_out/${TAG}sweep_<cfg>.json
for c in ${CFGS:-cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down cfg4_vit_b16_ffn_up cfg4_vit_b16_ffn_down}; do
  timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e --no-per-linear --no-gate --config $c $EXTRA > gpurun_out/${TAG}sweep_$c.json 2>/dev/null
done
