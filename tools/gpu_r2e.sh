export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up; do echo "== $c"; timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split; done > gpurun_out/t_variants.txt 2>&1
