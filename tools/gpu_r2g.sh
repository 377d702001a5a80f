export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for c in cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down cfg4_vit_b16_ffn_down cfg4_vit_b16_ffn_up; do echo "== $c"; timeout 300 python tools/exp_bwd.py $c 2>&1 | grep -v -i Warn; done > gpurun_out/l_bwd.txt 2>&1
