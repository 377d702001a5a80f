timeout 600 python -m pytest tests -m gpu -q -x -k "bitsplit or backward or full_size" 2>&1 | tail -2
for c in cfg2_bert_base_ffn1 cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up; do echo == $c; timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split; echo " G=2:"; I4_BS_G=2 timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split | head -3; done
timeout 300 python tools/gs_stamps.py cfg2_bert_base_ffn1 cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up 2>&1 | tail -18
