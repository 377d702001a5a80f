# grad_split variant timings (build_variants/*.so) at unit size auto and G=2
for c in ${CFGS:-cfg2_bert_base_ffn1 cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up}; do
  echo == $c; timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split
  echo " G=2:"; I4_BS_G=2 timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split
done
