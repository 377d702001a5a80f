#!/bin/bash
# grad_split timing: fast phase 2, phase 1 only, no-Philox, generic phase 2
for c in ${CFGS:-cfg3_bert_large_ffn_up cfg2_bert_base_ffn1}; do
  echo "== $c"
  echo -n " fast    "; timeout 120 python tools/exp_variants.py $c 2>&1 | grep grad_split
  echo -n " phase1  "; I4_BS_EXP=1 timeout 120 python tools/exp_variants.py $c 2>&1 | grep grad_split
  echo -n " noRNG   "; I4_BS_EXP=2 timeout 120 python tools/exp_variants.py $c 2>&1 | grep grad_split
  echo -n " generic "; I4_BS_GENERIC=1 timeout 120 python tools/exp_variants.py $c 2>&1 | grep grad_split
done
