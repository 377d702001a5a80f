#!/bin/bash
# Phase timing of the GEMM and the sampler from globaltimer stamps (run under gpurun from
# the repo root, after `tools/build_variants.sh stamps:"-DI4_STAMPS=1"`).
mkdir -p gpurun_out
export I4_LIB_OVERRIDE=$PWD/build_variants/stamps.so
( timeout 200 python tools/gemm_stamps.py bmm 12 512 512 64 5
  timeout 200 python tools/gemm_stamps.py bmm 48 128 128 64 5
  timeout 200 python tools/gemm_stamps.py linear cfg3_bert_large_ffn_up
  timeout 200 python tools/gemm_stamps.py linear cfg3_bert_large_qkv
  timeout 200 python tools/gemm_stamps.py linear cfg2_bert_base_ffn1
  timeout 300 python tools/smp_stamps.py cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down \
      cfg3_bert_large_qkv:dense cfg3_bert_large_ffn_up:dense cfg3_bert_large_ffn_down:dense
  timeout 200 python tools/bmm_stamps.py 12 512 512 64 5 ) > gpurun_out/stamps.txt 2>&1
