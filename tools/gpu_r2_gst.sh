#!/bin/bash
mkdir -p gpurun_out
export I4_LIB_OVERRIDE=$PWD/build_variants/stamps.so
( timeout 200 python tools/gemm_stamps.py bmm 12 512 512 64 5
  timeout 200 python tools/gemm_stamps.py linear cfg3_bert_large_ffn_up
  timeout 200 python tools/gemm_stamps.py linear cfg2_bert_base_ffn1 ) > gpurun_out/gemm_stamps.txt 2>&1
