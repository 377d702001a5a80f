#!/bin/bash
# Build library variants with different -D knobs into build_variants/<name>.so (for tools/exp_variants.py)
# Usage: tools/build_variants.sh name1:"-DX=1 -DY=2" name2:"..."
cd "$(dirname "$0")/.."
mkdir -p build_variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -fmad=false $defs \
    -o build_variants/$name.so paper_2306_11987_b200/csrc/{api,quant,sampler,compact,gemm,lsq,adaptive_k}.cu &
done
wait
ls build_variants
