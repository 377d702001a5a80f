#!/bin/bash
# Per-round ncu evidence (run under gpurun from the repo root):
#  1. launch list of the default bench command (per-launch device time, cold, serialised)
#  2. one full capture of each kernel of the step (grad_split, sampler, compact, the three GEMMs, hadamard_quant)
# Usage: tools/profile_round.sh r02 [config]
R=${1:-r02}
CFG=${2:-cfg2_bert_base_ffn1}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e --config $CFG \
    > gpurun_out/${R}_launches.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grad_split|gemm_i8|hadamard_quant|lss_sampler|compact" \
    -s 7 -c 7 -o gpurun_out/${R}_full -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config $CFG \
    > gpurun_out/${R}_full.out 2>&1
ls -la gpurun_out | grep ${R}
