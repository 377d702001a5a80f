#!/bin/bash
# Round-end evidence on one GPU (run under gpurun from the repo root):
#   tests, the default bench line, the one-step ncu launch list of the cfg5 stack and
#   --set full captures of one layer's backwards and forwards.
# Usage: tools/final_profile.sh <round tag, e.g. r2f>
R=${1:-r2f}
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${R}_tests.txt 2>&1; tail -2 gpurun_out/${R}_tests.txt
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; tail -1 gpurun_out/${R}_bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python tools/stack_step.py > gpurun_out/${R}_launches.out 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"grad_split|gemm_i8|hadamard_quant|lss_sampler|compact" -s 213 -c 12 \
    -o gpurun_out/${R}_full -f python tools/stack_step.py > gpurun_out/${R}_full.out 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"gemm_i8|hadamard_quant" -s 0 -c 6 \
    -o gpurun_out/${R}_fwd -f python tools/stack_step.py > gpurun_out/${R}_fwd.out 2>&1
ls -la gpurun_out | grep ${R}
