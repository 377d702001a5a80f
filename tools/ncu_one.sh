#!/bin/bash
# One ncu --set full capture of one kernel of the bench step (run under gpurun from the repo root).
# Usage: tools/ncu_one.sh <kernel-regex> <config> <out-name> [extra bench args]
K=$1; CFG=$2; OUT=$3; shift 3
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-2} -c 1 \
    -o gpurun_out/$OUT -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --config $CFG "$@" \
    > gpurun_out/$OUT.out 2>&1
ls -la gpurun_out/$OUT.ncu-rep
