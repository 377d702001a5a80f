#!/bin/bash
mkdir -p gpurun_out
I4_LIB_OVERRIDE=$PWD/build_variants/stamps.so timeout 300 python tools/bmm_stamps.py 12 512 512 64 5 > gpurun_out/bmm_stamps.txt 2>&1
I4_LIB_OVERRIDE=$PWD/build_variants/stamps.so timeout 300 python tools/bmm_stamps.py 48 128 128 64 5 >> gpurun_out/bmm_stamps.txt 2>&1
for cfg in "12 512 512 64 5" "48 128 128 64 5"; do
  timeout 300 python tools/bench_bmm.py $cfg >> gpurun_out/bmm_bench.jsonl 2>>gpurun_out/bmm_bench.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bmm_launches.csv python tools/bmm_step.py 12 512 512 64 5 3 > gpurun_out/bmm_step.log 2>&1
