#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --launch-skip 14 --launch-count 7 -o gpurun_out/bmm_full -f python tools/bmm_step.py 12 512 512 64 5 3 > gpurun_out/bmm_full.log 2>&1
