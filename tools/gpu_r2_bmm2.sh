#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bmm_launches.csv python tools/bmm_step.py 12 512 512 64 5 3 > gpurun_out/bmm_step.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bmm_launches48.csv python tools/bmm_step.py 48 128 128 64 5 3 >> gpurun_out/bmm_step.log 2>&1
