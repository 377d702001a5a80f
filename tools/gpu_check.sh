#!/bin/bash
# one GPU round trip: smoke, gpu tests, bench (used with gpurun)
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -${TAILN:-6}
timeout 300 python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
