#!/bin/bash
# batched attention BMM: parity tests, bench_bmm lines, the whole GPU suite, the default bench (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bmm.py -x -q 2>&1 | tail -30 > gpurun_out/bmm_tests.log
for cfg in "12 512 512 64 5" "48 128 128 64 5"; do
  timeout 300 python tools/bench_bmm.py $cfg >> gpurun_out/bmm_bench.jsonl 2>>gpurun_out/bmm_bench.err
done
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
