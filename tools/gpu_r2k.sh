export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/n_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/n_pytest.txt 2>&1
timeout 900 python bench.py > gpurun_out/n_bench.json 2> gpurun_out/n_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/n_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-per-linear --no-gate > gpurun_out/n_launches.out 2>&1
