export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/g_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/g_pytest.txt 2>&1
TAG=g_ STEPS=20 bash tools/sweep.sh
