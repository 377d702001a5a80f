export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_nvls.py -m gpu -q -rs -p no:cacheprovider > gpurun_out/p_nvls.txt 2>&1
timeout 900 python bench.py > gpurun_out/p_bench.json 2> gpurun_out/p_bench.err
