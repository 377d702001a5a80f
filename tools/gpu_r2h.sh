export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
python tools/gemm_sk.py > gpurun_out/i_gemm_sk.txt 2>&1
timeout 300 ncu --set full -k regex:gemm_i8 -s 6 -c 2 -o gpurun_out/i_sk -f python tools/gemm_sk.py > /dev/null 2>&1
