export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on -k regex:gemm_i8 -s 3 -c 1 -o gpurun_out/k_bwd_ffndown -f python tools/one_step.py cfg3_bert_large_ffn_down sparse 2 > gpurun_out/k_ncu.txt 2>&1
