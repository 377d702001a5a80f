export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_launches.csv python tools/stack_step.py > gpurun_out/r2s_launches.out 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"grad_split|gemm_i8|hadamard_quant|lss_sampler|compact" -s 213 -c 12 -o gpurun_out/r2s_full -f python tools/stack_step.py > gpurun_out/r2s_full.out 2>&1
