export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/b_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/b_pytest.txt 2>&1
for c in cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grad_split -s 1 -c 1 -o gpurun_out/b_gs_$c -f python tools/one_step.py $c sparse 2 > gpurun_out/b_ncu_$c.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"hadamard_quant|compact|lss_sampler" -s 3 -c 3 -o gpurun_out/b_misc_ffnup -f python tools/one_step.py cfg3_bert_large_ffn_up sparse 2 > gpurun_out/b_ncu_misc.txt 2>&1
