export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -x -p no:cacheprovider -k "bitsplit or subnormal or backward_parity or status or binding" > gpurun_out/c_pytest.txt 2>&1
for c in cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg4_vit_b16_ffn_up; do echo "== $c"; timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split; done > gpurun_out/c_variants.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
