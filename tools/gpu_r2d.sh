export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_r2.py -m gpu -q -x -p no:cacheprovider -k "bitsplit or subnormal or status" > gpurun_out/e_pytest.txt 2>&1
for c in cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down; do echo "== $c"; timeout 200 python tools/exp_variants.py $c 2>&1 | grep grad_split; done > gpurun_out/e_variants.txt 2>&1
