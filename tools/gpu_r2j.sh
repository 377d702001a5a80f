export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lsq_grad.py tests/test_gpu_parity_r2.py -m gpu -q -x -p no:cacheprovider -k "hadamard or forward or status or lsq or low_hadamard" > gpurun_out/m_pytest.txt 2>&1
CF="cfg2_bert_base_ffn1 cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down cfg4_vit_b16_ffn_up cfg4_vit_b16_ffn_down cfgT_transformer_base_qkv"
timeout 300 python tools/hq_time.py $CF > gpurun_out/m_hq.txt 2>&1
I4_LIB_OVERRIDE=$PWD/build_variants/oldhq.so timeout 300 python tools/hq_time.py $CF >> gpurun_out/m_hq.txt 2>&1
