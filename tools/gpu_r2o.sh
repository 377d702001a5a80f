export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s_pytest.txt 2>&1
for c in cfg3_bert_large_ffn_down cfg4_vit_b16_ffn_down cfg3_bert_large_qkv; do echo "== $c"; timeout 300 python tools/exp_bwd.py $c 2>&1 | grep -v -i Warn; done > gpurun_out/s_bwd.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
