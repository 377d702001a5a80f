export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py --smoke > gpurun_out/o_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/o_pytest.txt 2>&1
for c in cfg3_bert_large_ffn_up cfg3_bert_large_qkv; do echo "== $c"; timeout 300 python tools/exp_bwd.py $c 2>&1 | grep -v -i Warn; done > gpurun_out/o_bwd.txt 2>&1
