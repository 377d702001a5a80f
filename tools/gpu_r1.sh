export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/a_smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/a_pytest.txt 2>&1
CFGS="cfg3_bert_large_qkv cfg3_bert_large_ffn_up cfg3_bert_large_ffn_down cfg4_vit_b16_ffn_up" STEPS=20 bash tools/sweep.sh
for c in cfg3_bert_large_qkv cfg3_bert_large_ffn_up; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --config $c --grad dense > gpurun_out/sweep_dense_$c.json 2>/dev/null; done
