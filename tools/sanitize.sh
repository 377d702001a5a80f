# compute-sanitizer over one small fwd + bwd (smoke: BASELINE configs[0]) and a
# mid-size backward: memcheck, racecheck (shared memory), synccheck
export PYTHONUNBUFFERED=1
for tool in memcheck racecheck synccheck; do
  echo "== $tool (smoke)"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python __graft_entry__.py --smoke 2>&1 | grep -E "ERROR SUMMARY|smoke ok|Error|error" | head -5
done
echo "== memcheck (backward shapes, repeated bit split)"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "backward_parity_shapes or bitsplit_repeated" 2>&1 | grep -E "ERROR SUMMARY|passed|failed" | head -5
