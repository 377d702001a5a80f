export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
./tools/mb/cvt_tput > gpurun_out/d_cvt.txt 2>&1
for v in cvt0 cvt1; do
I4_LIB_OVERRIDE=$PWD/build_variants/$v.so timeout 300 ncu --set full -k regex:grad_split -s 1 -c 1 -o gpurun_out/d_gs_$v -f python tools/one_step.py cfg3_bert_large_ffn_up sparse 2 > /dev/null 2>&1
done
timeout 300 ncu --set full -k regex:grad_split -s 1 -c 1 -o gpurun_out/d_gs_cvt2 -f python tools/one_step.py cfg3_bert_large_ffn_up sparse 2 > /dev/null 2>&1
