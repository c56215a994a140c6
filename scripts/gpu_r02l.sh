# attention backward: packed-P dS phase (btp_attn_tune(3, 2)) vs the default kernel
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 600 python scripts/microbench/attn_bwd_variants.py 3 0,2 12 > gpurun_out/r02l_bwd_ab.log 2>&1; echo "ab rc=$?"; grep -E "worst|median" gpurun_out/r02l_bwd_ab.log
for v in 0 2 0 2; do
timeout 600 python bench.py --no-baselines --no-cpu-baseline --no-attention-ab --attn-bwd-variant $v > gpurun_out/r02l_bench_v$v.json 2> gpurun_out/r02l_bench_v$v.err; echo "bench v$v rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02l_bench_v$v.json')); print('v$v', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', d['breakdown'])"
done
