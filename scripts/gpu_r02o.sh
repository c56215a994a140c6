# up to 8 problems per GEMM launch (q|k|v dgrad + weight gradients merged): GEMM + block parity, bench x2
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_ckpt.py tests/test_gpu_baselines.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r02o_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed|Error" gpurun_out/r02o_pytest.log | tail -8
for i in 1 2; do
timeout 900 python bench.py --no-attention-ab > gpurun_out/r02o_bench_$i.json 2> gpurun_out/r02o_bench_$i.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02o_bench_$i.json')); r=d['roofline']; print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), d['breakdown'], round(r['frac'],3), r['gemm_launches_per_step'], r['traffic'], {k: round(v['ms_per_step'],3) for k,v in d['baselines'].items() if isinstance(v, dict) and 'ms_per_step' in v})"
done
timeout 800 python scripts/microbench/gpu_merge_bwd_ab.py 16 2>&1 | tail -2
