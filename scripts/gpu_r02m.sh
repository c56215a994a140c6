# backward dgrad + weight-gradient launches merged (default) vs separate; parity of the affected paths
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
for m in merged split merged split; do
  flag=""; [ $m = split ] && flag="--no-merge-bwd-gemms"
  timeout 600 python bench.py --no-baselines --no-cpu-baseline --no-attention-ab $flag > gpurun_out/r02m_bench_$m.json 2> gpurun_out/r02m_bench_$m.err; echo "bench $m rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/r02m_bench_$m.json')); r=d['roofline']; print('$m', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), 'gemm', round(d['breakdown']['gemm_ms'],3), 'frac', round(r['frac'],3), 'launches/step', r.get('gemm_launches_per_step'), 'gpu_launches', d['gpu_launches'])"
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_ckpt.py tests/test_gpu_model.py tests/test_gpu_lax.py tests/test_gpu_tp2.py -q -m gpu -x -p no:cacheprovider > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed|Error" gpurun_out/r02m_pytest.log | tail -8
