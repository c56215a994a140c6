# full-step A/B: bench with cuDNN attention vs the native kernels (+ native block parity tests)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_bench_parity.py -q -x 2>&1 | grep -E "passed|failed|Error|assert" | tail -5
for a in cudnn native cudnn native; do
  timeout 600 python bench.py --attn $a > gpurun_out/step_$a.json 2> gpurun_out/step_$a.err
  python -c "import json; d=json.load(open('gpurun_out/step_$a.json')); print('$a', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'Mtok/s e2e', round(d['e2e']['value']/1e6,3), d.get('breakdown'))"
done
