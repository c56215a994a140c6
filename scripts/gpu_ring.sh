timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_baselines.py -q -x 2>&1 | tail -2
timeout 120 python tests/gpu_profile_kernels.py up_resid 3 2>&1 | tail -1
timeout 300 python tests/gpu_gemm_pair_bench.py 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bring.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bring.json')); print(round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
