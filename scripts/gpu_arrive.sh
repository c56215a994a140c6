timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for k in qkv_up down_sigma dgrad_gu; do timeout 120 python scripts/microbench/gpu_profile_kernels.py $k 3 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/barr.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/barr.json')); print(round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
