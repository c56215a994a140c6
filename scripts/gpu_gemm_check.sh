timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for k in qkv_up down_sigma up_resid; do timeout 120 python tests/gpu_profile_kernels.py $k 3 2>&1 | tail -1; done
timeout 300 python tests/gpu_gemm_pair_bench.py 2>&1 | tail -24
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --dump-gemms gpurun_out/gemms_new.json > gpurun_out/b_new.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/b_new.json')); print('block', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks'])"
