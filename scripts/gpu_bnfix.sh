timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 600 python tests/gpu_gemm_bn.py
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --dump-gemms gpurun_out/gemms_bn.json > gpurun_out/bbn.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bbn.json')); print(round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
