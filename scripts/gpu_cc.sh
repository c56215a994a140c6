timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for i in 1 2; do
for m in "" "--serial-wgrad"; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline $m > gpurun_out/bcc.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bcc.json')); print('$m', round(d['ms_per_step'],3), round(d['value']), 'e2e', round(d['e2e']['value']), 'gemm', round(d['roofline']['achieved']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
done
timeout 600 python bench.py --model --layers 24 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/model_cc.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/model_cc.json')); print('model24', round(d['ms_per_step'],2), round(d['value']), d['clocks'])"
