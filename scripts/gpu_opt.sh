#!/bin/bash
# optimizer tests + parity suites + one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 400 python bench.py --steps 10 --warmup 3 --cpu-seconds 15 > gpurun_out/bench_opt.json 2>gpurun_out/bench_opt.err; echo B1 $?
tail -3 gpurun_out/bench_opt.err
python -c "import json; d=json.load(open('gpurun_out/bench_opt.json')); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'gemm',d['roofline']['achieved'], d['roofline']['frac'], 'cpu', d.get('cpu_baseline',{}).get('value'), 'clk', d['clocks'])"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-optimizer > gpurun_out/bench_noopt.json 2>&1; echo B2 $?
python -c "import json; d=json.load(open('gpurun_out/bench_noopt.json')); print('noopt value',d['value'],'ms',d['ms_per_step'])"
