#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x -k sigma 2>&1 | tail -3
for m in "" "--no-fuse-sigma"; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $m --dump-gemms gpurun_out/gemms$m.json > gpurun_out/bench_sig$m.json 2>gpurun_out/bench_sig.err; echo B1 $?
python -c "import json; d=json.load(open('gpurun_out/bench_sig$m.json')); print('$m value',d['value'],'ms',d['ms_per_step'],'gemm',d['roofline']['achieved'], d['roofline']['avg_launch_us']*d['roofline']['gemm_launches_per_step'])"
done
