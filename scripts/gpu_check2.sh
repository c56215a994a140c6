timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py -q -m gpu -x 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --dump-gemms gpurun_out/gemms.json > gpurun_out/bench_p.json 2>gpurun_out/bench_p.err; echo B1 $?; tail -3 gpurun_out/bench_p.err; python -c "import json; d=json.load(open('gpurun_out/bench_p.json')); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'],'gemm',d['roofline']['achieved'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 140 --csv --log-file gpurun_out/launches3.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo NCU $?
