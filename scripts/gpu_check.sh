# GPU validation + perf pass (run under gpurun from the repo root)
timeout 300 python tests/gpu_gemm_probe.py 2>&1 | grep -E "rel=[0-9.e-]+|BAD|timing|Error|error" | awk '{ if ($0 ~ /rel=/) { split($0,a,"rel="); if (a[2]+0 > 0.01) print "BADREL " $0 } else print }'
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py -q -m gpu -x 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo BENCH $?; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 2 -o gpurun_out/gemm_full python tests/gpu_gemm_shapes.py > gpurun_out/ncu_gemm.log 2>&1; echo NCU $?
