# model step tests + NCCL test (verbose) + model bench
timeout 600 python -m pytest tests/test_gpu_nccl.py -q -x 2>&1 | grep -v "^$" | tail -40
timeout 900 python -m pytest tests/test_gpu_model.py -q -x 2>&1 | tail -30
timeout 600 python bench.py --model --layers 4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/model_l4.json 2>gpurun_out/model_l4.err; echo rc=$?; tail -5 gpurun_out/model_l4.err; cat gpurun_out/model_l4.json
