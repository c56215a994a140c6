timeout 600 python -m pytest tests/test_gpu_nccl.py tests/test_gpu_tp2.py -q -x 2>&1 | grep -v "^$" | tail -15
