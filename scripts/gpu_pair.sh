timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -x 2>&1 | tail -15
timeout 300 python tests/gpu_gemm_pair_bench.py 2>&1 | tail -15
