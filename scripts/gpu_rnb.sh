timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baselines.py tests/test_gpu_model.py -q -x 2>&1 | tail -2
for k in rmsnorm_bwd rmsnorm dot; do timeout 120 python tests/gpu_profile_kernels.py $k 3 2>&1 | tail -1; done
