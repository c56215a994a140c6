cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=power.limit,power.default_limit,power.max_limit,clocks.max.sm,clocks.max.mem --format=csv
timeout 300 python scripts/microbench/gpu_gemm_power_probe.py 2>&1 | tail -8
timeout 300 python scripts/microbench/gpu_profile_kernels.py qkv_up 3 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_qkv_up_r02 python scripts/microbench/gpu_profile_kernels.py qkv_up 3 > /dev/null 2>&1 || echo "ncu failed"
