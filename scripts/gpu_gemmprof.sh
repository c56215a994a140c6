# --set full of selected GEMM launches (scripts/microbench/gpu_profile_kernels.py shapes)
for k in ${KS:-qkv_up dgrad_gu down_gu}; do
  timeout 120 python scripts/microbench/gpu_profile_kernels.py $k 3 2>&1 | tail -1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_$k python scripts/microbench/gpu_profile_kernels.py $k 3 > /dev/null 2>&1 || echo "ncu $k failed"
done
