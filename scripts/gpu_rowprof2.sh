for k in rmsnorm rmsnorm_bwd dot; do timeout 120 python tests/gpu_profile_kernels.py $k 3 2>&1 | tail -1; done
for k in rmsnorm_bwd dot; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"rmsnorm_bwd|dot_kernel" -s 3 -c 1 -o gpurun_out/full_$k python tests/gpu_profile_kernels.py $k 3 > /dev/null 2>&1 || echo "ncu $k failed"
done
