for k in adamw rmsnorm fixup_bwd; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"adamw|rmsnorm_residual|fixup_sigma_bwd" -s 3 -c 1 -o gpurun_out/full_$k python tests/gpu_profile_kernels.py $k 3 > /dev/null 2>&1 || echo "ncu $k failed"
done
ls gpurun_out/*.ncu-rep
