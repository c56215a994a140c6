timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 200 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r01b.log 2>&1; echo NCU $?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
for k in qkv_up down_sigma up_resid dgrad_gu rmsnorm rmsnorm_bwd swiglu swiglu_bwd fixup_bwd adamw; do
  timeout 300 ncu --metrics $M --clock-control none -k regex:"gemm_kernel|rmsnorm|swiglu|fixup|adamw" -s 3 -c 1 --csv --log-file gpurun_out/kmet2_$k.csv python scripts/microbench/gpu_profile_kernels.py $k 3 > /dev/null 2>&1 || echo "ncu $k failed"
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --dump-gemms gpurun_out/gemms_r01b.json > gpurun_out/b_r01b.json 2>/dev/null; cat gpurun_out/b_r01b.json | head -c 600
