# per-kernel: event timing, ncu key metrics (1 launch after 3 warm-up), and --set full for the GEMMs
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed
for k in qkv_up down_sigma up_resid rmsnorm swiglu swiglu_bwd fixup_bwd adamw xent peer_fwd peer_bwd; do
  timeout 120 python scripts/microbench/gpu_profile_kernels.py $k 3 2>&1 | tail -1
  timeout 300 ncu --metrics $M --clock-control none -s 3 -c 1 --csv --log-file gpurun_out/kmet_$k.csv python scripts/microbench/gpu_profile_kernels.py $k 3 > /dev/null 2>&1 || echo "ncu $k failed"
done
for k in qkv_up down_sigma up_resid; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/full_$k python scripts/microbench/gpu_profile_kernels.py $k 3 > gpurun_out/full_$k.log 2>&1 || echo "ncu full $k failed"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:peer_boundary -s 3 -c 1 -o gpurun_out/full_peer_fwd python scripts/microbench/gpu_profile_kernels.py peer_fwd 3 > gpurun_out/full_peer.log 2>&1 || echo "ncu full peer failed"
ls gpurun_out
