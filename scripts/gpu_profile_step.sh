# per-launch device time + DRAM traffic + tensor-pipe of every libbtp GEMM in one eager step
# (skip the 3 warm-up steps' 72 GEMM launches)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel -s 72 -c 24 --csv --log-file gpurun_out/gemm_traffic.csv python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline > gpurun_out/ncu_traffic.log 2>&1; echo NCU1 $?
