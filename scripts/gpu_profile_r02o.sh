# profiles of the merged-backward-GEMM step (16 btp_gemm launches): launch list of graph-replayed
# bench steps and per-GEMM DRAM traffic + tensor pipe of one eager step
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline --no-baselines --no-attention-ab"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 200 --csv --log-file gpurun_out/r02o_launches.csv $B --steps 4 --warmup 3 > gpurun_out/r02o_ncu_launches.log 2>&1; echo NCU-launches $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel -s 48 -c 16 --csv --log-file gpurun_out/r02o_gemm_traffic.csv $B --steps 1 --warmup 3 --no-graph > gpurun_out/r02o_ncu_traffic.log 2>&1; echo NCU-traffic $?
ls -la gpurun_out/ | tail -6
