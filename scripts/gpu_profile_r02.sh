# round-2 profiles: launch list of graph-replayed bench steps, per-GEMM DRAM traffic + tensor pipe of
# one eager step, and --set full of the residual-epilogue up-projection GEMM
cd $GRAFT_REPO_ROOT 2>/dev/null || true
B="python bench.py --no-cpu-baseline --no-baselines"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 200 --csv --log-file gpurun_out/r02_launches.csv $B --steps 4 --warmup 3 > gpurun_out/r02_ncu_launches.log 2>&1; echo NCU-launches $?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_kernel -s 72 -c 24 --csv --log-file gpurun_out/r02_gemm_traffic.csv $B --steps 1 --warmup 3 --no-graph > gpurun_out/r02_ncu_traffic.log 2>&1; echo NCU-traffic $?
KS="up_resid" timeout 900 bash scripts/gpu_gemmprof.sh
ls -la gpurun_out/ | tail -8
