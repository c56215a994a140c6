#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tests/gpu_sigma_probe.py both 20
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/sigma_full -f python tests/gpu_sigma_probe.py sigma 1 > gpurun_out/ncu_sig.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu_sig.log
