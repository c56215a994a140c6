timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/up_full python tests/gpu_gemm_shapes.py up > gpurun_out/ncu_up.log 2>&1; echo NCU $?
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 -o gpurun_out/down_full python tests/gpu_gemm_shapes.py down > gpurun_out/ncu_down.log 2>&1; echo NCU $?
