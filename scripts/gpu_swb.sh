for bn in 0 128 256; do timeout 120 python tests/gpu_swb_shape.py $bn; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/swb_full python tests/gpu_swb_shape.py 256 > gpurun_out/ncu_swb.log 2>&1; echo NCU $?
