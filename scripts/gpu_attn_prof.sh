# ncu captures of the own attention kernels at the CoLA-1B bench shape (b4 s4096 h32 hd64)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
SHAPE=${SHAPE:-"4 4096 32 64"}
TAG=${TAG:-r02}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd -s 1 -c 1 -f -o gpurun_out/${TAG}_attn_bwd python scripts/microbench/attn_one.py $SHAPE > gpurun_out/${TAG}_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 1 -c 1 -f -o gpurun_out/${TAG}_attn_fwd python scripts/microbench/attn_one.py $SHAPE > gpurun_out/${TAG}_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
tail -3 gpurun_out/${TAG}_ncu_bwd.log
