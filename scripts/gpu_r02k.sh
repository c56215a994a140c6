# TP=8 whole-tensor vs per-shard margins (bf16 and fp32 forward boundaries)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tp2.py -q -m gpu -s -p no:cacheprovider -k "whole_tensor or fp32_boundary_margin" > gpurun_out/r02k_margin.log 2>&1; echo "pytest rc=$?"; grep -E "TP=8|passed|failed|Error" gpurun_out/r02k_margin.log | tail -12
