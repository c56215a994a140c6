# attention kernels: parity tests + timing vs cuDNN + pipeline traces (full logs in gpurun_out/)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | grep -E "passed|failed|Error|error|assert" | tail -6
timeout 300 python scripts/microbench/gpu_attn_bench.py > gpurun_out/attn_bench.log 2>&1
timeout 120 python scripts/microbench/attn_trace.py > gpurun_out/attn_trace_bwd.log 2>&1
timeout 120 python scripts/microbench/attn_fwd_trace.py > gpurun_out/attn_trace_fwd.log 2>&1
cat gpurun_out/attn_bench.log
