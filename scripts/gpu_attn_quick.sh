# attention kernels: parity tests + timing vs cuDNN + bwd pipeline trace
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 300 python -m pytest tests/test_gpu_attention.py -q -x 2>&1 | grep -E "passed|failed|Error|error|assert" | tail -6
timeout 300 python scripts/microbench/gpu_attn_bench.py 2>&1 | tail -12
timeout 120 python scripts/microbench/attn_trace.py 2>&1 | sed -n '1,2p;8,11p;$p'
