# attention evidence for profiles/attention: tests, fwd/bwd A/B vs cuDNN, traces, pipe + MMA rates
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out/attn
timeout 300 python -m pytest tests/test_gpu_attention.py -q 2>&1 | tail -2 > gpurun_out/attn/pytest.log
timeout 300 python scripts/microbench/gpu_attn_bench.py > gpurun_out/attn/bench.log 2>&1
timeout 120 python scripts/microbench/attn_trace.py > gpurun_out/attn/trace_bwd.log 2>&1
timeout 120 python scripts/microbench/attn_fwd_trace.py > gpurun_out/attn/trace_fwd_split_row.log 2>&1
timeout 60 ./scripts/microbench/pipe_rates > gpurun_out/attn/pipe_rates.log 2>&1
timeout 60 ./scripts/microbench/mma_rates > gpurun_out/attn/mma_rates.log 2>&1
timeout 60 ./scripts/microbench/mma_pair_rates > gpurun_out/attn/mma_pair_rates.log 2>&1
cat gpurun_out/attn/pytest.log; tail -9 gpurun_out/attn/bench.log
