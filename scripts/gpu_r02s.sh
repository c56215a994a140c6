# 8-problem GEMM launches: unit tests (compute-sanitizer is closed on this pool since round 2's later
# sessions: runs under it left GPUs needing a reset; coverage comes from the torch fp32 comparisons)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -m gpu -p no:cacheprovider -k "eight or split or randomised" 2>&1 | tail -2
