cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python scripts/microbench/gpu_gemm_resid_ab.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py tests/test_gpu_ckpt.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
timeout 900 python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_r02b.err; cat gpurun_out/bench_r02b.json
timeout 900 python scripts/margin_probe2.py 2>&1 | grep -E "world=|Error|error" | head -20
timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python -m pytest tests/test_gpu_gemm.py -q -x -k "residual or randomised" > gpurun_out/san_racecheck_gemm.txt 2>&1; echo "racecheck gemm rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/san_racecheck_gemm.txt | tail -5
