# round-2 check: fixed model tests, margin probe (fp32 vs bf16 boundary reductions), new bench line, racecheck
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_ckpt.py -q -rf -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
timeout 900 python scripts/margin_probe2.py 2>&1 | grep -E "world=|Error|error" | head -20
timeout 900 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_r02a.err; cat gpurun_out/bench_r02a.json
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -q -x -k "residual or randomised" > gpurun_out/san_racecheck_gemm.txt 2>&1; echo "racecheck gemm rc=$?"; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed|hazard" gpurun_out/san_racecheck_gemm.txt | tail -5
