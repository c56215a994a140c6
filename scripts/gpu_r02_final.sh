# round-2 full check: every GPU test, smoke, default bench (+ a second run), reference arm, sanitizers on the new GEMM modes
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02_pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py > gpurun_out/r02_bench_$i.json 2> gpurun_out/r02_bench_$i.err; echo "bench rc=$?"; cat gpurun_out/r02_bench_$i.json | head -c 600; echo; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02_ref.json 2>gpurun_out/r02_ref.err; echo "ref rc=$?"; cat gpurun_out/r02_ref.json | head -c 1500; echo
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_gemm.py -q -x -k "epi or residual or split or randomised" > gpurun_out/san_memcheck_gemm.txt 2>&1; echo "memcheck gemm rc=$?"
timeout 900 compute-sanitizer --tool racecheck --print-limit 30 python -m pytest tests/test_gpu_gemm.py -q -x -k "residual or randomised" > gpurun_out/san_racecheck_gemm.txt 2>&1; echo "racecheck gemm rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_memcheck_gemm.txt gpurun_out/san_racecheck_gemm.txt | tail -6
