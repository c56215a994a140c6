# round-2 re-entry check: every GPU test, smoke, default bench
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02r_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02r_pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench rc=$?"; head -c 3000 gpurun_out/r02r_bench.json; echo
