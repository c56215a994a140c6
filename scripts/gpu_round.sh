# full GPU check: tests, smoke, default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x -rf 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo BENCH $?; tail -3 gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
