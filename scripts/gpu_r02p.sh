# round-2 regression after the merged backward GEMM launches: GPU tests, smoke, default bench, reference arm
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02p_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02p_pytest_gpu.log | tail -6
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r02p_bench_1.json 2> gpurun_out/r02p_bench_1.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02p_bench_1.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), d['breakdown'], d['roofline']['frac'], d['clocks'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02p_ref.json 2>gpurun_out/r02p_ref.err; echo "ref rc=$?"; head -c 600 gpurun_out/r02p_ref.json; echo
