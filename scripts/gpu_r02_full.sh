# round-2 full check after the attention work: every GPU test, smoke, default bench x2, native-attention bench, reference arm
cd $GRAFT_REPO_ROOT 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02g_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02g_pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py > gpurun_out/r02g_bench_$i.json 2> gpurun_out/r02g_bench_$i.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02g_bench_$i.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), d['breakdown'], d['roofline']['frac'])"; done
timeout 600 python bench.py --attn native > gpurun_out/r02g_bench_native.json 2> gpurun_out/r02g_bench_native.err; echo "bench native rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02g_bench_native.json')); print(round(d['ms_per_step'],3), 'ms', d['breakdown'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02g_ref.json 2>gpurun_out/r02g_ref.err; echo "ref rc=$?"; head -c 400 gpurun_out/r02g_ref.json; echo
