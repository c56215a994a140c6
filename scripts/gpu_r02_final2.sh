# round-2 final (re-entry session): default bench x2 on the fresh box, then the GPU suite, smoke,
# a bench after the suite, and the reference arm
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
show() { python -c "import json; d=json.load(open('$1')); r=d['roofline']; print('$1', round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), {k: round(v,3) for k,v in d['breakdown'].items()}, 'gemm frac', round(r['frac'],3), 'launches', r['gemm_launches_per_step'], 'traffic', r['traffic'], d['clocks'], {k: round(v['ms_per_step'],3) for k,v in d['baselines'].items() if isinstance(v, dict) and 'ms_per_step' in v})"; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r02z_bench_$i.json 2> gpurun_out/r02z_bench_$i.err; echo "bench rc=$?"; show gpurun_out/r02z_bench_$i.json; done
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02z_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02z_pytest_gpu.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02z_bench_3.json 2> gpurun_out/r02z_bench_3.err; echo "bench rc=$?"; show gpurun_out/r02z_bench_3.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02z_ref.json 2>gpurun_out/r02z_ref.err; echo "ref rc=$?"; head -c 400 gpurun_out/r02z_ref.json; echo
