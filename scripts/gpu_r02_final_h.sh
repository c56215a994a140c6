# round-2 final check after the hybrid-attention default: smoke, default bench x2, cuDNN-both and
# native-both benches, reference arm, launch list of the default step (pytest ran separately)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 2400 python -m pytest tests -q -m gpu -rf -p no:cacheprovider > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/r02i_pytest_gpu.log | tail -4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py > gpurun_out/r02i_bench_$i.json 2> gpurun_out/r02i_bench_$i.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02i_bench_$i.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), d['breakdown'], d['roofline']['frac'], d['config'].get('attention'))"; done
timeout 600 python bench.py --attn cudnn --no-attention-ab > gpurun_out/r02i_bench_cudnn.json 2> gpurun_out/r02i_bench_cudnn.err; echo "bench cudnn rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02i_bench_cudnn.json')); print(round(d['ms_per_step'],3), 'ms', d['breakdown'])"
timeout 600 python bench.py --attn native --no-attention-ab > gpurun_out/r02i_bench_native.json 2> gpurun_out/r02i_bench_native.err; echo "bench native rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02i_bench_native.json')); print(round(d['ms_per_step'],3), 'ms', d['breakdown'])"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02i_ref.json 2>gpurun_out/r02i_ref.err; echo "ref rc=$?"; head -c 300 gpurun_out/r02i_ref.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02i_launches.csv python bench.py --steps 2 --warmup 1 --no-attention-ab > gpurun_out/r02i_ncu_bench.log 2>&1; echo "ncu rc=$?"
