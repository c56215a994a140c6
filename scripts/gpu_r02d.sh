cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python scripts/microbench/gpu_gemm_resid_ab.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_nccl.py tests/test_gpu_tp2.py -q -rf -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
for m in 1 3; do timeout 300 python bench.py --no-cpu-baseline --no-baselines --emulate-tp 8 --config 7b --gemm-res $m > gpurun_out/em8_$m.json 2>gpurun_out/em8_$m.err; python -c "import json;d=json.load(open('gpurun_out/em8_$m.json'));print('7b emulated tp8 res=$m', round(d['ms_per_step'],3), 'ms', round(d['roofline']['achieved']), 'TF/s gemm', d['breakdown'])"; done
timeout 1500 python scripts/margin_probe2.py --cfg P7B --bs 1,256 --worlds 1,8 --modes none,fwd 2>&1 | grep -E "world=|Error|error" | head -20
