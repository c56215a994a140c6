# baselines with merged backward launches: parity + the default bench line (baselines included)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_baselines.py tests/test_gpu_tp2.py tests/test_gpu_lax.py tests/test_gpu_ckpt.py -q -m gpu -p no:cacheprovider -k "vanilla or full or naive or baseline or lax or ckpt" > gpurun_out/r02n_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "^FAILED|passed|failed|Error" gpurun_out/r02n_pytest.log | tail -8
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; echo "bench rc=$?"; python -c "import json; d=json.load(open('gpurun_out/r02n_bench.json')); print(round(d['ms_per_step'],3), 'ms', round(d['value']/1e6,3), 'M', 'e2e', round(d['e2e']['value']/1e6,3), d['breakdown'], round(d['roofline']['frac'],3), d['roofline']['traffic'], {k: round(v['ms_per_step'],3) for k,v in d['baselines'].items() if isinstance(v, dict) and 'ms_per_step' in v})"
