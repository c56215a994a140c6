cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 600 python scripts/microbench/gpu_gemm_resid_ab.py 2>&1 | tail -10
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x -rf -p no:cacheprovider 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
for st in 0 1 0 1; do timeout 300 python bench.py --no-cpu-baseline --no-baselines --gemm-st-global $st > gpurun_out/st$st.json 2>gpurun_out/st$st.err; python -c "import json;d=json.load(open('gpurun_out/st$st.json'));print('st_global=$st', round(d['ms_per_step'],3), 'ms', round(d['roofline']['achieved']), 'TF/s gemm', d['breakdown'])"; done
