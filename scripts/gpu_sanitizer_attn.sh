# compute-sanitizer over the attention kernels (memcheck + racecheck), small shapes
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -x -k "not block_step and not variants" > gpurun_out/san_memcheck_attn.txt 2>&1; echo "memcheck attn rc=$?"
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -x -k "variants and 64 and poly0 or bwd_hd64" > gpurun_out/san_memcheck_attn_variants.txt 2>&1; echo "memcheck attn variants rc=$?"
timeout 1500 compute-sanitizer --tool racecheck --print-limit 30 python -m pytest tests/test_gpu_attention.py -q -x -k "matches_fp32 and 1-128-1" > gpurun_out/san_racecheck_attn.txt 2>&1; echo "racecheck attn rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_memcheck_attn.txt gpurun_out/san_memcheck_attn_variants.txt gpurun_out/san_racecheck_attn.txt | tail -8
