# compute-sanitizer over the persistent hd-64 attention backward (memcheck + racecheck), small shapes
cd $GRAFT_REPO_ROOT 2>/dev/null || true
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_attention.py -q -x -k "persistent_walk and not 1024-80 and not 4096" > gpurun_out/san_memcheck_attn_persist.txt 2>&1; echo "memcheck persist rc=$?"
timeout 1200 compute-sanitizer --tool racecheck --print-limit 30 python -m pytest tests/test_gpu_attention.py -q -x -k "persistent_walk and (1-128-3 or 2-256-5)" > gpurun_out/san_racecheck_attn_persist.txt 2>&1; echo "racecheck persist rc=$?"
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/san_memcheck_attn_persist.txt gpurun_out/san_racecheck_attn_persist.txt | tail -8
