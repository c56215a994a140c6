# compute-sanitizer over the device path at small shapes (memcheck: out-of-bounds / misaligned /
# leaks; synccheck: illegal barrier use; racecheck: shared-memory hazards)
cd $GRAFT_REPO_ROOT 2>/dev/null || true
S=compute-sanitizer
timeout 900 $S --tool memcheck --leak-check full --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.txt 2>&1; echo "memcheck smoke rc=$?"
timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rowops.py -q -x -k "2048 or 64" > gpurun_out/san_memcheck_rowops.txt 2>&1; echo "memcheck rowops rc=$?"
timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_model.py -q -x -k "matches_oracle and not tp2" > gpurun_out/san_memcheck_model.txt 2>&1; echo "memcheck model rc=$?"
timeout 900 $S --tool synccheck --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_synccheck_smoke.txt 2>&1; echo "synccheck smoke rc=$?"
timeout 900 $S --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_rowops.py -q -x -k "2048" > gpurun_out/san_racecheck_rowops.txt 2>&1; echo "racecheck rowops rc=$?"
for f in gpurun_out/san_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|LEAK SUMMARY|passed|failed|Error" $f | tail -4; done
# round-1 additions: residual-staging GEMM (kSlots 4) + split-K tails, the lax variant, vanilla ckpt
timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_gemm.py -q -x -k "epi or residual or split or randomised" > gpurun_out/san_memcheck_gemm.txt 2>&1; echo "memcheck gemm rc=$?"
timeout 900 $S --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_lax.py -q -x -k "train_step and not tp2" > gpurun_out/san_memcheck_lax.txt 2>&1; echo "memcheck lax rc=$?"
timeout 900 $S --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_gemm.py -q -x -k "residual or randomised" > gpurun_out/san_racecheck_gemm.txt 2>&1; echo "racecheck gemm rc=$?"
for f in gpurun_out/san_memcheck_gemm.txt gpurun_out/san_memcheck_lax.txt gpurun_out/san_racecheck_gemm.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|Error" $f | tail -4; done
