# round-2 refresh: per-rank compute of TP=2/4/8 plans (emulated, collectives not executed), current code
# (NCCL one-rank tests run in the full suite)
run() { tag=$1; shift; timeout 400 python bench.py --no-cpu-baseline --steps 10 --warmup 3 "$@" > gpurun_out/emu2_$tag.json 2>gpurun_out/emu2_$tag.err; echo "$tag rc=$?"; tail -2 gpurun_out/emu2_$tag.err | grep -v "^$" ; python -c "import json; d=json.load(open('gpurun_out/emu2_$tag.json')); r=d['roofline']; print('$tag', 'ms', round(d['ms_per_step'],3), 'tok/s', round(d['value']), 'gemm TF/s', round(r['achieved']), 'gemm share', round(r['gemm_share_of_step'],3), 'step frac', round(r['step_frac_of_peak'],3))" 2>&1 | tail -1; }
run 1b_btp_tp2 --emulate-tp 2
run 1b_van_tp2 --emulate-tp 2 --strategy vanilla
run 1b_full_tp2 --emulate-tp 2 --strategy full-rank
run 7b_btp_tp8 --emulate-tp 8 --config 7b
run 7b_van_tp8 --emulate-tp 8 --config 7b --strategy vanilla
run 7b_full_tp8 --emulate-tp 8 --config 7b --strategy full-rank
run 7b_btp_tp4_s8192_ckpt --emulate-tp 4 --config 7b --b 1 --s 8192 --ckpt
run 7b_btp_tp4_s8192 --emulate-tp 4 --config 7b --b 1 --s 8192
run 7b_btp_tp1 --config 7b
run 1b_btp_tp1_nofuse --no-fuse-sigma
