run() { tag=$1; shift; timeout 400 python bench.py --no-cpu-baseline --steps 10 --warmup 3 "$@" > gpurun_out/emu2_$tag.json 2>gpurun_out/emu2_$tag.err; python -c "import json; d=json.load(open('gpurun_out/emu2_$tag.json')); r=d['roofline']; print('$tag', 'ms', round(d['ms_per_step'],3), 'tok/s', round(d['value']), 'gemm TF/s', round(r['achieved']), 'step frac', round(r['step_frac_of_peak'],3), d['clocks']['reasons'])" 2>&1 | tail -1; }
run 1b_btp_tp2 --emulate-tp 2
run 1b_van_tp2 --emulate-tp 2 --strategy vanilla
run 1b_full_tp2 --emulate-tp 2 --strategy full-rank
run 7b_btp_tp8 --emulate-tp 8 --config 7b
run 7b_van_tp8 --emulate-tp 8 --config 7b --strategy vanilla
run 7b_full_tp8 --emulate-tp 8 --config 7b --strategy full-rank
run 7b_btp_tp4_s8192_ckpt --emulate-tp 4 --config 7b --b 1 --s 8192 --ckpt
run 7b_btp_tp4_s8192 --emulate-tp 4 --config 7b --b 1 --s 8192
run 7b_btp_tp1 --config 7b
run 1b_full_tp1 --strategy full-rank
timeout 900 python bench.py --model --layers 24 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/emu2_model_l24.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/emu2_model_l24.json')); print('model24', round(d['ms_per_step'],2), round(d['value']), d['clocks'])"
timeout 900 python bench.py --model --layers 24 --ckpt --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/emu2_model_l24_ckpt.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/emu2_model_l24_ckpt.json')); print('model24ckpt', round(d['ms_per_step'],2), round(d['value']), d['clocks'])"
