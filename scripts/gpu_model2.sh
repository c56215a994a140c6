timeout 600 python -m pytest tests/test_gpu_nccl.py -q -x 2>&1 | grep -v "^$" | tail -25
for L in 24; do
timeout 900 python bench.py --model --layers $L --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/model_l$L.json 2>gpurun_out/model_l$L.err; echo rc=$?; tail -3 gpurun_out/model_l$L.err
python -c "import json; d=json.load(open('gpurun_out/model_l$L.json')); print('L$L', d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['step_frac_of_peak'], d['clocks'])"
done
timeout 900 python bench.py --model --layers 24 --ckpt --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/model_l24_ckpt.json 2>gpurun_out/model_l24_ckpt.err; echo rc=$?; tail -3 gpurun_out/model_l24_ckpt.err
python -c "import json; d=json.load(open('gpurun_out/model_l24_ckpt.json')); print('L24ckpt', d['ms_per_step'], d['value'], d['roofline']['step_frac_of_peak'])"
python -c "
import torch,sys; sys.path.insert(0,'.')
" 
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_clk.json; python -c "import json; d=json.load(open('gpurun_out/b_clk.json')); print('block', d['ms_per_step'], d['value'], d['clocks'])"
