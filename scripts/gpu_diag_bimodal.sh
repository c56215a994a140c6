set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for i in 1 2 3 4; do timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/d1_b$i.json 2>gpurun_out/d1_b$i.err; tail -c 400 gpurun_out/d1_b$i.json | head -c 0; python -c "import json;d=json.load(open('gpurun_out/d1_b$i.json'));print($i,d['ms_per_step'],d['clocks'],d['roofline']['frac'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 200 --csv --log-file gpurun_out/d1_launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/d1_ncu.log 2>&1; echo NCU $?
for i in 5 6; do timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/d1_b$i.json 2>gpurun_out/d1_b$i.err; python -c "import json;d=json.load(open('gpurun_out/d1_b$i.json'));print($i,d['ms_per_step'],d['clocks'],d['roofline']['frac'])"; done
