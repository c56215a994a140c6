# launch list of graph-replayed default bench steps (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 200 --csv --log-file gpurun_out/launches_cur.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cur.log 2>&1; echo NCU $?
tail -3 gpurun_out/ncu_cur.log
