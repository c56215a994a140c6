# For an 8 x B200 (NVSwitch) box: the TP scaling runs the driver does (N = 1, 2, 4, 8, NCCL
# boundaries), then the peer-memory and NVLS boundary forms at TP = 8, each with NCCL's own log
# (NCCL_DEBUG=INFO shows the algorithm / protocol / NVLS use of every communicator), the NVLink
# GB/s of the boundary all-reduces (the bench line's "comm" object), the two-process peer / NVLS
# tests and an ncu launch list of one TP=8 rank. Outputs: gpurun_out/scale_*.json / *.log.
cd $GRAFT_REPO_ROOT 2>/dev/null || true
export NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,COLL,TUNING
for n in 1 2 4 8; do
  timeout 900 python bench.py --gpus $n --steps 20 --warmup 5 > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.log
  echo "N=$n rc=$?"; python -c "import json;d=json.load(open('gpurun_out/scale_n$n.json'));print(d['value'],d['ms_per_step'],d.get('baselines',{}).get('btp_over_naive_tp'),d.get('baselines',{}).get('btp_over_full_rank'),d.get('comm',{}).get('bus_gbs'))"
done
for bd in peer nvls; do
  timeout 900 python bench.py --gpus 8 --boundary $bd --no-baselines > gpurun_out/scale_n8_$bd.json 2> gpurun_out/scale_n8_$bd.log; echo "N=8 $bd rc=$?"
done
timeout 900 python bench.py --gpus 8 --config 7b --no-cpu-baseline > gpurun_out/scale_7b_n8.json 2> gpurun_out/scale_7b_n8.log; echo "7b N=8 rc=$?"
timeout 900 python bench.py --gpus 8 --config 7b --boundary-dtype fp32 --no-cpu-baseline --no-baselines > gpurun_out/scale_7b_n8_fp32.json 2> gpurun_out/scale_7b_n8_fp32.log; echo "7b N=8 fp32 rc=$?"
grep -h "NVLS\|Algo\|algorithm" gpurun_out/scale_n8.log | sort | uniq -c | sort -rn | head -20
timeout 900 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_peer_ipc.py -q -rs 2>&1 | tail -5
