# refresh after the merged backward GEMM launches: emulated per-rank TP=2/4/8 compute and the 24-layer model
cd $GRAFT_REPO_ROOT 2>/dev/null || true
mkdir -p gpurun_out
sed 's/emu2_/emu3_/g' scripts/gpu_emulate_r02.sh > /tmp/emu3.sh && bash /tmp/emu3.sh
for ck in "" "--ckpt"; do
  tag=model_l24${ck:+_ckpt}
  timeout 900 python bench.py --no-cpu-baseline --no-baselines --no-attention-ab --model --layers 24 $ck > gpurun_out/emu3_$tag.json 2> gpurun_out/emu3_$tag.err; echo "$tag rc=$?"
  python -c "import json; d=json.load(open('gpurun_out/emu3_$tag.json')); print('$tag', round(d['ms_per_step'],2), 'ms', round(d['value']), 'tok/s', d['clocks'])"
done
