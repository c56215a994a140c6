# N>1 bench path on ONE GPU (ranks share cuda:0 over gloo): catches failures in the multi-rank code
# path (trainer, e2e fit, GEMM timing, baselines, comm profile, rank-0 line) before a real scaling run.
cd $GRAFT_REPO_ROOT 2>/dev/null || true
for cfg in "2 --b 4" "4 --b 2" "8 --b 1 --s 2048"; do
  set -- $cfg; n=$1; shift
  timeout 900 python bench.py --gpus $n --share-gpu --steps 2 --warmup 3 --cpu-seconds 3 "$@" > gpurun_out/share_n$n.json 2> gpurun_out/share_n$n.err
  echo "N=$n rc=$?"; tail -2 gpurun_out/share_n$n.err | cut -c1-300
  python -c "import json; d=json.load(open('gpurun_out/share_n$n.json')); print(sorted(d.keys())); print('n_gpus', d['n_gpus'], 'baselines', list((d.get('baselines') or {}).keys()), 'comm', (d.get('comm') or {}).keys() if d.get('comm') else None, 'cpu', (d.get('cpu_baseline') or {}).get('value'))" 2>&1 | tail -3
done
