timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | grep -v "^\s*$" | tail -6
for k in peer_fwd; do timeout 120 python scripts/microbench/gpu_profile_kernels.py $k 3 2>&1 | tail -1; done
