timeout 1200 python -m pytest tests/test_gpu_peer.py -q -x 2>&1 | grep -v "^$" | tail -30
