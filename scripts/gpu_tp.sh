#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_tp2.py -q -m gpu -x -k c60m 2>&1 | tail -15
