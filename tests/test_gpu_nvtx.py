"""BTP_NVTX=1 wraps every executor stage in an NVTX range (for Nsight Systems); the step still runs."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = """
import sys; sys.path.insert(0, '.')
import torch
from tests.gpu_util import SMALL, inputs
from paper_2512_12131_b200 import executor as E
from paper_2512_12131_b200.api import train_step
from paper_2512_12131_b200.model import RunShape, Variant
from paper_2512_12131_b200.plan import Strategy, plan
assert E._NVTX
blk, x, G, _ = inputs(SMALL, Variant.COLA, 2, 64)
pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(2, 64, 1), Variant.COLA, online_norm=True, grouping=True)
st = train_step(pl, blk, x, G)
print("ok", st.loss)
"""


def test_nvtx_ranges_step_runs():
    env = dict(os.environ, BTP_NVTX="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().startswith("ok")
