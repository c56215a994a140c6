"""Parity at the configuration bench.py measures: the CoLA-1B block (d 2048, d_ff 5472, r 512,
32 heads) at b = 4, s = 4096 (T = 16384; BASELINE.json configs[1] shape), BTP + online RMSNorm +
grouping, bf16 — run through the bench's own object (`BlockTrainer`, graph-captured step) and
compared, after a graph REPLAY, with the float64 oracle (lean attention) on y, the loss, dx and
every weight gradient at the north_star bar (2e-2 relative).

This is the shape where the weight-gradient GEMMs run split-K over K = T = 16384 and cuDNN picks
its s = 4096 attention kernels — neither is reached by the short-sequence parity tests.
Reference semantics: simulator.py:550-714 (forward), norms.py:67-96 (online norm)."""

import numpy as np
import pytest
import torch

from oracle import btp_oracle as O
from paper_2512_12131_b200.api import BlockTrainer
from paper_2512_12131_b200.model import RunShape, Variant, preset
from paper_2512_12131_b200.plan import Strategy, plan
from tests.gpu_util import BF16_TOL, inputs, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("attn", ["cudnn", "native", "hybrid"])
@pytest.mark.parametrize("b,s", [(4, 4096)])
def test_bench_config_block_vs_oracle(b, s, attn):
    cfg = preset("1b")
    T = b * s
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    tr = BlockTrainer(pl, blk, optimizer=False, attn_backend=attn)
    xd, gd = tr.device_inputs(x.values, G.values)
    tr.step_device(xd, gd)          # eager step (allocates), then capture
    tr.step_device(xd, gd)          # first replay
    torch.cuda.synchronize()
    assert tr.graphed
    ex = tr.ex
    y = tr._y.double().cpu().numpy().reshape(T, cfg.d)
    loss = float(tr.loss_buf.item())
    dx = tr._dx.double().cpu().numpy().reshape(T, cfg.d)
    grads = ex.weight_grads_by_name()

    x2, G2 = x.values.reshape(T, cfg.d), G.values.reshape(T, cfg.d)
    y_ref, cache = O.block_forward(oblk, x2, b, s, cfg.heads, lean=True)
    g_ref = O.block_backward(oblk, cache, G2, b, s, cfg.heads)
    loss_ref = float(np.sum(y_ref * G2))
    del cache

    errs = {"y": rel(y, y_ref), "loss": abs(loss - loss_ref) / abs(loss_ref)}
    errs["dx"] = rel(dx, g_ref["dx"])
    for n in O.PROJECTIONS:
        errs[f"A_{n}"] = rel(grads["A"][n], g_ref["A"][n])
        errs[f"B_{n}"] = rel(grads["B"][n], g_ref["B"][n])
    errs["gamma1"] = rel(grads["gamma1"], g_ref["dgamma1"])
    errs["gamma2"] = rel(grads["gamma2"], g_ref["dgamma2"])
    worst = max(errs, key=errs.get)
    print(f"bench-config parity (1b b{b} s{s}, attention {attn}): worst {worst} = {errs[worst]:.3e}; "
          + ", ".join(f"{k}={v:.2e}" for k, v in sorted(errs.items())))
    bad = {k: v for k, v in errs.items() if v > BF16_TOL}
    assert not bad, bad
