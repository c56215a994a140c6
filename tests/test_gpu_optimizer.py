"""Fused AdamW (btp_adamw) against torch.optim.AdamW in fp32, and the trainer's in-graph optimizer
step: a replayed CUDA graph must keep advancing the device-side step count (bias correction)."""

import numpy as np
import pytest
import torch

from paper_2512_12131_b200 import kernels as K
from paper_2512_12131_b200.api import BlockTrainer
from paper_2512_12131_b200.model import RunShape, Variant
from paper_2512_12131_b200.plan import Strategy, plan

from .gpu_util import SMALL, inputs

pytestmark = pytest.mark.gpu

HP = dict(lr=3e-3, b1=0.9, b2=0.95, eps=1e-8, wd=0.1)


def torch_adamw(p0, grads, **hp):
    """Reference: torch.optim.AdamW on CPU fp32 (decoupled weight decay), one step per gradient."""
    p = torch.nn.Parameter(p0.detach().cpu().float().clone())
    opt = torch.optim.AdamW([p], lr=hp["lr"], betas=(hp["b1"], hp["b2"]), eps=hp["eps"], weight_decay=hp["wd"])
    for g in grads:
        p.grad = g.detach().cpu().float().clone()
        opt.step()
    return p.detach()


@pytest.mark.parametrize("work_dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("on_device_step", [False, True])
def test_adamw_kernel_matches_torch(work_dtype, on_device_step):
    n = 8 * 12345
    gen = torch.Generator().manual_seed(0)
    p0 = torch.randn(n, generator=gen)
    grads = [torch.randn(n, generator=gen) * 0.1 for _ in range(3)]
    dev = "cuda"
    master = p0.to(dev).clone()
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    work = torch.empty(n, dtype=work_dtype, device=dev)
    ctr = torch.ones(1, dtype=torch.int32, device=dev)
    for i, g in enumerate(grads):
        gd = g.to(dev)
        if on_device_step:
            K.adamw(master, m, v, gd, work, step_dev=ctr, **HP)
            K.counter_add(ctr, 1)
        else:
            K.adamw(master, m, v, gd, work, step=i + 1, **HP)
    torch.cuda.synchronize()
    want = torch_adamw(p0, grads, **HP)
    err = (master.cpu() - want).abs().max().item()
    assert err < 1e-5, err
    # the working copy is the master rounded to the operand dtype
    assert torch.equal(work.cpu(), master.cpu().to(work_dtype))
    if on_device_step:
        assert int(ctr.item()) == len(grads) + 1


def test_adamw_rejects_misaligned():
    n = 8 * 100
    t = lambda: torch.zeros(n, device="cuda")  # noqa: E731
    with pytest.raises(Exception):
        K.adamw(t(), t(), t(), t(), t()[1:], lr=1e-3, step=1)  # length mismatch
    with pytest.raises(Exception):
        K.adamw(t()[:n - 4], t()[:n - 4], t()[:n - 4], t()[:n - 4], t()[:n - 4], lr=1e-3, step=1)  # n % 8


@pytest.mark.parametrize("use_graph", [True, False])
def test_trainer_steps_apply_adamw(use_graph):
    """Two trainer steps (graph replays when use_graph): the fp32 master equals torch AdamW fed the
    two gradients the steps produced, so the device step counter advanced inside the graph."""
    cfg, b, s = SMALL, 2, 128
    blk, x, G, _ = inputs(cfg, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    tr = BlockTrainer(pl, blk, adamw=HP, use_graph=use_graph)
    xd, gd = tr.device_inputs(x.values, G.values)
    ex = tr.ex
    p0 = ex.w_flat.float().cpu().clone()
    gam0 = ex.gam_flat.cpu().clone()
    grads, gam_grads, losses = [], [], []
    for _ in range(3):
        tr.step_device(xd, gd)
        torch.cuda.synchronize()
        grads.append(ex.g_flat.cpu().clone())
        gam_grads.append(ex.gam_grad_flat.cpu().clone())
        losses.append(float(tr.loss_buf.item()))
    master = ex.opt["master"].cpu()
    want = torch_adamw(p0, grads, **HP)
    assert (master - want).abs().max().item() < 1e-5
    want_g = torch_adamw(gam0, gam_grads, **{**HP, "wd": 0.0})
    assert (ex.gam_flat.cpu() - want_g).abs().max().item() < 1e-5
    assert int(ex.opt["step"].item()) == 4
    # the weights the next forward reads are the updated ones (views of the flat working copy)
    assert torch.equal(ex.w_flat.cpu(), master.to(ex.w_flat.dtype))
    # the update moves the loss: three distinct step losses
    assert len(set(np.round(losses, 6))) == 3
