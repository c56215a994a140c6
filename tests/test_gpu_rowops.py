"""Row kernels against plain PyTorch fp32 references across the widths the model zoo produces
(TP shards of 60M..30B d and d_ff) — in particular the TMA row-pipeline RMSNorm kernels, whose
stage count depends on the row size (with and without the residual branch)."""

import pytest
import torch

from paper_2512_12131_b200 import kernels as K

pytestmark = pytest.mark.gpu
WIDTHS = [64, 256, 512, 1536, 2048, 3072, 4096, 5120, 8192]


def _rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm())


@pytest.mark.parametrize("width", WIDTHS)
@pytest.mark.parametrize("branch", [False, True])
@pytest.mark.parametrize("rows", [1, 37, 3000])
def test_rmsnorm_residual_widths(width, branch, rows):
    torch.manual_seed(width + rows)
    x = torch.randn(rows, width, device="cuda").bfloat16()
    br = torch.randn(rows, width, device="cuda").bfloat16() if branch else None
    g = torch.rand(width, device="cuda") + 0.5
    n = torch.empty_like(x)
    xo = torch.empty_like(x) if branch else None
    ss = torch.empty(rows, device="cuda")
    rl = torch.empty(rows, device="cuda")
    K.rmsnorm_residual(x, g, branch=br, x_out=xo, n_out=n, ss_out=ss, rl_out=rl, eps=1e-6)
    v = (x.float() + br.float()).bfloat16().float() if branch else x.float()
    ss_ref = (v * v).sum(1)
    rl_ref = torch.sqrt(ss_ref / width + 1e-6)
    assert _rel(ss, ss_ref) < 1e-5 and _rel(rl, rl_ref) < 1e-5
    assert _rel(n, v * g / rl_ref[:, None]) < 1e-2
    if branch:
        assert torch.equal(xo, v.bfloat16())


@pytest.mark.parametrize("width", WIDTHS)
@pytest.mark.parametrize("dres", [False, True])
def test_rmsnorm_bwd_widths(width, dres):
    torch.manual_seed(width)
    rows = 1500
    dh, x = (torch.randn(rows, width, device="cuda").bfloat16() for _ in range(2))
    dr = torch.randn(rows, width, device="cuda").bfloat16() if dres else None
    g = torch.rand(width, device="cuda") + 0.5
    dss = torch.randn(rows, device="cuda")
    dx = torch.empty_like(x)
    parts = torch.empty(4 * K.num_sms(), width, device="cuda")
    nb = K.rmsnorm_bwd(dh, x, g, dss, dx, parts, dres=dr)
    dg = parts[:nb].sum(0)
    ref = dh.float() * g + 2 * x.float() * dss[:, None] + (dr.float() if dres else 0)
    assert _rel(dx, ref) < 1e-2
    assert _rel(dg, (dh.float() * x.float()).sum(0)) < 1e-4
