"""Pin the oracle's analytic backward (the reference has none) against torch float64
autograd of an independent torch restatement of the block forward."""

import numpy as np
import pytest
import torch

from oracle import btp_oracle as O

PROJ = O.PROJECTIONS


def torch_block(blk, x, b, s, heads, eps=1e-6, h_prev=None):
    """Independent float64 torch forward (same math as reference model.py:256-305)."""
    var = blk["variant"]
    H = {n: torch.tensor(h, requires_grad=True) for n, h in h_prev.items()} if h_prev is not None else None
    P = {g: {k: torch.tensor(v, dtype=torch.float64, requires_grad=True) for k, v in blk[g].items()}
         for g in ("A", "B", "W")}
    g1 = torch.tensor(blk["gamma1"], requires_grad=True)
    g2 = torch.tensor(blk["gamma2"], requires_grad=True)
    xt = torch.tensor(x, requires_grad=True)

    def norm(v, g):
        return v * g / torch.sqrt((v * v).mean(-1, keepdim=True) + eps)

    def sig(z):
        if var != "cola":
            return z
        h = z.shape[-1] // 2
        u, w = z[:, :h], z[:, h:]
        return torch.cat([torch.nn.functional.silu(u) * w, torch.nn.functional.silu(w) * u], -1)

    def proj(n, inp):
        if var == "full-rank":
            return inp @ P["W"][n].T
        z = inp @ P["B"][n].T
        if var == "lax" and H is not None:
            return (z + H[n]) @ P["A"][n].T
        return sig(z) @ P["A"][n].T

    d = x.shape[1]
    hd = d // heads
    n1 = norm(xt, g1)
    q, k, v = (proj(n, n1).reshape(b, s, heads, hd).transpose(1, 2) for n in "qkv")
    att = torch.softmax(q @ k.transpose(-1, -2) / hd**0.5, -1) @ v
    att = att.transpose(1, 2).reshape(b * s, d)
    xm = xt + proj("o", att)
    n2 = norm(xm, g2)
    act = torch.nn.functional.silu(proj("gate", n2)) * proj("up", n2)
    y = xm + proj("down", act)
    return (y, P, g1, g2, xt) if H is None else (y, P, g1, g2, xt, H)


@pytest.mark.parametrize("variant", ["cola", "svd", "full-rank"])
def test_backward_matches_autograd(variant):
    d, d_ff, r, heads, b, s = 32, 80, 8, 4, 2, 8
    blk = O.build_block(d, d_ff, r, variant, 3, scale_fan_in=3.0)
    x = O.seeded_fill((b * s, d), 10003)
    G = O.loss_projection((b * s, d), 30003)
    y, cache = O.block_forward(blk, x, b, s, heads)
    g = O.block_backward(blk, cache, G, b, s, heads)
    yt, P, g1, g2, xt = torch_block(blk, x, b, s, heads)
    np.testing.assert_allclose(yt.detach().numpy(), y, rtol=0, atol=1e-12)
    (yt * torch.tensor(G)).sum().backward()
    np.testing.assert_allclose(g["dx"], xt.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(g["dgamma1"], g1.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(g["dgamma2"], g2.grad.numpy(), rtol=0, atol=1e-11)
    for grp in ("A", "B", "W"):
        for n, t in P[grp].items():
            np.testing.assert_allclose(g[grp][n], t.grad.numpy(), rtol=0, atol=1e-11, err_msg=f"{grp}{n}")


def test_sharded_grads_are_slices():
    d, d_ff, r = 32, 80, 8
    blk = O.build_block(d, d_ff, r, "cola", 3)
    g = {"dgamma1": np.arange(d), "dgamma2": np.arange(d), "dx": np.zeros((4, d)),
         "A": {n: blk["A"][n] for n in PROJ}, "B": {n: blk["B"][n] for n in PROJ}}
    sh = O.grads_for_rank(g, 2, 1, d, d_ff)
    assert sh["A"]["gate"].shape == (40, 8) and sh["B"]["down"].shape == (8, 40)
    assert sh["A"]["q"].shape == (16, 8) and sh["B"]["q"].shape == (8, 16)
    assert np.array_equal(sh["dgamma1"], np.arange(16, 32))


def test_lax_backward_matches_autograd():
    """lax with a seeded h bundle: parameter grads, dx and dL/dh_prev per projection."""
    d, d_ff, r, heads, b, s = 32, 80, 8, 4, 2, 8
    blk = O.build_block(d, d_ff, r, "lax", 3, scale_fan_in=3.0)
    x = O.seeded_fill((b * s, d), 10003)
    G = O.loss_projection((b * s, d), 30003)
    hp = {n: h.reshape(b * s, r) for n, h in O.seeded_h_prev(b, s, r, 5).items()}
    y, cache = O.block_forward(blk, x, b, s, heads, h_prev=hp)
    g = O.block_backward(blk, cache, G, b, s, heads)
    yt, P, g1, g2, xt, H = torch_block(blk, x, b, s, heads, h_prev=hp)
    np.testing.assert_allclose(yt.detach().numpy(), y, rtol=0, atol=1e-12)
    (yt * torch.tensor(G)).sum().backward()
    np.testing.assert_allclose(g["dx"], xt.grad.numpy(), rtol=0, atol=1e-11)
    np.testing.assert_allclose(g["dgamma1"], g1.grad.numpy(), rtol=0, atol=1e-11)
    for grp in ("A", "B"):
        for n, t in P[grp].items():
            np.testing.assert_allclose(g[grp][n], t.grad.numpy(), rtol=0, atol=1e-11, err_msg=f"{grp}{n}")
    for n in PROJ:
        np.testing.assert_allclose(g["dh_prev"][n], H[n].grad.numpy(), rtol=0, atol=1e-11, err_msg=n)
