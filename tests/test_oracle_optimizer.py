"""The oracle's AdamW (CPU arm of the bench) against torch.optim.AdamW, float64."""

import numpy as np
import torch

from oracle import btp_oracle as O


def test_oracle_adamw_matches_torch():
    blk = O.build_block(64, 160, 16, "cola", 0, scale_fan_in=3.0)
    x = O.seeded_fill((2 * 8, 64), 10000)
    G = O.loss_projection((2 * 8, 64))
    hp = dict(lr=1e-2, b1=0.9, b2=0.95, eps=1e-8, wd=0.1)
    p0 = {("A", n): blk["A"][n].copy() for n in blk["A"]}
    p0[("g1",)] = blk["gamma1"].copy()
    tparams = {k: torch.nn.Parameter(torch.from_numpy(v.copy())) for k, v in p0.items()}
    opt = torch.optim.AdamW([{"params": [v for k, v in tparams.items() if k[0] == "A"], "weight_decay": hp["wd"]},
                             {"params": [tparams[("g1",)]], "weight_decay": 0.0}],
                            lr=hp["lr"], betas=(hp["b1"], hp["b2"]), eps=hp["eps"])
    state = {}
    for _ in range(3):
        _, cache = O.block_forward(blk, x, 2, 8, 4)
        grads = O.block_backward(blk, cache, G, 2, 8, 4)
        for k, p in tparams.items():
            p.grad = torch.from_numpy((grads["A"][k[1]] if k[0] == "A" else grads["dgamma1"]).copy())
        O.adamw_step(blk, grads, state, **hp)
        opt.step()
    assert state["t"] == 3
    for k, p in tparams.items():
        got = blk["A"][k[1]] if k[0] == "A" else blk["gamma1"]
        np.testing.assert_allclose(got, p.detach().numpy(), rtol=1e-10, atol=1e-12)
        assert not np.array_equal(got, p0[k])
