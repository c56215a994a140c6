"""Shared helpers for the GPU parity tests: oracle runs, error metrics, config builders."""

import numpy as np

from oracle import btp_oracle as O
from paper_2512_12131_b200.model import ModelConfig, RunShape, Variant, build_block, fan_in_scaled
from paper_2512_12131_b200.tensor import seeded_fill

SMALL = ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)
C60M = ModelConfig(layers=8, heads=8, d=512, d_ff=1376, r=128)
P7B = ModelConfig(layers=32, heads=32, d=4096, d_ff=11008, r=1024)  # the paper's CoLA-7B block widths
BF16_TOL = 2e-2  # north_star: bf16 mode within 2e-2 relative on activations, gradients and loss


def rel(got, want):
    got = np.asarray(got, dtype=np.float64).reshape(np.shape(want))
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def inputs(cfg, variant, b, s, seed=0):
    blk = fan_in_scaled(build_block(cfg, variant, seed))
    x = seeded_fill((b, s, cfg.d), seed + 10000)
    G = seeded_fill((b, s, cfg.d), seed + 30000)
    oblk = O.build_block(cfg.d, cfg.d_ff, cfg.r, variant.value, seed, scale_fan_in=3.0)
    return blk, x, G, oblk


def oracle_step(oblk, x, G, cfg, b, s, tp=1, online=True, sharded=True, h_prev=None):
    """h_prev (lax): {projection: Tensor/array [b, s, r]}; grads then hold dh_prev and the
    returned cache's h_cur is in grads["h_cur"]."""
    T = b * s
    x2 = x.values.reshape(T, cfg.d)
    G2 = G.values.reshape(T, cfg.d)
    hp = None
    if h_prev is not None:
        hp = {n: np.asarray(getattr(v, "values", v)).reshape(T, cfg.r) for n, v in h_prev.items()}
    y, cache = O.block_forward(oblk, x2, b, s, cfg.heads, h_prev=hp)
    grads = O.block_backward(oblk, cache, G2, b, s, cfg.heads)
    if "h_cur" in cache:
        grads["h_cur"] = cache["h_cur"]
    ws = O.btp_forward_sharded(oblk, x2, b, s, cfg.heads, tp, online=online, h_prev=hp)[1] if sharded else None
    loss = float(np.sum(y * G2))
    return y, grads, ws, loss
