"""Probe: does a concurrent 64 MiB pinned H2D per step slow the graph-replayed block step (L2 / HBM
interference)? Device time of 20 replays, without and with the copy on a side stream."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200.api import BlockTrainer  # noqa: E402
from paper_2512_12131_b200.model import RunShape, Variant, build_block, fan_in_scaled, preset  # noqa: E402
from paper_2512_12131_b200.plan import Strategy, plan  # noqa: E402
from paper_2512_12131_b200.tensor import seeded_fill  # noqa: E402

cfg = preset("1b")
b, s = 4, 4096
blk = fan_in_scaled(build_block(cfg, Variant.COLA, 0))
pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
tr = BlockTrainer(pl, blk, adamw=dict(lr=1e-4, b1=0.9, b2=0.95, eps=1e-8, wd=0.1))
x = seeded_fill((b, s, cfg.d), 10000).values
G = seeded_fill((b, s, cfg.d), 30000).values
xd, gd = tr.device_inputs(x, G)
for _ in range(3):
    tr.step_device(xd, gd)
torch.cuda.synchronize()
host = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
dev = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
side = torch.cuda.Stream()
for mode in ("none", "h2d", "none", "h2d", "d2d"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        if mode != "none":
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                if mode == "h2d":
                    dev.copy_(host, non_blocking=True)
                else:
                    dev.copy_(dev.flip(0) if False else dev, non_blocking=True)
        tr.step_device(xd, gd)
    e1.record()
    torch.cuda.synchronize()
    print(f"{mode}: {e0.elapsed_time(e1) / 20:.3f} ms/step", flush=True)
