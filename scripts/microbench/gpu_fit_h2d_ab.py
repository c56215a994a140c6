"""A/B of BlockTrainer.fit's first-batch H2D split over 1 vs 4 copy streams: 10-step fit() calls on
the bench step (CoLA-1B b4 s4096 TP=1), host wall time around each call (it includes every H2D and
the loss read-back, as bench.py's e2e), alternating, median over rounds."""
import sys
import time

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
x = seeded_fill((b, s, cfg.d), 10000).values
G = seeded_fill((b, s, cfg.d), 30000).values
tr = BlockTrainer(pl, blk, adamw=dict(lr=1e-4, b1=0.9, b2=0.95, eps=1e-8, wd=0.1))
xh, gh = tr.pinned_host_inputs(x, G)
xh2 = xh.clone().pin_memory()
batches = [xh if i % 2 == 0 else xh2 for i in range(10)]
tr.fit([xh, xh2, xh], gh)
torch.cuda.synchronize()
times = {1: [], 4: []}
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
    for n in ((1, 4) if r % 2 == 0 else (4, 1)):
        BlockTrainer.FIRST_COPY_STREAMS = n
        tr._slots = None  # re-create the copy streams for this setting
        tr.fit([xh], gh)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tr.fit(batches, gh)
        times[n].append((time.perf_counter() - t0) / len(batches) * 1e3)
for n, t in times.items():
    t = sorted(t)
    print(f"first-batch copy streams {n}: median {t[len(t)//2]:.4f} ms/step (e2e), min {t[0]:.4f}, "
          f"max {t[-1]:.4f} over {len(t)}; {b * s / t[len(t)//2] * 1e3 / 1e6:.3f} M tok/s", flush=True)
