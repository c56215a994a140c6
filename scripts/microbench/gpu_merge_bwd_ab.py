"""In-process A/B: backward dgrad + weight-gradient GEMMs merged into one launch per chunk (default)
vs separate launches. Two graph-captured BlockTrainers on the bench step (CoLA-1B b4 s4096 TP=1),
replays alternating in rounds of 10 steps (CUDA events), median over rounds."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import executor as E  # noqa: E402
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
trainers = {}
for mode in ("merged", "split"):
    E.ExecutorBase.merge_bwd_gemms = mode == "merged"
    tr = BlockTrainer(pl, blk, adamw=dict(lr=1e-4, b1=0.9, b2=0.95, eps=1e-8, wd=0.1))
    xd, gd = tr.device_inputs(x, G)
    for _ in range(3):  # warm-up + graph capture with this mode
        tr.step_device(xd, gd)
    torch.cuda.synchronize()
    trainers[mode] = (tr, xd, gd)
times = {m: [] for m in trainers}
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    for mode in (("merged", "split") if r % 2 == 0 else ("split", "merged")):
        tr, xd, gd = trainers[mode]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            tr.step_device(xd, gd)
        e1.record()
        torch.cuda.synchronize()
        times[mode].append(e0.elapsed_time(e1) / 10)
for mode, t in times.items():
    t = sorted(t)
    print(f"{mode}: median {t[len(t)//2]:.4f} ms/step, min {t[0]:.4f}, max {t[-1]:.4f} over {len(t)} rounds", flush=True)
