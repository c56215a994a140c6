"""In-process A/B of the merged-launch split-K policy: "behind" (executor._pick_splits_behind, the
round-robin makespan model with the dgrad tiles ahead) vs "plain" (_pick_splits on the weight-gradient
tiles alone, as if launched separately). One graph-captured BlockTrainer per policy on the bench step,
replays alternating in rounds of 10 steps, median over rounds; prints the split counts chosen."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import executor as E  # noqa: E402
from paper_2512_12131_b200.api import BlockTrainer  # noqa: E402
from paper_2512_12131_b200.model import RunShape, Variant, build_block, fan_in_scaled, preset  # noqa: E402
from paper_2512_12131_b200.plan import Strategy, plan  # noqa: E402
from paper_2512_12131_b200.tensor import seeded_fill  # noqa: E402

vals = sys.argv[1].split(",")
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = preset("1b")
b, s = 4, 4096
blk = fan_in_scaled(build_block(cfg, Variant.COLA, 0))
pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
x = seeded_fill((b, s, cfg.d), 10000).values
G = seeded_fill((b, s, cfg.d), 30000).values
orig = E._pick_splits_behind
trainers = {}
for v in vals:
    chosen = []
    pol = orig if v == "behind" else (lambda ahead, w, kb, units: E._pick_splits(w, kb, units))
    E._pick_splits_behind = lambda *a, _o=pol, _c=chosen: (_c.append(_o(*a)) or _c[-1])
    tr = BlockTrainer(pl, blk, adamw=dict(lr=1e-4, b1=0.9, b2=0.95, eps=1e-8, wd=0.1))
    xd, gd = tr.device_inputs(x, G)
    for _ in range(3):
        tr.step_device(xd, gd)
    torch.cuda.synchronize()
    E._pick_splits_behind = orig
    print(f"policy {v}: splits chosen {chosen[:9]}", flush=True)
    trainers[v] = (tr, xd, gd)
times = {v: [] for v in vals}
for r in range(rounds):
    for v in (vals if r % 2 == 0 else vals[::-1]):
        tr, xd, gd = trainers[v]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            tr.step_device(xd, gd)
        e1.record()
        torch.cuda.synchronize()
        times[v].append(e0.elapsed_time(e1) / 10)
for v, t in times.items():
    t = sorted(t)
    print(f"policy {v}: median {t[len(t)//2]:.4f} ms/step, min {t[0]:.4f}, max {t[-1]:.4f}", flush=True)
