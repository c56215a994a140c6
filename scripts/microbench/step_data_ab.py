"""Same step, two data sets: the bench's trainer (fan-in-scaled seeded weights, seeded_fill inputs)
vs unscaled build_block weights with standard-normal inputs — graph replays interleaved in one
process (10 steps per sample, 10 rounds), SM clock and power from NVML per sample. Checks whether
the data (bit toggling -> power -> clock under the power cap) moves the step time."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200.api import BlockTrainer  # noqa: E402
from paper_2512_12131_b200.model import PRESETS, RunShape, Variant, build_block, fan_in_scaled  # noqa: E402
from paper_2512_12131_b200.plan import Strategy, plan  # noqa: E402
from paper_2512_12131_b200.tensor import seeded_fill  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
cfg = PRESETS["1b"]
b, s = 4, 4096
pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
ADAMW = {"lr": 1e-4, "b1": 0.9, "b2": 0.95, "eps": 1e-8, "wd": 0.1}
sets = {}
blk = fan_in_scaled(build_block(cfg, Variant.COLA, 0))
sets["bench"] = (blk, seeded_fill((b, s, cfg.d), 10000).values, seeded_fill((b, s, cfg.d), 30000).values)
rng = np.random.default_rng(0)
sets["normal"] = (build_block(cfg, Variant.COLA, 0), rng.standard_normal((b, s, cfg.d)).astype(np.float32),
                  rng.standard_normal((b, s, cfg.d)).astype(np.float32) / 100)
for k, (bl, x, G) in sets.items():
    print(k, "x absmean", float(np.abs(x).mean()), "G absmean", float(np.abs(G).mean()), flush=True)
tr = {}
for k, (bl, x, G) in sets.items():
    t = BlockTrainer(pl, bl, adamw=ADAMW)
    xd, gd = t.device_inputs(x, G)
    for _ in range(3):
        t.step_device(xd, gd)
    tr[k] = (t, xd, gd)
torch.cuda.synchronize()
times = {k: [] for k in tr}
for r in range(10):
    for k in (list(tr) if r % 2 == 0 else list(tr)[::-1]):
        t, xd, gd = tr[k]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            t.step_device(xd, gd)
        e1.record()
        torch.cuda.synchronize()
        times[k].append(e0.elapsed_time(e1) / 10)
        sm = pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM)
        pw = pynvml.nvmlDeviceGetPowerUsage(hdl) // 1000
        print(f"round {r} {k:6s} {times[k][-1]:.3f} ms/step  sm {sm} MHz  {pw} W", flush=True)
for k in tr:
    v = sorted(times[k])
    print(f"{k}: median {v[len(v) // 2]:.3f} ms/step, min {v[0]:.3f}, max {v[-1]:.3f}")
