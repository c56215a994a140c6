"""Why do the step's GEMMs take longer back to back (67.7 us / launch) than in ncu's isolated
replay (59.7 us at a LOWER clock)? Probe (not a pytest module):  python scripts/microbench/gpu_gemm_power_probe.py

(a) the step's 24 GEMM launches as one graph, replayed hot back to back;
(b) the same graph replayed once after the GPU idled 0.5 s (cool);
(c) every GEMM followed by a ~20 us spin kernel (per-GEMM events): launch gaps and power both relax;
(d) every GEMM bracketed by events with no spin (the bench's per-launch timing)."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402
from paper_2512_12131_b200.api import BlockTrainer  # noqa: E402
from paper_2512_12131_b200.model import RunShape, Variant, build_block, fan_in_scaled, preset  # noqa: E402
from paper_2512_12131_b200.plan import Strategy, plan  # noqa: E402
from paper_2512_12131_b200.tensor import seeded_fill  # noqa: E402

cfg = preset("1b")
b, s = 4, 4096
pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
tr = BlockTrainer(pl, fan_in_scaled(build_block(cfg, Variant.COLA, 0)), optimizer=False)
x, g = tr.device_inputs(seeded_fill((b, s, cfg.d), 10000).values, seeded_fill((b, s, cfg.d), 30000).values)
tr.step_device(x, g)
tr.ex.gemm_log = []
tr._eager(x, g)
log, tr.ex.gemm_log = tr.ex.gemm_log, None
torch.cuda.synchronize()
fl = sum(f for _, f in log)


def capture(fn):
    gph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(gph, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    gph.replay()
    torch.cuda.synchronize()
    return gph


def seq():
    for probs, _ in log:
        K.gemm(*probs)


evs = []


def seq_ev(spin):
    evs.clear()
    for probs, _ in log:
        e0 = torch.cuda.Event(enable_timing=True, external=True)
        e1 = torch.cuda.Event(enable_timing=True, external=True)
        e0.record()
        K.gemm(*probs)
        e1.record()
        evs.append((e0, e1))
        if spin:
            torch.cuda._sleep(spin)


def timed(gph, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


g_seq = capture(seq)
hot = timed(g_seq, 20)
time.sleep(0.5)
cool = timed(g_seq, 1)
hot2 = timed(g_seq, 20)
print(f"(a) hot  back-to-back: {hot * 1e3:7.1f} us / step-of-GEMMs = {hot * 1e3 / len(log):5.1f} us/launch, {fl / hot / 1e9:6.0f} TF/s")
print(f"(b) cool single replay: {cool * 1e3:7.1f} us ({cool * 1e3 / len(log):5.1f} us/launch); hot again {hot2 * 1e3:7.1f}")
for spin in (0, 40000):
    gph = capture(lambda: seq_ev(spin))
    for _ in range(3):
        gph.replay()
    torch.cuda.synchronize()
    per = [a.elapsed_time(b_) * 1e3 for a, b_ in evs]
    tot = timed(gph, 5)
    per = [a.elapsed_time(b_) * 1e3 for a, b_ in evs]
    print(f"({'c' if spin else 'd'}) per-GEMM events, spin={spin}: sum {sum(per):7.1f} us ({sum(per) / len(per):5.1f}/launch, "
          f"{fl / sum(per) / 1e6:6.0f} TF/s); graph total {tot * 1e3:7.1f} us")
print("per-launch (spin) us:", " ".join(f"{v:.1f}" for v in per))
