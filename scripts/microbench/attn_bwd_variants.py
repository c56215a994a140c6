"""Backward A/B over one btp_attn_tune knob (key, values): parity of dq / dk / dv against torch fp32
autograd on a small shape, then device time at the bench shape (b4 s4096 h32 hd64; CUDA events,
median of 3 x 20 calls), values alternating. usage: attn_bwd_variants.py KEY v1,v2,... [rounds]"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import _native  # noqa: E402
from paper_2512_12131_b200 import kernels as K  # noqa: E402


def timeit(fn, n=20):
    fn()
    torch.cuda.synchronize()
    res = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / n)
    return sorted(res)[1]


def bufs(b, s, h, hd, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = h * hd
    q, k, v, do = (torch.randn(b * s, w, device="cuda", generator=g).bfloat16() for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(b, h, s, device="cuda")
    D = torch.empty(b, h, s, device="cuda")
    acc = torch.empty(b * s, w, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    return q, k, v, do, o, lse, D, acc, dq, dk, dv


def check(b, s, h, hd):
    q, k, v, do, o, lse, D, acc, dq, dk, dv = bufs(b, s, h, hd, seed=s + h)
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
    v4 = lambda t: t.float().view(b, s, h, hd).transpose(1, 2).requires_grad_(True)
    Q, Kk, V = v4(q), v4(k), v4(v)
    out = torch.softmax(Q @ Kk.transpose(-1, -2) / math.sqrt(hd), -1) @ V
    out.backward(v4(do).detach())
    back = lambda t: t.transpose(1, 2).reshape(b * s, h * hd)
    rel = lambda a, r: float((a.float() - r).norm() / r.norm())
    return max(rel(dq, back(Q.grad)), rel(dk, back(Kk.grad)), rel(dv, back(V.grad)))


def main():
    key = int(sys.argv[1])
    vals = [int(x) for x in sys.argv[2].split(",")]
    rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    lib = _native.load()
    prev = lib.btp_attn_tune(key, -1)
    b, s, h, hd = 4, 4096, 32, 64
    q, k, v, do, o, lse, D, acc, dq, dk, dv = bufs(b, s, h, hd)
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    flops = 2.5 * 4 * b * h * s * s * hd
    for val in vals:
        lib.btp_attn_tune(key, val)
        err = max(check(2, 512, 2, 64), check(1, 1024, 3, 64), check(2, 256, 5, 64))
        print(f"key {key} = {val}: worst rel err {err:.2e}", flush=True)
    try:
        import pynvml

        pynvml.nvmlInit()
        hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
        clk = lambda: (pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                       pynvml.nvmlDeviceGetPowerUsage(hdl) // 1000)
    except Exception:  # noqa: BLE001
        clk = lambda: (0, 0)
    times = {v_: [] for v_ in vals}
    fn = lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
    for r in range(rounds):  # fine-grained alternation: the box drifts by ~10 % under sustained load
        for val in (vals if r % 2 == 0 else vals[::-1]):
            lib.btp_attn_tune(key, val)
            fn()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            times[val].append(e0.elapsed_time(e1) / 10)
            if r % 4 == 0:
                sm, pw = clk()
                print(f"  round {r} key {key} = {val}: {times[val][-1]*1e3:.1f} us  sm {sm} MHz  {pw} W", flush=True)
    for val in vals:
        t = sorted(times[val])
        print(f"key {key} = {val}: median {t[len(t)//2]*1e3:.1f} us ({flops/t[len(t)//2]/1e9:.0f} TF/s), "
              f"min {t[0]*1e3:.1f}, max {t[-1]*1e3:.1f} over {len(t)}", flush=True)
    lib.btp_attn_tune(key, prev)


if __name__ == "__main__":
    main()
