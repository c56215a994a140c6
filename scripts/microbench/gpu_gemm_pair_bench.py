"""Pair (cta_group::2) vs single-CTA tiles on the CoLA-1B step's GEMM shapes (run on the box)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2512_12131_b200 import kernels as K

dev = "cuda"
bf = torch.bfloat16
T, d, r, f = 16384, 2048, 512, 5472


def mk(*s):
    return torch.randn(*s, device=dev, dtype=bf)


cases = {
    "down_qkv  [T x 1536, K=2048]": lambda: [K.Gemm(mk(T, d), mk(3 * r, d), torch.empty(T, 3 * r, device=dev, dtype=bf))],
    "up_qkv  3x[T x 2048, K=512]": lambda: [K.Gemm(mk(T, r), mk(d, r), torch.empty(T, d, device=dev, dtype=bf)) for _ in range(3)],
    "down_o    [T x 512, K=2048]": lambda: [K.Gemm(mk(T, d), mk(r, d), torch.empty(T, r, device=dev, dtype=bf))],
    "up_gu   2x[T x 5472, K=512]": lambda: [K.Gemm(mk(T, r), mk(f, r), torch.empty(T, f, device=dev, dtype=bf)) for _ in range(2)],
    "down_d    [T x 512, K=5472]": lambda: [K.Gemm(mk(T, f), mk(r, f), torch.empty(T, r, device=dev, dtype=bf))],
    "dgrad dh  [T x 2048, K=1536] (B MN)": lambda: [K.Gemm(mk(T, 3 * r), mk(3 * r, d), torch.empty(T, d, device=dev, dtype=bf), b_mn=True)],
    "dgrad dact[T x 5472, K=512] (B MN)": lambda: [K.Gemm(mk(T, r), mk(r, f), torch.empty(T, f, device=dev, dtype=bf), b_mn=True)],
    "wgrad  [1536 x 2048, K=T] split3": lambda: [K.Gemm(mk(T, 3 * r), mk(T, d), torch.zeros(3 * r, d, device=dev), a_mn=True, b_mn=True, splits=3)],
    "wgrad 2x[5472 x 512, K=T] split4": lambda: [K.Gemm(mk(T, f), mk(T, r), torch.zeros(f, r, device=dev), a_mn=True, b_mn=True, splits=4) for _ in range(2)],
    "up_o +resid [T x 2048, K=512]": lambda: [K.Gemm(mk(T, r), mk(d, r), torch.empty(T, d, device=dev, dtype=bf), resid=mk(T, d))],
}
for name, mkcase in cases.items():
    probs = mkcase()
    fl = 0
    for p in probs:
        M = p.a.shape[1] if p.a_mn else p.a.shape[0]
        Kd = p.a.shape[0] if p.a_mn else p.a.shape[1]
        N = p.b.shape[1] if p.b_mn else p.b.shape[0]
        fl += 2 * M * N * Kd
    res = []
    for pair in (False, True):
        K.set_pair_mode(pair)
        for _ in range(3):
            K.gemm(*probs)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            K.gemm(*probs)
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / 20 * 1e3
        res.append(f"{'pair' if pair else 'single'} {us:7.1f} us {fl / us / 1e6:6.0f} TF/s")
    print(f"{name:38s} " + " | ".join(res), flush=True)
K.set_pair_mode(True)
