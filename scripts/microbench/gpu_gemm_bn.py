"""N-tile A/B (BN 128 vs 256) on the step's weakest GEMM launches (run on the box)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402

dev, bf = "cuda", torch.bfloat16
T, d, r, f = 16384, 2048, 512, 5472


def mk(*s):
    return torch.randn(*s, device=dev, dtype=bf)


def timeit(probs, bn, reps=20):
    for _ in range(3):
        K.gemm(*probs, bn=bn)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.gemm(*probs, bn=bn)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


cases = {
    "dgrad_gu 2x[T x 512, K=5472] B MN": (lambda: [K.Gemm(mk(T, f), mk(f, r), torch.empty(T, r, device=dev, dtype=bf), b_mn=True) for _ in range(2)], 2 * 2 * T * r * f),
    "dgrad_o [T x 2048, K=512] B MN": (lambda: [K.Gemm(mk(T, r), mk(r, d), torch.empty(T, d, device=dev, dtype=bf), b_mn=True)], 2 * T * d * r),
    "down_o [T x 512, K=2048]": (lambda: [K.Gemm(mk(T, d), mk(r, d), torch.empty(T, r, device=dev, dtype=bf))], 2 * T * r * d),
    "dgrad_qkv 3x[T x 512, K=2048] B MN": (lambda: [K.Gemm(mk(T, d), mk(d, r), torch.empty(T, r, device=dev, dtype=bf), b_mn=True) for _ in range(3)], 3 * 2 * T * r * d),
    "down_d [T x 512, K=5472]": (lambda: [K.Gemm(mk(T, f), mk(r, f), torch.empty(T, r, device=dev, dtype=bf))], 2 * T * r * f),
}
for name, (mkc, fl) in cases.items():
    probs = mkc()
    line = []
    for bn in (0, 128, 256):
        us = timeit(probs, bn)
        line.append(f"bn={bn or 'auto'}: {us:6.1f} us {fl / us / 1e6:5.0f} TF/s")
    print(f"{name:38s} " + " | ".join(line))
