"""Probe (run on the box): the TP=1 down-projection qkv GEMM [16384 x 1536, K=2048] with the
plain epilogue vs the fused sigma epilogue, CUDA-event timed; `ncu` target with argv[1]."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402

T, d, r = 16384, 2048, 512
bf = torch.bfloat16
n = torch.randn(T, d, device="cuda", dtype=bf)
W = torch.randn(3 * r, d, device="cuda", dtype=bf) * 0.02
P = torch.empty(T, 3 * r, device="cuda", dtype=bf)
A = torch.empty(T, 3 * r, device="cuda", dtype=bf)
which = sys.argv[1] if len(sys.argv) > 1 else "both"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def run(mode, bn=0):
    if mode == "plain":
        K.gemm(K.Gemm(n, W, P), bn=bn)
    else:
        K.gemm(K.Gemm(n, W, P, sigma=(A, r // 2)), bn=bn)


for mode in (["plain", "sigma"] if which == "both" else [which]):
    for bn in (0, 128):
        for _ in range(3):
            run(mode, bn)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run(mode, bn)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        print(f"{mode} bn={bn}: {us:.1f} us  {2 * T * 3 * r * d / us / 1e6:.0f} TF/s", flush=True)
