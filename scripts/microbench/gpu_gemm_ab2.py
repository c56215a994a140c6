"""Split-K sweep for the step's multi-problem weight-gradient launches (run on the box)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402
from scripts.microbench.gpu_gemm_ab import flops, mk, timeit  # noqa: E402

T = 16384
for (M, N, n) in ((5472, 512, 2), (2048, 512, 3), (5472, 512, 1), (512, 5472, 1), (1024, 2048, 1), (512, 2048, 1)):
    pairs = [(mk(T, M), mk(T, N)) for _ in range(n)]
    line = []
    for sp in (1, 2, 3, 4, 5, 6, 8, 9, 12):
        outs = [torch.zeros(M, N, device="cuda") for _ in range(n)]
        probs = [K.Gemm(a, b, o, a_mn=True, b_mn=True, splits=sp) for (a, b), o in zip(pairs, outs)]
        us = timeit(probs)
        line.append(f"s{sp}:{us:6.1f}")
    print(f"{n}x[{M}x{N}]", " ".join(line))
