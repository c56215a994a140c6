"""Own tcgen05 attention vs torch SDPA (cuDNN) on the bench shapes, same [T, h*hd] strided layout.
Prints per-call device time (CUDA events, median of 3 x 20 back-to-back calls) and TFLOP/s."""
import math
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

sys.path.insert(0, ".")
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


def main():
    shapes = [(4, 4096, 32, 64), (4, 4096, 4, 128), (4, 4096, 16, 64), (1, 8192, 8, 128)]
    for b, s, h, hd in shapes:
        w = h * hd
        q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
        o = torch.empty_like(q)
        lse = torch.empty(b, h, s, device="cuda")
        flops = 4 * b * h * s * s * hd
        t_own = timeit(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
        v4 = lambda t: t.view(b, s, h, hd).transpose(1, 2)
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            t_cud = timeit(lambda: F.scaled_dot_product_attention(v4(q), v4(k), v4(v), scale=1 / math.sqrt(hd)))
            ref = F.scaled_dot_product_attention(v4(q), v4(k), v4(v), scale=1 / math.sqrt(hd))
        err = float((o.float() - ref.transpose(1, 2).reshape(b * s, w).float()).norm() / ref.float().norm())
        print(f"b{b} s{s} h{h} hd{hd}: own fwd {t_own*1e3:.1f} us ({flops/t_own/1e9:.0f} TF/s)  "
              f"cudnn fwd {t_cud*1e3:.1f} us ({flops/t_cud/1e9:.0f} TF/s)  rel err vs cudnn {err:.2e}", flush=True)


if __name__ == "__main__":
    main()
