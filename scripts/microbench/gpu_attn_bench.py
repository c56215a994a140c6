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


def poly_sweep():
    from paper_2512_12131_b200 import _native
    lib = _native.load()
    b, s, h, hd = 4, 4096, 32, 64
    w = h * hd
    q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(b, h, s, device="cuda")
    flops = 4 * b * h * s * s * hd
    for var in (0, 4):
        lib.btp_attn_tune(1, var)
        for n in (0, 2):
            lib.btp_attn_tune(0, n)
            t_own = timeit(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
            print(f"  fwd variant {var} poly every {n}: {t_own*1e3:.1f} us ({flops/t_own/1e9:.0f} TF/s)", flush=True)
    lib.btp_attn_tune(0, 0)
    lib.btp_attn_tune(1, 0)
    do = torch.randn(b * s, w, device="cuda").bfloat16()
    D = torch.empty(b, h, s, device="cuda")
    acc = torch.empty(b * s, w, device="cuda")
    dq, dk, dv = (torch.empty_like(q) for _ in range(3))
    prev = lib.btp_attn_tune(3, -1)
    for var in (0, 1, 0, 1):
        lib.btp_attn_tune(3, var)
        t_b = timeit(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
        print(f"  bwd variant {var}: {t_b*1e3:.1f} us ({2.5*flops/t_b/1e9:.0f} TF/s)", flush=True)
    lib.btp_attn_tune(3, prev)


def main():
    poly_sweep()
    shapes = [(4, 4096, 32, 64), (4, 4096, 4, 128), (4, 4096, 16, 64), (1, 8192, 8, 128)]
    for b, s, h, hd in shapes:
        w = h * hd
        q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
        o = torch.empty_like(q)
        lse = torch.empty(b, h, s, device="cuda")
        flops = 4 * b * h * s * s * hd
        t_own = timeit(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
        view4 = lambda t: t.view(b, s, h, hd).transpose(1, 2)
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            t_cud = timeit(lambda: F.scaled_dot_product_attention(view4(q), view4(k), view4(v), scale=1 / math.sqrt(hd)))
            ref = F.scaled_dot_product_attention(view4(q), view4(k), view4(v), scale=1 / math.sqrt(hd))
        err = float((o.float() - ref.transpose(1, 2).reshape(b * s, w).float()).norm() / ref.float().norm())
        print(f"b{b} s{s} h{h} hd{hd}: own fwd {t_own*1e3:.1f} us ({flops/t_own/1e9:.0f} TF/s)  "
              f"cudnn fwd {t_cud*1e3:.1f} us ({flops/t_cud/1e9:.0f} TF/s)  rel err vs cudnn {err:.2e}", flush=True)
        # backward: 2.5x the forward FLOPs (5 GEMMs)
        do = torch.randn(b * s, w, device="cuda").bfloat16()
        D = torch.empty(b, h, s, device="cuda")
        acc = torch.empty(b * s, w, device="cuda")
        dq, dk, dv = (torch.empty_like(q) for _ in range(3))
        t_ob = timeit(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
        q4, k4, v4 = (view4(t).detach().requires_grad_() for t in (q, k, v))
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            out = F.scaled_dot_product_attention(q4, k4, v4, scale=1 / math.sqrt(hd))
            t_cb = timeit(lambda: torch.autograd.grad(out, (q4, k4, v4), view4(do), retain_graph=True))
            gq, gk, gv = torch.autograd.grad(out, (q4, k4, v4), view4(do), retain_graph=True)
        e = [float((a.float() - g_.transpose(1, 2).reshape(b * s, w).float()).norm() / g_.float().norm())
             for a, g_ in ((dq, gq), (dk, gk), (dv, gv))]
        bfl = 2.5 * flops
        print(f"    own bwd {t_ob*1e3:.1f} us ({bfl/t_ob/1e9:.0f} TF/s)  cudnn bwd {t_cb*1e3:.1f} us ({bfl/t_cb/1e9:.0f} TF/s)"
              f"  rel err dq/dk/dv vs cudnn {e[0]:.2e}/{e[1]:.2e}/{e[2]:.2e}", flush=True)


if __name__ == "__main__":
    main()
