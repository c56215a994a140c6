"""Forward-kernel variants x exp2 split (btp_attn_tune keys 1 / 0): parity vs torch fp32 on a small
shape, then device time at the bench shape (CUDA events, median of 3 x 20 calls) beside cuDNN.
usage: python scripts/microbench/attn_fwd_variants.py [variants, e.g. 4,5] [poly list, e.g. 0,2,4]"""
import math
import sys

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

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


def check(b, s, h, hd, scale=1.0):
    w = h * hd
    g = torch.Generator(device="cuda").manual_seed(0)
    q, k, v = (torch.randn(b * s, w, device="cuda", generator=g).mul(scale).bfloat16() for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    view4 = lambda t: t.float().view(b, s, h, hd).transpose(1, 2)
    sc = view4(q) @ view4(k).transpose(-1, -2) / math.sqrt(hd)
    ref = torch.softmax(sc, -1) @ view4(v)
    ref_lse = torch.logsumexp(sc, -1) / math.log(2)
    eo = float((view4(o) - ref).norm() / ref.norm())
    el = float((lse - ref_lse).abs().max())
    return eo, el


def main():
    variants = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,5").split(",")]
    polys = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,2,4").split(",")]
    lib = _native.load()
    pv, pp = lib.btp_attn_tune(1, -1), lib.btp_attn_tune(0, -1)
    b, s, h, hd = 4, 4096, 32, 64
    w = h * hd
    q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
    o = torch.empty_like(q)
    lse = torch.empty(b, h, s, device="cuda")
    flops = 4 * b * h * s * s * hd
    for var in variants:
        for n in polys:
            lib.btp_attn_tune(1, var)
            lib.btp_attn_tune(0, n)
            errs = [check(2, 512, 4, 64), check(1, 1024, 2, 64, scale=3.0), check(1, 256, 3, 64)]
            t = timeit(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
            worst_o = max(e[0] for e in errs)
            worst_l = max(e[1] for e in errs)
            print(f"variant {var} poly {n}: {t*1e3:.1f} us ({flops/t/1e9:.0f} TF/s)  "
                  f"o rel err {worst_o:.2e}  lse abs err {worst_l:.2e}", flush=True)
    lib.btp_attn_tune(1, pv)
    lib.btp_attn_tune(0, pp)
    view4 = lambda t: t.view(b, s, h, hd).transpose(1, 2)
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        t_cud = timeit(lambda: F.scaled_dot_product_attention(view4(q), view4(k), view4(v), scale=1 / math.sqrt(hd)))
    print(f"cudnn: {t_cud*1e3:.1f} us ({flops/t_cud/1e9:.0f} TF/s)", flush=True)


if __name__ == "__main__":
    main()
