"""Attention forward at the bench shape: each split-row variant full vs handshake-only (wrong results)."""
import sys
import torch
sys.path.insert(0, ".")
from scripts.microbench.gpu_attn_bench import timeit  # noqa: E402
from paper_2512_12131_b200 import _native, kernels as K  # noqa: E402
lib = _native.load()
b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
o = torch.empty_like(q); lse = torch.empty(b, h, s, device="cuda")
pv = lib.btp_attn_tune(1, -1)
for var in (1, 3, 4):
    lib.btp_attn_tune(1, var)
    for dry in (0, 1):
        lib.btp_attn_tune(6, dry)
        t = timeit(lambda: K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd))
        print(f"fwd variant {var} dry={dry}: {t*1e3:.1f} us", flush=True)
lib.btp_attn_tune(6, 0)
lib.btp_attn_tune(1, pv)
