"""MMA-warp timeline of the split-role backward in handshake-only mode (dry=1): where the issuing
warp spends each query-tile iteration when no compute is on the critical path."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import _native  # noqa: E402
from paper_2512_12131_b200 import kernels as K  # noqa: E402

lib = _native.load()
b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q); lse = torch.empty(b, h, s, device="cuda")
D = torch.empty(b, h, s, device="cuda"); acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
P = lambda t: ctypes.c_void_p(t.data_ptr())
pv = lib.btp_attn_tune(3, 1)
for dry in (1, 0):
    lib.btp_attn_tune(4, dry)
    tr = torch.zeros(s // 128, 16, dtype=torch.int64, device="cuda")
    for _ in range(2):
        _native.call("btp_attn_bwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(do), w, P(lse), P(D), P(acc), w,
                     P(dq), w, P(dk), w, P(dv), w, b, s, h, hd, P(tr), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    t = tr.cpu()
    print(f"dry={dry}: per-iteration MMA-warp segments (cycles): at-P -> P seen | -> dP read | -> dS seen | -> dq free | -> next at-P")
    for i in range(8, 14):
        a = [int(t[i, e]) for e in (7, 8, 9, 10, 11)] + [int(t[i + 1, 7])]
        print(f"  iter {i}: " + " ".join(f"{a[j + 1] - a[j]:6d}" for j in range(5)) + f"   total {a[5] - a[0]}")
lib.btp_attn_tune(4, 0)
lib.btp_attn_tune(3, pv)
