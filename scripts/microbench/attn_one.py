"""One forward + one backward of the own attention kernels at a bench shape (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import kernels as K  # noqa: E402

b, s, h, hd = (int(x) for x in (sys.argv[1:5] if len(sys.argv) >= 5 else (4, 4096, 32, 64)))
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(b, h, s, device="cuda")
D = torch.empty(b, h, s, device="cuda")
acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
import os
from paper_2512_12131_b200 import _native  # noqa: E402
if os.environ.get("FWD_VARIANT"):
    _native.load().btp_attn_tune(1, int(os.environ["FWD_VARIANT"]))
for _ in range(2):
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
torch.cuda.synchronize()
print("ok")
