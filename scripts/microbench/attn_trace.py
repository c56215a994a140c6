"""Pipeline timeline of the attention backward kernel (clock64 stamps of CTA 0, btp_attn_bwd_trace)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import _native  # noqa: E402
from paper_2512_12131_b200 import kernels as K  # noqa: E402

b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(b, h, s, device="cuda")
D = torch.empty(b, h, s, device="cuda")
acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
tr = torch.zeros(s // 128, 16, dtype=torch.int64, device="cuda")
K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
P = lambda t: ctypes.c_void_p(t.data_ptr())
for _ in range(3):
    _native.call("btp_attn_bwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(do), w, P(lse), P(D), P(acc), w,
                 P(dq), w, P(dk), w, P(dv), w, b, s, h, hd, P(tr), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
t = tr.cpu()
t0 = int(t[t > 0].min())
from paper_2512_12131_b200 import _native as N2  # noqa: E402
if N2.load().btp_attn_tune(3, -1) == 1:  # split-role kernel
    names = {0: "P0 S seen", 2: "P0 P done", 4: "dS dP,P seen", 6: "dS ld0", 14: "dS c0 done", 12: "dS ld1",
             15: "dS c1 done", 5: "dS done", 8: "mma P seen", 10: "mma dS seen", 11: "mma dq free", 13: "red dQ"}
else:
    names = {0: "g0 S ready", 1: "g0 P done", 2: "g0 dP ready", 3: "g0 dS done", 4: "g1 S ready", 5: "g1 P done",
             6: "g1 dP ready", 7: "g1 dS done", 8: "mma P seen", 9: "mma [3][1] issued", 10: "mma dS seen",
             11: "mma dq free", 12: "mma [2] issued", 13: "red dQ ready", 14: "g0 S in regs", 15: "g0 P computed"}
print("iter " + " ".join(f"{names[e][:12]:>12}" for e in sorted(names)))
for i in range(t.shape[0]):
    print(f"{i:4d} " + " ".join(f"{(int(t[i, e]) - t0) if t[i, e] else 0:12d}" for e in sorted(names)))
per = [(int(t[i + 1, 8]) - int(t[i, 8])) for i in range(4, t.shape[0] - 2)]
print("clk per query tile (mma P seen deltas):", sorted(per)[len(per) // 2])
