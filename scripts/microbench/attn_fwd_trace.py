"""Pipeline timeline of the split-row attention forward (clock64 stamps of CTA 0, btp_attn_fwd_trace)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import _native  # noqa: E402

b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty(b, h, s, device="cuda")
tr = torch.zeros(s // 128, 16, dtype=torch.int64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
_native.load().btp_attn_tune(1, 1)  # the stamps live in the split-row kernel
for _ in range(3):
    _native.call("btp_attn_fwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(lse), b, s, h, hd, P(tr),
                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
t = tr.cpu()
t0 = int(t[t > 0].min())
names = {0: "g0 S ready", 1: "g0 max done", 2: "g0 P done", 4: "g1 S ready", 5: "g1 max done", 6: "g1 P done",
         8: "mma P seen", 9: "mma PV issued", 10: "mma S+2 issued"}
print("iter " + " ".join(f"{names[e][:13]:>13}" for e in sorted(names)))
for i in list(range(0, 4)) + list(range(12, 16)):
    print(f"{i:4d} " + " ".join(f"{(int(t[i, e]) - t0) if t[i, e] else 0:13d}" for e in sorted(names)))
per = [(int(t[i + 1, 2]) - int(t[i, 2])) for i in range(4, t.shape[0] - 2)]
print("clk per key tile (g0 P done deltas):", sorted(per)[len(per) // 2])
