"""Pipeline timeline of the P-apart forward (variant 5): clock64 stamps of CTA 0 (btp_attn_fwd_trace)."""
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
lib = _native.load()
lib.btp_attn_tune(1, int(sys.argv[2]) if len(sys.argv) > 2 else 5)
if len(sys.argv) > 1:
    lib.btp_attn_tune(0, int(sys.argv[1]))
for _ in range(3):
    _native.call("btp_attn_fwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(lse), b, s, h, hd, P(tr),
                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
t = tr.cpu()
t0 = int(t[0, 12])  # CTA start
names = {0: "u0 S ready", 1: "u0 max done", 3: "u0 PV-1 done", 2: "u0 P done", 4: "u1 S ready", 5: "u1 max done",
         7: "u1 PV-1 done", 6: "u1 P done", 8: "mma P0 seen", 9: "mma S0+2", 10: "mma P1 seen", 11: "mma S1+2"}
order = [0, 1, 3, 2, 4, 5, 7, 6, 8, 9, 10, 11]
print("iter " + " ".join(f"{names[e][:12]:>12}" for e in order))
n = s // 128
for i in list(range(0, 6)) + list(range(n - 6, n)):
    print(f"{i:4d} " + " ".join(f"{(int(t[i, e]) - t0) if t[i, e] else 0:12d}" for e in order))
for u in (0, 1):
    per = [(int(t[i + 1, 4 * u + 2]) - int(t[i, 4 * u + 2])) for i in range(4, n - 2)]
    print(f"u{u}: clk per key tile (P done deltas): median {sorted(per)[len(per) // 2]}")
    seg = lambda a, b_: sorted(int(t[i, b_]) - int(t[i, a]) for i in range(4, n - 2))[(n - 6) // 2]
    print(f"   S ready->max {seg(4*u, 4*u+1)}  max->PV-1 wait done {seg(4*u+1, 4*u+3)}  ->P done {seg(4*u+3, 4*u+2)}")
    wait = sorted(int(t[i + 1, 4 * u]) - int(t[i, 4 * u + 2]) for i in range(4, n - 2))[(n - 6) // 2]
    print(f"   P done -> next S ready (softmax idle) {wait}")
print(f"CTA start 0, barriers+TMEM {int(t[0, 13]) - t0}, first S ready {int(t[0, 0]) - t0}, "
      f"last P done {int(t[n - 1, 6]) - t0}, epilogue stored {int(t[0, 14]) - t0}, CTA done {int(t[0, 15]) - t0}")
