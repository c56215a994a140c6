"""Per-CTA timeline of the hd-64 attention backward (btp_attn_bwd_trace): every CTA stamps its SM id and
clock64 at start, last MMA issued, compute walk done, dQ reduce loop done, its last bulk reduce
completed, thread 0 past the final __syncthreads, and dK / dV stored. Per SM (one CTA resident at a
time) the CTAs are ordered by start: prints the distribution of each segment and of the gap between
one CTA's last stamp and the next CTA's start on the same SM."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_12131_b200 import _native  # noqa: E402

b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q)
lse = torch.empty(b, h, s, device="cuda")
D = torch.empty(b, h, s, device="cuda")
acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
from paper_2512_12131_b200 import kernels as K  # noqa: E402

K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
n_q = s // 128
n_cta = (s // 128) * h * b
tr = torch.zeros(n_q * 16 + 8 * n_cta, dtype=torch.int64, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    _native.call("btp_attn_bwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(do), w, P(lse), P(D), P(acc), w,
                 P(dq), w, P(dk), w, P(dv), w, b, s, h, hd, P(tr), st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_native.call("btp_attn_bwd_trace", P(q), w, P(k), w, P(v), w, P(o), w, P(do), w, P(lse), P(D), P(acc), w,
             P(dq), w, P(dk), w, P(dv), w, b, s, h, hd, P(tr), st)
e1.record()
torch.cuda.synchronize()
print(f"kernel+prep+convert: {e0.elapsed_time(e1) * 1e3:.1f} us")
c = tr[n_q * 16:].view(n_cta, 8).cpu().tolist()
by_sm = {}
for row in c:
    by_sm.setdefault(row[0], []).append(row[1:])
seg = {k: [] for k in ("start -> last MMA issued", "start -> compute walk done", "compute done -> dK/dV stored",
                       "compute done -> reduce loop done", "reduce loop done -> bulk reduce complete",
                       "thread 0 past sync - compute done", "CTA (start -> last stamp)", "gap last stamp -> next start")}
spans = []
for sm, lst in by_sm.items():
    lst.sort()
    prev_end = None
    for t0, t_mma, t_cmp, t_red, t_bulk, t_sync, t_dkv in lst:
        end = max(t_mma, t_cmp, t_red, t_bulk, t_sync, t_dkv)
        seg["start -> last MMA issued"].append(t_mma - t0)
        seg["start -> compute walk done"].append(t_cmp - t0)
        seg["compute done -> dK/dV stored"].append(t_dkv - t_cmp)
        seg["compute done -> reduce loop done"].append(t_red - t_cmp)
        seg["reduce loop done -> bulk reduce complete"].append(t_bulk - t_red)
        seg["thread 0 past sync - compute done"].append(t_sync - t_cmp)
        seg["CTA (start -> last stamp)"].append(end - t0)
        if prev_end is not None:
            seg["gap last stamp -> next start"].append(t0 - prev_end)
        prev_end = end
    spans.append(len(lst))


def q(xs, name):
    xs = sorted(xs)
    n = len(xs)
    print(f"{name:42s} n={n:5d} min {xs[0]:8d} p10 {xs[n // 10]:8d} median {xs[n // 2]:8d} p90 {xs[9 * n // 10]:8d} "
          f"max {xs[-1]:8d}")


for k_, v_ in seg.items():
    q(v_, k_)
print("CTAs per SM: min", min(spans), "max", max(spans), "SMs", len(spans))
