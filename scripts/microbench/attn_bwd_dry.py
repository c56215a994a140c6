"""Split-role hd-64 backward at the bench shape: full kernel vs diagnostic variants (wrong results):
dry 1 = handshakes only; diag bits: 1 no dS st.shared, 2 no proxy fence, 4 no lse/D shared loads."""
import sys
import torch
sys.path.insert(0, ".")
from scripts.microbench.gpu_attn_bench import timeit  # noqa: E402
from paper_2512_12131_b200 import _native, kernels as K  # noqa: E402
lib = _native.load()
b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q); lse = torch.empty(b, h, s, device="cuda")
K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
D = torch.empty(b, h, s, device="cuda"); acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
prev_variant = lib.btp_attn_tune(3, 1)  # the split-role kernel carries the diagnostic modes
cases = [(0, 0), (1, 0), (0, 1), (0, 2), (0, 3), (0, 4), (0, 7), (0, 0)]
for dry, diag in cases:
    lib.btp_attn_tune(4, dry)
    lib.btp_attn_tune(5, diag)
    t = timeit(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
    print(f"split-role bwd dry={dry} diag={diag}: {t*1e3:.1f} us", flush=True)
lib.btp_attn_tune(4, 0)
lib.btp_attn_tune(5, 0)
lib.btp_attn_tune(3, prev_variant)
lib.btp_attn_tune(3, 0)
t0 = timeit(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
print(f"default (shared-warp) bwd kernel: {t0*1e3:.1f} us")
