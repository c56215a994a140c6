import sys, torch
sys.path.insert(0, ".")
from scripts.microbench.gpu_attn_bench import timeit
from paper_2512_12131_b200 import kernels as K
b, s, h, hd = 4, 4096, 32, 64
w = h * hd
q, k, v, do = (torch.randn(b * s, w, device="cuda").bfloat16() for _ in range(4))
o = torch.empty_like(q); lse = torch.empty(b, h, s, device="cuda")
K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
D = torch.empty(b, h, s, device="cuda"); acc = torch.empty(b * s, w, device="cuda")
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
for _ in range(3):
    t = timeit(lambda: K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd))
    print(f"bwd {t*1e3:.1f} us", flush=True)
