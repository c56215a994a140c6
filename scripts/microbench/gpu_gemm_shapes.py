"""GEMM shapes of the CoLA-1B BTP step (TP=1) for ncu --set full captures (run on the box)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2512_12131_b200 import kernels as K

T, d, r, f = 16384, 2048, 512, 5472
dev = "cuda"
bf = torch.bfloat16
a = torch.randn(T, r, device=dev, dtype=bf)
W_up = torch.randn(d, r, device=dev, dtype=bf)
out = torch.empty(T, d, device=dev, dtype=bf)
n = torch.randn(T, d, device=dev, dtype=bf)
W_dn = torch.randn(3 * r, d, device=dev, dtype=bf)
P = torch.empty(T, 3 * r, device=dev, dtype=bf)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for _ in range(3):
    if which in ("all", "up"):
        K.gemm(K.Gemm(a, W_up, out))                   # up-projection [16384x2048], K=512
    if which in ("all", "down"):
        K.gemm(K.Gemm(n, W_dn, P))                     # grouped down qkv [16384x1536], K=2048
torch.cuda.synchronize()
print("done")
