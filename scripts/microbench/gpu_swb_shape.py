"""Time / profile the fused SwiGLU-backward GEMM epilogue at the CoLA-1B shape (run on the box)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2512_12131_b200 import kernels as K

T, r, f = 16384, 512, 5472
dP = torch.randn(T, r, device="cuda").bfloat16()
Wd = torch.randn(r, f, device="cuda").bfloat16()
g = torch.randn(T, f, device="cuda").bfloat16()
u = torch.randn(T, f, device="cuda").bfloat16()
dg = torch.empty(T, f, device="cuda", dtype=torch.bfloat16)
du = torch.empty_like(dg)
dact = torch.empty_like(dg)
bn = int(sys.argv[1]) if len(sys.argv) > 1 else 0
def fused():
    K.gemm(K.Gemm(dP, Wd, dg, b_mn=True, swiglu_bwd=(g, u, du)), bn=bn)
def plain():
    K.gemm(K.Gemm(dP, Wd, dact, b_mn=True), bn=bn)
def resid():
    K.gemm(K.Gemm(dP, Wd, dact, b_mn=True, resid=g), bn=bn)
for name, fn in (("fused", fused), ("plain", plain), ("resid", resid)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    print(name, bn, f"{s.elapsed_time(e) / 10 * 1e3:.1f} us", flush=True)
