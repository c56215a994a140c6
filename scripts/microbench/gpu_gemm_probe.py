"""Ad-hoc GEMM probe (run on the GPU box): every layout / epilogue vs torch fp32."""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2512_12131_b200 import kernels as K

torch.manual_seed(0)
dev = "cuda"
def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()

def run(M, N, Kd, a_mn, b_mn, bn=0, out=torch.bfloat16, splits=1, rs=False, cs=False, res=False):
    A = torch.randn(M, Kd, device=dev).bfloat16()
    B = torch.randn(N, Kd, device=dev).bfloat16()
    a_arg = A.t().contiguous() if a_mn else A
    b_arg = B.t().contiguous() if b_mn else B
    ref = A.float() @ B.float().t()
    row = torch.rand(M, device=dev) + 0.5 if rs else None
    col = torch.rand(N, device=dev) + 0.5 if cs else None
    R = torch.randn(M, N, device=dev).bfloat16() if res else None
    if row is not None: ref = ref * row[:, None]
    if col is not None: ref = ref * col[None, :]
    if R is not None: ref = ref + R.float()
    if splits > 1:
        C = torch.empty(M, N, device=dev)
        K.zero(C)
        K.gemm(K.Gemm(a_arg, b_arg, C, a_mn=a_mn, b_mn=b_mn, row_scale=row, col_scale=col, splits=splits), bn=bn)
        Cs = C
    else:
        C = torch.zeros(M, N, device=dev, dtype=out)
        K.gemm(K.Gemm(a_arg, b_arg, C, a_mn=a_mn, b_mn=b_mn, row_scale=row, col_scale=col, resid=R), bn=bn)
        Cs = C
    torch.cuda.synchronize()
    e = rel(Cs, ref)
    print(f"M={M} N={N} K={Kd} a_mn={a_mn} b_mn={b_mn} bn={bn} out={out} splits={splits} rs={rs} cs={cs} res={res}: rel={e:.3e}", flush=True)
    return e

bad = 0
for (M, N, Kd) in [(128, 128, 64), (256, 256, 128), (296, 200, 72), (1024, 512, 512), (2048, 1536, 2048)]:
    for a_mn, b_mn in [(False, False), (False, True), (True, True), (True, False)]:
        for bn in (128, 192, 256):
            e = run(M, N, Kd, a_mn, b_mn, bn)
            bad += e > 1e-2
e = run(1000, 640, 512, False, False, 0, out=torch.float32, rs=True, cs=True); bad += e > 1e-2
e = run(1000, 640, 512, False, False, 0, res=True); bad += e > 1e-2
e = run(512, 2048, 4096, True, True, 0, splits=4); bad += e > 1e-2
# grouped launch
A = [torch.randn(2048, 512, device=dev).bfloat16() for _ in range(3)]
B = [torch.randn(768, 512, device=dev).bfloat16() for _ in range(3)]
C = [torch.empty(2048, 768, device=dev).bfloat16() for _ in range(3)]
K.gemm(*[K.Gemm(a, b, c) for a, b, c in zip(A, B, C)])
torch.cuda.synchronize()
for a, b, c in zip(A, B, C):
    e = rel(c, a.float() @ b.float().t()); print("grouped", e); bad += e > 1e-2
# mixed majors in one launch: a dgrad-like (K, MN) problem + a split-K wgrad-like (MN, MN) problem
dY = torch.randn(4096, 1024, device=dev).bfloat16()
W = torch.randn(1024, 512, device=dev).bfloat16()      # [K=1024, N=512] -> MN-major B
X = torch.randn(4096, 512, device=dev).bfloat16()
dA = torch.empty(4096, 512, device=dev).bfloat16()
dW = torch.empty(1024, 512, device=dev); K.zero(dW)
K.gemm(K.Gemm(dY, W, dA, b_mn=True), K.Gemm(dY, X, dW, a_mn=True, b_mn=True, splits=4))
torch.cuda.synchronize()
e1 = rel(dA, dY.float() @ W.float()); e2 = rel(dW, dY.float().t() @ X.float())
print("mixed-major dgrad", e1, "wgrad", e2); bad += (e1 > 1e-2) + (e2 > 1e-2)
# timing
for (M, N, Kd) in [(16384, 2048, 512), (16384, 1536, 2048), (8192, 8192, 8192)]:
    A = torch.randn(M, Kd, device=dev).bfloat16(); B = torch.randn(N, Kd, device=dev).bfloat16()
    C = torch.empty(M, N, device=dev).bfloat16()
    for _ in range(3): K.gemm(K.Gemm(A, B, C))
    torch.cuda.synchronize()
    s, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): K.gemm(K.Gemm(A, B, C))
    e_.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e_) / 20
    s.record()
    for _ in range(20): torch.matmul(A, B.t())
    e_.record(); torch.cuda.synchronize()
    ms_t = s.elapsed_time(e_) / 20
    print(f"timing {M}x{N}x{Kd}: btp {ms*1e3:.1f} us = {2*M*N*Kd/ms/1e9:.0f} TF/s ; torch {ms_t*1e3:.1f} us = {2*M*N*Kd/ms_t/1e9:.0f} TF/s")
print("BAD", bad)
