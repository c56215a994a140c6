"""Residual-epilogue layouts must agree BITWISE (same fp32 accumulation, one bf16 rounding of
acc + residual): modes 0/1/2/3 x store paths on step-like shapes (not a pytest module)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402

torch.manual_seed(0)
for M, N, Kd in [(64, 256, 64), (64, 256, 640), (4096, 256, 64), (1000, 640, 512), (16384, 512, 1024)]:
    A = torch.randn(M, Kd, device="cuda").bfloat16()
    B = (torch.randn(N, Kd, device="cuda") * 0.05).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    outs = {}
    for mode in (0, 1, 2, 3):
        for st in (0, 1):
            K.set_res4(mode)
            K.set_st_global(bool(st))
            C = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
            K.gemm(K.Gemm(A, B, C, resid=R))
            torch.cuda.synchronize()
            outs[(mode, st)] = C
    K.set_res4(3)
    K.set_st_global(False)
    ref = outs[(1, 0)]
    exact = (A.float() @ B.float().t() + R.float())
    for k, C in outs.items():
        diff = (C.float() != ref.float()).sum().item()
        nan = torch.isnan(C.float()).sum().item()
        err = ((C.float() - exact).norm() / exact.norm()).item()
        print(f"[{M}x{N} K={Kd}] mode={k[0]} st={k[1]}: differs from (1,0) in {diff} elements, nan={nan}, rel={err:.2e}")
