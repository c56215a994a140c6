"""A/B of the residual-epilogue GEMM against the plain one at the TP=8 / TP=1 up-projection
shapes (not a pytest module):  python tests/gpu_gemm_resid_ab.py"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402


def t(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for M, N, Kd in [(16384, 512, 1024), (16384, 2048, 512), (16384, 1024, 512)]:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = torch.randn(N, Kd, device="cuda").bfloat16()
    r = torch.randn(M, N, device="cuda").bfloat16()
    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * Kd
    for pair in (1, 2):
        K.set_pair_mode(pair)
        for bn in (0, 256):
            tp = t(lambda: K.gemm(K.Gemm(a, w, o), bn=bn))
            K.set_res4(False)
            tr0 = t(lambda: K.gemm(K.Gemm(a, w, o, resid=r), bn=bn))
            K.set_res4(True)
            tr = t(lambda: K.gemm(K.Gemm(a, w, o, resid=r), bn=bn))
            print(f"[{M}x{N} K={Kd}] pair={pair} bn={bn or 'auto'}: plain {tp:6.1f} us ({fl / tp / 1e6:5.0f} TF/s)"
                  f"  resid/chunk {tr0:6.1f} us  resid/tile {tr:6.1f} us ({fl / tr / 1e6:5.0f} TF/s)")
    K.set_pair_mode(1)
