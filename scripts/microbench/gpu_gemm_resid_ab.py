"""A/B of the residual-epilogue GEMM layouts against the plain epilogue at the TP=8 / TP=1
up-projection shapes (not a pytest module):  python scripts/microbench/gpu_gemm_resid_ab.py
Residual modes (btp_gemm_set_res4): 0 per-chunk prefetch, 1 whole-tile staging, 2 pipelined
residual slots fed by a producer warp (pair tiles)."""
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


for M, N, Kd in [(16384, 512, 1024), (16384, 2048, 512), (16384, 1024, 512), (16384, 4096, 1024)]:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    w = torch.randn(N, Kd, device="cuda").bfloat16()
    r = torch.randn(M, N, device="cuda").bfloat16()
    o = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ref = (a.float() @ w.float().t() + r.float())
    fl = 2 * M * N * Kd
    K.set_pair_mode(2)
    for st in (0, 1):
        K.set_st_global(st)
        tp = t(lambda: K.gemm(K.Gemm(a, w, o)))
        res = {}
        for mode in (0, 1, 2, 3):
            K.set_res4(mode)
            res[mode] = t(lambda: K.gemm(K.Gemm(a, w, o, resid=r)))
            err = float((o.float() - ref).norm() / ref.norm())
            assert err < 1e-2, (mode, err)
        K.set_res4(3)
        print(f"[{M}x{N} K={Kd}] st_global={st} plain {tp:6.1f} us ({fl / tp / 1e6:5.0f} TF/s) | resid chunk "
              f"{res[0]:6.1f}  tile {res[1]:6.1f}  pipe {res[2]:6.1f}  auto {res[3]:6.1f} us "
              f"({fl / res[3] / 1e6:5.0f} TF/s)", flush=True)
    K.set_st_global(0)
