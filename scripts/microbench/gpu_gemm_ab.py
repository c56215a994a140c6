"""A/B timings of GEMM configurations on the CoLA-1B step's weakest shapes (run on the box):
residual up-projections single-CTA vs CTA-pair, and weight-gradient split-K counts."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402

dev, bf = "cuda", torch.bfloat16
T, d, r, f = 16384, 2048, 512, 5472


def mk(*s):
    return torch.randn(*s, device=dev, dtype=bf)


def timeit(probs, reps=20):
    for _ in range(3):
        K.gemm(*probs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        K.gemm(*probs)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def flops(probs):
    tot = 0
    for p in probs:
        M = p.a.shape[1] if p.a_mn else p.a.shape[0]
        Kd = p.a.shape[0] if p.a_mn else p.a.shape[1]
        N = p.b.shape[1] if p.b_mn else p.b.shape[0]
        tot += 2 * M * N * Kd
    return tot



def main():
    res_case = [K.Gemm(mk(T, r), mk(d, r), torch.empty(T, d, device=dev, dtype=bf), resid=mk(T, d))]
    for mode in (1, 2, 0):
        K.set_pair_mode(mode)
        us = timeit(res_case)
        print(f"up_o+resid [T x 2048, K=512] pair_mode={mode}: {us:7.1f} us  {flops(res_case) / us / 1e6:6.0f} TF/s")
    K.set_pair_mode(1)
    for (M, N) in ((1024, 2048), (512, 2048), (2048, 512), (1536, 2048), (f, r)):
        a, b = mk(T, M), mk(T, N)
        for sp in (2, 3, 4, 6, 8, 9, 12, 16):
            out = torch.zeros(M, N, device=dev)
            probs = [K.Gemm(a, b, out, a_mn=True, b_mn=True, splits=sp)]
            us = timeit(probs)
            print(f"wgrad [{M} x {N}, K=T] splits={sp:2d}: {us:7.1f} us  {flops(probs) / us / 1e6:6.0f} TF/s")


if __name__ == "__main__":
    main()
