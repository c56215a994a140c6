"""Plain-epilogue GEMMs with narrow outputs (the step's N = 512 launches): TMA bulk-tensor stores vs
coalesced st.global stores from the staging chunk (btp_gemm_set_st_global)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import kernels as K  # noqa: E402
from scripts.microbench.gpu_gemm_resid_ab import t  # noqa: E402

cases = [  # (M, N, K, b_mn, nprob)
    (16384, 512, 2048, True, 1),   # dgrad of an up factor at 1B TP=1: dA = dY U
    (16384, 512, 2048, True, 3),   # q|k|v grouped dgrad
    (16384, 512, 2048, False, 1),
    (16384, 512, 5472, True, 1),
    (16384, 1024, 2048, False, 1),
    (16384, 256, 2048, True, 1),   # TP=2 shapes
    (16384, 128, 4096, True, 1),
]
for M, N, Kd, bmn, npb in cases:
    a = torch.randn(M, Kd, device="cuda").bfloat16()
    ws = [(torch.randn(Kd, N, device="cuda") if bmn else torch.randn(N, Kd, device="cuda")).bfloat16() for _ in range(npb)]
    outs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(npb)]
    probs = [K.Gemm(a, w, o, b_mn=bmn) for w, o in zip(ws, outs)]
    fl = 2 * M * N * Kd * npb
    res = {}
    for st in (0, 1):
        K.set_st_global(st)
        res[st] = t(lambda: K.gemm(*probs))
        ref = a.float() @ (ws[0].float() if bmn else ws[0].float().t())
        err = float((outs[0].float() - ref).norm() / ref.norm())
        assert err < 1e-2, err
    K.set_st_global(0)
    print(f"[{M}x{N} K={Kd} b_mn={int(bmn)} x{npb}] TMA store {res[0]:6.1f} us ({fl/res[0]/1e6:5.0f} TF/s)  "
          f"st.global {res[1]:6.1f} us ({fl/res[1]/1e6:5.0f} TF/s)", flush=True)
