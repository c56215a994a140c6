"""Standalone launches of the step's kernels at CoLA-1B (b4 s4096, TP=1) shapes — and of the
peer-memory boundary at CoLA-7B TP=8 shapes (tp virtual peer buffers on one GPU) — for ncu
captures on the box:  python scripts/microbench/gpu_profile_kernels.py <name> [reps]   (not a pytest module)."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2512_12131_b200 import _native  # noqa: E402
from paper_2512_12131_b200 import kernels as K  # noqa: E402

T, d, r, f, V = 16384, 2048, 512, 5472, 32000
dev, bf, f32 = "cuda", torch.bfloat16, torch.float32
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.manual_seed(0)


def rnd(*shape, dtype=bf):
    return torch.randn(*shape, device=dev, dtype=dtype)


if name == "qkv_up":          # grouped up-projection q|k|v: 3 x [16384 x 2048], K = 512
    a, w, o = rnd(3, T, r), rnd(3, d, r), torch.empty(3, T, d, device=dev, dtype=bf)
    run = lambda: K.gemm(*[K.Gemm(a[i], w[i], o[i]) for i in range(3)])  # noqa: E731
elif name == "down_sigma":    # grouped down q|k|v with the crossgate epilogue (TP = 1): [16384 x 1536], K = 2048
    n, w = rnd(T, d), rnd(3 * r, d)
    P, A = torch.empty(T, 3 * r, device=dev, dtype=bf), torch.empty(T, 3 * r, device=dev, dtype=bf)
    run = lambda: K.gemm(K.Gemm(n, w, P, sigma=(A, r // 2)))  # noqa: E731
elif name == "up_resid":      # o up-projection + residual: [16384 x 2048], K = 512
    a, w, x, o = rnd(T, r), rnd(d, r), rnd(T, d), torch.empty(T, d, device=dev, dtype=bf)
    run = lambda: K.gemm(K.Gemm(a, w, o, resid=x))  # noqa: E731
elif name == "dgrad_gu":      # gate|up up-projection dgrad: 2 x [16384 x 512], K = 5472, B MN-major
    dg, w, o = rnd(2, T, f), rnd(2, f, r), torch.empty(2, T, r, device=dev, dtype=bf)
    run = lambda: K.gemm(*[K.Gemm(dg[i], w[i], o[i], b_mn=True) for i in range(2)])  # noqa: E731
elif name == "down_gu":       # gate|up down + sigma at TP=1: [16384 x 1024], K = 2048
    n, w = rnd(T, d), rnd(2 * r, d)
    P, A = torch.empty(T, 2 * r, device=dev, dtype=bf), torch.empty(T, 2 * r, device=dev, dtype=bf)
    run = lambda: K.gemm(K.Gemm(n, w, P, sigma=(A, r // 2)))  # noqa: E731
elif name in ("down7b_plain", "down7b_scatter"):  # 7B TP=8 q|k|v down GEMM [16384 x 3072], K=512
    n7, w7 = rnd(T, 512), rnd(3072, 512)
    if name == "down7b_plain":
        P7 = torch.empty(T, 3072, device=dev, dtype=bf)
        run = lambda: K.gemm(K.Gemm(n7, w7, P7))  # noqa: E731
    else:  # reduce-added into 8 owners' fp32 [2048 x 3072] buffers (virtual peers: same GPU)
        owners = [torch.zeros(T // 8, 3072, device=dev, dtype=f32) for _ in range(8)]
        run = lambda: K.gemm_scatter(K.Gemm(n7, w7, None), owners=[o.data_ptr() for o in owners],  # noqa: E731
                                     rows_per_owner=T // 8, width=3072, ld=3072, col0=[0])
elif name == "rmsnorm":
    x, g = rnd(T, d), rnd(d, dtype=f32)
    n, ss, rl = torch.empty_like(x), torch.empty(T, device=dev, dtype=f32), torch.empty(T, device=dev, dtype=f32)
    run = lambda: K.rmsnorm_residual(x, g, n_out=n, ss_out=ss, rl_out=rl)  # noqa: E731
elif name == "rmsnorm_bwd":   # dx = dres + dh*gamma + 2 x dss, dgamma partials [16384 x 2048]
    dh, x, dres, g = rnd(T, d), rnd(T, d), rnd(T, d), rnd(d, dtype=f32)
    dss, dx = torch.rand(T, device=dev, dtype=f32), torch.empty(T, d, device=dev, dtype=bf)
    parts = torch.empty(4 * 148, d, device=dev, dtype=f32)
    run = lambda: K.rmsnorm_bwd(dh, x, g, dss, dx, parts, dres=dres)  # noqa: E731
elif name == "dot":           # loss partials <y, G> over [16384 x 2048]
    y, G2 = rnd(T, d), rnd(T, d)
    part = torch.empty(4 * 148, device=dev, dtype=f32)
    run = lambda: K.dot(y, G2, part)  # noqa: E731
elif name == "swiglu":
    g, u, a = rnd(T, f), rnd(T, f), torch.empty(T, f, device=dev, dtype=bf)
    run = lambda: K.swiglu(g, u, a)  # noqa: E731
elif name == "swiglu_bwd":
    g, u, da = rnd(T, f), rnd(T, f), rnd(T, f)
    dg, du = torch.empty_like(g), torch.empty_like(u)
    run = lambda: K.swiglu_bwd(g, u, da, dg, du)  # noqa: E731
elif name == "fixup_bwd":     # sigma-bwd of the q|k|v chunk [16384 x 1536]
    z, da, s = rnd(T, 3 * r), rnd(T, 3 * r), torch.rand(T, device=dev, dtype=f32) + 0.5
    dss = torch.empty(T, device=dev, dtype=f32)
    run = lambda: K.fixup_sigma_bwd(z, da, da, r=r, nproj=3, variant=1, s=s, d=d, dss=dss)  # noqa: E731
elif name == "adamw":         # the block's 19.9 M low-rank parameters
    n = 11 * d * r + 3 * f * r
    n = -(-n // 8) * 8
    mst, m, v, g = (torch.zeros(n, device=dev, dtype=f32) for _ in range(4))
    w = torch.zeros(n, device=dev, dtype=bf)
    run = lambda: K.adamw(mst, m, v, g, w, lr=1e-4, step=1)  # noqa: E731
elif name == "xent":          # fused cross-entropy over [16384 x 32000] logits
    lg = rnd(T, V)
    tg = torch.randint(0, V, (T,), device=dev, dtype=torch.int32)
    rows = torch.empty(T, device=dev, dtype=f32)
    run = lambda: K.cross_entropy(lg, tg, rows, dlogits=lg, scale=1.0 / T)  # noqa: E731
elif name == "peer_fwd":      # CoLA-7B TP=8 q|k|v boundary: T=16384, W=3r=3072, 8 virtual peers
    tp, r7, d7 = 8, 1024, 4096
    W = 3 * r7
    P = [rnd(T, W) for _ in range(tp)]
    ss = [torch.rand(T, device=dev, dtype=f32) * d7 for _ in range(tp)]
    A = [torch.empty(T, W, device=dev, dtype=bf) for _ in range(tp)]
    z = torch.empty(T // tp, W, device=dev, dtype=bf)
    s_own = torch.empty(T // tp, device=dev, dtype=f32)
    ptr = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)  # noqa: E731
    pP, pS, pA = ptr(P), ptr(ss), ptr(A)
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    run = lambda: _native.call("btp_peer_boundary_fwd", vp(pP), vp(pS), tp, 3, T, W, r7, 1, d7,  # noqa: E731
                               ctypes.c_float(1e-6), vp(z), vp(s_own), vp(pA), st())
elif name == "peer_bwd":
    tp, r7, d7 = 8, 1024, 4096
    W = 3 * r7
    dA = [rnd(T, W) for _ in range(tp)]
    dP = [torch.empty(T, W, device=dev, dtype=bf) for _ in range(tp)]
    dss = [torch.empty(T, device=dev, dtype=f32) for _ in range(tp)]
    z, s_own = rnd(T // tp, W), torch.rand(T // tp, device=dev, dtype=f32) + 0.5
    ptr = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)  # noqa: E731
    pA, pP, pD = ptr(dA), ptr(dP), ptr(dss)
    st = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
    vp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    run = lambda: _native.call("btp_peer_boundary_bwd", vp(pA), tp, 3, T, W, r7, 1, d7, vp(z), vp(s_own),  # noqa: E731
                               vp(pP), vp(pD), st())
else:
    raise SystemExit(f"unknown kernel {name}")

for _ in range(reps):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
print(f"{name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/launch (CUDA events, 20 back-to-back)")
