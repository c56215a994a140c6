"""tcgen05 GEMM kernel (libbtp.so `btp_gemm`) against a torch fp32 reference of the same op:
every operand-major combination and N tile, grouped launches, mixed majors in one launch,
split-K via TMA reduce-add, row/col scales, the TMA residual epilogue and the fused SwiGLU
backward epilogue. bf16 inputs, fp32 accumulation: tolerance 1e-2 relative Frobenius."""

import pytest
import torch

from paper_2512_12131_b200 import kernels as K

pytestmark = pytest.mark.gpu
TOL = 1e-2


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def _mk(*shape):
    return torch.randn(*shape, device="cuda").bfloat16()


@pytest.mark.parametrize("M,N,Kd", [(128, 128, 64), (296, 200, 72), (1024, 512, 512), (2048, 1536, 2048)])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True), (True, False)])
@pytest.mark.parametrize("bn", [128, 192, 256])
def test_layouts(M, N, Kd, a_mn, b_mn, bn):
    A, B = _mk(M, Kd), _mk(N, Kd)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    K.gemm(K.Gemm(A.t().contiguous() if a_mn else A, B.t().contiguous() if b_mn else B, C, a_mn=a_mn, b_mn=b_mn),
           bn=bn)
    assert rel(C, A.float() @ B.float().t()) < TOL


def test_scales_fp32_out_and_residual():
    A, B = _mk(1000, 512), _mk(640, 512)
    row = torch.rand(1000, device="cuda") + 0.5
    col = torch.rand(640, device="cuda") + 0.5
    C = torch.empty(1000, 640, device="cuda")
    K.gemm(K.Gemm(A, B, C, row_scale=row, col_scale=col))
    assert rel(C, (A.float() @ B.float().t()) * row[:, None] * col[None, :]) < 1e-5
    R = _mk(1000, 640)
    Cb = torch.empty(1000, 640, device="cuda", dtype=torch.bfloat16)
    K.gemm(K.Gemm(A, B, Cb, resid=R))
    assert rel(Cb, A.float() @ B.float().t() + R.float()) < TOL
    # residual aliasing the output (in-place accumulate, used by chained dgrads)
    K.gemm(K.Gemm(A, B, Cb, resid=Cb))
    assert rel(Cb, 2 * (A.float() @ B.float().t()) + R.float()) < TOL


@pytest.mark.parametrize("splits", [2, 4, 9, 13, 64])
def test_split_k_reduce_add(splits):
    """K = 4096 = 64 k-blocks: 9 splits of 8 (and 13 of 5) leave trailing splits empty — they are
    dropped, not reduce-added as an unwritten accumulator."""
    dY, X = _mk(4096, 512), _mk(4096, 2048)
    dW = torch.empty(512, 2048, device="cuda")
    K.zero(dW)
    cs = torch.rand(2048, device="cuda") + 0.5
    K.gemm(K.Gemm(dY, X, dW, a_mn=True, b_mn=True, splits=splits, col_scale=cs))
    assert rel(dW, (dY.float().t() @ X.float()) * cs[None, :]) < 1e-5


def test_grouped_and_mixed_majors():
    A = [_mk(2048, 512) for _ in range(3)]
    B = [_mk(768, 512) for _ in range(3)]
    C = [torch.empty(2048, 768, device="cuda", dtype=torch.bfloat16) for _ in range(3)]
    K.gemm(*[K.Gemm(a, b, c) for a, b, c in zip(A, B, C)])
    for a, b, c in zip(A, B, C):
        assert rel(c, a.float() @ b.float().t()) < TOL
    dY, W, X = _mk(4096, 1024), _mk(1024, 512), _mk(4096, 512)
    dA = torch.empty(4096, 512, device="cuda", dtype=torch.bfloat16)
    dW = torch.empty(1024, 512, device="cuda")
    K.zero(dW)
    K.gemm(K.Gemm(dY, W, dA, b_mn=True), K.Gemm(dY, X, dW, a_mn=True, b_mn=True, splits=4))
    assert rel(dA, dY.float() @ W.float()) < TOL
    assert rel(dW, dY.float().t() @ X.float()) < 1e-5


@pytest.mark.parametrize(
    "shapes",
    [
        [(16384, 2048, 512)] * 3,  # the q|k|v up-projection launch at the bench config
        [(4096, 5472, 512)] * 2,  # gate|up widths (N tail: 5472 = 21.375 x 256)
        [(1000, 640, 200), (296, 2048, 512), (2560, 136, 64)],  # M / N / K tails in one launch
        [(300, 4096, 448)],  # fewer M blocks than CTA pairs
    ],
)
def test_grouped_short_k_launches(shapes):
    """Grouped K <= 512 launches (the forward up-projections) with ragged M / N / K, against torch fp32."""
    A = [_mk(m, kd) for m, n, kd in shapes]
    B = [_mk(n, kd) for m, n, kd in shapes]
    C = [torch.empty(m, n, device="cuda", dtype=torch.bfloat16) for m, n, kd in shapes]
    K.gemm(*[K.Gemm(a, b, c) for a, b, c in zip(A, B, C)])
    torch.cuda.synchronize()
    for a, b, c in zip(A, B, C):
        assert rel(c, a.float() @ b.float().t()) < TOL


@pytest.mark.parametrize("N", [640, 5472])
def test_swiglu_bwd_epilogue(N):
    T, r = 1024, 512
    dP, Wd = _mk(T, r), _mk(r, N)          # dact = dP @ Wd  (B operand MN-major)
    g, u = _mk(T, N), _mk(T, N)
    dg = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    du = torch.empty_like(dg)
    K.gemm(K.Gemm(dP, Wd, dg, b_mn=True, swiglu_bwd=(g, u, du)))
    dact = dP.float() @ Wd.float()
    gf, uf = g.float(), u.float()
    sg = torch.sigmoid(gf)
    assert rel(dg, dact * uf * sg * (1 + gf * (1 - sg))) < TOL
    assert rel(du, dact * gf * sg) < TOL


def test_rejects_misaligned():
    A, B = _mk(64, 60), _mk(64, 60)
    C = torch.empty(64, 64, device="cuda", dtype=torch.bfloat16)
    from paper_2512_12131_b200._native import NativeError

    with pytest.raises(NativeError):
        K.gemm(K.Gemm(A, B, C))


def _crossgate_ref(z, r):
    """[silu(u) v, silu(v) u] per r-wide projection, from the bf16-rounded z (as the epilogue)."""
    z = z.float()
    out = torch.empty_like(z)
    for p in range(z.shape[1] // r):
        u, v = z[:, p * r:p * r + r // 2], z[:, p * r + r // 2:(p + 1) * r]
        out[:, p * r:p * r + r // 2] = torch.nn.functional.silu(u) * v
        out[:, p * r + r // 2:(p + 1) * r] = torch.nn.functional.silu(v) * u
    return out


@pytest.mark.parametrize("M,r,nproj,Kd", [(300, 128, 3, 512), (2048, 512, 3, 2048), (1000, 256, 2, 1024),
                                          (4096, 512, 1, 5472), (256, 1024, 1, 512)])
@pytest.mark.parametrize("pair", [True, False])
@pytest.mark.parametrize("bn", [0, 128])
def test_sigma_epilogue(M, r, nproj, Kd, pair, bn):
    """z = scale * (X @ B^T) and a = crossgate(z) from one launch (the TP = 1 rank-r boundary)."""
    X, B = _mk(M, Kd), _mk(nproj * r, Kd) * 0.05
    row = torch.rand(M, device="cuda") + 0.5
    Z = torch.empty(M, nproj * r, device="cuda", dtype=torch.bfloat16)
    Aout = torch.full((M, nproj * r), float("nan"), device="cuda", dtype=torch.bfloat16)
    prev = K.set_pair_mode(pair)
    try:
        K.gemm(K.Gemm(X, B, Z, row_scale=row, sigma=(Aout, r // 2)), bn=bn)
    finally:
        K.set_pair_mode(prev)
    z_ref = (X.float() @ B.float().t()) * row[:, None]
    assert rel(Z, z_ref) < TOL
    assert rel(Aout, _crossgate_ref(Z, r)) < TOL
    assert not torch.isnan(Aout.float()).any()


def test_sigma_epilogue_rejects_bad_shapes():
    X, B = _mk(256, 512), _mk(192, 512)
    Z = torch.empty(256, 192, device="cuda", dtype=torch.bfloat16)
    A = torch.empty_like(Z)
    with pytest.raises(Exception):
        K.gemm(K.Gemm(X, B, Z, sigma=(A, 96)))  # half-width not a multiple of 64
    X, B = _mk(256, 512), _mk(128, 512)
    Z = torch.empty(256, 128, device="cuda", dtype=torch.bfloat16)
    A = torch.empty_like(Z)
    with pytest.raises(Exception):
        K.gemm(K.Gemm(X, B, Z, sigma=(A, 64)), bn=256)  # a 256-wide tile would straddle two projections
    with pytest.raises(Exception):
        K.gemm(K.Gemm(X, B.t().contiguous(), Z, b_mn=True, sigma=(A, 64)))  # B must be K-major


@pytest.mark.parametrize("M,N,Kd,nprob,b_mn,tp", [(128, 64, 128, 3, True, 2), (256, 192, 256, 1, False, 2),
                                                 (512, 64, 512, 2, True, 4), (2048, 512, 256, 1, False, 8),
                                                 (16384, 3072, 512, 1, False, 8)])
def test_gemm_scatter_reduce_into_owners(M, N, Kd, nprob, b_mn, tp):
    """btp_gemm_scatter: each problem's rows are reduce-added (fp32) into the owning rank's buffer
    at its column offset; two launches accumulate (the owners' buffers start at zero)."""
    torch.manual_seed(M + N)
    A = [_mk(M, Kd) for _ in range(nprob)]
    B = [_mk(Kd, N) if b_mn else _mk(N, Kd) for _ in range(nprob)]
    W = nprob * N
    owners = [torch.zeros(M // tp, W, device="cuda") for _ in range(tp)]
    probs = [K.Gemm(A[i], B[i], None, b_mn=b_mn) for i in range(nprob)]
    for _ in range(2):
        K.gemm_scatter(*probs, owners=[o.data_ptr() for o in owners], rows_per_owner=M // tp, width=W, ld=W,
                       col0=[i * N for i in range(nprob)])
    torch.cuda.synchronize()
    full = torch.cat(owners, 0)
    for i in range(nprob):
        ref = A[i].float() @ (B[i].float() if b_mn else B[i].float().t())
        assert rel(full[:, i * N:(i + 1) * N] / 2, ref) < TOL


def test_randomised_shapes_against_torch():
    """Seeded sweep over problem counts, shapes (multiples of 8, incl. tails of every tile size),
    operand majors, split-K, residual and row/col scales, against torch fp32 of the same op."""
    import random

    rng = random.Random(1234)
    for case in range(40):
        nprob = rng.choice([1, 1, 2, 3, 4])
        probs, checks = [], []
        fp32_split = rng.random() < 0.3
        for _ in range(nprob):
            M = rng.choice([8, 96, 128, 200, 256, 1000, 2048])
            N = 8 * rng.randint(1, 96)
            Kd = 8 * rng.randint(1, 160)
            a_mn, b_mn = rng.random() < 0.3, rng.random() < 0.5
            A, B = _mk(M, Kd), _mk(N, Kd)
            Aop = A.t().contiguous() if a_mn else A
            Bop = B.t().contiguous() if b_mn else B
            ref = A.float() @ B.float().t()
            if fp32_split:
                splits = rng.choice([1, 2, 3, 5])
                C = torch.zeros(M, N, device="cuda")
                cs = torch.rand(N, device="cuda") + 0.5
                probs.append(K.Gemm(Aop, Bop, C, a_mn=a_mn, b_mn=b_mn, splits=splits, reduce_add=True, col_scale=cs))
                checks.append((C, ref * cs[None, :], 1e-5))
            else:
                rs = torch.rand(M, device="cuda") + 0.5 if rng.random() < 0.3 else None
                R = _mk(M, N) if rng.random() < 0.3 else None
                C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
                probs.append(K.Gemm(Aop, Bop, C, a_mn=a_mn, b_mn=b_mn, row_scale=rs, resid=R))
                want = ref * (rs[:, None] if rs is not None else 1.0) + (R.float() if R is not None else 0.0)
                checks.append((C, want, TOL))
        K.gemm(*probs, bn=rng.choice([0, 0, 128, 192, 256]))
        for C, want, tol in checks:
            assert rel(C, want) < tol, (case, tuple(C.shape))


@pytest.mark.parametrize("res_mode", [0, 1, 2, 3])
@pytest.mark.parametrize("st_global", [0, 1])
def test_residual_layouts_and_store_paths(res_mode, st_global):
    """Every residual-epilogue layout (0 per-chunk, 1 whole tile, 2 producer-warp pipeline, 3 by
    width) x both store paths (TMA bulk / coalesced st.global), incl. M / N tails, a grouped launch
    mixing residual and plain problems, in-place accumulation (resid aliasing C, the chained dgrads)
    and the sigma / fp32 / split-K epilogues that must ignore the store switch."""
    prev_r, prev_s = K.set_res4(res_mode), K.set_st_global(bool(st_global))
    try:
        for M, N, Kd in [(1000, 640, 512), (16384, 512, 1024), (2048, 2048, 512), (296, 1000, 72)]:
            A, B, R = _mk(M, Kd), _mk(N, Kd), _mk(M, N)
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            K.gemm(K.Gemm(A, B, C, resid=R))
            ref = A.float() @ B.float().t()
            assert rel(C, ref + R.float()) < TOL, (M, N, Kd)
            K.gemm(K.Gemm(A, B, C, resid=C))                      # in place: C = A B^T + C
            assert rel(C, 2 * ref + R.float()) < TOL, (M, N, Kd, "in-place")
        # grouped: residual + plain problems in one launch
        A1, B1, R1 = _mk(1024, 512), _mk(768, 512), _mk(1024, 768)
        A2, B2 = _mk(1024, 512), _mk(512, 512)
        C1 = torch.empty(1024, 768, device="cuda", dtype=torch.bfloat16)
        C2 = torch.empty(1024, 512, device="cuda", dtype=torch.bfloat16)
        K.gemm(K.Gemm(A1, B1, C1, resid=R1), K.Gemm(A2, B2, C2))
        assert rel(C1, A1.float() @ B1.float().t() + R1.float()) < TOL
        assert rel(C2, A2.float() @ B2.float().t()) < TOL
        # fp32 output and split-K reduce-add (TMA reduce regardless of the store switch)
        Cf = torch.zeros(512, 640, device="cuda")
        dY, X = _mk(4096, 512), _mk(4096, 640)
        K.gemm(K.Gemm(dY, X, Cf, a_mn=True, b_mn=True, splits=4))
        assert rel(Cf, dY.float().t() @ X.float()) < 1e-5
        Cp = torch.empty(1000, 640, device="cuda")
        A3, B3 = _mk(1000, 256), _mk(640, 256)
        K.gemm(K.Gemm(A3, B3, Cp))
        assert rel(Cp, A3.float() @ B3.float().t()) < 1e-5
        # sigma epilogue (TP = 1 boundary): z and crossgate(z) both through the store path
        n_in, W = _mk(2048, 512), _mk(1024, 512) * 0.05
        z = torch.empty(2048, 1024, device="cuda", dtype=torch.bfloat16)
        a = torch.empty_like(z)
        K.gemm(K.Gemm(n_in, W, z, sigma=(a, 256)))
        assert rel(z, n_in.float() @ W.float().t()) < TOL
        assert rel(a, _crossgate_ref(z, 512)) < TOL
    finally:
        K.set_res4(prev_r)
        K.set_st_global(bool(prev_s))


@pytest.mark.parametrize("n_probs", [5, 6, 8])
def test_up_to_eight_problems_dgrad_and_split_wgrad(n_probs):
    """The merged backward launches (executor._dgrad_wgrad): up to 8 problems in ONE launch, bf16
    dgrads (B MN-major) ahead of fp32 split-K weight gradients (both operands MN-major, TMA
    reduce-add into zeroed outputs, with and without a column scale), ragged shapes included."""
    T = 1536
    probs, checks = [], []
    n_d = n_probs // 2
    for i in range(n_d):  # dgrads: dA[T, r] = dY[T, w] @ W[r, w]^T... with W read MN-major
        w, r = 384 + 64 * i, 128 + 32 * i
        dY, W = _mk(T, w), _mk(w, r)
        out = torch.empty(T, r, device="cuda", dtype=torch.bfloat16)
        probs.append(K.Gemm(dY, W, out, b_mn=True))
        checks.append((out, dY.float() @ W.float(), TOL))
    for i in range(n_probs - n_d):  # weight gradients: dW[m, n] = dY^T X over the T tokens, split-K 3
        m, n = 256 + 96 * i, 320 + 64 * i
        dY, X = _mk(T, m), _mk(T, n)
        dW = torch.empty(m, n, device="cuda")
        K.zero(dW)
        cs = (torch.rand(n, device="cuda") + 0.5) if i % 2 else None
        probs.append(K.Gemm(dY, X, dW, a_mn=True, b_mn=True, splits=3, col_scale=cs))
        ref = dY.float().t() @ X.float()
        checks.append((dW, ref * cs[None, :] if cs is not None else ref, 1e-5))
    K.gemm(*probs)
    for got, want, tol in checks:
        assert rel(got, want) < tol
