"""The tcgen05 / TMEM attention kernels (csrc/attn.cu) against a plain PyTorch fp32 reference of the
reference's unmasked per-head SDPA (model.py:205-230 `sdpa_values`: heads as contiguous feature
slices of [T, heads*hd]).

Tolerances: bf16 inputs, fp32 statistics, P rounded to bf16 before the PV MMA (as every
flash-attention kernel does) -> 1e-2 relative Frobenius on o (measured ~3e-3), 1e-5 absolute on the
log-sum-exp."""

import math

import pytest
import torch

from paper_2512_12131_b200 import kernels as K

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm())


def _ref(q, k, v, b, s, h, hd):
    def v4(t):
        return t.float().view(b, s, h, hd).transpose(1, 2)

    sc = v4(q) @ v4(k).transpose(-1, -2) / math.sqrt(hd)
    lse = torch.logsumexp(sc, dim=-1)  # natural log, [b, h, s]
    o = torch.softmax(sc, dim=-1) @ v4(v)
    return o.transpose(1, 2).reshape(b * s, h * hd), lse


def _inputs(b, s, h, hd, scale=1.0, ld_pad=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = h * hd
    out = []
    for _ in range(3):
        t = torch.randn(b * s, w + ld_pad, device="cuda", generator=g) * scale
        out.append(t.bfloat16()[:, :w])
    return out


@pytest.mark.parametrize("hd", [64, 128])
@pytest.mark.parametrize("b,s,h", [(1, 128, 1), (2, 256, 3), (1, 1024, 4), (2, 512, 2)])
def test_attn_fwd_matches_fp32(b, s, h, hd):
    q, k, v = _inputs(b, s, h, hd, seed=b * 1000 + s + h)
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    torch.cuda.synchronize()
    o_ref, lse_ref = _ref(q, k, v, b, s, h, hd)
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse * math.log(2.0), lse_ref, atol=1e-4, rtol=1e-5)


@pytest.mark.parametrize("hd", [64, 128])
def test_attn_fwd_large_scores_rescale_and_strided_views(hd):
    """Scores spread over ~+-60 so the running max grows by more than 2^8 across key tiles (the lazy
    O rescale path), on q/k/v/o views with padded row strides (the [T, width] column slices)."""
    b, s, h = 2, 512, 2
    q, k, v = _inputs(b, s, h, hd, scale=3.0, ld_pad=64, seed=7)
    # a key tile late in the sequence carries the largest scores for half the queries
    k[b * s // 2 - 128 : b * s // 2] *= 2.0
    obuf = torch.zeros(b * s, h * hd + 32, device="cuda", dtype=torch.bfloat16)
    o = obuf[:, : h * hd]
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    torch.cuda.synchronize()
    o_ref, lse_ref = _ref(q, k, v, b, s, h, hd)
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse * math.log(2.0), lse_ref, atol=1e-3, rtol=1e-5)
    assert torch.count_nonzero(obuf[:, h * hd :]) == 0  # nothing written past the view


def test_attn_fwd_rejects_bad_shapes():
    q, k, v = _inputs(1, 128, 1, 64)
    o = torch.empty_like(q)
    lse = torch.empty(1, 1, 128, device="cuda")
    with pytest.raises(Exception):
        K.attn_fwd(q, k, v, o, lse, b=1, s=100, heads=1, head_dim=64)
    with pytest.raises(Exception):
        K.attn_fwd(q, k, v, o, lse, b=1, s=128, heads=1, head_dim=32)


def _ref_bwd(q, k, v, do, b, s, h, hd):
    qf, kf, vf = (t.float().detach().requires_grad_(True) for t in (q, k, v))
    o, _ = _ref(qf, kf, vf, b, s, h, hd)
    o.backward(do.float())
    return qf.grad, kf.grad, vf.grad


@pytest.mark.parametrize("hd", [64, 128])
@pytest.mark.parametrize("b,s,h", [(1, 128, 1), (2, 256, 3), (1, 1024, 2)])
def test_attn_bwd_matches_fp32(b, s, h, hd):
    q, k, v = _inputs(b, s, h, hd, seed=11 * s + h)
    do = torch.randn(b * s, h * hd, device="cuda").bfloat16()
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    D = torch.empty(b, h, s, device="cuda")
    acc = torch.empty(b * s, h * hd, device="cuda")
    dq, dk, dv = (torch.empty_like(o) for _ in range(3))
    K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
    torch.cuda.synchronize()
    rq, rk, rv = _ref_bwd(q, k, v, do, b, s, h, hd)
    errs = {"dq": _rel(dq, rq), "dk": _rel(dk, rk), "dv": _rel(dv, rv)}
    assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("grouping", [True, False])
def test_block_step_native_attention_vs_oracle(grouping):
    """The BTP CoLA-60M block (8 heads of 64) fwd+bwd with the native attention kernels inside the
    executor, against the float64 oracle (reference model.py:205-230 attention inside
    simulator.py:550-714), at the north_star bf16 bar."""
    from paper_2512_12131_b200.api import train_step
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan
    from tests.gpu_util import BF16_TOL, C60M, inputs, oracle_step, rel

    b, s = 2, 256
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=grouping)
    st = train_step(pl, blk, x, G, attn_backend="native")
    torch.cuda.synchronize()
    assert st.executor.attn.native
    y_ref, g_ref, _, _ = oracle_step(oblk, x, G, C60M, b, s)
    errs = {"y": rel(st.y.values, y_ref), "dx": rel(st.dx, g_ref["dx"])}
    for n in g_ref["A"]:
        errs[f"A_{n}"] = rel(st.grads["A"][n], g_ref["A"][n])
        errs[f"B_{n}"] = rel(st.grads["B"][n], g_ref["B"][n])
    worst = max(errs, key=errs.get)
    assert errs[worst] < BF16_TOL, errs


@pytest.mark.parametrize("grouping", [True])
def test_block_step_hybrid_attention_vs_oracle(grouping):
    """The same block with the "hybrid" attention (cuDNN forward + its log-sum-exp converted to log2,
    then the native tcgen05 backward) against the float64 oracle."""
    from paper_2512_12131_b200.api import train_step
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan
    from tests.gpu_util import BF16_TOL, C60M, inputs, oracle_step, rel

    b, s = 2, 256
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=grouping)
    st = train_step(pl, blk, x, G, attn_backend="hybrid")
    torch.cuda.synchronize()
    assert st.executor.attn.hybrid
    y_ref, g_ref, _, _ = oracle_step(oblk, x, G, C60M, b, s)
    errs = {"y": rel(st.y.values, y_ref), "dx": rel(st.dx, g_ref["dx"])}
    for n in g_ref["A"]:
        errs[f"A_{n}"] = rel(st.grads["A"][n], g_ref["A"][n])
        errs[f"B_{n}"] = rel(st.grads["B"][n], g_ref["B"][n])
    worst = max(errs, key=errs.get)
    assert errs[worst] < BF16_TOL, errs


@pytest.mark.parametrize("hd", [64, 128])
@pytest.mark.parametrize("b,s,h", [(1, 256, 3), (2, 1024, 4), (3, 384, 5)])
def test_hybrid_attention_matches_fp32(b, s, h, hd):
    """Attention(backend="hybrid") forward + backward against torch fp32 autograd."""
    from paper_2512_12131_b200.attention import Attention

    q, k, v = _inputs(b, s, h, hd, scale=1.5, seed=31 * s + h)
    do = torch.randn(b * s, h * hd, device="cuda").bfloat16()
    att = Attention(b, s, h, hd, "hybrid")
    out, ctx = att.forward(q, k, v)
    dq, dk, dv = att.backward(do, ctx)
    torch.cuda.synchronize()
    o_ref, _ = _ref(q, k, v, b, s, h, hd)
    rq, rk, rv = _ref_bwd(q, k, v, do, b, s, h, hd)
    errs = {"o": _rel(out, o_ref), "dq": _rel(dq, rq), "dk": _rel(dk, rk), "dv": _rel(dv, rv)}
    assert max(errs.values()) < 2e-2, errs


def test_native_attention_rejects_unsupported_shapes():
    from paper_2512_12131_b200.attention import Attention

    with pytest.raises(ValueError):
        Attention(1, 100, 2, 64, "native")
    with pytest.raises(ValueError):
        Attention(1, 128, 2, 32, "native")
    with pytest.raises(ValueError):
        Attention(1, 100, 2, 64, "hybrid")


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 5, 6])
@pytest.mark.parametrize("poly", [0, 3, 4])
@pytest.mark.parametrize("hd", [64, 128])
def test_attn_fwd_kernel_variants(variant, poly, hd):
    """Every forward kernel variant behind btp_attn_tune (single S buffer / split rows double-buffered /
    4 key groups / split rows single-buffered / two query tiles per CTA / two query tiles with P apart
    from S, hd 64) and the polynomial exp2 share, against torch fp32."""
    from paper_2512_12131_b200 import _native

    lib = _native.load()
    b, s, h = 2, 512, 2
    q, k, v = _inputs(b, s, h, hd, scale=2.0, seed=variant * 10 + poly)
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    prev_v, prev_p = lib.btp_attn_tune(1, variant), lib.btp_attn_tune(0, poly)
    try:
        K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
        torch.cuda.synchronize()
    finally:
        lib.btp_attn_tune(1, prev_v)
        lib.btp_attn_tune(0, prev_p)
    o_ref, lse_ref = _ref(q, k, v, b, s, h, hd)
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse * math.log(2.0), lse_ref, atol=2e-3, rtol=1e-5)


@pytest.mark.parametrize("variant", [4, 5, 6])
def test_attn_fwd_growing_row_max(variant):
    """Scores that grow along the keys (every key tile raises the row max) plus one dominant key in
    the last tile (a late jump far above the 2^8 lazy-rescale threshold): the O / l rescale paths of
    the two-query-tile kernels, against torch fp32."""
    from paper_2512_12131_b200 import _native

    lib = _native.load()
    b, s, h, hd = 1, 1024, 2, 64
    q, k, v = _inputs(b, s, h, hd, seed=11)
    ramp = torch.linspace(0.2, 3.0, s, device="cuda").repeat(b).unsqueeze(1)
    k = (k.float() * ramp).bfloat16()
    k[s - 5] = (q[3].float() * 6.0).bfloat16()  # query row 3 (both heads) meets a huge score late
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    prev = lib.btp_attn_tune(1, variant)
    try:
        K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
        torch.cuda.synchronize()
    finally:
        lib.btp_attn_tune(1, prev)
    o_ref, lse_ref = _ref(q, k, v, b, s, h, hd)
    assert torch.isfinite(o.float()).all()
    assert _rel(o, o_ref) < 1e-2
    assert torch.allclose(lse * math.log(2.0), lse_ref, atol=2e-3, rtol=1e-5)


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("b,s,h", [(1, 256, 2), (2, 1024, 2)])
def test_attn_bwd_hd64_kernel_variants(variant, b, s, h):
    """Both hd-64 backward kernels behind btp_attn_tune(3, v) (shared P/dS warps, split roles) vs torch fp32."""
    from paper_2512_12131_b200 import _native

    lib = _native.load()
    hd = 64
    q, k, v = _inputs(b, s, h, hd, seed=3 * s + variant)
    do = torch.randn(b * s, h * hd, device="cuda").bfloat16()
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    D = torch.empty(b, h, s, device="cuda")
    acc = torch.empty(b * s, h * hd, device="cuda")
    dq, dk, dv = (torch.empty_like(o) for _ in range(3))
    prev = lib.btp_attn_tune(3, variant)
    try:
        K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
        torch.cuda.synchronize()
    finally:
        lib.btp_attn_tune(3, prev)
    rq, rk, rv = _ref_bwd(q, k, v, do, b, s, h, hd)
    errs = {"dq": _rel(dq, rq), "dk": _rel(dk, rk), "dv": _rel(dv, rv)}
    assert max(errs.values()) < 2e-2, errs


@pytest.mark.parametrize("poly", [2, 0])
@pytest.mark.parametrize("persist", [1, 0])
@pytest.mark.parametrize("b,s,h", [(1, 128, 3), (2, 256, 5), (3, 384, 7), (2, 640, 33), (2, 1024, 80), (1, 4096, 2)])
def test_attn_bwd_hd64_persistent_walk(persist, b, s, h, poly):
    """The hd-64 backward's persistent walk (btp_attn_tune(7, 1), default: one CTA per SM taking key-tile
    items x, x + grid, ...) and the one-CTA-per-item grid, with and without the polynomial exp2 share
    (btp_attn_tune(2, 2), default), vs torch fp32: fewer query tiles than ring stages (s = 128, 256),
    an odd number of query tiles per item (s = 384, 640: the per-item phase parity alternates), item
    counts that do not divide by the grid (2 x 8 x 80 = 1280, 2 x 5 x 33 = 330 items), and fewer items
    than SMs."""
    from paper_2512_12131_b200 import _native

    lib = _native.load()
    hd = 64
    q, k, v = _inputs(b, s, h, hd, seed=7 * s + h)
    do = torch.randn(b * s, h * hd, device="cuda").bfloat16()
    o = torch.empty(b * s, h * hd, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, h, s, device="cuda")
    K.attn_fwd(q, k, v, o, lse, b=b, s=s, heads=h, head_dim=hd)
    D = torch.empty(b, h, s, device="cuda")
    acc = torch.empty(b * s, h * hd, device="cuda")
    dq, dk, dv = (torch.empty_like(o) for _ in range(3))
    prev, prev_p = lib.btp_attn_tune(7, persist), lib.btp_attn_tune(2, poly)
    try:
        K.attn_bwd(q, k, v, o, do, lse, D, acc, dq, dk, dv, b=b, s=s, heads=h, head_dim=hd)
        torch.cuda.synchronize()
    finally:
        lib.btp_attn_tune(7, prev)
        lib.btp_attn_tune(2, prev_p)
    rq, rk, rv = _ref_bwd(q, k, v, do, b, s, h, hd)
    errs = {"dq": _rel(dq, rq), "dk": _rel(dk, rk), "dv": _rel(dv, rv)}
    assert max(errs.values()) < 2e-2, errs


def test_paper_7b_width_block_native_attention_vs_oracle():
    """CoLA-7B block widths (32 heads of hd 128: the hd-128 forward / backward kernels) with native
    attention inside the BTP block, fwd + bwd vs the float64 oracle."""
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.api import train_step
    from paper_2512_12131_b200.model import RunShape, Variant, preset
    from paper_2512_12131_b200.plan import Strategy, plan
    from tests.gpu_util import BF16_TOL, inputs, oracle_step, rel

    cfg = preset("7b")
    b, s = 1, 256
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    st = train_step(pl, blk, x, G, attn_backend="native")
    assert st.executor.attn.native and st.executor.attn.hd == 128
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, cfg, b, s, sharded=False)
    errs = {"y": rel(st.y.values.reshape(-1, cfg.d), y_ref), "loss": abs(st.loss - loss_ref) / abs(loss_ref),
            "dx": rel(st.dx, g_ref["dx"])}
    for n in O.PROJECTIONS:
        errs[f"A_{n}"] = rel(st.grads["A"][n], g_ref["A"][n])
        errs[f"B_{n}"] = rel(st.grads["B"][n], g_ref["B"][n])
    bad = {k: v for k, v in errs.items() if v > BF16_TOL}
    assert not bad, bad


@pytest.mark.parametrize("ckpt", [False, True])
def test_model_step_native_attention_vs_oracle(ckpt):
    """The 2-layer model step (embedding -> BTP blocks -> head -> cross-entropy) with native attention
    in every block (and with low-rank checkpointing: the recompute runs the native forward again),
    fwd + bwd vs the float64 oracle model."""
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import ModelConfig, RunShape, Variant, build_model, token_batch
    from paper_2512_12131_b200.model_executor import model_train_step
    from paper_2512_12131_b200.plan import Strategy, plan
    from tests.gpu_util import BF16_TOL, SMALL, rel

    layers, V, b, s = 2, 256, 2, 128
    cfg = ModelConfig(layers=layers, heads=SMALL.heads, d=SMALL.d, d_ff=SMALL.d_ff, r=SMALL.r)
    mw = build_model(cfg, Variant.COLA, 0, V)
    om = O.build_model(cfg.d, cfg.d_ff, cfg.r, "cola", 0, V, layers)
    ids, tg = token_batch(b, s, V)
    loss_ref, cache = O.model_forward(om, ids, tg, b, s, cfg.heads)
    g_ref = O.model_backward(om, cache, b, s, cfg.heads)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True,
              lowrank_ckpt=ckpt)
    loss, ex = model_train_step(pl, mw, ids, tg, attn_backend="native")
    assert all(blk.attn.native for blk in ex.blocks)
    assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
    got = ex.model_grads()
    assert rel(got["dhead"], g_ref["dhead"]) < BF16_TOL
    assert rel(got["dembedding"], g_ref["dembedding"]) < BF16_TOL
    for l in range(layers):
        gr, gb = g_ref["blocks"][l], got["blocks"][l]
        for n in O.PROJECTIONS:
            assert rel(gb["A"][n], gr["A"][n]) < BF16_TOL, (l, "A", n)
            assert rel(gb["B"][n], gr["B"][n]) < BF16_TOL, (l, "B", n)
