"""TP = 2 end to end on ONE GPU: two processes (one per TP rank) share cuda:0 and talk over the
gloo backend (the box has a single GPU; NCCL refuses two ranks on one device). Every compute
site runs in libbtp.so on each rank's shard; the all-reduces / rider / gather go through the
same TPComm code the NCCL path uses. Outputs, the loss, per-rank dx shards and per-rank weight
gradient shards are compared with the float64 oracle sliced to each rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, strategy, grouping, online, ckpt, q, cfg_name="SMALL", bs=(2, 64), bdt="bf16",
               attn="auto"):
    try:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        import datetime

        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
        from tests import gpu_util
        from tests.gpu_util import inputs
        from paper_2512_12131_b200.api import make_executor, train_step
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.plan import Strategy, plan

        b, s = bs
        cfg = getattr(gpu_util, cfg_name)
        variant = Variant.FULL_RANK if strategy == "full-rank" else Variant.COLA
        blk, x, G, _ = inputs(cfg, variant, b, s)
        pl = plan(Strategy(strategy), cfg, RunShape(b, s, world), None if strategy == "full-rank" else variant,
                  online_norm=online, grouping=grouping, lowrank_ckpt=ckpt)
        ex = make_executor(pl, blk, boundary_dtype=bdt, attn_backend=attn) if (bdt != "bf16" or attn != "auto") else None
        st = train_step(pl, blk, x, G, executor=ex)
        q.put((rank, st.y.values, st.loss, st.dx, st.grads, st.trace.record_tuples("forward"),
               st.trace.record_tuples("backward"), st.trace.record_tuples("reforward"), None))
        dist.destroy_process_group()
    except Exception as exc:  # surface the failure to the parent instead of hanging it
        import traceback

        q.put((rank, None, None, None, None, None, None, None, traceback.format_exc()))


def _run_tp2(strategy, grouping, online, ckpt, world=2, cfg_name="SMALL", bs=(2, 64), bdt="bf16", attn="auto"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, strategy, grouping, online, ckpt, q, cfg_name, bs,
                                                  bdt, attn))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            item = q.get(timeout=600)
            res[item[0]] = item
            assert item[-1] is None, f"rank {item[0]} failed:\n{item[-1]}"  # fail fast; peers are killed below
    finally:
        for p in procs:
            p.join(timeout=60 if len(res) == len(procs) else 1)
            if p.is_alive():
                p.kill()
    return res


def _assert_closed_form_volume(fwd_records, strategy, b, s):
    """Traced forward block volume == the closed form (reference test_costs.py:129-145)."""
    from tests.gpu_util import SMALL
    from paper_2512_12131_b200.model import RunShape
    from paper_2512_12131_b200.plan import Strategy
    from paper_2512_12131_b200.trace import tp_block_volume

    # the closed form counts the boundary tensors; sync-norm statistics ([T] each) come on top
    traced = sum(rec[3] for rec in fwd_records if rec[2] == "block" and not rec[0].endswith("-stat"))
    assert traced == tp_block_volume(Strategy(strategy), SMALL, RunShape(b, s, 2)), (strategy, traced)


@pytest.mark.parametrize("grouping,online,ckpt", [(True, True, False), (False, True, False), (True, False, True)])
def test_btp_tp2_matches_oracle(grouping, online, ckpt):
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

    b, s = 2, 64
    res = _run_tp2("btp", grouping, online, ckpt)
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=2, online=online)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 2), Variant.COLA, online_norm=online, grouping=grouping)
    pred = [(p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]
    for rank, (_, y, loss, dx, grads, fwd, bwd, refwd, _) in res.items():
        assert rel(y.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
        gr = O.grads_for_rank(g_ref, 2, rank, SMALL.d, SMALL.d_ff)
        assert rel(dx, gr["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(grads["A"][n], gr["A"][n]) < BF16_TOL, (rank, "A", n)
            assert rel(grads["B"][n], gr["B"][n]) < BF16_TOL, (rank, "B", n)
        assert rel(grads["gamma1"], gr["dgamma1"]) < BF16_TOL
        assert rel(grads["gamma2"], gr["dgamma2"]) < BF16_TOL
        assert fwd == pred                      # real collectives == the plan's prediction
        _assert_closed_form_volume(fwd, "btp", b, s)
        assert sum(rec[3] for rec in bwd) == 7 * b * s * SMALL.r  # backward moves only rank-r tensors
        assert refwd == []                      # checkpoint recompute is collective-free


@pytest.mark.parametrize("strategy", ["vanilla"])
def test_vanilla_tp2_matches_oracle(strategy):
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant
    from paper_2512_12131_b200.plan import cola_pair_indices

    b, s = 2, 64
    res = _run_tp2(strategy, True, False, False)
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False)
    for rank, (_, y, loss, dx, grads, *_rest) in res.items():
        assert rel(y.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
        assert rel(dx, g_ref["dx"]) < BF16_TOL
        idx = cola_pair_indices(SMALL.r, 2, rank)
        for n in O.PROJECTIONS:
            assert rel(grads["B"][n], g_ref["B"][n][idx, :]) < BF16_TOL, (rank, "B", n)
            assert rel(grads["A"][n], g_ref["A"][n][:, idx]) < BF16_TOL, (rank, "A", n)
        _assert_closed_form_volume(_rest[0], "vanilla", b, s)


def test_full_rank_tp2_matches_oracle():
    """Megatron column->row TP=2 of the full-rank block (the comparison point) vs the oracle."""
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant

    b, s = 2, 64
    res = _run_tp2("full-rank", True, False, False)
    blk, x, G, oblk = inputs(SMALL, Variant.FULL_RANK, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False)
    dl, fl = SMALL.d // 2, SMALL.d_ff // 2
    for rank, (_, y, loss, dx, grads, fwd, bwd, *_r) in res.items():
        assert rel(y.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
        assert rel(dx, g_ref["dx"]) < BF16_TOL
        sl, fsl = slice(rank * dl, (rank + 1) * dl), slice(rank * fl, (rank + 1) * fl)
        want = {"q": g_ref["W"]["q"][sl], "k": g_ref["W"]["k"][sl], "v": g_ref["W"]["v"][sl],
                "o": g_ref["W"]["o"][:, sl], "gate": g_ref["W"]["gate"][fsl], "up": g_ref["W"]["up"][fsl],
                "down": g_ref["W"]["down"][:, fsl]}
        for n, w in want.items():
            assert rel(grads["W"][n], w) < BF16_TOL, (rank, n)
        assert [r[0] for r in fwd] == ["attn", "mlp"]
        _assert_closed_form_volume(fwd, "full-rank", b, s)


@pytest.mark.parametrize("world", [4, 8])
def test_btp_tp4_tp8_c60m_matches_oracle(world):
    """CoLA-60M (d512, 8 heads, d_ff 1376, r128) at TP=4 and TP=8, one process per rank on one GPU:
    at TP=8 each rank owns 64 residual columns, one head and 172 d_ff columns (zero-padded to 176
    for 16-byte TMA strides)."""
    from tests.gpu_util import BF16_TOL, C60M, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

    b, s = 2, 128  # (2, 64) has a near-cancelling loss (-1.43 out of sum|y*G| = 16379): ill-conditioned
    res = _run_tp2("btp", True, True, False, world=world, cfg_name="C60M", bs=(b, s))
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, C60M, b, s, tp=world, online=True, sharded=False)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, world), Variant.COLA, online_norm=True, grouping=True)
    pred = [(p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]
    assert len(res) == world
    for rank, (_, y, loss, dx, grads, fwd, bwd, _refwd, _) in res.items():
        assert rel(y.reshape(-1, C60M.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
        gr = O.grads_for_rank(g_ref, world, rank, C60M.d, C60M.d_ff)
        assert rel(dx, gr["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(grads["A"][n], gr["A"][n]) < BF16_TOL, (rank, "A", n)
            assert rel(grads["B"][n], gr["B"][n]) < BF16_TOL, (rank, "B", n)
        assert rel(grads["gamma1"], gr["dgamma1"]) < BF16_TOL
        assert rel(grads["gamma2"], gr["dgamma2"]) < BF16_TOL
        assert fwd == pred
        assert sum(rec[3] for rec in bwd) == 7 * b * s * C60M.r


def test_btp_tp2_sliced_forward_boundaries():
    """T = 2048: the forward chunk boundaries pipeline over two token slices (async all-reduce of
    slice 0 under the down GEMM of slice 1), across two real ranks."""
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

    b, s = 2, 1024
    res = _run_tp2("btp", True, True, False, bs=(b, s))
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=2, sharded=False)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 2), Variant.COLA, online_norm=True, grouping=True)
    pred = [(p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]
    # L = sum(y * G) nearly cancels at this shape (|L| ~ 2 of sum|y*G| ~ 1e5): judge the loss error
    # against the magnitude of its terms
    scale = float(np.sum(np.abs(y_ref * G.values.reshape(-1, SMALL.d))))
    for rank, (_, y, loss, dx, grads, fwd, _bwd, _rf, _) in res.items():
        assert rel(y.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / scale < BF16_TOL
        gr = O.grads_for_rank(g_ref, 2, rank, SMALL.d, SMALL.d_ff)
        assert rel(dx, gr["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(grads["A"][n], gr["A"][n]) < BF16_TOL, (rank, "A", n)
            assert rel(grads["B"][n], gr["B"][n]) < BF16_TOL, (rank, "B", n)
        assert fwd == pred  # one record per chunk boundary although each is issued in slices


@pytest.mark.parametrize("world,ckpt", [(2, False), (8, False), (4, True)])
def test_btp_tp2_paper_7b_widths(world, ckpt):
    """CoLA-7B block widths (d 4096, d_ff 11008, r 1024) at TP=2 and TP=8 (BASELINE configs[2]'s
    sharding), short sequence: a TP=8 rank owns 512 residual columns, 4 heads, 1376 d_ff columns;
    TP=4 with the low-rank checkpoint is configs[4]'s path (its re-forward must stay collective-free)."""
    from tests.gpu_util import BF16_TOL, P7B, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant

    b, s = 1, 256
    res = _run_tp2("btp", True, True, ckpt, world=world, cfg_name="P7B", bs=(b, s))
    assert len(res) == world
    blk, x, G, oblk = inputs(P7B, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, P7B, b, s, tp=world, sharded=False)
    for rank, (_, y, loss, dx, grads, fwd, bwd, *_r) in res.items():
        assert rel(y.reshape(-1, P7B.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / abs(loss_ref) < BF16_TOL
        gr = O.grads_for_rank(g_ref, world, rank, P7B.d, P7B.d_ff)
        assert rel(dx, gr["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(grads["A"][n], gr["A"][n]) < BF16_TOL, (rank, "A", n)
            assert rel(grads["B"][n], gr["B"][n]) < BF16_TOL, (rank, "B", n)
        if ckpt:
            assert _r[0] == []  # re-forward records no collective


@pytest.mark.parametrize("cfg_name,bs", [("C60M", (2, 128)), ("P7B", (1, 256))])
def test_btp_tp8_fp32_boundary_margin(cfg_name, bs):
    """TP = 8 with the forward rank-r boundaries reduced in fp32 (boundary_dtype="fp32": one bf16
    rounding of the cross-rank sum instead of one per ring hop): every tensor within 1.7e-2 — the
    bf16 bar (2e-2) with >= 15 % headroom (bf16 boundaries: 1.98e-2 at C60M, 1.86e-2 at 7B widths;
    scripts/margin_probe2.py)."""
    from tests import gpu_util
    from tests.gpu_util import inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant

    cfg = getattr(gpu_util, cfg_name)
    b, s = bs
    world = 8
    res = _run_tp2("btp", True, True, False, world=world, cfg_name=cfg_name, bs=(b, s), bdt="fp32")
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, cfg, b, s, tp=world, sharded=False)
    worst = {}
    for rank, (_, y, loss, dx, grads, fwd, bwd, *_r) in res.items():
        gr = O.grads_for_rank(g_ref, world, rank, cfg.d, cfg.d_ff)
        errs = {"y": rel(y.reshape(-1, cfg.d), y_ref), "dx": rel(dx, gr["dx"]),
                "g1": rel(grads["gamma1"], gr["dgamma1"]), "g2": rel(grads["gamma2"], gr["dgamma2"])}
        for n in O.PROJECTIONS:
            errs["A_" + n] = rel(grads["A"][n], gr["A"][n])
            errs["B_" + n] = rel(grads["B"][n], gr["B"][n])
        for k, v in errs.items():
            worst[k] = max(worst.get(k, 0.0), v)
    top = max(worst, key=worst.get)
    print(f"{cfg_name} TP=8 fp32 boundaries: worst {top} = {worst[top]:.3e}")
    assert worst[top] < 1.7e-2, worst


@pytest.mark.parametrize("cfg_name,bs", [("C60M", (2, 128)), ("P7B", (1, 256))])
@pytest.mark.parametrize("bdt", ["bf16", "fp32"])
def test_btp_tp8_whole_tensor_margin(cfg_name, bs, bdt):
    """TP = 8, errors of the WHOLE gradient tensors (the north_star's "within 2e-2 relative on
    gradients"): the relative Frobenius error of the concatenated per-rank shards,
    sqrt(sum_r |got_r - ref_r|^2) / sqrt(sum_r |ref_r|^2). The per-shard worst case (above) is a
    stricter statistic: a TP=8 rank's d-shard of dgamma2 is only d/8 = 64 elements at C60M, so its
    relative error is a noisier small-sample estimate of the same per-element error. Measured
    (r02k): whole-tensor worst 1.87e-2 / 1.79e-2 (C60M / 7B widths, bf16 boundaries: the up-factor
    gradients dA, through a = sigma(z) of the bf16-reduced z), 1.40e-2 / 1.34e-2 with fp32 forward
    boundaries -- within ~10 % of the TP=1 level (1.27e-2 / 1.22e-2), which is bf16 storage
    (DESIGN.md section 4), so TP adds almost nothing once the forward boundary sums in fp32."""
    from tests import gpu_util
    from tests.gpu_util import inputs, oracle_step
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant

    cfg = getattr(gpu_util, cfg_name)
    b, s = bs
    world = 8
    res = _run_tp2("btp", True, True, False, world=world, cfg_name=cfg_name, bs=(b, s), bdt=bdt)
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, cfg, b, s, tp=world, sharded=False)
    num, den, shard_worst = {}, {}, {}

    def acc(key, got, want):
        got = np.asarray(got, dtype=np.float64).reshape(np.shape(want))
        want = np.asarray(want, dtype=np.float64)
        e, w = float(np.sum((got - want) ** 2)), float(np.sum(want ** 2))
        num[key] = num.get(key, 0.0) + e
        den[key] = den.get(key, 0.0) + w
        shard_worst[key] = max(shard_worst.get(key, 0.0), (e / max(w, 1e-300)) ** 0.5)

    for rank, (_, y, loss, dx, grads, *_r) in res.items():
        gr = O.grads_for_rank(g_ref, world, rank, cfg.d, cfg.d_ff)
        if rank == 0:
            acc("y", y.reshape(-1, cfg.d), y_ref)  # y is gathered on every rank
        acc("dx", dx, gr["dx"])
        acc("g1", grads["gamma1"], gr["dgamma1"])
        acc("g2", grads["gamma2"], gr["dgamma2"])
        for n in O.PROJECTIONS:
            acc("A_" + n, grads["A"][n], gr["A"][n])
            acc("B_" + n, grads["B"][n], gr["B"][n])
    whole = {k: (num[k] / max(den[k], 1e-300)) ** 0.5 for k in num}
    top, stop = max(whole, key=whole.get), max(shard_worst, key=shard_worst.get)
    print(f"{cfg_name} TP=8 {bdt} boundaries: whole-tensor worst {top} = {whole[top]:.3e}; "
          f"per-shard worst {stop} = {shard_worst[stop]:.3e}; whole g2 = {whole['g2']:.3e}")
    assert whole[top] < (2e-2 if bdt == "bf16" else 1.5e-2), whole
    assert shard_worst[stop] < (2e-2 if bdt == "bf16" else 1.7e-2), shard_worst


@pytest.mark.parametrize("attn", ["cudnn", "native", "hybrid"])
def test_btp_tp2_attention_backends_match_oracle(attn):
    """TP = 2 (two processes, gloo) at s = 128 with cuDNN ("auto") and with the native attention
    kernels on each rank's heads (2 of 4), fwd + bwd vs the float64 oracle sliced per rank. The loss
    L = sum(y * G) nearly cancels here (|L| ~ 1.5 against 65 k O(1) terms), so its error is bounded
    the well-conditioned way, |dL| <= ||dy|| ||G||, relative to ||y|| ||G||."""
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import Variant

    b, s = 2, 128
    res = _run_tp2("btp", True, True, False, bs=(b, s), attn=attn)
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=2, online=True)
    scale = float(np.linalg.norm(y_ref) * np.linalg.norm(G.values))
    for rank, (_, y, loss, dx, grads, *_rest) in res.items():
        assert rel(y.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(loss - loss_ref) / scale < BF16_TOL
        gr = O.grads_for_rank(g_ref, 2, rank, SMALL.d, SMALL.d_ff)
        assert rel(dx, gr["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(grads["A"][n], gr["A"][n]) < BF16_TOL, (rank, "A", n)
            assert rel(grads["B"][n], gr["B"][n]) < BF16_TOL, (rank, "B", n)
