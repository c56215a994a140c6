"""Multi-layer model step on the GPU vs the float64 oracle model: embedding
shard -> L BTP blocks -> tail all-gather -> final RMSNorm -> replicated LM head -> fused
cross-entropy, forward + backward, at the north_star bf16 tolerance; the graph-replayed trainer
with AdamW; and TP = 2 (two ranks on one GPU over gloo) vs the oracle sliced per rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

L, V, B, S = 2, 256, 2, 64


def _setup(variant="cola", layers=L):
    from tests.gpu_util import SMALL
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.model import ModelConfig, Variant, build_model, token_batch

    cfg = ModelConfig(layers=layers, heads=SMALL.heads, d=SMALL.d, d_ff=SMALL.d_ff, r=SMALL.r)
    mw = build_model(cfg, Variant(variant), 0, V)
    om = O.build_model(cfg.d, cfg.d_ff, cfg.r, variant, 0, V, layers)
    ids, tg = token_batch(B, S, V)
    loss, cache = O.model_forward(om, ids, tg, B, S, cfg.heads)
    g = O.model_backward(om, cache, B, S, cfg.heads)
    return cfg, mw, ids, tg, loss, g


def _check_grads(got, want, tp=1, rank=0, cfg=None):
    from tests.gpu_util import BF16_TOL, rel
    from oracle import btp_oracle as O

    dl = cfg.d // tp
    sl = slice(rank * dl, (rank + 1) * dl)
    assert rel(got["dhead"], want["dhead"]) < BF16_TOL
    assert rel(got["dfinal_gamma"], want["dfinal_gamma"]) < BF16_TOL
    assert rel(got["dembedding"], want["dembedding"][:, sl]) < BF16_TOL
    for l in range(len(want["blocks"])):
        gr = O.grads_for_rank(want["blocks"][l], tp, rank, cfg.d, cfg.d_ff)
        gb = got["blocks"][l]
        for n in O.PROJECTIONS:
            assert rel(gb["A"][n], gr["A"][n]) < BF16_TOL, (l, "A", n)
            assert rel(gb["B"][n], gr["B"][n]) < BF16_TOL, (l, "B", n)
        assert rel(gb["gamma1"], gr["dgamma1"]) < BF16_TOL, (l, "gamma1")
        assert rel(gb["gamma2"], gr["dgamma2"]) < BF16_TOL, (l, "gamma2")


@pytest.mark.parametrize("grouping,ckpt", [(True, False), (False, False), (True, True)])
def test_model_step_matches_oracle(grouping, ckpt):
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.model_executor import model_train_step
    from paper_2512_12131_b200.plan import Strategy, plan

    cfg, mw, ids, tg, loss_ref, g_ref = _setup()
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(B, S, 1), Variant.COLA, online_norm=True, grouping=grouping,
              lowrank_ckpt=ckpt)
    loss, ex = model_train_step(pl, mw, ids, tg)
    assert abs(loss - loss_ref) / abs(loss_ref) < 2e-2
    _check_grads(ex.model_grads(), g_ref, cfg=cfg)
    # collective log: every block's 4 (or 7) forward chunk boundaries, then the tail gather
    fwd = ex.comm.trace.record_tuples("forward")
    assert fwd[-1][0] == "final-gather" and len(fwd) == L * (4 if grouping else 7) + 1


@pytest.mark.parametrize("grouping,ckpt", [(True, False), (False, False), (True, True)])
def test_lax_model_chains_the_bundle(grouping, ckpt):
    """lax model: block l's h_cur feeds block l+1's merge, and dL/dh_prev flows back into block
    l's dz — every block's gradients against the oracle model (3 layers: two merges)."""
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.model_executor import model_train_step
    from paper_2512_12131_b200.plan import Strategy, plan

    cfg, mw, ids, tg, loss_ref, g_ref = _setup("lax", 3)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(B, S, 1), Variant.LAX, online_norm=True, grouping=grouping,
              lowrank_ckpt=ckpt)
    loss, ex = model_train_step(pl, mw, ids, tg)
    assert abs(loss - loss_ref) / abs(loss_ref) < 2e-2
    _check_grads(ex.model_grads(), g_ref, cfg=cfg)
    assert not ex.blocks[0].has_h_prev and ex.blocks[1].has_h_prev and ex.blocks[2].has_h_prev


def test_model_trainer_graph_replay_and_adamw():
    from paper_2512_12131_b200.api import ModelTrainer
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan

    cfg, mw, ids, tg, loss_ref, _ = _setup()
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(B, S, 1), Variant.COLA, online_norm=True, grouping=True)
    tr = ModelTrainer(pl, mw, adamw=dict(lr=2e-3, wd=0.0))
    x, g = tr.device_inputs(ids, tg)
    tr.step_device(x, g)                      # eager first step (allocates), then capture
    first = float(tr.loss_buf.item())
    assert abs(first - loss_ref) / loss_ref < 2e-2
    xh, gh = tr.pinned_host_inputs(ids, tg)
    losses = tr.fit([xh] * 12, gh)            # pinned packed (ids, targets) batches, graph replays
    assert tr.graphed
    assert all(np.isfinite(losses)) and losses[-1] < first - 0.05  # AdamW fits the fixed batch


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, q, variant="cola", layers=L):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.model_executor import model_train_step
        from paper_2512_12131_b200.plan import Strategy, plan

        cfg, mw, ids, tg, _, _ = _setup(variant, layers)
        pl = plan(Strategy.BOTTLENECK, cfg, RunShape(B, S, world), Variant(variant), online_norm=True, grouping=True)
        loss, ex = model_train_step(pl, mw, ids, tg)
        q.put((rank, loss, ex.model_grads(), ex.comm.trace.record_tuples("forward"), None))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, None, None, None, traceback.format_exc()))


@pytest.mark.parametrize("variant,layers", [("cola", L), ("lax", 3)])
def test_model_tp2_matches_oracle(variant, layers):
    cfg, _, _, _, loss_ref, g_ref = _setup(variant, layers)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, variant, layers)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            item = q.get(timeout=600)
            assert item[-1] is None, f"rank {item[0]} failed:\n{item[-1]}"
            res[item[0]] = item
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank, (_, loss, grads, fwd, _) in res.items():
        assert abs(loss - loss_ref) / abs(loss_ref) < 2e-2
        _check_grads(grads, g_ref, tp=2, rank=rank, cfg=cfg)
        assert fwd[-1][:3] == ("final-gather", "all-gather", "boundary")


def test_lowrank_ckpt_frees_device_memory():
    """with low-rank ckpt the recomputable activations of all blocks live in ONE
    scratch set shared by the blocks, so the model's peak device memory drops (not just the
    saved-tensor bookkeeping), and the step still matches the non-ckpt step closely."""
    import gc

    from paper_2512_12131_b200.model import ModelConfig, RunShape, Variant, build_model, token_batch
    from paper_2512_12131_b200.model_executor import model_train_step
    from paper_2512_12131_b200.plan import Strategy, plan

    layers, b, s = 6, 2, 512
    cfg = ModelConfig(layers=layers, heads=8, d=512, d_ff=1376, r=128)
    mw = build_model(cfg, Variant.COLA, 0, V)
    ids, tg = token_batch(b, s, V)
    peaks, losses = {}, {}
    for ckpt in (False, True):
        gc.collect()
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        base = torch.cuda.memory_allocated()
        torch.cuda.reset_peak_memory_stats()
        pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True,
                  lowrank_ckpt=ckpt)
        loss, ex = model_train_step(pl, mw, ids, tg)
        torch.cuda.synchronize()
        peaks[ckpt] = torch.cuda.max_memory_allocated() - base
        losses[ckpt] = loss
        del ex
    T = b * s
    # per block, ckpt drops at least qkv + attn + x_mid + 2 x gu + act + a_* (bf16) minus one shared set
    per_block = 2 * T * (3 * cfg.d + cfg.d + cfg.d + 3 * cfg.d_ff + 7 * cfg.r)
    assert peaks[False] - peaks[True] > 0.5 * (layers - 1) * per_block, peaks
    assert abs(losses[True] - losses[False]) <= 1e-3 * abs(losses[False])
