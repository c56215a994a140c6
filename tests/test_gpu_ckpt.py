"""Low-rank boundary checkpointing on the device, BTP vs the naive-TP baseline at TP = 2 (two
gloo ranks sharing the GPU), mirroring the reference's test_ckpt.py:79-125: the BTP re-forward is
collective-free, the vanilla one replays its chunk all-reduces (3 grouped / 6 ungrouped; the down
chunk's output feeds nothing backward needs), both rebuild every tensor BITWISE, BTP frees less
memory, and ΔMem / eff_ckpt order the two strategies as the reference itself does at this shape
(tests/golden/ckpt_small.json) — and the checkpointed training step still matches the oracle."""

import json
import os
import socket

from pathlib import Path

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

REF_CKPT = json.loads((Path(__file__).resolve().parent / "golden" / "ckpt_small.json").read_text())


def _port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _rank_main(rank, world, port, q):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
        from tests.gpu_util import SMALL, inputs
        from paper_2512_12131_b200.checkpointing import CkptPolicy, eff_ckpt, run_with_ckpt
        from paper_2512_12131_b200.model import RunShape, Variant, seeded_h_prev
        from paper_2512_12131_b200.plan import Strategy, plan

        b, s = 2, 64
        out = {}
        for strategy in ("btp", "vanilla"):
            for variant in ("svd", "lax", "cola"):
                for grouping in (True, False):
                    var = Variant(variant)
                    blk, x, _, _ = inputs(SMALL, var, b, s)
                    hp = seeded_h_prev(SMALL, RunShape(b, s, world), 5) if var is Variant.LAX else None
                    pl = plan(Strategy(strategy), SMALL, RunShape(b, s, world), var,
                              online_norm=strategy == "btp", grouping=grouping)
                    run = run_with_ckpt(pl, blk, x, CkptPolicy.LOWRANK_BOUNDARY, hp)
                    rp = run.report
                    out[(strategy, variant, grouping)] = dict(
                        ok=run.recompute_bitwise_ok, checks=run.recompute_checks, calls=rp.reforward_collectives,
                        ring=rp.reforward_ring_elements, dmem=rp.delta_mem_elements, eff=float(eff_ckpt(rp)),
                        flops=rp.recompute_flops)
        q.put((rank, out, None))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, None, traceback.format_exc()))


def test_ckpt_btp_vs_vanilla_tp2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in procs:
            rank, out, err = q.get(timeout=600)
            assert err is None, f"rank {rank} failed:\n{err}"
            res[rank] = out
    finally:
        for p in procs:
            p.join(timeout=60 if len(res) == 2 else 1)
            if p.is_alive():
                p.kill()
    for rank, out in res.items():
        for (strategy, variant, grouping), o in out.items():
            key = (rank, strategy, variant, grouping)
            assert o["ok"], (key, o["checks"])
            assert o["flops"] > 0, key
            if strategy == "btp":
                assert o["calls"] == 0 and o["ring"] == 0, key
            else:
                assert o["calls"] == (3 if grouping else 6) and o["ring"] > 0, key
        # the reference itself at this shape (tests/golden/ckpt_small.json, make_ckpt_golden.py):
        # same collective counts and ring elements; ΔMem and eff_ckpt in the reference's ORDER
        for (strategy, variant, grouping), o in out.items():
            ref = REF_CKPT[f"{strategy}/{variant}/{int(grouping)}"]
            assert o["calls"] == ref["reforward_collectives"], (strategy, variant, grouping)
            assert o["ring"] == ref["reforward_ring_elements"], (strategy, variant, grouping, o["ring"])
        for variant in ("svd", "lax", "cola"):
            van, btp = out[("vanilla", variant, True)], out[("btp", variant, True)]
            rv, rb = REF_CKPT[f"vanilla/{variant}/1"], REF_CKPT[f"btp/{variant}/1"]
            assert van["dmem"] > btp["dmem"] > 0, (rank, variant)
            assert rv["delta_mem_elements"] > rb["delta_mem_elements"]
            assert (btp["eff"] > van["eff"]) == (rb["eff_ckpt"] > rv["eff_ckpt"]), (rank, variant, btp, van)


def test_ckpt_vanilla_train_step_matches_oracle():
    """The checkpointed naive-TP step (re-forward in backward) at TP = 1 against the oracle."""
    from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
    from oracle import btp_oracle as O
    from paper_2512_12131_b200.api import train_step
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan

    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    for grouping in (True, False):
        pl = plan(Strategy.VANILLA, SMALL, RunShape(b, s, 1), Variant.COLA, grouping=grouping, lowrank_ckpt=True)
        st = train_step(pl, blk, x, G)
        y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False)
        assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
        assert rel(st.dx, g_ref["dx"]) < BF16_TOL
        for n in O.PROJECTIONS:
            assert rel(st.grads["A"][n], g_ref["A"][n]) < BF16_TOL, n
            assert rel(st.grads["B"][n], g_ref["B"][n]) < BF16_TOL, n
        assert len(st.trace.record_tuples("reforward")) == (3 if grouping else 6)


@pytest.mark.parametrize("variant", ["cola", "svd"])
@pytest.mark.parametrize("grouping", [True, False])
def test_ckpt_recompute_bitwise_with_fused_sigma_epilogue(variant, grouping):
    """TP = 1 at r = 128 (CoLA-60M widths): the forward's crossgate runs in the down-GEMM epilogue
    while the checkpoint recompute runs btp_fixup_sigma — both must use the same SiLU so the
    recomputed activations equal the forward's bitwise."""
    from tests.gpu_util import C60M, inputs
    from paper_2512_12131_b200 import executor as E
    from paper_2512_12131_b200.checkpointing import CkptPolicy, run_with_ckpt
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan

    assert E.FUSE_SIGMA
    b, s = 2, 128
    blk, x, _, _ = inputs(C60M, Variant(variant), b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant(variant), online_norm=True, grouping=grouping)
    run = run_with_ckpt(pl, blk, x, CkptPolicy.LOWRANK_BOUNDARY)
    assert run.recompute_bitwise_ok, run.recompute_checks
    assert run.report.reforward_collectives == 0
