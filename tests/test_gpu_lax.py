"""LaX variant on the device path (reference simulator.py:247-265, model.py:249-253): after each
chunk's reduction the up-projection consumes a = z + h_prev[projection] (btp_add), and the block
returns h_cur = z for the next layer. Checked against the float64 oracle (itself pinned to the
reference's lax goldens, tests/test_oracle_golden.py): every intermediate, the h_cur bundle, all
weight gradients, dx, the loss and dL/dh_prev; without a bundle lax must be bitwise the svd block
(reference test_model.py:182-192)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
from oracle import btp_oracle as O
from paper_2512_12131_b200.api import execute_forward, train_step
from paper_2512_12131_b200.model import RunShape, Variant, seeded_h_prev
from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4


def _check_step(st, y_ref, g_ref, loss_ref, tol, cfg=SMALL, grads_rank=None):
    assert rel(st.y.values.reshape(-1, cfg.d), y_ref) < tol
    assert abs(st.loss - loss_ref) / abs(loss_ref) < tol
    gr = g_ref if grads_rank is None else grads_rank
    errs = {"dx": rel(st.dx, gr["dx"]), "gamma1": rel(st.grads["gamma1"], gr["dgamma1"]),
            "gamma2": rel(st.grads["gamma2"], gr["dgamma2"])}
    for n in O.PROJECTIONS:
        errs[f"A_{n}"] = rel(st.grads["A"][n], gr["A"][n])
        errs[f"B_{n}"] = rel(st.grads["B"][n], gr["B"][n])
    for n in O.PROJECTIONS:
        errs[f"h_{n}"] = rel(st.h_cur[n].values, g_ref["h_cur"][n])
        if "dh_prev" in g_ref:
            errs[f"dh_{n}"] = rel(st.dh_prev[n], g_ref["dh_prev"][n])
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, bad


@pytest.mark.parametrize("online", [True, False])
@pytest.mark.parametrize("grouping", [True, False])
@pytest.mark.parametrize("hp_seed", [9, None])
def test_lax_forward_workspaces(online, grouping, hp_seed):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 1), hp_seed) if hp_seed is not None else None
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.LAX, online_norm=online, grouping=grouping)
    res = execute_forward(pl, blk, x, hp, capture_workspaces=True)
    y_ref, g_ref, ws_ref, _ = oracle_step(oblk, x, G, SMALL, b, s, online=online, h_prev=hp)
    assert rel(res.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
    bad = {n: rel(res.workspaces[0][n], w) for n, w in ws_ref[0].items() if n != "x"}
    bad = {n: e for n, e in bad.items() if e > BF16_TOL}
    assert not bad, bad
    assert set(ws_ref[0]) <= set(res.workspaces[0]), set(ws_ref[0]) - set(res.workspaces[0])
    for n in O.PROJECTIONS:
        assert rel(res.h_cur[n].values, g_ref["h_cur"][n]) < BF16_TOL, n
    assert res.trace.record_tuples("forward") == [
        (p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)
    ]


@pytest.mark.parametrize("grouping,online,ckpt", [(True, True, False), (False, True, False), (True, False, False),
                                                  (True, True, True), (False, False, True)])
def test_lax_train_step(grouping, online, ckpt):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 1), 5)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.LAX, online_norm=online, grouping=grouping,
              lowrank_ckpt=ckpt)
    st = train_step(pl, blk, x, G, h_prev=hp)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, online=online, h_prev=hp)
    _check_step(st, y_ref, g_ref, loss_ref, BF16_TOL)
    assert st.trace.record_tuples("reforward") == []


def test_lax_fp32_mode():
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 1), 5)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.LAX, online_norm=True, grouping=True)
    st = train_step(pl, blk, x, G, h_prev=hp, precision="fp32")
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, h_prev=hp)
    _check_step(st, y_ref, g_ref, loss_ref, FP32_TOL)


def test_lax_without_bundle_is_bitwise_svd():
    b, s = 2, 64
    out = {}
    for var in (Variant.SVD, Variant.LAX):
        blk, x, G, _ = inputs(SMALL, var, b, s)
        pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), var, online_norm=True, grouping=True)
        out[var] = train_step(pl, blk, x, G)
    a, l = out[Variant.SVD], out[Variant.LAX]
    assert np.array_equal(a.y.values, l.y.values) and np.array_equal(a.dx, l.dx) and a.loss == l.loss
    for fam in ("A", "B"):
        for n in O.PROJECTIONS:
            assert np.array_equal(a.grads[fam][n], l.grads[fam][n]), (fam, n)
    assert l.dh_prev is None and a.h_cur is None and set(l.h_cur) == set(O.PROJECTIONS)


def test_lax_ckpt_recompute_bitwise():
    from paper_2512_12131_b200.checkpointing import CkptPolicy, run_with_ckpt

    b, s = 2, 64
    blk, x, G, _ = inputs(SMALL, Variant.LAX, b, s)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.LAX, online_norm=True, grouping=True)
    run = run_with_ckpt(pl, blk, x, CkptPolicy.LOWRANK_BOUNDARY, seeded_h_prev(SMALL, RunShape(b, s, 1), 5))
    assert run.recompute_bitwise_ok, run.recompute_checks
    assert run.report.reforward_collectives == 0


# ---------------------------------------------------------------- TP = 2 (two gloo ranks on one GPU)
def _port():
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    p = sk.getsockname()[1]
    sk.close()
    return p


def _rank_main(rank, world, port, online, grouping, q, strategy="btp"):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=180))
        b, s = 2, 64
        blk, x, G, _ = inputs(SMALL, Variant.LAX, b, s)
        hp = seeded_h_prev(SMALL, RunShape(b, s, world), 5)
        pl = plan(Strategy(strategy), SMALL, RunShape(b, s, world), Variant.LAX, online_norm=online,
                  grouping=grouping)
        st = train_step(pl, blk, x, G, h_prev=hp)
        q.put((rank, dict(y=st.y.values, loss=st.loss, dx=st.dx, grads=st.grads,
                          h_cur={n: t.values for n, t in st.h_cur.items()}, dh_prev=st.dh_prev,
                          fwd=st.trace.record_tuples("forward")), None))
        dist.destroy_process_group()
    except Exception:
        import traceback

        q.put((rank, None, traceback.format_exc()))


def _spawn_tp2(online, grouping, strategy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, online, grouping, q, strategy)) for r in range(2)]
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
    return res


@pytest.mark.parametrize("online,grouping", [(True, True), (False, False)])
def test_lax_tp2_matches_oracle(online, grouping):
    res = _spawn_tp2(online, grouping, "btp")
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 2), 5)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, tp=2, online=online, h_prev=hp)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 2), Variant.LAX, online_norm=online, grouping=grouping)
    pred = [(p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]
    for rank, o in res.items():
        assert rel(o["y"].reshape(-1, SMALL.d), y_ref) < BF16_TOL
        assert abs(o["loss"] - loss_ref) / abs(loss_ref) < BF16_TOL
        gr = O.grads_for_rank(g_ref, 2, rank, SMALL.d, SMALL.d_ff)
        errs = {"dx": rel(o["dx"], gr["dx"])}
        for n in O.PROJECTIONS:
            errs[f"A_{n}"] = rel(o["grads"]["A"][n], gr["A"][n])
            errs[f"B_{n}"] = rel(o["grads"]["B"][n], gr["B"][n])
            errs[f"h_{n}"] = rel(o["h_cur"][n], g_ref["h_cur"][n])      # replicated on every rank
            errs[f"dh_{n}"] = rel(o["dh_prev"][n], g_ref["dh_prev"][n])  # the reduced da: replicated
        bad = {k: v for k, v in errs.items() if v > BF16_TOL}
        assert not bad, (rank, bad)
        assert o["fwd"] == pred


# ---------------------------------------------------------------- naive-TP baseline with lax
def _vanilla_check(o, g_ref, y_ref, loss_ref, tp, rank):
    from paper_2512_12131_b200.plan import col_shard_bounds

    lo, hi = col_shard_bounds(SMALL.r, tp, rank)
    assert rel(o["y"].reshape(-1, SMALL.d), y_ref) < BF16_TOL
    assert abs(o["loss"] - loss_ref) / abs(loss_ref) < BF16_TOL
    errs = {"dx": rel(o["dx"], g_ref["dx"])}   # replicated residual: full dx on every rank
    for n in O.PROJECTIONS:
        errs[f"A_{n}"] = rel(o["grads"]["A"][n], g_ref["A"][n][:, lo:hi])
        errs[f"B_{n}"] = rel(o["grads"]["B"][n], g_ref["B"][n][lo:hi, :])
        errs[f"h_{n}"] = rel(o["h_cur"][n], g_ref["h_cur"][n])       # gathered over the r-slices
        errs[f"dh_{n}"] = rel(o["dh_prev"][n], g_ref["dh_prev"][n])
    bad = {k: v for k, v in errs.items() if v > BF16_TOL}
    assert not bad, (rank, bad)


@pytest.mark.parametrize("grouping", [True, False])
def test_lax_vanilla_tp1(grouping):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 1), 5)
    pl = plan(Strategy.VANILLA, SMALL, RunShape(b, s, 1), Variant.LAX, online_norm=False, grouping=grouping)
    st = train_step(pl, blk, x, G, h_prev=hp)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False, h_prev=hp)
    o = dict(y=st.y.values, loss=st.loss, dx=st.dx, grads=st.grads, dh_prev=st.dh_prev,
             h_cur={n: t.values for n, t in st.h_cur.items()})
    _vanilla_check(o, g_ref, y_ref, loss_ref, 1, 0)


def test_lax_vanilla_tp2():
    res = _spawn_tp2(False, True, "vanilla")
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.LAX, b, s)
    hp = seeded_h_prev(SMALL, RunShape(b, s, 2), 5)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False, h_prev=hp)
    for rank, o in res.items():
        _vanilla_check(o, g_ref, y_ref, loss_ref, 2, rank)
