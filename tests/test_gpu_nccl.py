"""The NCCL code path of the TP communicator on the single-GPU box.

NCCL refuses two ranks on one device, so the multi-rank numerics are covered over gloo
(test_gpu_tp2.py). Here a ONE-rank NCCL process group runs the same step with every collective
really issued (`TPComm(force=True)`): in-place all-reduces, the coalesced bf16+fp32 rider inside
one NCCL group, the forward boundaries pipelined over token slices with async (coalesced)
all-reduces, the async backward all-reduce handles overlapping the weight-gradient GEMM, the
loss all-reduce and the tail all-gather. A one-rank sum is the identity, so y, the loss and dx must be
bit-identical to the record-only tp == 1 run (weight gradients to fp32 reduce-add order)."""

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


def _main(port, q):
    try:
        import datetime

        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, timeout=datetime.timedelta(seconds=120),
                                device_id=torch.device("cuda", 0))
        from tests.gpu_util import SMALL, inputs
        from paper_2512_12131_b200.api import BlockTrainer, make_executor, train_step
        from paper_2512_12131_b200.comm import TPComm
        from paper_2512_12131_b200.model import RunShape, Variant
        from paper_2512_12131_b200.plan import Strategy, plan
        from paper_2512_12131_b200.trace import Trace

        from paper_2512_12131_b200 import executor as E

        E.FUSE_SIGMA = False  # live collectives separate GEMM and sigma; compare like with like
        b, s = 4, 1024       # T = 4096: the forward boundaries pipeline over 4 token slices
        blk, x, G, _ = inputs(SMALL, Variant.COLA, b, s)
        out = {}
        for grouping in (True, False):
            pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.COLA, online_norm=True,
                      grouping=grouping)
            ref = train_step(pl, blk, x, G)
            ex = make_executor(pl, blk, comm=TPComm(1, 0, trace=Trace(), force=True))
            assert ex.comm.live and dist.get_backend() == "nccl"
            assert ex.fwd_slices == (4 if grouping else 1)
            got = train_step(pl, blk, x, G, executor=ex)
            torch.cuda.synchronize()
            same = {"y": np.array_equal(ref.y.values, got.y.values), "loss": ref.loss == got.loss,
                    "dx": np.array_equal(ref.dx, got.dx)}
            # weight gradients: split-K partials meet in an fp32 reduce-add whose order is not fixed
            for fam in ("A", "B"):
                for n, g in ref.grads[fam].items():
                    e = float(np.linalg.norm(g - got.grads[fam][n]) / np.linalg.norm(g))
                    # the q factors also inherit dQ's run-to-run rounding: the attention backward
                    # reduce-adds each key tile's fp32 dQ contribution in unfixed order before the bf16
                    # rounding, so a few dq elements differ by one bf16 ulp between runs (measured
                    # 1.1e-5 .. 1.2e-4 on dA_q / dB_q over 8 runs, every other factor <= 5e-7)
                    same[f"d{fam}_{n}"] = e < (5e-4 if n == "q" else 1e-4)
            out[grouping] = (same, got.trace.record_tuples("forward") == ref.trace.record_tuples("forward"),
                             len(got.trace.record_tuples("backward")))
        # the trainer loop with live NCCL collectives: CUDA-graph captured (NCCL kernels inside the
        # graph) vs eager launches from the same initial weights
        pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
        runs = {}
        for graphs in (True, False):
            tr = BlockTrainer(pl, blk, comm=TPComm(1, 0, trace=Trace(), force=True), adamw=dict(lr=1e-3),
                              graph_collectives=graphs)
            xh, gh = tr.pinned_host_inputs(x.values, G.values)
            losses = tr.fit([xh, xh, xh, xh], gh)
            runs[graphs] = (tr.graphed, losses)
        # a backend that refuses the capture: the trainer warns once and keeps running eagerly
        import warnings

        orig_graph = torch.cuda.graph

        def _refuse(*a, **k):
            raise RuntimeError("capture refused (test)")

        torch.cuda.graph = _refuse
        try:
            with warnings.catch_warnings(record=True) as caught:
                warnings.simplefilter("always")
                tr = BlockTrainer(pl, blk, comm=TPComm(1, 0, trace=Trace(), force=True), adamw=dict(lr=1e-3),
                                  graph_collectives=True)
                xh, gh = tr.pinned_host_inputs(x.values, G.values)
                losses = tr.fit([xh, xh, xh, xh], gh)
        finally:
            torch.cuda.graph = orig_graph
        runs["refused"] = (tr.graphed, tr.use_graph, losses,
                           sum("capture" in str(w.message) for w in caught))
        gathered = tr.ex.comm.all_gather_cols(torch.ones(4, 8, device="cuda"), "final-gather")
        out["trainer"] = (runs, tuple(gathered.shape))
        dist.destroy_process_group()
        q.put((out, None))
    except Exception:
        import traceback

        q.put((None, traceback.format_exc()))


def test_nccl_one_rank_step_is_bit_identical():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_main, args=(_port(), q))
    p.start()
    try:
        out, err = q.get(timeout=600)
    finally:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    assert err is None, err
    for grouping in (True, False):
        same, fwd_equal, n_bwd = out[grouping]
        assert all(same.values()), (grouping, {k: v for k, v in same.items() if not v})
        assert fwd_equal
        assert n_bwd == (4 if grouping else 7)
    runs, gshape = out["trainer"]
    (graphed, losses), (eager_graphed, eager_losses) = runs[True], runs[False]
    assert graphed and not eager_graphed        # the NCCL step was captured into a CUDA graph
    assert all(np.isfinite(losses)) and losses[0] != losses[-1]  # AdamW moved the weights
    # replay == eager up to the split-K fp32 reduce order, which AdamW can amplify where a gradient
    # element is ~0 (its normalised update flips sign): a loose relative bar
    np.testing.assert_allclose(losses, eager_losses, rtol=5e-3)
    r_graphed, r_use_graph, r_losses, n_warn = runs["refused"]
    assert not r_graphed and not r_use_graph and n_warn == 1  # fell back to eager launches, warned once
    np.testing.assert_allclose(r_losses, eager_losses, rtol=5e-3)
    assert gshape == (4, 8)
