"""GPU parity: the CUDA path (through the C-ABI) against the float64 CPU oracle on identical
seeded inputs — per intermediate (reference workspace names), every weight gradient, dx and the
loss, at the north_star bf16 tolerance (2e-2 relative Frobenius)."""

import numpy as np
import pytest
import torch

from tests.gpu_util import BF16_TOL, C60M, SMALL, inputs, oracle_step, rel
from oracle import btp_oracle as O
from paper_2512_12131_b200.api import execute_forward, train_step
from paper_2512_12131_b200.model import RunShape, Variant
from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

pytestmark = pytest.mark.gpu

WS_SKIP = {"x"}


def _check_ws(ws_gpu, ws_ref, tol=BF16_TOL):
    bad = {}
    for name, want in ws_ref.items():
        if name in WS_SKIP or name not in ws_gpu:
            continue
        e = rel(ws_gpu[name], want)
        if e > tol:
            bad[name] = e
    assert not bad, bad
    missing = {n for n in ws_ref if n not in ws_gpu}
    assert not missing, missing


@pytest.mark.parametrize("variant", [Variant.COLA, Variant.SVD])
@pytest.mark.parametrize("online", [True, False])
@pytest.mark.parametrize("grouping", [True, False])
def test_forward_workspaces_small(variant, online, grouping):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, variant, b, s)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), variant, online_norm=online, grouping=grouping)
    res = execute_forward(pl, blk, x, capture_workspaces=True)
    y_ref, _, ws_ref, _ = oracle_step(oblk, x, G, SMALL, b, s, online=online)
    assert rel(res.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
    _check_ws(res.workspaces[0], ws_ref[0])
    # the collective log equals the plan's prediction, tuple for tuple
    assert res.trace.record_tuples("forward") == [
        (p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)
    ]


@pytest.mark.parametrize("fuse_sigma", [True, False])
@pytest.mark.parametrize("online,grouping", [(True, True), (False, False)])
def test_forward_workspaces_c60m_sigma_epilogue(fuse_sigma, online, grouping, monkeypatch):
    """r = 128: z_* and a_in_* come straight out of the down-GEMM epilogue (fuse_sigma) or from
    the fix-up kernel; both must match the reference workspaces."""
    from paper_2512_12131_b200 import executor as E

    monkeypatch.setattr(E, "FUSE_SIGMA", fuse_sigma)
    b, s = 2, 128
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=online, grouping=grouping)
    res = execute_forward(pl, blk, x, capture_workspaces=True)
    y_ref, _, ws_ref, _ = oracle_step(oblk, x, G, C60M, b, s, online=online)
    assert rel(res.y.values.reshape(-1, C60M.d), y_ref) < BF16_TOL
    _check_ws(res.workspaces[0], ws_ref[0])
    assert res.trace.record_tuples("forward") == [
        (p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)
    ]


@pytest.mark.parametrize("variant", [Variant.COLA, Variant.SVD])
@pytest.mark.parametrize("grouping,online,ckpt", [(True, True, False), (False, True, False), (True, False, False),
                                                  (True, True, True), (False, False, True)])
def test_train_step_grads_small(variant, grouping, online, ckpt):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, variant, b, s)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), variant, online_norm=online, grouping=grouping,
              lowrank_ckpt=ckpt)
    st = train_step(pl, blk, x, G)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, online=online)
    assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL
    errs = {f"A_{n}": rel(st.grads["A"][n], g_ref["A"][n]) for n in O.PROJECTIONS}
    errs.update({f"B_{n}": rel(st.grads["B"][n], g_ref["B"][n]) for n in O.PROJECTIONS})
    errs["gamma1"] = rel(st.grads["gamma1"], g_ref["dgamma1"])
    errs["gamma2"] = rel(st.grads["gamma2"], g_ref["dgamma2"])
    bad = {k: v for k, v in errs.items() if v > BF16_TOL}
    assert not bad, bad
    # backward collectives: one [T, k*r] all-reduce per up-projection input grad
    bwd = st.trace.record_tuples("backward")
    T, r = b * s, SMALL.r
    assert sum(rec[3] for rec in bwd) == 7 * T * r
    # checkpointed recompute issues no collective (reference test_ckpt.py:79-87)
    assert st.trace.record_tuples("reforward") == []


@pytest.mark.parametrize("fuse_sigma,grouping,online,ckpt", [(True, True, True, False), (False, True, True, False),
                                                              (True, False, True, False), (True, True, False, True)])
def test_c60m_block_step(fuse_sigma, grouping, online, ckpt, monkeypatch):
    """CoLA-60M block (BASELINE config #1 shape) fwd+bwd vs the oracle. r = 128, so at TP = 1 the
    down-projections run the sigma-fused GEMM epilogue (fuse_sigma) or GEMM + fix-up kernel."""
    from paper_2512_12131_b200 import executor as E

    monkeypatch.setattr(E, "FUSE_SIGMA", fuse_sigma)
    b, s = 8, 256
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=online, grouping=grouping,
              lowrank_ckpt=ckpt)
    st = train_step(pl, blk, x, G)
    assert st.executor.fuse_sigma == fuse_sigma
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, C60M, b, s, sharded=False)
    assert rel(st.y.values.reshape(-1, C60M.d), y_ref) < BF16_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
    for n in O.PROJECTIONS:
        assert rel(st.grads["A"][n], g_ref["A"][n]) < BF16_TOL, n
        assert rel(st.grads["B"][n], g_ref["B"][n]) < BF16_TOL, n
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL


def test_run_with_ckpt_bitwise_and_collective_free():
    """Reference contract (test_ckpt.py:79-87): the BTP re-forward from the checkpoint set has
    zero collectives and reproduces the forward bitwise; it frees memory."""
    from paper_2512_12131_b200.checkpointing import CkptPolicy, eff_ckpt, run_with_ckpt

    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    run = run_with_ckpt(pl, blk, x, CkptPolicy.LOWRANK_BOUNDARY)
    assert run.recompute_bitwise_ok, run.recompute_checks
    assert run.report.reforward_collectives == 0
    assert run.report.delta_mem_bytes > 0
    assert eff_ckpt(run.report) > 0


FP32_TOL = 1e-4  # north_star: fp32 mode within 1e-4 relative on activations, gradients and loss


@pytest.mark.parametrize("variant", [Variant.COLA, Variant.SVD])
@pytest.mark.parametrize("online", [True, False])
def test_fp32_mode_forward_and_grads(variant, online):
    """fp32 parity mode (exact-fp32 SIMT GEMM + fp32 row kernels) against the float64 oracle."""
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, variant, b, s)
    pl = plan(Strategy.BOTTLENECK, SMALL, RunShape(b, s, 1), variant, online_norm=online, grouping=True)
    res = execute_forward(pl, blk, x, capture_workspaces=True, precision="fp32")
    y_ref, g_ref, ws_ref, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, online=online)
    _check_ws(res.workspaces[0], ws_ref[0], tol=FP32_TOL)
    st = train_step(pl, blk, x, G, precision="fp32")
    assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < FP32_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < FP32_TOL
    assert rel(st.dx, g_ref["dx"]) < FP32_TOL
    errs = {f"A_{n}": rel(st.grads["A"][n], g_ref["A"][n]) for n in O.PROJECTIONS}
    errs.update({f"B_{n}": rel(st.grads["B"][n], g_ref["B"][n]) for n in O.PROJECTIONS})
    errs["gamma1"] = rel(st.grads["gamma1"], g_ref["dgamma1"])
    errs["gamma2"] = rel(st.grads["gamma2"], g_ref["dgamma2"])
    bad = {k: v for k, v in errs.items() if v > FP32_TOL}
    assert not bad, bad


def test_fp32_mode_c60m_forward():
    """CoLA-60M block (BASELINE config #1) in fp32 mode vs the oracle, every intermediate."""
    b, s = 8, 256
    blk, x, G, oblk = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    res = execute_forward(pl, blk, x, capture_workspaces=True, precision="fp32")
    _, _, ws_ref, _ = oracle_step(oblk, x, G, C60M, b, s)
    _check_ws(res.workspaces[0], ws_ref[0], tol=FP32_TOL)


def test_concurrent_wgrad_stream_matches_serial(monkeypatch):
    """Weight-gradient GEMMs on the side stream (concurrent with dgrads / row kernels) give the same
    step as the serial schedule: y, loss, dx bit-identical, weight grads to reduce-add order."""
    import numpy as np

    from tests.gpu_util import C60M, inputs, rel
    from paper_2512_12131_b200 import executor as E
    from paper_2512_12131_b200.api import train_step
    from paper_2512_12131_b200.model import RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, plan

    b, s = 4, 256
    blk, x, G, _ = inputs(C60M, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, C60M, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    monkeypatch.setattr(E.ExecutorBase, "concurrent_wgrad", False)
    ser = train_step(pl, blk, x, G)
    monkeypatch.setattr(E.ExecutorBase, "concurrent_wgrad", True)
    con = train_step(pl, blk, x, G)
    assert np.array_equal(ser.y.values, con.y.values) and np.array_equal(ser.dx, con.dx)
    assert ser.loss == con.loss
    for fam in ("A", "B"):
        for n, g in ser.grads[fam].items():
            assert rel(con.grads[fam][n], g) < 1e-4, (fam, n)


@pytest.mark.parametrize("preset_name,b,s", [("1b", 1, 256), ("7b", 1, 256)])
def test_paper_width_blocks_vs_oracle(preset_name, b, s):
    """The paper's CoLA-1B / CoLA-7B block widths (d 2048/4096, d_ff 5472/11008, r 512/1024: the
    sigma epilogue with r/2 = 256/512, BN choices, the d_ff tail tile of 5472 = 21.4 x 256) at a
    short sequence, fwd + bwd against the float64 oracle."""
    from paper_2512_12131_b200.model import preset

    cfg = preset(preset_name)
    blk, x, G, oblk = inputs(cfg, Variant.COLA, b, s)
    pl = plan(Strategy.BOTTLENECK, cfg, RunShape(b, s, 1), Variant.COLA, online_norm=True, grouping=True)
    st = train_step(pl, blk, x, G)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, cfg, b, s, sharded=False)
    assert rel(st.y.values.reshape(-1, cfg.d), y_ref) < BF16_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL
    errs = {f"A_{n}": rel(st.grads["A"][n], g_ref["A"][n]) for n in O.PROJECTIONS}
    errs.update({f"B_{n}": rel(st.grads["B"][n], g_ref["B"][n]) for n in O.PROJECTIONS})
    errs["gamma1"] = rel(st.grads["gamma1"], g_ref["dgamma1"])
    errs["gamma2"] = rel(st.grads["gamma2"], g_ref["dgamma2"])
    bad = {k: v for k, v in errs.items() if v > BF16_TOL}
    assert not bad, bad
