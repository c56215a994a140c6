"""GPU: the INTEGRATION.md hook run with the reference's OWN objects — a `btpsim.ShardPlan`,
`btpsim.DecoderBlockWeights` and `btpsim.Tensor` go straight into our `execute_forward` /
`train_step` / `run_with_ckpt`, and the result is compared with `btpsim.execute_forward` itself
(the reference, float64, run in this process from baseline/_ref) and with the float64 oracle.

Tolerances per north_star: fp32 mode 1e-4 relative, bf16 mode 2e-2 relative."""

import dataclasses

import numpy as np
import pytest

import paper_2512_12131_b200 as btp
from tests.gpu_util import BF16_TOL, rel
from tests.refpkg import load_btpsim

bs = load_btpsim()
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(bs is None, reason="reference package btpsim not installed")]

FP32_TOL = 1e-4


def _ref_inputs(cfg, variant, b, s, seed=0):
    """The parity recipe applied to the reference's own block: dataclasses.replace on
    the frozen btpsim block, every factor times sqrt(3 / fan_in)."""
    blk = bs.build_block(cfg, variant, seed)

    def scale(g):
        return {k: bs.Tensor(v.values * np.sqrt(3.0 / v.values.shape[1]), v.element_bytes) for k, v in g.items()}

    blk = dataclasses.replace(blk, down_factors=scale(blk.down_factors), up_factors=scale(blk.up_factors))
    x = bs.seeded_fill((b, s, cfg.d), seed + 10000)
    return blk, x


@pytest.mark.parametrize("variant", ["cola", "svd"])
@pytest.mark.parametrize("online,grouping", [(True, True), (False, False)])
@pytest.mark.parametrize("precision,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
def test_hook_with_reference_objects_matches_btpsim(variant, online, grouping, precision, tol):
    cfg = bs.ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)
    b, s = 2, 32
    blk, x = _ref_inputs(cfg, bs.Variant(variant), b, s)
    pl = bs.plan(bs.Strategy.BOTTLENECK, cfg, bs.RunShape(b, s, 1), bs.Variant(variant), online_norm=online,
                 grouping=grouping)
    want = bs.execute_forward(pl, blk, x, model_tail=True)
    got = btp.execute_forward(pl, blk, x, model_tail=True, precision=precision, capture_workspaces=True)
    assert isinstance(got.y, btp.Tensor)
    assert rel(got.y.values, want.y.values) < tol
    # the y ≈ x residual path hides errors in the branches: compare the branch outputs too. In
    # fp32 mode that is the block's update y - x itself; in bf16 the update of this block is ~1 bf16
    # ulp of y (|y - x| ~ 1e-3 |x| for the raw reference gains), so the rounding of y alone exceeds
    # 2e-2 of it — the attention / MLP branch outputs are compared directly, as the reference's
    # workspace tensors (simulator.py:672-706)
    if precision == "fp32":
        assert rel(got.y.values - x.values, want.y.values - x.values) < tol
    for name in ("o", "mlp"):
        assert rel(got.workspaces[0][name], want.workspaces[0][name]) < tol, name
    # the routing is BTP: our collective log is the reference's own trace, record for record
    assert got.trace.record_tuples("forward") == [
        (r.chunk_id, r.kind, r.tag, r.elements, tuple((t, e) for t, e, _ in r.extras))
        for r in want.trace.records if r.pass_tag == "forward"]


def test_lax_bundle_and_ckpt_with_reference_objects():
    cfg = bs.ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)
    b, s = 2, 32
    blk, x = _ref_inputs(cfg, bs.Variant.LAX, b, s)
    shape = bs.RunShape(b, s, 1)
    from btpsim.model import seeded_h_prev

    hp = {k: bs.Tensor(v.values * 0.5, v.element_bytes) for k, v in seeded_h_prev(cfg, shape, 20000).items()}
    pl = bs.plan(bs.Strategy.BOTTLENECK, cfg, shape, bs.Variant.LAX, online_norm=True, grouping=True,
                 lowrank_ckpt=True)
    want = bs.execute_forward(pl, blk, x, hp)
    got = btp.execute_forward(pl, blk, x, hp, precision="fp32")
    assert rel(got.y.values - x.values, want.y.values - x.values) < FP32_TOL
    for k in want.h_cur:
        assert rel(got.h_cur[k].values, want.h_cur[k].values) < FP32_TOL
    run = btp.run_with_ckpt(pl, blk, x, bs.CkptPolicy.LOWRANK_BOUNDARY, hp)
    assert run.recompute_bitwise_ok and run.report.reforward_collectives == 0


def test_train_step_and_trainer_accept_reference_objects():
    cfg = bs.ModelConfig(layers=1, heads=4, d=256, d_ff=640, r=64)
    b, s = 2, 32
    blk, x = _ref_inputs(cfg, bs.Variant.COLA, b, s)
    pl = bs.plan(bs.Strategy.BOTTLENECK, cfg, bs.RunShape(b, s, 1), bs.Variant.COLA, online_norm=True, grouping=True)
    st = btp.train_step(pl, blk, x, precision="fp32")
    ours = btp.train_step(btp.interop.as_plan(pl), btp.interop.as_block(blk), btp.interop.as_tensor(x),
                          precision="fp32")
    assert np.array_equal(st.y.values, ours.y.values) and st.loss == ours.loss
    assert isinstance(st.executor, btp.executor.BTPBlockExecutor)
    tr = btp.BlockTrainer(pl, blk, use_graph=False)
    assert tr.pl.strategy is btp.Strategy.BOTTLENECK


def test_scenario_runs_on_device_and_matches_reference():
    """config API -> plan -> device forward, checked against the reference's own run of the same
    scenario (cli.py:351-372 semantics: model_tail=True, inputs from the scenario seeds)."""
    raw = {"name": "toy", "model": {"layers": 1, "heads": 4, "d": 256, "d_ff": 640, "r": 64}, "b": 2, "s": 32,
           "variant": "cola", "enable_grouping": True}
    scn = btp.scenario_from_dict(raw)
    res = btp.run_scenario(scn, scaled=True, precision="fp32")
    import btpsim.cli as rcli

    rscn = rcli.scenario_from_dict(raw)
    rpl = rcli.build_plan(rscn)
    rblk, rx, _ = rcli._block_inputs(rscn)

    def scale(g):
        return {k: bs.Tensor(v.values * np.sqrt(3.0 / v.values.shape[1]), v.element_bytes) for k, v in g.items()}

    rblk = dataclasses.replace(rblk, down_factors=scale(rblk.down_factors), up_factors=scale(rblk.up_factors))
    want = bs.execute_forward(rpl, rblk, rx, model_tail=True)
    assert rel(res.y.values - rx.values, want.y.values - rx.values) < FP32_TOL
