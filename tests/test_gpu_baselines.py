"""GPU parity of the two comparison strategies (naive low-rank TP, Megatron full-rank TP) on the
same kernels, against the float64 oracle (bf16 tolerance 2e-2)."""

import numpy as np
import pytest

from tests.gpu_util import BF16_TOL, SMALL, inputs, oracle_step, rel
from oracle import btp_oracle as O
from paper_2512_12131_b200.api import execute_forward, train_step
from paper_2512_12131_b200.model import RunShape, Variant
from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("variant", [Variant.COLA, Variant.SVD])
@pytest.mark.parametrize("grouping", [True, False])
def test_vanilla_step(variant, grouping):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, variant, b, s)
    pl = plan(Strategy.VANILLA, SMALL, RunShape(b, s, 1), variant, grouping=grouping)
    st = train_step(pl, blk, x, G)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s)
    assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL
    for n in O.PROJECTIONS:
        assert rel(st.grads["A"][n], g_ref["A"][n]) < BF16_TOL, ("A", n)
        assert rel(st.grads["B"][n], g_ref["B"][n]) < BF16_TOL, ("B", n)
    assert rel(st.grads["gamma1"], g_ref["dgamma1"]) < BF16_TOL
    assert rel(st.grads["gamma2"], g_ref["dgamma2"]) < BF16_TOL
    assert st.trace.record_tuples("forward") == [
        (p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]


@pytest.mark.parametrize("grouping", [True, False])
def test_full_rank_step(grouping):
    b, s = 2, 64
    blk, x, G, oblk = inputs(SMALL, Variant.FULL_RANK, b, s)
    pl = plan(Strategy.FULL_RANK, SMALL, RunShape(b, s, 1), grouping=grouping)
    st = train_step(pl, blk, x, G)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False)
    assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < BF16_TOL
    assert abs(st.loss - loss_ref) / abs(loss_ref) < BF16_TOL
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL
    for n in O.PROJECTIONS:
        assert rel(st.grads["W"][n], g_ref["W"][n]) < BF16_TOL, n
    assert st.trace.record_tuples("forward") == [
        (p.chunk_id, p.kind, p.tag, p.elements, p.extras) for p in enumerate_collectives(pl)]


@pytest.mark.parametrize("strategy", ["btp", "full-rank"])
def test_dff_shard_padding(strategy):
    """d_ff shard not a multiple of 8 (like CoLA-1B at TP=8: 5472/8 = 684): the executors pad the
    shard with zero rows/columns for TMA alignment; results must be unaffected."""
    from paper_2512_12131_b200.model import ModelConfig

    cfg = ModelConfig(layers=1, heads=4, d=256, d_ff=612, r=64)
    b, s = 2, 64
    variant = Variant.FULL_RANK if strategy == "full-rank" else Variant.COLA
    blk, x, G, oblk = inputs(cfg, variant, b, s)
    pl = plan(Strategy(strategy), cfg, RunShape(b, s, 1), None if strategy == "full-rank" else variant,
              online_norm=strategy == "btp", grouping=True)
    st = train_step(pl, blk, x, G)
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, cfg, b, s, sharded=False)
    assert rel(st.y.values.reshape(-1, cfg.d), y_ref) < BF16_TOL
    assert rel(st.dx, g_ref["dx"]) < BF16_TOL
    grp = ("W",) if strategy == "full-rank" else ("A", "B")
    for gname in grp:
        for n in O.PROJECTIONS:
            assert st.grads[gname][n].shape == g_ref[gname][n].shape, (gname, n)
            assert rel(st.grads[gname][n], g_ref[gname][n]) < BF16_TOL, (gname, n)


@pytest.mark.parametrize("strategy", ["vanilla", "full-rank"])
def test_baselines_fp32_mode(strategy):
    b, s = 2, 64
    variant = Variant.FULL_RANK if strategy == "full-rank" else Variant.COLA
    blk, x, G, oblk = inputs(SMALL, variant, b, s)
    pl = plan(Strategy(strategy), SMALL, RunShape(b, s, 1), None if strategy == "full-rank" else variant)
    st = train_step(pl, blk, x, G, precision="fp32")
    y_ref, g_ref, _, loss_ref = oracle_step(oblk, x, G, SMALL, b, s, sharded=False)
    assert rel(st.y.values.reshape(-1, SMALL.d), y_ref) < 1e-4
    assert rel(st.dx, g_ref["dx"]) < 1e-4
    grp = "W" if strategy == "full-rank" else "A"
    for n in O.PROJECTIONS:
        assert rel(st.grads[grp][n], g_ref[grp][n]) < 1e-4, n
