"""CPU: the reference's own objects cross the drop-in boundary unchanged.

A btpsim ShardPlan / DecoderBlockWeights / Tensor / enum members are normalised by value and
fields (interop.py), never by identity, so BTP plans keep routing to the BTP executor."""

import numpy as np
import pytest

import paper_2512_12131_b200 as btp
from paper_2512_12131_b200 import interop
from tests.refpkg import load_btpsim

bs = load_btpsim()
needs_ref = pytest.mark.skipif(bs is None, reason="reference package btpsim not available")


@needs_ref
@pytest.mark.parametrize("strategy,variant,online,grouping,ckpt", [
    ("btp", "cola", True, True, False),
    ("btp", "svd", False, False, True),
    ("vanilla", "lax", True, True, True),      # online falls back with a warning
    ("full-rank", None, False, True, True),    # ckpt ignored with a warning
])
def test_reference_plan_is_rebuilt_identically(strategy, variant, online, grouping, ckpt):
    cfg = bs.ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
    ref = bs.plan(bs.Strategy(strategy), cfg, bs.RunShape(2, 8, 2), None if variant is None else bs.Variant(variant),
                  online_norm=online, grouping=grouping, lowrank_ckpt=ckpt)
    ours = interop.as_plan(ref)
    assert isinstance(ours, btp.ShardPlan)
    assert ours.strategy is btp.Strategy(strategy)           # identity on OUR enum: routing is right
    assert ours.norm_mode.value == ref.norm_mode.value
    assert ours.warnings == tuple(ref.warnings)
    assert [(c.chunk_id, c.ops, c.payload_elements, c.rider_elements) for c in ours.chunks] == \
           [(c.chunk_id, c.ops, c.payload_elements, c.rider_elements) for c in ref.chunks]
    assert ours.block_volume_elements == ref.block_volume_elements
    # our plan() accepts the reference's enums / config / shape directly, too
    direct = btp.plan(bs.Strategy(strategy), cfg, bs.RunShape(2, 8, 2),
                      None if variant is None else bs.Variant(variant), online_norm=online, grouping=grouping,
                      lowrank_ckpt=ckpt)
    assert direct == ours


@needs_ref
def test_reference_block_and_tensor_are_accepted():
    cfg = bs.ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
    ref_blk = bs.build_block(cfg, bs.Variant.COLA, 5)
    blk = interop.as_block(ref_blk)
    assert isinstance(blk, btp.DecoderBlockWeights) and blk.variant is btp.Variant.COLA
    ours = btp.build_block(btp.ModelConfig(2, 4, 16, 40, 4), btp.Variant.COLA, 5)
    for g in ("down_factors", "up_factors"):
        for k in ours.down_factors:
            assert np.array_equal(getattr(blk, g)[k].values, getattr(ours, g)[k].values)
    assert np.array_equal(blk.gamma1.values, ours.gamma1.values)
    x = bs.seeded_fill((2, 8, 16), 10005)
    assert not isinstance(x, btp.Tensor)
    t = interop.as_tensor(x)
    assert isinstance(t, btp.Tensor) and np.array_equal(t.values, x.values) and t.element_bytes == x.element_bytes
    assert interop.values_of(x) is x.values
    # build_block accepts the reference's config / enum
    again = btp.build_block(cfg, bs.Variant.COLA, 5)
    assert np.array_equal(again.up_factors["down"].values, ours.up_factors["down"].values)


@needs_ref
def test_api_normalises_reference_objects_before_routing():
    """execute_forward / train_step / make_executor / run_with_ckpt go through api._normalise: a
    btpsim BTP plan routes to the BTP executor (identity tests misrouted it)."""
    from paper_2512_12131_b200.api import _check_inputs, _normalise

    cfg = bs.ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
    ref_pl = bs.plan(bs.Strategy.BOTTLENECK, cfg, bs.RunShape(2, 8, 1), bs.Variant.COLA, online_norm=True,
                     grouping=True)
    pl, blk = _normalise(ref_pl, bs.build_block(cfg, bs.Variant.COLA, 0))
    assert pl.strategy is btp.Strategy.BOTTLENECK and blk.variant is pl.variant
    xv = _check_inputs(pl, blk, bs.seeded_fill((2, 8, 16), 10000))
    assert xv.shape == (2, 8, 16)


def test_enum_and_tensor_coercion_without_reference():
    assert interop.as_strategy("btp") is btp.Strategy.BOTTLENECK
    assert interop.as_variant("lax") is btp.Variant.LAX
    with pytest.raises(ValueError, match="not a valid Strategy"):
        interop.as_strategy("megatron")
    assert interop.as_tensor([[1, 2]]).values.dtype == np.float64
