"""Host-side TP-strategy switch: plans, collective prediction and describe() text must equal
the reference's (golden vectors produced by the reference itself, tests/golden/)."""

import json
from pathlib import Path

import pytest

from paper_2512_12131_b200.model import ModelConfig, RunShape, Variant, preset, PRESETS
from paper_2512_12131_b200.plan import (
    NormMode, PlanError, Strategy, apply_grouping, cola_pair_indices, describe, enumerate_collectives, plan,
)

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "btpsim_golden.json").read_text())
TOY = ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)


@pytest.mark.parametrize("key", sorted(GOLD["describe"]))
def test_describe_matches_reference(key):
    strategy, variant, tp, online, grouping = key.split("|")
    v = None if strategy == "full-rank" else Variant(variant)
    pl = plan(Strategy(strategy), TOY, RunShape(2, 8, int(tp)), v, online_norm=bool(int(online)),
              grouping=bool(int(grouping)), lowrank_ckpt=True)
    assert describe(pl) == GOLD["describe"][key]


@pytest.mark.parametrize("entry", GOLD["combos"], ids=lambda e: e["tag"])
def test_enumerate_equals_reference_trace(entry):
    """The reference's traced records (its simulator ran the plan) equal our static prediction."""
    v = None if entry["strategy"] == "full-rank" else Variant(entry["variant"])
    pl = plan(Strategy(entry["strategy"]), TOY, RunShape(2, 8, entry["tp"]), v, online_norm=entry["online"],
              grouping=entry["grouping"])
    pred = [[p.chunk_id, p.kind, p.tag, p.elements, [list(e) for e in p.extras]]
            for p in enumerate_collectives(pl, model_tail=True)]
    assert pred == entry["records"]


def test_presets_and_validation():
    assert (preset("7b").d, preset("7b").r) == (4096, 1024)
    assert set(PRESETS) == {"1b", "3b", "7b", "13b", "30b"}
    with pytest.raises(KeyError):
        preset("70b")
    with pytest.raises(PlanError, match="heads"):
        plan(Strategy.BOTTLENECK, ModelConfig(1, 6, 48, 96, 8), RunShape(1, 4, 4), Variant.SVD)
    with pytest.raises(PlanError, match="d_ff"):
        plan(Strategy.BOTTLENECK, ModelConfig(1, 4, 16, 42, 4), RunShape(1, 4, 4), Variant.SVD)
    with pytest.raises(PlanError, match="r/2"):
        plan(Strategy.VANILLA, TOY, RunShape(1, 4, 4), Variant.COLA)
    with pytest.raises(PlanError, match="cannot shard"):
        plan(Strategy.FULL_RANK, TOY, RunShape(1, 4, 1), Variant.SVD)


def test_online_fallback_and_ckpt_warnings():
    pl = plan(Strategy.VANILLA, TOY, RunShape(2, 8, 2), Variant.SVD, online_norm=True)
    assert pl.norm_mode is NormMode.REPLICATED and pl.warnings
    fr = plan(Strategy.FULL_RANK, TOY, RunShape(2, 8, 2), lowrank_ckpt=True)
    assert not fr.lowrank_ckpt and any("ignored" in w for w in fr.warnings)


def test_grouping_preserves_volume_and_cuts_collectives():
    for strat, var in [(Strategy.BOTTLENECK, Variant.COLA), (Strategy.VANILLA, Variant.SVD)]:
        pl = plan(strat, TOY, RunShape(2, 8, 2), var, online_norm=True)
        g = apply_grouping(pl)
        assert g.block_volume_elements == pl.block_volume_elements
        assert len(g.chunks) < len(pl.chunks)
    btp = plan(Strategy.BOTTLENECK, preset("7b"), RunShape(4, 4096, 8), Variant.COLA, online_norm=True)
    assert btp.boundary_volume_elements == 7 * 4 * 4096 * 1024


def test_cola_pair_indices():
    idx = cola_pair_indices(8, 2, 1)
    assert list(idx) == [2, 3, 6, 7]


def test_closed_form_block_volume_matches_plan():
    """The plan's predicted forward collectives sum to the closed form of reference costs.py:28-44
    for every strategy, tp and grouping (the device traces are checked against the plan on the GPU)."""
    from paper_2512_12131_b200.model import ModelConfig, RunShape, Variant
    from paper_2512_12131_b200.plan import Strategy, enumerate_collectives, plan
    from paper_2512_12131_b200.trace import tp_block_volume

    cfg = ModelConfig(layers=2, heads=4, d=16, d_ff=40, r=4)
    for strategy, var in ((Strategy.FULL_RANK, None), (Strategy.VANILLA, Variant.SVD), (Strategy.BOTTLENECK, Variant.SVD),
                          (Strategy.BOTTLENECK, Variant.COLA)):
        for tp in (1, 2, 4):
            for grouping in (False, True):
                for b, s in ((1, 4), (2, 8)):
                    shape = RunShape(b, s, tp)
                    pl = plan(strategy, cfg, shape, var, online_norm=True, grouping=grouping)
                    got = sum(p.elements for p in enumerate_collectives(pl) if p.tag == "block")
                    assert got == tp_block_volume(strategy, cfg, shape), (strategy, tp, grouping, b, s)
