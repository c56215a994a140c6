"""CPU: the reference's scenario / config API (btpsim.cli, cli.py:55-304) — key names, defaults,
the TP-strategy switch and its contradictions, overrides — ported from the reference's own
pkg/tests/test_cli.py cases (:102-185), minus the CLI commands and report writers."""

import argparse
import json

import pytest

import paper_2512_12131_b200.cli as cli
from paper_2512_12131_b200 import NormMode, PlanError, Strategy, Variant

TOY_TOML = """\
name = "toy"
b = 2
s = 8
tp = 2
variant = "svd"
seed = 7

[model]
layers = 2
heads = 4
d = 16
d_ff = 40
r = 4
"""

TOY_JSON = {"name": "toy-json", "model": {"layers": 2, "heads": 4, "d": 16, "d_ff": 40, "r": 4},
            "b": 2, "s": 8, "tp": 2, "variant": "svd", "seed": 7}


@pytest.fixture
def toy_toml(tmp_path):
    p = tmp_path / "toy.toml"
    p.write_text(TOY_TOML)
    return str(p)


def test_toml_and_json_load_the_same_scenario(toy_toml, tmp_path):
    pj = tmp_path / "toy.json"
    pj.write_text(json.dumps(TOY_JSON))
    a, b = cli.load_scenario(toy_toml), cli.load_scenario(str(pj))
    assert a.name == "toy" and b.name == "toy-json"
    assert a.to_dict() | {"name": None} == b.to_dict() | {"name": None}
    # defaults of the reference (cli.py:225-246): BTP resolved, online norm on only for BTP
    assert a.strategy is Strategy.BOTTLENECK and a.enable_btp
    assert a.enable_online_rmsnorm and not a.enable_grouping and not a.enable_lowrank_ckpt
    assert a.element_bytes == 2 and a.eps == 1e-6 and a.lax_h_prev == "zero"


def test_unknown_key_is_config_error(tmp_path):
    bad = tmp_path / "bad.toml"
    bad.write_text('model = "7b"\nwhatever = 1\n')
    with pytest.raises(cli.ConfigError, match="unknown config keys"):
        cli.load_scenario(str(bad))
    with pytest.raises(cli.ConfigError, match="unknown model keys"):
        cli.scenario_from_dict({"model": {"layers": 1, "heads": 1, "d": 4, "d_ff": 8, "rank": 2}})
    with pytest.raises(cli.ConfigError, match="missing keys"):
        cli.scenario_from_dict({"model": {"layers": 1, "heads": 1}})
    with pytest.raises(cli.ConfigError, match="unknown model preset"):
        cli.scenario_from_dict({"model": "9b"})
    with pytest.raises(cli.ConfigError, match="needs a model"):
        cli.scenario_from_dict({"b": 1})


def test_json_parse_error_names_line_and_column(tmp_path):
    bad = tmp_path / "bad.json"
    bad.write_text('{"model": "7b", "b": }')
    with pytest.raises(cli.ConfigError, match="bad.json:1:22"):
        cli.load_scenario(str(bad))


def test_missing_file_and_bad_suffix(tmp_path):
    with pytest.raises(cli.ConfigError, match="not found"):
        cli.load_scenario(str(tmp_path / "nope.toml"))
    bad = tmp_path / "cfg.yaml"
    bad.write_text("model: 7b")
    with pytest.raises(cli.ConfigError, match=".toml or .json"):
        cli.load_scenario(str(bad))


def test_type_checks():
    for raw, msg in ((dict(model="7b", b=True), "b must be an integer"),
                     (dict(model="7b", enable_grouping=1), "enable_grouping must be a boolean"),
                     (dict(model="7b", element_bytes=3), "element_bytes must be one of"),
                     (dict(model="7b", eps="x"), "eps must be a number"),
                     (dict(model="7b", lax_h_prev="rand"), "lax_h_prev"),
                     (dict(model="7b", variant="lora"), "unknown variant"),
                     (dict(model="7b", strategy="zero"), "unknown strategy"),
                     (dict(model="7b", b=0), "b must be positive"),
                     (dict(model={"layers": 1, "heads": 1, "d": 4, "d_ff": 8}, variant="cola"), "needs a bottleneck rank")):
        with pytest.raises(cli.ConfigError, match=msg):
            cli.scenario_from_dict(raw)


def test_strategy_resolution_and_contradictions(tmp_path):
    """Reference pkg/tests/test_cli.py:140-158."""
    implicit_vanilla = tmp_path / "v.toml"
    implicit_vanilla.write_text('model = "7b"\nvariant = "svd"\nenable_btp = false\n')
    scn = cli.load_scenario(str(implicit_vanilla))
    assert scn.strategy.value == "vanilla"
    assert not scn.enable_online_rmsnorm        # online default is on only for BTP

    explicit = tmp_path / "e.toml"
    explicit.write_text('model = "7b"\nvariant = "svd"\nstrategy = "vanilla"\n')
    assert cli.load_scenario(str(explicit)).strategy.value == "vanilla"

    contra = tmp_path / "c.toml"
    contra.write_text('model = "7b"\nvariant = "svd"\nstrategy = "vanilla"\nenable_btp = true\n')
    with pytest.raises(cli.ConfigError, match="contradicts"):
        cli.load_scenario(str(contra))

    fullrank_lowrank = tmp_path / "f.toml"
    fullrank_lowrank.write_text('model = "7b"\nvariant = "svd"\nstrategy = "full-rank"\n')
    with pytest.raises(cli.ConfigError, match="full-rank"):
        cli.load_scenario(str(fullrank_lowrank))

    with pytest.raises(cli.ConfigError, match="contradicts enable_btp=false"):
        cli.scenario_from_dict(dict(model="7b", strategy="btp", enable_btp=False))
    with pytest.raises(cli.ConfigError, match="requires a low-rank variant"):
        cli.scenario_from_dict(dict(model="7b", variant="full-rank", strategy="btp"))
    # a full-rank block resolves to Megatron TP whatever enable_btp says when no strategy is given
    assert cli.scenario_from_dict(dict(model="7b", variant="full-rank")).strategy is Strategy.FULL_RANK
    assert cli._resolve_strategy(Variant.COLA, None, None) is Strategy.BOTTLENECK
    assert cli._resolve_strategy(Variant.COLA, None, False) is Strategy.VANILLA


def test_flag_overrides_change_resolved_strategy(toy_toml):
    """Reference pkg/tests/test_cli.py:161-174, through argparse with the reference's flag names."""
    ap = cli.add_config_flags(argparse.ArgumentParser())
    args = ap.parse_args(["--lowrank-architecture-type", "lax", "--no-enable-btp", "--enable-grouping"])
    scn = cli.apply_overrides(cli.load_scenario(toy_toml), args)
    assert scn.variant is Variant.LAX and scn.strategy is Strategy.VANILLA and scn.enable_grouping
    pl = cli.build_plan(scn)
    assert pl.grouping and len(pl.chunks) == 4
    # no flags: the file wins unchanged
    same = cli.apply_overrides(cli.load_scenario(toy_toml), ap.parse_args([]))
    assert same == cli.load_scenario(toy_toml)
    # switching BTP back on re-resolves the strategy
    back = cli.apply_overrides(scn, argparse.Namespace(enable_btp=True))
    assert back.strategy is Strategy.BOTTLENECK
    seeded = cli.apply_overrides(scn, argparse.Namespace(seed=11, element_bytes=4, enable_lowrank_ckpt=True))
    assert (seeded.seed, seeded.element_bytes, seeded.enable_lowrank_ckpt) == (11, 4, True)


def test_online_norm_fallback_warns_and_ckpt_ignored_under_full_rank():
    """Reference test_cli.py:177-184 and plan.py:309-325: online norm requested under vanilla falls
    back to replicated with a warning; low-rank ckpt under full-rank is ignored with a warning."""
    scn = cli.scenario_from_dict(dict(model={"layers": 2, "heads": 4, "d": 16, "d_ff": 40, "r": 4}, variant="svd",
                                      enable_btp=False, enable_online_rmsnorm=True))
    pl = cli.build_plan(scn)
    assert pl.norm_mode is NormMode.REPLICATED and any("falling back" in w for w in pl.warnings)
    fr = cli.scenario_from_dict(dict(model="7b", variant="full-rank", enable_lowrank_ckpt=True))
    pl = cli.build_plan(fr)
    assert not pl.lowrank_ckpt and any("ignored" in w for w in pl.warnings)


def test_infeasible_plan_raises_plan_error():
    """Reference test_cli.py:124-131 (exit code 3 there): cola gate pairs cannot split 4 ways at r=4."""
    scn = cli.scenario_from_dict(dict(model={"layers": 2, "heads": 4, "d": 16, "d_ff": 40, "r": 4}, variant="cola",
                                      tp=4, enable_btp=False))
    with pytest.raises(PlanError, match="gate pairs"):
        cli.build_plan(scn)


def test_scenario_inputs_match_reference_seeding():
    """Block and input seeds follow cli.py:307-320 (x from seed + 10000, lax seeded bundle + 20000)."""
    from paper_2512_12131_b200 import build_block, seeded_fill

    scn = cli.scenario_from_dict(dict(TOY_JSON, variant="lax", lax_h_prev="seeded"))
    block, x, h = cli.scenario_inputs(scn)
    ref = build_block(scn.cfg, Variant.LAX, 7)
    assert (block.down_factors["q"].values == ref.down_factors["q"].values).all()
    assert (x.values == seeded_fill((2, 8, 16), 10007).values).all()
    assert set(h) == {"q", "k", "v", "o", "gate", "up", "down"}
    assert (h["q"].values == seeded_fill((2, 8, 4), 20007).values).all()
