"""The reference's scenario / config API: the `enable_*` switches and the TP-strategy switch
(reference `btpsim.cli`, cli.py:55-304), without its CLI commands or report writers.

Same key names, defaults, validation and error messages as the reference:

* `_SCENARIO_KEYS` / `_MODEL_KEYS` and unknown-key rejection (cli.py:55-73, :189-192);
* `Scenario` (cli.py:76-114) and `scenario_from_dict` / `load_scenario` (.toml / .json,
  cli.py:189-266);
* `_resolve_strategy` — `enable_btp` true => BTP, false => naive (vanilla) TP, contradictions
  with an explicit `strategy` rejected (cli.py:155-186);
* defaults: online RMSNorm on only under BTP, grouping and low-rank ckpt off (cli.py:225-246);
* `apply_overrides` (flags win over the file, cli.py:269-291) and `build_plan` (cli.py:294-304).

On top of that, `add_config_flags` registers the reference's override flags on an argparse
parser (cli.py:638-660, names only — no subcommands), and `run_scenario` executes a scenario on
the GPU through `execute_forward` / `run_with_ckpt` (the device counterpart of cli.py:360-372).
"""

from __future__ import annotations

import argparse
import json
from dataclasses import dataclass, replace
from pathlib import Path

try:
    import tomllib
except ModuleNotFoundError:  # py3.10
    import tomli as tomllib

from .model import EPS_DEFAULT, PRESETS, ModelConfig, RunShape, Variant
from .plan import ShardPlan, Strategy, plan
from .tensor import VALID_ELEMENT_BYTES

INPUT_SEED_OFFSET = 10_000   # x = seeded_fill((b, s, d), seed + 10000)   (cli.py:40)
HPREV_SEED_OFFSET = 20_000   # lax seeded bundle seed                        (cli.py:41)


class ConfigError(Exception):
    """Bad scenario configuration (reference cli.py:51-52; the CLI maps it to exit code 2)."""


_SCENARIO_KEYS = frozenset({
    "name", "model", "b", "s", "tp", "p", "variant", "strategy", "seed", "element_bytes", "eps",
    "enable_btp", "enable_online_rmsnorm", "enable_grouping", "enable_lowrank_ckpt", "lax_h_prev",
})
_MODEL_KEYS = frozenset({"layers", "heads", "d", "d_ff", "r"})


@dataclass(frozen=True)
class Scenario:
    name: str
    cfg: ModelConfig
    shape: RunShape
    variant: Variant
    strategy: Strategy
    seed: int = 0
    element_bytes: int = 2
    eps: float = EPS_DEFAULT
    enable_online_rmsnorm: bool = True
    enable_grouping: bool = False
    enable_lowrank_ckpt: bool = False
    lax_h_prev: str = "zero"

    @property
    def enable_btp(self) -> bool:
        return self.strategy is Strategy.BOTTLENECK

    def to_dict(self) -> dict:
        c = self.cfg
        return {
            "name": self.name,
            "model": {"layers": c.layers, "heads": c.heads, "d": c.d, "d_ff": c.d_ff, "r": c.r},
            "b": self.shape.b, "s": self.shape.s, "tp": self.shape.tp, "p": self.shape.p,
            "variant": self.variant.value, "strategy": self.strategy.value, "seed": self.seed,
            "element_bytes": self.element_bytes, "eps": self.eps,
            "enable_online_rmsnorm": self.enable_online_rmsnorm, "enable_grouping": self.enable_grouping,
            "enable_lowrank_ckpt": self.enable_lowrank_ckpt, "lax_h_prev": self.lax_h_prev,
        }


def _require(cond: bool, msg: str) -> None:
    if not cond:
        raise ConfigError(msg)


def _int_key(raw: dict, key: str, default: int) -> int:
    v = raw.get(key, default)
    _require(isinstance(v, int) and not isinstance(v, bool), f"{key} must be an integer")
    return v


def _bool_key(raw: dict, key: str, default: bool) -> bool:
    v = raw.get(key, default)
    _require(isinstance(v, bool), f"{key} must be a boolean")
    return v


def _model(raw) -> ModelConfig:
    if isinstance(raw, str):
        _require(raw in PRESETS, f"unknown model preset {raw!r}; expected one of {sorted(PRESETS)}")
        return PRESETS[raw]
    _require(isinstance(raw, dict), "model must be a preset name or a table of dimensions")
    extra = sorted(set(raw) - _MODEL_KEYS)
    _require(not extra, f"unknown model keys: {extra}")
    missing = sorted(k for k in ("layers", "heads", "d", "d_ff") if k not in raw)
    _require(not missing, f"model table is missing keys: {missing}")
    try:
        return ModelConfig(layers=raw["layers"], heads=raw["heads"], d=raw["d"], d_ff=raw["d_ff"], r=raw.get("r"))
    except (ValueError, TypeError) as exc:
        raise ConfigError(str(exc)) from exc


def _resolve_strategy(variant: Variant, raw_strategy, enable_btp: bool | None) -> Strategy:
    """The TP-strategy switch (reference cli.py:155-186). enable_btp=None: the key was absent,
    so an explicit strategy cannot contradict it; with no strategy, full-rank blocks get
    Megatron TP and low-rank blocks BTP unless enable_btp is false (then naive TP)."""
    variant = Variant(getattr(variant, "value", variant))
    if raw_strategy is None:
        if variant is Variant.FULL_RANK:
            return Strategy.FULL_RANK
        return Strategy.BOTTLENECK if (enable_btp is None or enable_btp) else Strategy.VANILLA
    _require(isinstance(raw_strategy, str), "strategy must be a string")
    try:
        strategy = Strategy(raw_strategy)
    except ValueError:
        raise ConfigError(
            f"unknown strategy {raw_strategy!r}; expected one of {[s.value for s in Strategy]}") from None
    if strategy is Strategy.FULL_RANK:
        _require(variant is Variant.FULL_RANK, f"strategy full-rank requires variant full-rank, got {variant.value}")
    else:
        _require(variant is not Variant.FULL_RANK, f"strategy {strategy.value} requires a low-rank variant")
    if enable_btp is not None:
        if strategy is Strategy.VANILLA and enable_btp:
            raise ConfigError("strategy vanilla contradicts enable_btp=true")
        if strategy is Strategy.BOTTLENECK and not enable_btp:
            raise ConfigError("strategy btp contradicts enable_btp=false")
    return strategy


def scenario_from_dict(raw: dict, default_name: str = "scenario") -> Scenario:
    """Validate a scenario table (reference cli.py:189-246)."""
    _require(isinstance(raw, dict), "top-level config must be a table/object")
    extra = sorted(set(raw) - _SCENARIO_KEYS)
    _require(not extra, f"unknown config keys: {extra}")
    _require("model" in raw, "config needs a model (preset name or dimension table)")
    cfg = _model(raw["model"])
    name = raw.get("name", default_name)
    _require(isinstance(name, str), "name must be a string")
    vraw = raw.get("variant", "svd")
    try:
        variant = Variant(vraw)
    except ValueError:
        raise ConfigError(f"unknown variant {vraw!r}; expected one of {[v.value for v in Variant]}") from None
    enable_btp = _bool_key(raw, "enable_btp", True) if "enable_btp" in raw else None
    strategy = _resolve_strategy(variant, raw.get("strategy"), enable_btp)
    try:
        shape = RunShape(b=_int_key(raw, "b", 1), s=_int_key(raw, "s", 8), tp=_int_key(raw, "tp", 1),
                         p=_int_key(raw, "p", 1))
    except ValueError as exc:
        raise ConfigError(str(exc)) from exc
    eb = _int_key(raw, "element_bytes", 2)
    _require(eb in VALID_ELEMENT_BYTES, f"element_bytes must be one of {VALID_ELEMENT_BYTES}, got {eb}")
    eps = raw.get("eps", EPS_DEFAULT)
    _require(isinstance(eps, (int, float)) and not isinstance(eps, bool), "eps must be a number")
    lax_h_prev = raw.get("lax_h_prev", "zero")
    _require(lax_h_prev in ("zero", "seeded"), "lax_h_prev must be 'zero' or 'seeded'")
    if variant is not Variant.FULL_RANK:
        _require(cfg.r is not None, f"variant {variant.value} needs a bottleneck rank r")
    return Scenario(
        name=name, cfg=cfg, shape=shape, variant=variant, strategy=strategy,
        seed=_int_key(raw, "seed", 0), element_bytes=eb, eps=float(eps),
        # the online norm exists only where the norm input is sharded (BTP): default it on there only
        enable_online_rmsnorm=_bool_key(raw, "enable_online_rmsnorm", strategy is Strategy.BOTTLENECK),
        enable_grouping=_bool_key(raw, "enable_grouping", False),
        enable_lowrank_ckpt=_bool_key(raw, "enable_lowrank_ckpt", False),
        lax_h_prev=lax_h_prev,
    )


def load_scenario(path: str) -> Scenario:
    """A scenario from a .toml or .json file (reference cli.py:249-266)."""
    p = Path(path)
    if not p.exists():
        raise ConfigError(f"config file not found: {path}")
    text = p.read_bytes()
    suffix = p.suffix.lower()
    if suffix == ".json":
        try:
            raw = json.loads(text)
        except json.JSONDecodeError as exc:
            raise ConfigError(f"{path}:{exc.lineno}:{exc.colno}: {exc.msg}") from exc
    elif suffix == ".toml":
        try:
            raw = tomllib.loads(text.decode("utf-8"))
        except tomllib.TOMLDecodeError as exc:
            raise ConfigError(f"{path}: {exc}") from exc
    else:
        raise ConfigError(f"config must be .toml or .json, got {p.suffix!r}")
    return scenario_from_dict(raw, default_name=p.stem)


def apply_overrides(scn: Scenario, args) -> Scenario:
    """Flags win over the file (reference cli.py:269-291). `args` is an argparse Namespace (or any
    object) whose absent / None attributes leave the scenario's value in place."""
    cfg, variant, strategy = scn.cfg, scn.variant, scn.strategy
    arch = getattr(args, "lowrank_architecture_type", None)
    if arch:
        variant = Variant(arch)
        _require(cfg.r is not None, f"variant {variant.value} needs a bottleneck rank r")
    enable_btp = strategy is Strategy.BOTTLENECK
    if getattr(args, "enable_btp", None) is not None:
        enable_btp = args.enable_btp
    if variant is not scn.variant or enable_btp != (strategy is Strategy.BOTTLENECK):
        strategy = _resolve_strategy(variant, None, enable_btp)
    updates = {"variant": variant, "strategy": strategy}
    for key in ("seed", "element_bytes", "enable_online_rmsnorm", "enable_grouping", "enable_lowrank_ckpt"):
        v = getattr(args, key, None)
        if v is not None:
            updates[key] = v
    return replace(scn, **updates)


def build_plan(scn: Scenario) -> ShardPlan:
    """The scenario's ShardPlan (reference cli.py:294-304)."""
    return plan(scn.strategy, scn.cfg, scn.shape,
                variant=None if scn.strategy is Strategy.FULL_RANK else scn.variant,
                online_norm=scn.enable_online_rmsnorm, grouping=scn.enable_grouping,
                lowrank_ckpt=scn.enable_lowrank_ckpt)


def add_config_flags(ap: argparse.ArgumentParser) -> argparse.ArgumentParser:
    """The reference's scenario override flags (cli.py:638-660), for `apply_overrides`."""
    ap.add_argument("--seed", type=int, help="override the scenario seed")
    ap.add_argument("--element-bytes", type=int, choices=list(VALID_ELEMENT_BYTES),
                    help="override the accounting element width")
    ap.add_argument("--lowrank-architecture-type", choices=[v.value for v in Variant if v is not Variant.FULL_RANK],
                    help="override the low-rank variant")
    ap.add_argument("--enable-btp", action=argparse.BooleanOptionalAction, default=None)
    ap.add_argument("--enable-online-rmsnorm", action=argparse.BooleanOptionalAction, default=None)
    ap.add_argument("--enable-grouping", action=argparse.BooleanOptionalAction, default=None)
    ap.add_argument("--enable-lowrank-ckpt", action=argparse.BooleanOptionalAction, default=None)
    return ap


def scenario_inputs(scn: Scenario, *, scaled: bool = False):
    """(block, x, h_prev) exactly as the reference builds them (cli.py:307-320); scaled applies
    the bf16 parity recipe (model.fan_in_scaled) to the factors."""
    from .model import build_block, fan_in_scaled, seeded_h_prev, zero_h_prev
    from .tensor import seeded_fill

    block = build_block(scn.cfg, scn.variant, scn.seed, element_bytes=scn.element_bytes)
    if scaled:
        block = fan_in_scaled(block)
    x = seeded_fill((scn.shape.b, scn.shape.s, scn.cfg.d), scn.seed + INPUT_SEED_OFFSET, scn.element_bytes)
    h_prev = None
    if scn.variant is Variant.LAX:
        if scn.lax_h_prev == "seeded":
            h_prev = seeded_h_prev(scn.cfg, scn.shape, scn.seed + HPREV_SEED_OFFSET, element_bytes=scn.element_bytes)
        else:
            h_prev = zero_h_prev(scn.cfg, scn.shape, element_bytes=scn.element_bytes)
    return block, x, h_prev


def run_scenario(scn: Scenario, *, scaled: bool = True, precision: str = "bf16", model_tail: bool = True):
    """Execute a scenario's block forward on this rank's GPU (the device counterpart of the
    reference's `_simulate`, cli.py:351-372): low-rank ckpt on => `run_with_ckpt` (returns a
    CkptRun), else `execute_forward` (returns a SimResult). At tp > 1 every rank calls it."""
    from .api import execute_forward
    from .checkpointing import CkptPolicy, run_with_ckpt

    pl = build_plan(scn)
    block, x, h_prev = scenario_inputs(scn, scaled=scaled)
    if scn.enable_lowrank_ckpt and pl.lowrank_ckpt:
        return run_with_ckpt(pl, block, x, CkptPolicy.LOWRANK_BOUNDARY, h_prev, eps=scn.eps, model_tail=model_tail)
    return execute_forward(pl, block, x, h_prev, eps=scn.eps, model_tail=model_tail, precision=precision)
