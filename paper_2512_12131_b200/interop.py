"""Accept the reference package's own objects at the public API (drop-in boundary).

A `btpsim` caller hands over `btpsim.ShardPlan`, `btpsim.DecoderBlockWeights`, `btpsim.Tensor`,
`btpsim.Strategy` / `Variant` / `CkptPolicy` members and `btpsim.ModelConfig` / `RunShape`.
Those are different classes from ours, so identity tests (`x is Strategy.BOTTLENECK`) and
`isinstance(x, Tensor)` would misroute them. Every public entry point therefore normalises its
arguments here first:

* enums by their `.value` string (both packages use the same values, reference plan.py:33-42,
  model.py:31-37, checkpointing.py:39-41);
* tensors by duck type: anything with a `.values` float array (reference tensor.py:31-60);
* dataclasses by their fields only (reference model.py:48-123, :140-156; plan.py:105-118).

A foreign plan is rebuilt with our `plan()` from its strategy / config / shape / variant / flags
and must reproduce the foreign chunk table exactly; a mismatch raises `PlanError` rather than
executing a different plan.
"""

from __future__ import annotations

import numpy as np

from .model import DecoderBlockWeights, ModelConfig, RunShape, Variant
from .plan import NormMode, PlanError, ShardPlan, Strategy, plan
from .tensor import Tensor


def _enum(cls, v):
    if isinstance(v, cls):
        return v
    try:
        return cls(getattr(v, "value", v))
    except ValueError:
        raise ValueError(f"{v!r} is not a valid {cls.__name__}") from None


def as_strategy(v) -> Strategy:
    return _enum(Strategy, v)


def as_variant(v) -> Variant:
    return _enum(Variant, v)


def as_norm_mode(v) -> NormMode:
    return _enum(NormMode, v)


def as_config(cfg) -> ModelConfig:
    if isinstance(cfg, ModelConfig):
        return cfg
    return ModelConfig(layers=cfg.layers, heads=cfg.heads, d=cfg.d, d_ff=cfg.d_ff, r=getattr(cfg, "r", None))


def as_shape(shape) -> RunShape:
    if isinstance(shape, RunShape):
        return shape
    return RunShape(b=shape.b, s=shape.s, tp=getattr(shape, "tp", 1), p=getattr(shape, "p", 1))


def is_tensor_like(x) -> bool:
    return isinstance(x, Tensor) or (hasattr(x, "values") and isinstance(getattr(x, "values"), np.ndarray))


def as_tensor(x, element_bytes: int = 2) -> Tensor:
    """Tensor from ours, a reference Tensor (duck-typed on `.values`), or any array-like."""
    if isinstance(x, Tensor):
        return x
    if is_tensor_like(x):
        return Tensor(np.asarray(x.values, dtype=np.float64), int(getattr(x, "element_bytes", element_bytes)))
    return Tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float64)), element_bytes)


def values_of(x) -> np.ndarray:
    """The float64 values of a Tensor-like or array-like input."""
    if is_tensor_like(x):
        return np.asarray(x.values)
    return np.asarray(x)


def element_bytes_of(x, default: int = 2) -> int:
    return int(getattr(x, "element_bytes", default)) if is_tensor_like(x) else default


def as_block(block) -> DecoderBlockWeights:
    if isinstance(block, DecoderBlockWeights):
        return block

    def group(g):
        return {k: as_tensor(v) for k, v in (g or {}).items()}

    return DecoderBlockWeights(
        as_config(block.cfg),
        as_variant(block.variant),
        group(getattr(block, "full", None)),
        group(getattr(block, "down_factors", None)),
        group(getattr(block, "up_factors", None)),
        None if block.gamma1 is None else as_tensor(block.gamma1),
        None if block.gamma2 is None else as_tensor(block.gamma2),
    )


def _chunk_table(pl) -> tuple:
    return tuple((c.chunk_id, tuple(c.ops), int(c.payload_elements), int(c.rider_elements)) for c in pl.chunks)


def as_plan(pl) -> ShardPlan:
    """Our ShardPlan for ours or a reference one (rebuilt and cross-checked chunk by chunk)."""
    if isinstance(pl, ShardPlan):
        return pl
    strategy = as_strategy(pl.strategy)
    variant = None if strategy is Strategy.FULL_RANK else as_variant(pl.variant)
    ours = plan(strategy, as_config(pl.cfg), as_shape(pl.shape), variant,
                online_norm=as_norm_mode(pl.norm_mode) is NormMode.ONLINE,
                grouping=bool(pl.grouping), lowrank_ckpt=bool(pl.lowrank_ckpt))
    if _chunk_table(ours) != _chunk_table(pl):
        raise PlanError("foreign plan's chunk table differs from the plan rebuilt from its fields")
    if tuple(getattr(pl, "warnings", ())) != ours.warnings:
        from dataclasses import replace

        ours = replace(ours, warnings=tuple(pl.warnings))
    return ours


def as_h_prev(h_prev):
    if h_prev is None:
        return None
    return {k: as_tensor(v) for k, v in h_prev.items()}
