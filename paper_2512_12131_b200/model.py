"""Block configuration, presets and deterministic weights — the reference's config API.

Same names, fields, validation and seeding as `btpsim.model` (pkg/src/btpsim/model.py), so
a scenario built for the reference builds the identical block here:

* `ModelConfig` (:58-89), `PRESETS`/`preset` (:93-106), `RunShape` (:109-123)
* `projection_dims` (:126-137), `DecoderBlockWeights` (:140-155), `build_block` (:158-186)

Factor naming follows the reference: the DOWN factor B[r, d_in] is applied first, the UP
factor A[d_out, r] second. `cola` is the rank-preserving crossgate sigma
[silu(u)*v, silu(v)*u] on the two halves of the rank-r activation (model.py:189-196).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from enum import Enum
from fractions import Fraction

import numpy as np

from .tensor import DivisibilityError, Tensor, seeded_fill

EPS_DEFAULT = 1e-6
PROJECTIONS = ("q", "k", "v", "o", "gate", "up", "down")


class Variant(str, Enum):
    FULL_RANK = "full-rank"
    SVD = "svd"
    COLA = "cola"
    LAX = "lax"


LOWRANK_VARIANTS = (Variant.SVD, Variant.COLA, Variant.LAX)


@dataclass(frozen=True)
class ModelConfig:
    layers: int
    heads: int
    d: int
    d_ff: int
    r: int | None = None

    def __post_init__(self):
        for name in ("layers", "heads", "d", "d_ff"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.d % self.heads:
            raise DivisibilityError(f"d={self.d} not divisible by heads={self.heads}")
        if self.r is not None and self.r <= 0:
            raise ValueError("r must be positive when set")

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    @property
    def alpha(self) -> Fraction:
        return Fraction(self.d_ff, self.d)

    @property
    def beta(self) -> Fraction:
        if self.r is None:
            raise ValueError("beta undefined without r")
        return Fraction(self.d, self.r)


PRESETS: dict[str, ModelConfig] = {
    name: ModelConfig(layers=l, heads=h, d=d, d_ff=ff, r=r)
    for name, (l, h, d, ff, r) in {
        "1b": (24, 32, 2048, 5472, 512),
        "3b": (28, 24, 3072, 8192, 768),
        "7b": (32, 32, 4096, 11008, 1024),
        "13b": (40, 40, 5120, 13824, 1280),
        "30b": (36, 64, 8192, 22016, 2048),
    }.items()
}

# LLaMA-60M (CoLA paper's smallest model); not a reference preset, built explicitly.
COLA_60M = ModelConfig(layers=8, heads=8, d=512, d_ff=1376, r=128)


def preset(name: str) -> ModelConfig:
    try:
        return PRESETS[name.lower()]
    except KeyError:
        raise KeyError(f"unknown preset {name!r}; choose from {sorted(PRESETS)}") from None


@dataclass(frozen=True)
class RunShape:
    b: int
    s: int
    tp: int = 1
    p: int = 1

    def __post_init__(self):
        for name in ("b", "s", "tp", "p"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")

    @property
    def tokens(self) -> int:
        return self.b * self.s


def projection_dims(cfg: ModelConfig) -> dict[str, tuple[int, int]]:
    """(d_out, d_in) per projection."""
    d, f = cfg.d, cfg.d_ff
    return {"q": (d, d), "k": (d, d), "v": (d, d), "o": (d, d), "gate": (f, d), "up": (f, d), "down": (d, f)}


@dataclass(frozen=True)
class DecoderBlockWeights:
    cfg: ModelConfig
    variant: Variant
    full: dict[str, Tensor] = field(default_factory=dict)          # W[d_out, d_in]
    down_factors: dict[str, Tensor] = field(default_factory=dict)  # B[r, d_in]
    up_factors: dict[str, Tensor] = field(default_factory=dict)    # A[d_out, r]
    gamma1: Tensor | None = None
    gamma2: Tensor | None = None

    def linear_parameter_count(self) -> int:
        groups = (self.full, self.down_factors, self.up_factors)
        return sum(t.elements for g in groups for t in g.values())


def build_block(cfg: ModelConfig, variant: Variant, seed: int, element_bytes: int = 2) -> DecoderBlockWeights:
    """Deterministic weights: seed+i per full matrix, or seed+2i (B) / seed+2i+1 (A) per factor pair;
    gamma1/gamma2 from seed+101/102 (reference model.py:158-186)."""
    variant = Variant(getattr(variant, "value", variant))
    if not isinstance(cfg, ModelConfig):
        cfg = ModelConfig(layers=cfg.layers, heads=cfg.heads, d=cfg.d, d_ff=cfg.d_ff, r=getattr(cfg, "r", None))
    dims = projection_dims(cfg)
    full: dict[str, Tensor] = {}
    down: dict[str, Tensor] = {}
    up: dict[str, Tensor] = {}
    if variant is Variant.FULL_RANK:
        for i, name in enumerate(PROJECTIONS):
            full[name] = seeded_fill(dims[name], seed + i, element_bytes)
    else:
        if cfg.r is None:
            raise ValueError(f"variant {variant.value} needs cfg.r")
        if variant is Variant.COLA and cfg.r % 2:
            raise DivisibilityError(f"r={cfg.r} must be even for the cola gate split")
        for i, name in enumerate(PROJECTIONS):
            d_out, d_in = dims[name]
            down[name] = seeded_fill((cfg.r, d_in), seed + 2 * i, element_bytes)
            up[name] = seeded_fill((d_out, cfg.r), seed + 2 * i + 1, element_bytes)
    g1 = seeded_fill((cfg.d,), seed + 101, element_bytes)
    g2 = seeded_fill((cfg.d,), seed + 102, element_bytes)
    return DecoderBlockWeights(cfg, variant, full, down, up, g1, g2)


def zero_h_prev(cfg: ModelConfig, shape: RunShape, element_bytes: int = 2) -> dict[str, Tensor]:
    """The lax first-layer boundary bundle: zeros for all seven projections (model.py:308-315)."""
    if cfg.r is None:
        raise ValueError("h bundle needs cfg.r")
    return {n: Tensor(np.zeros((shape.b, shape.s, cfg.r)), element_bytes) for n in PROJECTIONS}


def seeded_h_prev(cfg: ModelConfig, shape: RunShape, seed: int, element_bytes: int = 2) -> dict[str, Tensor]:
    """Deterministic nonzero lax bundle: projection i gets fill((b, s, r), seed + 7 i) (model.py:318-325)."""
    if cfg.r is None:
        raise ValueError("h bundle needs cfg.r")
    return {n: seeded_fill((shape.b, shape.s, cfg.r), seed + 7 * i, element_bytes) for i, n in enumerate(PROJECTIONS)}


def fan_in_scaled(block: DecoderBlockWeights, gain: float = 3.0) -> DecoderBlockWeights:
    """The parity recipe: every linear factor times sqrt(gain / fan_in).

    The reference's raw uniform(-1, 1) factors blow activations up to ~1e14 at real widths,
    which no bf16 pipeline can reproduce; scaling by sqrt(3/fan_in) gives unit-variance
    outputs. Both the oracle and the GPU path consume the same scaled block.
    """

    def scale(group: dict[str, Tensor]) -> dict[str, Tensor]:
        return {
            k: Tensor(v.values * np.sqrt(gain / v.shape[1]), v.element_bytes) for k, v in group.items()
        }

    return dataclasses.replace(
        block, full=scale(block.full), down_factors=scale(block.down_factors), up_factors=scale(block.up_factors)
    )


# ----------------------------------------------------------------------------- model boundary
# SURVEY §8f row 1 (absent in the reference, whose executor stops at one block + the tail
# all-gather, simulator.py:710-714): L blocks chained through the d-sharded residual, fed by a
# d-sharded token embedding (the paper shards the embedding output so the first down-projection
# is row-split), a final RMSNorm and a replicated LM head with mean next-token
# cross-entropy. Builder-defined seeding: block l from seed + 1000*l, embedding / final gain /
# head from seed + 50000 / 50001 / 50002 (head fan-in scaled like the blocks).
LAYER_SEED_STRIDE = 1000


@dataclass(frozen=True)
class ModelWeights:
    cfg: ModelConfig
    variant: Variant
    vocab: int
    blocks: tuple[DecoderBlockWeights, ...]
    embedding: Tensor      # [vocab, d]
    final_gamma: Tensor    # [d]
    head: Tensor           # [vocab, d]

    @property
    def layers(self) -> int:
        return len(self.blocks)


def build_model(cfg: ModelConfig, variant: Variant, seed: int, vocab: int, layers: int | None = None,
                scaled: bool = True, element_bytes: int = 2) -> ModelWeights:
    """`layers` defaults to cfg.layers; `scaled` applies the parity recipe (fan_in_scaled) to every block."""
    n = cfg.layers if layers is None else layers
    if vocab <= 0 or n <= 0:
        raise ValueError("vocab and layers must be positive")
    blocks = []
    for l in range(n):
        blk = build_block(cfg, variant, seed + LAYER_SEED_STRIDE * l, element_bytes)
        blocks.append(fan_in_scaled(blk) if scaled else blk)
    head = seeded_fill((vocab, cfg.d), seed + 50002, element_bytes)
    if scaled:
        head = Tensor(head.values * np.sqrt(3.0 / cfg.d), element_bytes)
    return ModelWeights(cfg, variant, vocab, tuple(blocks), seeded_fill((vocab, cfg.d), seed + 50000, element_bytes),
                        seeded_fill((cfg.d,), seed + 50001, element_bytes), head)


def token_batch(b: int, s: int, vocab: int, seed: int = 40000) -> tuple[np.ndarray, np.ndarray]:
    """Synthetic next-token data: SplitMix64 stream mod vocab, [b, s+1] -> (inputs, targets), each int64 [b*s]."""
    from .tensor import splitmix64

    raw = splitmix64(seed, b * (s + 1))
    ids = (raw % np.uint64(vocab)).astype(np.int64).reshape(b, s + 1)
    return ids[:, :-1].reshape(-1), ids[:, 1:].reshape(-1)
