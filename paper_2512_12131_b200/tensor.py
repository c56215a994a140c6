"""Host-side tensor wrapper, error types and the deterministic SplitMix64 fill.

Mirrors the reference's host data model (`btpsim.tensor`, pkg/src/btpsim/tensor.py): a
frozen float64 array plus a byte-accounting width, and `seeded_fill`, so blocks and inputs
built here are bit-identical to the reference's for the same (shape, seed). The arithmetic
of the block itself never runs here; it runs in libbtp.so on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

VALID_ELEMENT_BYTES = (1, 2, 4, 8)


class DimensionError(ValueError):
    """Operands do not conform (reference tensor.py:23-24)."""


class DivisibilityError(ValueError):
    """A dimension does not split as required; the message names it (reference tensor.py:27-28)."""


@dataclass(frozen=True)
class Tensor:
    """Row-major float64 host array with an accounting element width (reference tensor.py:31-60)."""

    values: np.ndarray
    element_bytes: int = 2

    def __post_init__(self):
        if self.element_bytes not in VALID_ELEMENT_BYTES:
            raise ValueError(f"element_bytes must be one of {VALID_ELEMENT_BYTES}, got {self.element_bytes}")
        if not isinstance(self.values, np.ndarray) or self.values.dtype != np.float64:
            raise TypeError("Tensor values must be a float64 ndarray")
        if not self.values.flags["C_CONTIGUOUS"]:
            object.__setattr__(self, "values", np.ascontiguousarray(self.values))

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(self.values.shape)

    @property
    def elements(self) -> int:
        return int(self.values.size)

    @property
    def logical_nbytes(self) -> int:
        return self.elements * self.element_bytes


def tensor(data, element_bytes: int = 2) -> Tensor:
    return Tensor(np.ascontiguousarray(np.asarray(data, dtype=np.float64)), element_bytes)


def zeros(shape: tuple[int, ...], element_bytes: int = 2) -> Tensor:
    return Tensor(np.zeros(shape, dtype=np.float64), element_bytes)


# SplitMix64 (Steele, Lea & Flood, OOPSLA 2014): Weyl increment + two xor-shift-multiply rounds.
_GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """uint64 outputs 1..count of SplitMix64 seeded with `seed` (state_i = seed + i*gamma)."""
    with np.errstate(over="ignore"):
        state = np.arange(1, count + 1, dtype=np.uint64) * _GOLDEN_GAMMA + np.uint64(seed % (1 << 64))
        state ^= state >> np.uint64(30)
        state *= _MIX1
        state ^= state >> np.uint64(27)
        state *= _MIX2
        state ^= state >> np.uint64(31)
    return state


def seeded_fill(shape: tuple[int, ...], seed: int, element_bytes: int = 2) -> Tensor:
    """Row-major fill in [-1, 1): u = (z >> 11) * 2^-53, value = 2u - 1 (reference tensor.py:197-209)."""
    n = int(np.prod(shape, dtype=np.int64)) if len(shape) else 1
    bits = splitmix64(seed, n) >> np.uint64(11)
    unit = bits.astype(np.float64) * (2.0**-53)
    return Tensor((unit * 2.0 - 1.0).reshape(shape), element_bytes)
