"""Collective log with the reference's record schema (reference simulator.py:47-120).

Every collective the executor issues — real NCCL/gloo calls, or the record-only no-op at
tp == 1 (the reference records even single-rank collectives, simulator.py:153-161) — appends
one CollectiveRecord with the LOGICAL payload (element count of the reduced / gathered
tensor, no ring factor). `record_tuples` is what tests compare against
`plan.enumerate_collectives`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

# Fixed per-element costs of non-GEMM work (reference simulator.py:37-44); relative scale only.
EW_FLOPS = {"rmsnorm": 4, "swiglu": 5, "crossgate": 5, "add": 1, "softmax": 5, "scale": 1}


@dataclass(frozen=True)
class CollectiveRecord:
    kind: str        # all-reduce | all-reduce-coalesced | all-gather
    chunk_id: str
    tag: str         # block | fused-stat | boundary
    elements: int
    nbytes: int
    pass_tag: str    # forward | reforward | backward
    extras: tuple[tuple[str, int, int], ...] = ()

    def payloads(self) -> tuple[tuple[str, int, int], ...]:
        return ((self.tag, self.elements, self.nbytes), *self.extras)


@dataclass
class Trace:
    element_bytes: int = 2
    records: list[CollectiveRecord] = field(default_factory=list)
    gemm_launches: int = 0
    gemm_flops: int = 0
    elementwise_flops: int = 0

    def add_ew(self, kind: str, elements: int) -> None:
        self.elementwise_flops += EW_FLOPS[kind] * elements

    def add_gemm(self, flops: int, launches: int = 1) -> None:
        self.gemm_flops += flops
        self.gemm_launches += launches

    def emit(self, kind: str, chunk_id: str, tag: str, elements: int, pass_tag: str, extras=()) -> None:
        eb = self.element_bytes
        self.records.append(
            CollectiveRecord(kind, chunk_id, tag, int(elements), int(elements) * eb, pass_tag,
                             tuple((t, int(e), int(e) * eb) for t, e in extras))
        )

    def volume(self, tag: str | None = None, pass_tag: str | None = None) -> tuple[int, int, int]:
        """(elements, bytes, calls) over payloads matching tag and pass; a coalesced record is one call."""
        el = nb = calls = 0
        for rec in self.records:
            if pass_tag is not None and rec.pass_tag != pass_tag:
                continue
            hits = [(e, b) for t, e, b in rec.payloads() if tag is None or t == tag]
            if hits:
                calls += 1
                el += sum(e for e, _ in hits)
                nb += sum(b for _, b in hits)
        return el, nb, calls

    def record_tuples(self, pass_tag: str | None = None) -> list[tuple]:
        return [
            (r.chunk_id, r.kind, r.tag, r.elements, tuple((t, e) for t, e, _ in r.extras))
            for r in self.records
            if pass_tag is None or r.pass_tag == pass_tag
        ]


def trace_volume(trace: Trace, tag: str | None = None, pass_tag: str | None = None) -> tuple[int, int, int]:
    return trace.volume(tag=tag, pass_tag=pass_tag)


def ring_transfer_elements(trace: Trace, tp: int, pass_tag: str | None = None) -> int:
    """2*(tp-1)*payload per record, summed (reference simulator.py:107-120)."""
    return sum(
        2 * (tp - 1) * e
        for rec in trace.records
        if pass_tag is None or rec.pass_tag == pass_tag
        for _, e, _ in rec.payloads()
    )


def tp_block_volume(strategy, cfg, shape) -> int:
    """Closed-form forward all-reduce elements per block (logical payload, no ring factor) that
    the traced collectives must equal exactly — reference costs.py:28-44: full-rank two [T, d]
    boundaries, naive TP five [T, d] + two [T, d_ff] full-width partials, BTP seven [T, r]."""
    from .plan import Strategy

    strategy = Strategy(getattr(strategy, "value", strategy))
    t = shape.b * shape.s
    if strategy is Strategy.FULL_RANK:
        return 2 * t * cfg.d
    if strategy is Strategy.VANILLA:
        return 5 * t * cfg.d + 2 * t * cfg.d_ff
    if strategy is Strategy.BOTTLENECK:
        if cfg.r is None:
            raise ValueError("btp volume needs a bottleneck rank r")
        return 7 * t * cfg.r
    raise ValueError(f"unknown strategy {strategy!r}")
