"""Low-rank boundary activation checkpointing on the device path (reference `btpsim.checkpointing`,
pkg/src/btpsim/checkpointing.py:1-163, and the re-forward sweeps simulator.py:720-921).

Policy LOWRANK_BOUNDARY keeps, per block and rank, only the block input shard x_i, the seven
reduced rank-r tensors z_* (replicated [T, r]) and the per-row global RMS s1/s2 (fp32 [T]; the
reference keeps them only in sync mode, but backward needs them and recovering them would cost
a collective). Everything else is recomputed in backward from that set with ZERO collectives
under BTP (the vanilla layout would have to replay its chunk all-reduces).

`run_with_ckpt` mirrors the reference contract: forward once, then re-materialise from the
checkpoint set and compare BITWISE with the forward's tensors (the device kernels are
deterministic, so any mismatch is a defect), and report the memory freed against the
recompute cost proxy (FLOPs + 64 x ring-transferred elements, reference :34-36).
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from enum import Enum
from fractions import Fraction

import torch

from .model import EPS_DEFAULT, DecoderBlockWeights
from .plan import PlanError, ShardPlan, Strategy
from .trace import ring_transfer_elements

COMM_FLOP_EQUIV_PER_ELEMENT = 64


class CkptPolicy(str, Enum):
    NONE = "none"
    LOWRANK_BOUNDARY = "lowrank-boundary"


@dataclass(frozen=True)
class CkptReport:
    policy: CkptPolicy
    stored_bytes_without: int      # activations kept for backward by a plain forward (this rank)
    stored_bytes_with: int         # ... under the low-rank boundary policy
    recompute_flops: int
    reforward_collectives: int
    reforward_ring_elements: int

    @property
    def delta_mem_bytes(self) -> int:
        return self.stored_bytes_without - self.stored_bytes_with

    @property
    def time_proxy(self) -> int:
        return self.recompute_flops + COMM_FLOP_EQUIV_PER_ELEMENT * self.reforward_ring_elements

    def to_dict(self) -> dict:
        return {
            "policy": self.policy.value,
            "stored_bytes_without": self.stored_bytes_without,
            "stored_bytes_with": self.stored_bytes_with,
            "delta_mem_bytes": self.delta_mem_bytes,
            "recompute_flops": self.recompute_flops,
            "reforward_collectives": self.reforward_collectives,
            "reforward_ring_elements": self.reforward_ring_elements,
            "time_proxy": self.time_proxy,
            "eff_ckpt": float(eff_ckpt(self)) if self.policy is CkptPolicy.LOWRANK_BOUNDARY else None,
        }


def eff_ckpt(report: CkptReport) -> Fraction:
    """Memory freed per unit of recompute-time proxy (reference checkpointing.py:75-79)."""
    if report.time_proxy == 0:
        raise ValueError("nothing was recomputed; eff_ckpt is undefined")
    return Fraction(report.delta_mem_bytes, report.time_proxy)


@dataclass
class CkptRun:
    y: torch.Tensor
    report: CkptReport
    recompute_bitwise_ok: bool
    recompute_checks: dict


_RECOMPUTED = ("x_mid", "gu", "act", "qkv", "attn", "a_o", "a_gu", "a_d", "a_qkv")


def run_with_ckpt(pl: ShardPlan, block: DecoderBlockWeights, x, policy: CkptPolicy, h_prev=None, *,
                  eps: float = EPS_DEFAULT, model_tail: bool = False) -> CkptRun:
    """Device analogue of the reference's run_with_ckpt (checkpointing.py:109-163)."""
    from .api import _check_inputs, _stage_h_prev, make_executor, shard_input

    if policy is CkptPolicy.LOWRANK_BOUNDARY and pl.strategy is Strategy.FULL_RANK:
        raise PlanError("lowrank-boundary checkpointing stores rank-r tensors; the full-rank strategy has none")
    if pl.strategy is not Strategy.BOTTLENECK:
        raise PlanError("the device re-forward is implemented for the btp strategy")
    xv = _check_inputs(pl, block, x)
    full_pl = replace(pl, lowrank_ckpt=False)
    ex = make_executor(full_pl, block, eps=eps)
    _stage_h_prev(ex, block, h_prev)
    x_sh = shard_input(ex, xv)
    y = ex.forward(x_sh).clone()
    without = ex.saved_activation_bytes()
    if policy is CkptPolicy.NONE:
        rep = CkptReport(policy, without, without, 0, 0, 0)
        return CkptRun(y, rep, True, {})
    reference = {}
    for name in _RECOMPUTED:
        v = ex.saved[name]
        reference[name] = [t.clone() for t in v] if isinstance(v, list) else v.clone()

    ck_pl = replace(pl, lowrank_ckpt=True)
    ck = make_executor(ck_pl, block, eps=eps)
    _stage_h_prev(ck, block, h_prev)
    ck.forward(x_sh)
    with_ = ck.saved_activation_bytes()
    f0 = ck.stats.gemm_flops
    ck._recompute_mlp_inputs()
    ck._recompute_attn_inputs()
    torch.cuda.synchronize()
    attn_flops = 4 * pl.shape.b * pl.shape.s * pl.shape.s * (pl.cfg.d // pl.shape.tp)
    recompute_flops = ck.stats.gemm_flops - f0 + attn_flops
    checks = {}
    for name, want in reference.items():
        got = ck.saved[name]
        if isinstance(want, list):
            checks[name] = all(torch.equal(a, b) for a, b in zip(got, want))
        else:
            checks[name] = bool(torch.equal(got, want))
    _, _, calls = ck.comm.trace.volume(pass_tag="reforward")
    ring = ring_transfer_elements(ck.comm.trace, pl.shape.tp, pass_tag="reforward")
    rep = CkptReport(policy, without, with_, recompute_flops, calls, ring)
    return CkptRun(y, rep, all(checks.values()), checks)
