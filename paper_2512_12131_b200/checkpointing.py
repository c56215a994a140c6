"""Low-rank boundary activation checkpointing on the device path (reference `btpsim.checkpointing`,
pkg/src/btpsim/checkpointing.py:1-163, and the re-forward sweeps simulator.py:720-921).

Policy LOWRANK_BOUNDARY keeps, per block and rank, only the block input shard x_i, the seven
reduced rank-r tensors z_* (replicated [T, r]) and the per-row global RMS s1/s2 (fp32 [T]; the
reference keeps them only in sync mode, but backward needs them and recovering them would cost
a collective). Everything else is recomputed in backward from that set with ZERO collectives
under BTP. The naive-TP baseline keeps x and its rank-local z shards and must replay the
all-reduces of its up-projection partials (qkv, o, gate_up: 3 grouped, 6 ungrouped), which is
the comparison the reference's checkpointing tests make (test_ckpt.py:90-125).

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
    """Reference checkpointing.py:45-72, field for field, in the reference's all-rank units:
    stored elements and recompute FLOPs summed over the TP ranks (replicated z charged once per
    rank), ring elements 2(tp-1) x payload per re-run collective. The device also reports bytes
    (bf16 activations + fp32 statistics). The kept set is what the device backward reads, not the
    reference's workspace inventory, so ΔMem / eff are comparable in ordering, not digit for digit."""

    policy: CkptPolicy
    stored_elements_without: int   # activation elements a plain forward keeps for backward (all ranks)
    stored_elements_with: int      # ... under the low-rank boundary policy
    recompute_flops: int
    reforward_collectives: int
    reforward_ring_elements: int
    stored_bytes_without: int = 0
    stored_bytes_with: int = 0

    @property
    def delta_mem_elements(self) -> int:
        return self.stored_elements_without - self.stored_elements_with

    @property
    def delta_mem_bytes(self) -> int:
        return self.stored_bytes_without - self.stored_bytes_with

    @property
    def time_proxy(self) -> int:
        return self.recompute_flops + COMM_FLOP_EQUIV_PER_ELEMENT * self.reforward_ring_elements

    def to_dict(self) -> dict:
        return {
            "policy": self.policy.value,
            "stored_elements_without": self.stored_elements_without,
            "stored_elements_with": self.stored_elements_with,
            "delta_mem_elements": self.delta_mem_elements,
            "recompute_flops": self.recompute_flops,
            "reforward_collectives": self.reforward_collectives,
            "reforward_ring_elements": self.reforward_ring_elements,
            "time_proxy": self.time_proxy,
            "eff_ckpt": float(eff_ckpt(self)) if self.policy is CkptPolicy.LOWRANK_BOUNDARY else None,
            "stored_bytes_without": self.stored_bytes_without,
            "stored_bytes_with": self.stored_bytes_with,
        }


def eff_ckpt(report: CkptReport) -> Fraction:
    """Memory freed per unit of recompute-time proxy, as an exact rational (reference
    checkpointing.py:75-79)."""
    if report.time_proxy == 0:
        raise ValueError("nothing was recomputed; eff_ckpt is undefined")
    return Fraction(report.delta_mem_elements, report.time_proxy)


@dataclass
class CkptRun:
    result: object                 # SimResult of the plain forward (reference checkpointing.py:83-87)
    report: CkptReport
    recompute_bitwise_ok: bool
    recompute_checks: dict

    @property
    def y(self):
        return self.result.y


# what each executor's re-forward rebuilds, compared bitwise with the plain forward's tensors
_RECOMPUTED_BTP = ("x_mid", "gu", "act", "qkv", "attn", "a_o", "a_gu", "a_d", "a_qkv")


def _all_ranks(ex, *counts) -> tuple[int, ...]:
    """Per-rank counts summed over the TP group — the reference's all-rank convention
    (checkpointing.py:1-8: memory summed over ranks, replicated storage charged once per rank;
    trace FLOPs summed over ranks). Live group: an all-reduce; record-only: ranks are symmetric."""
    if ex.tp == 1:
        return tuple(int(c) for c in counts)
    if ex.comm.live:
        import torch.distributed as dist

        t = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=ex.dev)
        dist.all_reduce(t, group=ex.comm.group)
        return tuple(int(v) for v in t.tolist())
    return tuple(int(c) * ex.tp for c in counts)


def _snapshot(ex, names) -> dict:
    out = {}
    for name in names:
        v = ex.saved[name]
        out[name] = [t.clone() for t in v] if isinstance(v, list) else v.clone()
    return out


def run_with_ckpt(pl: ShardPlan, block: DecoderBlockWeights, x, policy: CkptPolicy, h_prev=None, *,
                  eps: float = EPS_DEFAULT, model_tail: bool = False) -> CkptRun:
    """Device analogue of the reference's run_with_ckpt (checkpointing.py:109-163): BTP re-forwards
    with zero collectives; the naive-TP baseline replays its chunk all-reduces (3 grouped / 6 not)."""
    from .api import SimResult, _check_inputs, _gather_y, _h_cur, _normalise, _stage_h_prev, make_executor, shard_input
    from .tensor import Tensor

    pl, block = _normalise(pl, block)
    policy = CkptPolicy(getattr(policy, "value", policy))

    if policy is CkptPolicy.LOWRANK_BOUNDARY and pl.strategy is Strategy.FULL_RANK:
        raise PlanError("lowrank-boundary checkpointing stores rank-r tensors; the full-rank strategy has none")
    xv = _check_inputs(pl, block, x)
    b, s, d = xv.shape
    full_pl = replace(pl, lowrank_ckpt=False)
    ex = make_executor(full_pl, block, eps=eps)
    _stage_h_prev(ex, block, h_prev)
    x_sh = shard_input(ex, xv)
    y_sh = ex.forward(x_sh)
    h_cur = _h_cur(ex, b, s)
    y = _gather_y(ex, y_sh, model_tail)
    result = SimResult(Tensor(y.double().cpu().numpy().reshape(b, s, d)), h_cur, ex.comm.trace,
                       [dict() for _ in range(pl.shape.tp)], pl)
    without_e, without_b = _all_ranks(ex, ex.saved_activation_elements(), ex.saved_activation_bytes())
    if policy is CkptPolicy.NONE:
        rep = CkptReport(policy, without_e, without_e, 0, 0, 0, without_b, without_b)
        return CkptRun(result, rep, True, {})
    names = getattr(ex, "RECOMPUTED", _RECOMPUTED_BTP)
    reference = _snapshot(ex, names)

    ck_pl = replace(pl, lowrank_ckpt=True)
    ck = make_executor(ck_pl, block, eps=eps)
    _stage_h_prev(ck, block, h_prev)
    ck.forward(x_sh)
    with_e, with_b = _all_ranks(ck, ck.saved_activation_elements(), ck.saved_activation_bytes())
    f0 = ck.stats.gemm_flops
    if pl.strategy is Strategy.BOTTLENECK:
        ck._recompute_mlp_inputs()
        ck._recompute_attn_inputs()
        heads_dim = pl.cfg.d // pl.shape.tp   # heads are split h/tp
    else:
        ck._reforward()
        heads_dim = pl.cfg.d                  # replicated attention
    torch.cuda.synchronize()
    # GEMM FLOPs + the re-run attention's (4 b s^2 x its width, the reference's sdpa_values
    # count, model.py:205-230), summed over ranks like the reference's trace; elementwise FLOPs
    # (the reference's EW_FLOPS, simulator.py:37) are not counted on the device path
    recompute_flops = _all_ranks(ck, ck.stats.gemm_flops - f0 + 4 * b * s * s * heads_dim)[0]
    checks = {}
    for name, want in reference.items():
        got = ck.saved[name]
        if isinstance(want, list):
            checks[name] = all(torch.equal(a, b_) for a, b_ in zip(got, want))
        else:
            checks[name] = bool(torch.equal(got, want))
    _, _, calls = ck.comm.trace.volume(pass_tag="reforward")
    ring = ring_transfer_elements(ck.comm.trace, pl.shape.tp, pass_tag="reforward")
    rep = CkptReport(policy, without_e, with_e, recompute_flops, calls, ring, without_b, with_b)
    return CkptRun(result, rep, all(checks.values()), checks)
