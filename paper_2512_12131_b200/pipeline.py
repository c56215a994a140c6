"""Pipeline parallelism (PP) with the 1F1B schedule around the BTP model stages.

The reference has PP only as a closed form: `costs.iter_volume("pp") = 2 * p * b * s * d` elements
per iteration (costs.py:63-64, PAPER.md:581, :631 — "pipeline activations of size [b, s, d] traverse
stage boundaries in forward / backward"); the paper's runs put TP inside a node and PP across nodes
with 1F1B scheduling and low-rank activation checkpointing. Here that layout is
executed: world = P stages x TP ranks, rank = stage * TP + tp_rank.

* Stage s owns blocks [s L/P, (s+1) L/P) of the model as a `ModelExecutor` over the MICRO-batch
  shape (b/m sequences); stage 0 also runs the d-sharded embedding, the last stage the tail
  all-gather, final RMSNorm, replicated LM head and cross-entropy. Inside a stage every block is the
  BTP block of executor.py on the stage's own TP group (its rank-r boundary all-reduces).
* Stage boundaries move this TP rank's residual shard [T_mb, d/TP] (bf16) point to point to the same
  TP rank of the next stage (forward) and its gradient back (backward): per iteration 2 (P - 1) m
  transfers of T_mb * d elements over the TP group, i.e. 2 (P - 1) b s d elements — the reference's
  2 p b s d with the P - 1 real edges counted (both are recorded in the trace as "p2p" records).
* 1F1B: stage s runs min(P - s - 1, m) warm-up forwards, then alternates one forward and one
  backward, then drains the remaining backwards; at most min(P - s, m) micro-batches are in flight
  on stage s, each in its own activation SLOT (the executors' per-block persistent buffers and
  saved tensors are switched per slot; temporaries stay shared). With low-rank checkpointing a slot
  holds only x, the seven z and the norm statistics per block — the paper's reason to combine the
  two.
* Gradients of the m micro-batches are accumulated into one fp32 buffer per executor (the
  cross-entropy is scaled by 1/m so the step's gradient is the full batch's mean-loss gradient),
  then the fused AdamW step runs once per stage.

Sends are asynchronous (isend) and receives blocking, so the 1F1B order cannot deadlock; with the
gloo backend (CPU tests, several ranks on one GPU) tensors are staged through host memory, with
NCCL they go device to device over NVLink.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch
import torch.distributed as dist

from . import kernels as K
from .comm import TPComm
from .model import ModelWeights, RunShape
from .model_executor import ModelExecutor
from .plan import PlanError, ShardPlan, Strategy, plan
from .trace import Trace


def schedule_1f1b(stage: int, stages: int, microbatches: int) -> list[tuple[str, int]]:
    """The 1F1B order of one stage: [("F", j) | ("B", j)] (PipeDream-flush / Megatron 1F1B)."""
    if not 0 <= stage < stages or microbatches <= 0:
        raise ValueError(f"bad stage {stage} of {stages} / microbatches {microbatches}")
    warm = min(stages - stage - 1, microbatches)
    out = [("F", j) for j in range(warm)]
    for i in range(microbatches - warm):
        out += [("F", warm + i), ("B", i)]
    out += [("B", j) for j in range(microbatches - warm, microbatches)]
    return out


def pp_boundary_elements(cfg, shape: RunShape, stages: int) -> int:
    """Elements moved across the stage boundaries per iteration (forward + backward, all TP ranks):
    2 (P - 1) b s d. The reference's closed form (costs.py:63-64) counts 2 p b s d."""
    return 2 * (stages - 1) * shape.b * shape.s * cfg.d


class _Slotted:
    """Switches an executor's per-block persistent buffers, saved tensors and per-forward
    attributes between in-flight micro-batch slots (temporaries in the shared scratch are not
    slotted)."""

    ATTRS = ("_ids", "_tg", "_y_full")

    def __init__(self, ex):
        self.ex = ex
        self.state = {0: self._get()}
        self.cur = 0

    def _get(self):
        ex = self.ex
        return {"_buf": ex._buf, "saved": ex.saved, **{a: getattr(ex, a, None) for a in self.ATTRS}}

    def use(self, k: int) -> None:
        ex = self.ex
        shared = ex._scratch is ex._buf
        self.state[self.cur] = self._get()
        st = self.state.setdefault(k, {"_buf": {}, "saved": {}, **{a: None for a in self.ATTRS}})
        for key, v in st.items():
            setattr(ex, key, v)
        if shared:
            ex._scratch = ex._buf
        self.cur = k


class PipelineStageExecutor(ModelExecutor):
    """One (stage, tp_rank) process's share of the model for a micro-batch shape."""

    def __init__(self, pl_mb: ShardPlan, mw: ModelWeights, stage: int, stages: int, comm: TPComm,
                 device="cuda", eps: float = 1e-6, attn_backend: str = "auto"):
        if mw.layers % stages:
            raise PlanError(f"layers={mw.layers} must divide into {stages} pipeline stages")
        if mw.variant.value == "lax":
            raise PlanError("lax bundles do not cross pipeline stages here (the h bundle is block-to-block)")
        per = mw.layers // stages
        sub = dataclasses.replace(mw, blocks=tuple(mw.blocks[stage * per:(stage + 1) * per]))
        super().__init__(pl_mb, sub, comm, device, eps, attn_backend)
        self.stage, self.stages = stage, stages
        self.first, self.last = stage == 0, stage == stages - 1
        self.layer0 = stage * per
        self._slots = [_Slotted(self)] + [_Slotted(ex) for ex in self.blocks]
        self._acc = None

    # ---------------------------------------------------------------- slots / accumulation
    def use_slot(self, k: int) -> None:
        for s in self._slots:
            s.use(k)

    def _flat_grads(self):
        out = []
        for ex in [self] + self.blocks:
            out += [ex.g_flat, ex.gam_grad_flat]
        return out

    def accumulate(self, j: int, m: int) -> None:
        """After micro-batch j's backward: acc (+)= grads; after the last one grads = acc."""
        gs = self._flat_grads()
        if self._acc is None:
            self._acc = [torch.empty_like(g) for g in gs]
        for a, g in zip(self._acc, gs):
            if j == 0:
                a.copy_(g)
            else:
                K.add(a.view(1, -1), g.view(1, -1), a.view(1, -1))
                self.stats.kernel_launches += 1
            if j == m - 1:
                g.copy_(a)

    # ---------------------------------------------------------------- stage pieces
    def stage_forward(self, x_or_ids: torch.Tensor) -> torch.Tensor:
        """Stage 0: int32 ids [T_mb] -> embedding -> blocks; others: the received residual shard."""
        self.comm.pass_tag = "forward"
        if self.first:
            return ModelExecutor.forward(self, x_or_ids)
        x = x_or_ids
        for ex in self.blocks:
            x = ex.forward(x)
        self.comm.pass_tag = "forward"
        return x

    def stage_backward(self, dy_sh: torch.Tensor | None) -> torch.Tensor:
        """Last stage: from the loss (dy_sh None); others: the received gradient shard. Returns the
        gradient of this stage's input shard (stage 0: after the embedding backward)."""
        if self.last:
            dy_sh = self._head_backward()
        dy_sh = self._blocks_backward(dy_sh)
        if self.first:
            self._embedding_backward(dy_sh)
        self._join_side()
        return dy_sh

    def backward(self, targets=None):  # the whole-model backward of a single-stage model only
        if not (self.first and self.last):
            raise PlanError("use stage_backward on a multi-stage pipeline")
        return ModelExecutor.backward(self)


class PipelineTrainer:
    """TP x PP training step of the BTP model with the 1F1B schedule (one process per GPU; world =
    stages x TP). `step(ids, targets)` runs the m micro-batches through this rank's stage and one
    AdamW update (unless optimizer=False), and returns the mean loss on the last stage (None
    elsewhere). Inputs are host int32 [b, s] arrays (every rank gets the full batch; stage 0 reads
    the ids, the last stage the targets)."""

    def __init__(self, pl: ShardPlan, mw: ModelWeights, *, stages: int, microbatches: int, eps: float = 1e-6,
                 attn_backend: str = "auto", adamw: dict | None = None, optimizer: bool = True):
        if pl.strategy is not Strategy.BOTTLENECK:
            raise PlanError("the pipeline runs BTP stages")
        if not dist.is_initialized():
            raise RuntimeError("PipelineTrainer needs an initialised torch.distributed process group")
        world, rank = dist.get_world_size(), dist.get_rank()
        if world % stages:
            raise PlanError(f"world size {world} is not a multiple of {stages} stages")
        tp = world // stages
        if pl.shape.tp != tp:
            raise PlanError(f"plan tp={pl.shape.tp} but world {world} / {stages} stages = TP {tp}")
        b, m = pl.shape.b, microbatches
        if m <= 0 or b % m:
            raise PlanError(f"batch b={b} must split into {m} micro-batches")
        self.stages, self.m, self.tp = stages, m, tp
        self.stage, self.tp_rank = rank // tp, rank % tp
        groups = [dist.new_group(list(range(s * tp, (s + 1) * tp))) for s in range(stages)]
        self.group = groups[self.stage]
        self.trace = Trace()
        comm = TPComm(tp, self.tp_rank, self.group if tp > 1 else None, self.trace)
        self.pl_mb = plan(pl.strategy, pl.cfg, RunShape(b // m, pl.shape.s, tp, stages), pl.variant,
                          online_norm=pl.norm_mode.value == "online", grouping=pl.grouping,
                          lowrank_ckpt=pl.lowrank_ckpt)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ex = PipelineStageExecutor(self.pl_mb, mw, self.stage, stages, comm, dev, eps, attn_backend)
        self.ex.loss_scale = 1.0 / m  # the step's gradient is the full batch's mean-loss gradient
        self.adamw = dict(adamw or {}) if optimizer else None
        self.dev = dev
        self.T_mb = (b // m) * pl.shape.s
        self.dl = pl.cfg.d // tp
        self.prev = rank - tp if self.stage > 0 else None
        self.next = rank + tp if self.stage < stages - 1 else None
        self.gloo = dist.get_backend() == "gloo"
        self._pending: list = []
        self.losses: list[float] = []

    # ---------------------------------------------------------------- point to point
    def _send(self, t: torch.Tensor, peer: int, chunk: str) -> None:
        self.trace.emit("p2p", chunk, "pp", t.numel(), self.ex.comm.pass_tag)
        src = t.contiguous().cpu() if self.gloo else t.contiguous()
        self._pending.append((dist.isend(src, peer), src))

    def _recv(self, peer: int) -> torch.Tensor:
        shape = (self.T_mb, self.dl)
        if self.gloo:
            buf = torch.empty(shape, dtype=self.ex.act)
            dist.recv(buf, peer)
            return buf.to(self.dev)
        buf = torch.empty(shape, dtype=self.ex.act, device=self.dev)
        dist.recv(buf, peer)
        return buf

    def _drain(self) -> None:
        for w, _ in self._pending:
            w.wait()
        self._pending.clear()

    # ---------------------------------------------------------------- the step
    def step(self, ids: np.ndarray, targets: np.ndarray):
        ex, m = self.ex, self.m
        ids = np.asarray(ids, dtype=np.int32).reshape(m, -1)
        targets = np.asarray(targets, dtype=np.int32).reshape(m, -1)
        n_slots = min(self.stages - self.stage, m)
        losses = []
        for op, j in schedule_1f1b(self.stage, self.stages, m):
            ex.use_slot(j % n_slots)
            if op == "F":
                if ex.first:
                    inp = torch.as_tensor(ids[j]).to(self.dev)
                else:
                    inp = self._recv(self.prev)  # block 0 keeps it alive in its saved x
                y = ex.stage_forward(inp)
                if ex.last:
                    tg = torch.as_tensor(targets[j]).to(self.dev)
                    losses.append(ex.loss_device(y, tg).clone())  # the slot's loss buffer is reused
                else:
                    self._send(y, self.next, "pp-activation")
            else:
                dy = None if ex.last else self._recv(self.next)
                ex.comm.pass_tag = "backward"
                dx = ex.stage_backward(dy)
                if not ex.first:
                    self._send(dx, self.prev, "pp-gradient")
                ex.accumulate(j, m)
        self._drain()
        if self.adamw is not None:
            ex.optimizer_step(**self.adamw)
        if ex.last:
            loss = float(torch.stack([l.view(()) for l in losses]).mean().item())
            self.losses.append(loss)
            return loss
        return None

    def stage_grads(self) -> dict:
        """This rank's accumulated gradients (float64 host copies), blocks keyed by GLOBAL layer."""
        g = self.ex.model_grads()
        return {"blocks": {self.ex.layer0 + i: gb for i, gb in enumerate(g["blocks"])},
                "dembedding": g["dembedding"] if self.ex.first else None,
                "dhead": g["dhead"] if self.ex.last else None,
                "dfinal_gamma": g["dfinal_gamma"] if self.ex.last else None}


__all__ = ["PipelineStageExecutor", "PipelineTrainer", "pp_boundary_elements", "schedule_1f1b"]
