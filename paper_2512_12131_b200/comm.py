"""TP communicator: the collective sub-boundary of the reference (`SimGroup`,
simulator.py:123-186) over torch.distributed — NCCL over NVLink/NVSwitch on the GPU box,
gloo for the multi-process CPU tests.

* `all_reduce`            — in-place sum of one buffer (chunk boundary [T, k*r]).
* `all_reduce_coalesced`  — the BTP online-norm rider: the bf16 [T, k*r] partial and the fp32
                            [T] sum-of-squares reduced under ONE record, issued inside one NCCL
                            group (one launch), so the statistic never costs its own collective.
* `all_gather`            — model-tail gather of the d-sharded residual along the feature axis.

At tp == 1 nothing is sent, but the record is still written, exactly like the reference's
single-rank group. Every call records into a `Trace` with the current pass tag.

Two non-default modes, neither used by the training path:
* `force=True`  — issue the torch.distributed calls even at tp == 1 (a one-rank NCCL group on
                  the single-GPU box exercises the NCCL code path: coalescing manager, async
                  work handles, stream ordering).
* `emulate=True` — `TPComm.emulated(tp, rank)`: one rank's share of a tp-way plan on a single
                  GPU with NO data exchange (records only). The numbers are wrong by design;
                  it exists to time the per-rank compute of TP=4/8 shapes on one GPU
                  (`bench.py --emulate-tp`), and is labelled compute-only wherever reported.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .trace import Trace


class TPComm:
    def __init__(self, tp: int = 1, rank: int = 0, group=None, trace: Trace | None = None, *,
                 force: bool = False, emulate: bool = False, peer=None):
        self.tp = tp
        self.rank = rank
        self.group = group
        self.trace = trace if trace is not None else Trace()
        self.pass_tag = "forward"
        self.emulate = emulate
        # peer: a peer.PeerComm — the BTP chunk boundaries then run as fused reduce-scatter /
        # fix-up / all-gather kernels over peer memory instead of NCCL all-reduces
        self.peer = peer
        if peer is not None and (peer.tp != tp or peer.rank != rank):
            raise ValueError("peer communicator disagrees on (tp, rank)")
        if (tp > 1 or force) and not emulate and peer is None and not dist.is_initialized():
            raise RuntimeError("tp > 1 needs an initialised torch.distributed process group")
        if emulate and not 0 <= rank < tp:
            raise ValueError(f"rank {rank} outside tp={tp}")
        # issue real torch.distributed collectives? (a peer-only group has no process group)
        self.live = (tp > 1 or force) and not emulate and dist.is_initialized()

    @classmethod
    def emulated(cls, tp: int, rank: int = 0, trace: Trace | None = None) -> "TPComm":
        return cls(tp, rank, None, trace, emulate=True)

    @classmethod
    def from_env(cls, tp: int | None = None, trace: Trace | None = None) -> "TPComm":
        if not dist.is_initialized():
            return cls(1, 0, None, trace)
        world = dist.get_world_size()
        tp = world if tp is None else tp
        if tp != world:
            raise ValueError(f"tp={tp} must equal the process-group size {world} (one TP group per job)")
        return cls(tp, dist.get_rank(), None, trace)

    # ------------------------------------------------------------------ collectives
    def all_reduce(self, buf: torch.Tensor, chunk_id: str, tag: str = "block") -> torch.Tensor:
        if self.live:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        self.trace.emit("all-reduce", chunk_id, tag, buf.numel(), self.pass_tag)
        return buf

    def record(self, kind: str, chunk_id: str, elements: int, tag: str = "block", extras=()) -> None:
        """One logical collective record (for collectives issued in several slices)."""
        self.trace.emit(kind, chunk_id, tag, elements, self.pass_tag, extras=extras)

    def all_reduce_start(self, buf: torch.Tensor, chunk_id: str, tag: str = "block", record: bool = True):
        """Asynchronous in-place all-reduce: NCCL runs on its own stream (ordered after the work
        already queued on the current stream) while the caller keeps launching independent
        kernels; `wait(handle)` orders the current stream after the reduction."""
        work = dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group, async_op=True) if self.live else None
        if record:
            self.trace.emit("all-reduce", chunk_id, tag, buf.numel(), self.pass_tag)
        return work

    def all_reduce_coalesced_start(self, main: torch.Tensor, stat: torch.Tensor, chunk_id: str, tag: str = "block",
                                   stat_tag: str = "fused-stat", record: bool = True):
        """Asynchronous form of `all_reduce_coalesced` (bf16 payload + fp32 rider in one NCCL
        group); returns a handle (or a list of handles) for `wait`."""
        work = None
        if self.live:
            pg = self.group if self.group is not None else dist.distributed_c10d._get_default_group()
            if dist.get_backend(pg) == "nccl" and hasattr(pg, "_start_coalescing"):
                pg._start_coalescing(main.device)
                dist.all_reduce(main, group=pg, async_op=True)  # queued into the open NCCL group
                dist.all_reduce(stat, group=pg, async_op=True)
                work = pg._end_coalescing(main.device)
            else:
                work = [dist.all_reduce(main, group=pg, async_op=True), dist.all_reduce(stat, group=pg, async_op=True)]
        if record:
            self.trace.emit("all-reduce-coalesced", chunk_id, tag, main.numel(), self.pass_tag,
                            extras=((stat_tag, stat.numel()),))
        return work

    @staticmethod
    def wait(handle) -> None:
        if isinstance(handle, list):
            for h in handle:
                if h is not None:
                    h.wait()
        elif handle is not None:
            handle.wait()

    def all_reduce_coalesced(self, main: torch.Tensor, stat: torch.Tensor, chunk_id: str,
                             tag: str = "block", stat_tag: str = "fused-stat"):
        if self.live:
            pg = self.group if self.group is not None else dist.distributed_c10d._get_default_group()
            if dist.get_backend(pg) == "nccl" and hasattr(pg, "_start_coalescing"):
                # one ncclGroupStart/End around a bf16 and an fp32 all-reduce: both ride one launch.
                # (dist._coalescing_manager's all-reduce fast path would hand both tensors to
                # allreduce_coalesced, which requires ONE dtype and raises for the bf16 + fp32 rider.)
                pg._start_coalescing(main.device)
                dist.all_reduce(main, group=pg, async_op=True)  # queued into the open NCCL group
                dist.all_reduce(stat, group=pg, async_op=True)
                work = pg._end_coalescing(main.device)
                if work is not None:
                    work.wait()  # stream-orders the caller after the grouped reduction
            else:
                dist.all_reduce(main, group=pg)
                dist.all_reduce(stat, group=pg)
        self.trace.emit("all-reduce-coalesced", chunk_id, tag, main.numel(), self.pass_tag,
                        extras=((stat_tag, stat.numel()),))
        return main, stat

    def all_gather_cols(self, shard: torch.Tensor, chunk_id: str, tag: str = "boundary") -> torch.Tensor:
        """Gather [rows, w] shards along the feature axis into [rows, tp*w]."""
        rows, w = shard.shape
        if self.live:
            stacked = torch.empty((self.tp * rows, w), dtype=shard.dtype, device=shard.device)
            dist.all_gather_into_tensor(stacked, shard.contiguous(), group=self.group)
            out = stacked.view(self.tp, rows, w).permute(1, 0, 2).reshape(rows, self.tp * w)
        elif self.tp > 1:  # emulated: shape-correct placeholder
            out = shard.repeat(1, self.tp)
        else:
            out = shard
        self.trace.emit("all-gather", chunk_id, tag, out.numel(), self.pass_tag)
        return out
