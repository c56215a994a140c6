"""Multi-layer model step around the BTP block executor ("next").

The reference executes one block (plus the tail all-gather, simulator.py:710-714); the paper's
model shards the embedding OUTPUT so the first block's down-projection is
row-split, chains the blocks through the d-sharded residual, and replicates the final
projection on every TP rank. Here, per rank:

  forward   ids -> btp_embedding_fwd (this rank's d-shard of the table, no collective)
            -> L x BTPBlockExecutor.forward (4 grouped rank-r all-reduces each)
            -> all-gather [T, d]  ("final-gather", the reference's model-tail boundary record)
            -> final RMSNorm (full width, replicated) -> LM head GEMM [T, V] (replicated)
            -> btp_cross_entropy: per-row loss AND dlogits = (softmax - onehot)/T in place
  backward  dhn = dlogits @ H (tcgen05) ; dH = dlogits^T hn (split-K) ; final-norm backward
            -> this rank's column slice of dy (the head is replicated, so no collective)
            -> L x BTPBlockExecutor.backward -> btp_embedding_bwd into the table-shard gradient

lax models chain the rank-r bundle: block l's h_cur (its reduced z, a device view that stays
resident) is block l+1's h_prev (zero bundle = none at l = 0, reference model.py:264-266); in
backward block l+1's dL/dh_prev arrives at block l as dL/dh_cur and joins dz before its sigma-bwd.

The block executors share this executor's communicator (one collective log) and launch
counters; every kernel is a libbtp.so entry point.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .comm import TPComm
from .executor import F32, ExecutorBase, BTPBlockExecutor, StepStats
from .model import ModelWeights
from .plan import PlanError, ShardPlan, Strategy


class ModelExecutor(ExecutorBase):
    """One TP rank's shard of an L-block low-rank model under a BTP plan."""

    def __init__(self, pl: ShardPlan, mw: ModelWeights, comm: TPComm | None = None, device="cuda",
                 eps: float = 1e-6, attn_backend: str = "auto", precision: str = "bf16"):
        if pl.strategy is not Strategy.BOTTLENECK:
            raise PlanError(f"ModelExecutor runs BTP plans, got {pl.strategy.value}")
        if mw.cfg.d != pl.cfg.d or mw.cfg.d_ff != pl.cfg.d_ff or mw.cfg.r != pl.cfg.r:
            raise PlanError("model weights and plan disagree on (d, d_ff, r)")
        if mw.vocab % 8:
            raise PlanError(f"vocab={mw.vocab} must be a multiple of 8 (16-byte TMA row strides)")
        self._setup(pl, comm, device, eps, precision)
        self.vocab = mw.vocab
        self.d, self.dl = pl.cfg.d, pl.cfg.d // self.tp
        self.blocks = [BTPBlockExecutor(pl, blk, self._block_comm(l), self.dev, eps, attn_backend, precision)
                       for l, blk in enumerate(mw.blocks)]
        self._block_scratch: dict = {}
        for ex in self.blocks:
            ex.stats = self.stats  # one launch/FLOP count for the whole step
            ex.share_scratch(self._block_scratch)  # one set of temporaries / recomputables for all blocks
        sl = slice(self.rank * self.dl, (self.rank + 1) * self.dl)
        self.W = {"embedding": self._dev(mw.embedding.values[:, sl]),   # [V, d/tp] (row-split first layer)
                  "head": self._dev(mw.head.values)}                    # [V, d] replicated
        self.gamma1 = self._dev(mw.final_gamma.values, F32)              # final norm gain (replicated)
        self.gamma2 = torch.zeros(8, device=self.dev, dtype=F32)         # unused slot of the flat layout
        self.grad = {k: torch.zeros(v.shape, device=self.dev, dtype=F32) for k, v in self.W.items()}
        self._flatten_params()
        self.final_gamma = self.gamma1
        self._ids = None

    def _block_comm(self, l: int) -> TPComm:
        """The communicator of block l: the model's own, except that peer-memory boundaries need a
        symmetric heap (and flag epochs) PER block — block l's boundary buffers hold activations
        its backward reads after later blocks have run. Same group, same collective log."""
        pc = getattr(self.comm, "peer", None)
        if pc is None or l == 0:
            return self.comm
        from .peer import PeerComm

        bpc = PeerComm(pc.tp, pc.rank, pc.dev, provider=pc.provider, group=pc.group, scatter=pc.scatter, nvls=pc.nvls)
        c = TPComm(self.comm.tp, self.comm.rank, self.comm.group, self.comm.trace, emulate=self.comm.emulate, peer=bpc)
        c.live = self.comm.live
        return c

    # ------------------------------------------------------------------ instrumentation
    @property
    def gemm_timer(self):
        return self._gemm_timer

    @gemm_timer.setter
    def gemm_timer(self, value):
        self._gemm_timer = value
        for ex in getattr(self, "blocks", ()):
            ex.gemm_timer = value

    _gemm_timer = None

    @property
    def gemm_log(self):
        return self._gemm_log

    @gemm_log.setter
    def gemm_log(self, value):
        self._gemm_log = value
        for ex in getattr(self, "blocks", ()):
            ex.gemm_log = value

    _gemm_log = None
    loss_scale = 1.0

    # ------------------------------------------------------------------ step pieces
    def forward(self, ids: torch.Tensor) -> torch.Tensor:
        """ids: int32 [T] token ids on the device, or int32 [2, T] = (ids, targets) packed as one
        per-step input (then loss_device uses the packed targets). Returns this rank's last
        residual shard [T, d/tp]."""
        T = self.T
        self._tg = None
        if ids.dim() == 2 and tuple(ids.shape) == (2, T):
            ids, self._tg = ids[0], ids[1]
        if ids.dtype != torch.int32 or tuple(ids.shape) != (T,):
            raise PlanError(f"ids must be int32 [{T}], got {ids.dtype} {tuple(ids.shape)}")
        self._ids = ids
        self.comm.pass_tag = "forward"
        x = self.buf("emb_out", (T, self.dl))
        K.embedding_fwd(ids, self.W["embedding"], x)
        self.stats.kernel_launches += 1
        h = None
        for ex in self.blocks:
            if ex.lax:
                ex.set_h_prev_device(h)
            x = ex.forward(x)
            h = ex.h_cur if ex.lax else None
        self.comm.pass_tag = "forward"
        return x

    def loss_device(self, y_sh: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        """Tail of the forward: gather, final norm, LM head, fused cross-entropy (the logits buffer
        is overwritten by dlogits/T). Returns the mean loss as a 1-element fp32 device tensor."""
        T, d, V = self.T, self.d, self.vocab
        if self._tg is not None:
            targets = self._tg
        if targets.dtype != torch.int32 or tuple(targets.shape) != (T,):
            raise PlanError(f"targets must be int32 [{T}], got {targets.dtype} {tuple(targets.shape)}")
        y = self.comm.all_gather_cols(y_sh, "final-gather", tag="boundary")
        if y.data_ptr() != y_sh.data_ptr() or not y.is_contiguous():
            y = y.contiguous()
        self._y_full = y
        hn = self.buf("hn", (T, d))
        rl = self.buf("final_rms", (T,), F32)
        K.rmsnorm_residual(y, self.final_gamma, n_out=hn, rl_out=rl, eps=self.eps)
        logits = self.buf("logits", (T, V))
        self._gemm(K.Gemm(hn, self.W["head"], logits))
        rows = self.buf("loss_rows", (T,), F32)
        # dlogits = (softmax - onehot) * loss_scale / T (loss_scale: 1/m for m pipeline micro-batches)
        K.cross_entropy(logits, targets, rows, dlogits=logits, scale=self.loss_scale / T)
        out = self.buf("loss", (1,), F32)
        inv_t = self._buf.get("inv_T")
        if inv_t is None:
            inv_t = self._buf["inv_T"] = torch.full((1,), 1.0 / T, device=self.dev, dtype=F32)
        K.reduce_rows(rows.view(T, 1, 1), out.view(1, 1), col_scale=inv_t)
        self.stats.kernel_launches += 3
        return out

    def backward(self, targets: torch.Tensor | None = None) -> torch.Tensor:
        """Backward of the whole model for the loss computed by loss_device. Returns dx of the
        embedding output shard and fills every gradient (blocks: ex.grad; here: self.grad)."""
        dy_sh = self._blocks_backward(self._head_backward())
        self._embedding_backward(dy_sh)
        self._join_side()
        return dy_sh

    def _head_backward(self) -> torch.Tensor:
        """LM head + final norm backward: this rank's column slice of dL/dy (no collective)."""
        T, d = self.T, self.d
        dlogits, hn, y = self._buf["logits"], self._buf["hn"], self._y_full
        self.comm.pass_tag = "backward"
        dhn = self.buf("dhn", (T, d))
        self._gemm(K.Gemm(dlogits, self.W["head"], dhn, b_mn=True))          # dhn = dlogits @ H
        self._wgrad([(dlogits, hn, self.grad["head"])])                        # dH = dlogits^T hn
        dss = self.buf("final_dss", (T,), F32)
        K.rmsnorm_bwd_prep(dhn, y, self.final_gamma, self._buf["final_rms"], dhn, dss)
        dy = self.buf("dy_full", (T, d))
        gparts = self.buf("final_gparts", (4 * self.sms, d), F32)
        nb = K.rmsnorm_bwd(dhn, y, self.final_gamma, dss, dy, gparts)
        K.reduce_rows(gparts[:nb].view(nb, 1, d), self.grad["gamma1"].view(1, d))
        self.stats.kernel_launches += 3
        return dy[:, self.rank * self.dl:(self.rank + 1) * self.dl]            # replicated head: local slice

    def _blocks_backward(self, dy_sh: torch.Tensor) -> torch.Tensor:
        self.comm.pass_tag = "backward"
        dh = None
        for ex in reversed(self.blocks):
            if ex.lax:
                ex.dh_cur_in = dh
            dy_sh = ex.backward(dy_sh)
            dh = ex.dh_prev if ex.lax else None
        return dy_sh

    def _embedding_backward(self, dy_sh: torch.Tensor) -> None:
        K.zero(self.grad["embedding"])
        K.embedding_bwd(self._ids, dy_sh, self.grad["embedding"])
        self.stats.kernel_launches += 2

    def optimizer_step(self, **hp) -> None:
        for ex in self.blocks:
            ex.optimizer_step(**hp)
        super().optimizer_step(**hp)

    # ------------------------------------------------------------------ host views
    def model_grads(self) -> dict:
        """float64 host copies: {'blocks': [per-block rank-local grads], 'dembedding' [V, d/tp],
        'dhead' [V, d], 'dfinal_gamma' [d]}."""
        return {"blocks": [ex.weight_grads_by_name() for ex in self.blocks],
                "dembedding": self.grad["embedding"].double().cpu().numpy(),
                "dhead": self.grad["head"].double().cpu().numpy(),
                "dfinal_gamma": self.grad["gamma1"].double().cpu().numpy()}

    def saved_activation_bytes(self) -> int:
        return sum(ex.saved_activation_bytes() for ex in self.blocks)


def model_train_step(pl: ShardPlan, mw: ModelWeights, ids: np.ndarray, targets: np.ndarray, *, executor=None,
                     eps: float = 1e-6, attn_backend: str = "auto", precision: str = "bf16"):
    """One forward + backward of the model on this rank; returns (loss, executor)."""
    ex = executor if executor is not None else ModelExecutor(pl, mw, TPComm.from_env(pl.shape.tp), eps=eps,
                                                             attn_backend=attn_backend, precision=precision)
    ids_d = torch.as_tensor(np.asarray(ids), dtype=torch.int32).to(ex.dev)
    tg_d = torch.as_tensor(np.asarray(targets), dtype=torch.int32).to(ex.dev)
    y = ex.forward(ids_d)
    loss = float(ex.loss_device(y, tg_d).item())
    ex.backward(tg_d)
    return loss, ex


__all__ = ["ModelExecutor", "model_train_step", "StepStats"]
