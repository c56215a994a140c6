"""The two comparison points of the metric, on the SAME kernels as BTP:

* VanillaExecutor  — naive low-rank TP (reference `_forward_vanilla`, simulator.py:412-543):
  factor pairs sharded along r (cola keeps each crossgate pair rank-local via
  `cola_pair_indices`, plan.py:419-428), sigma fused per rank, the up-projection produces a
  full-width PARTIAL [T, d_out] that is all-reduced; residual, norms and attention are
  replicated on every rank (the reference's semantics, :518-520).
* FullRankExecutor — Megatron column->row TP of the full-rank block (reference
  `_forward_full_rank`, simulator.py:323-398): 2 all-reduces of [T, d] per pass.

Both run forward + backward (the backward all-reduces the input gradient of every
row-split boundary) and report the same collective log schema as the BTP executor.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .attention import Attention
from .comm import TPComm
from .executor import F32, ExecutorBase
from .model import DecoderBlockWeights, Variant
from .plan import PlanError, ShardPlan, Strategy, cola_pair_indices, col_shard_bounds

_VAR = {Variant.SVD: 0, Variant.COLA: 1, Variant.LAX: 0}


class _ReplicatedNormMixin:
    """Full-width RMSNorm forward/backward for the replicated-residual strategies."""

    def _rnorm(self, x, gamma, tag, branch=None, x_out=None):
        T, d = self.T, self.d
        n = self.buf(f"n{tag}", (T, d))
        s = self.buf(f"s{tag}", (T,), F32)
        K.rmsnorm_residual(x, gamma, branch=branch, x_out=x_out, n_out=n, rl_out=s, eps=self.eps)
        self.stats.kernel_launches += 1
        return n, s

    def _rnorm_bwd(self, dn, x, gamma, s, dres, dx_out, gkey):
        T, d = self.T, self.d
        dss = self.buf("dss_r", (T,), F32)
        K.rmsnorm_bwd_prep(dn, x, gamma, s, dn, dss)
        gparts = self.buf("gparts", (4 * self.sms, d), F32)
        nb = K.rmsnorm_bwd(dn, x, gamma, dss, dx_out, gparts, dres=dres)
        K.reduce_rows(gparts[:nb].view(nb, 1, d), self.grad[gkey].view(1, d))
        self.stats.kernel_launches += 3


class VanillaExecutor(_ReplicatedNormMixin, ExecutorBase):
    residual_sharded = False

    def __init__(self, pl: ShardPlan, block: DecoderBlockWeights, comm: TPComm | None = None, device="cuda",
                 eps: float = 1e-6, attn_backend: str = "auto", precision: str = "bf16"):
        if pl.strategy is not Strategy.VANILLA:
            raise PlanError(f"VanillaExecutor needs a vanilla plan, got {pl.strategy.value}")
        if block.variant is not pl.variant or pl.variant not in _VAR:
            raise PlanError(f"vanilla device path supports svd/cola/lax blocks matching the plan")
        self._setup(pl, comm, device, eps, precision)
        cfg = self.cfg
        self.var = _VAR[pl.variant]
        # lax (simulator.py:440-447): each rank merges its r-slice of the bundle into its z shard
        self.lax = pl.variant is Variant.LAX
        self.ckpt = pl.lowrank_ckpt
        self.has_h_prev = False
        self.h_cur: dict = {}
        self.dh_prev: dict | None = None
        self.grouping = pl.grouping
        self.r, self.d, self.d_ff = cfg.r, cfg.d, cfg.d_ff
        self.rl = cfg.r // self.tp
        self.dl = cfg.d  # replicated residual
        self.attn = Attention(pl.shape.b, pl.shape.s, cfg.heads, cfg.head_dim,
                              "fp32" if precision == "fp32" else attn_backend)
        self.attn.stats = self.stats
        if pl.variant is Variant.COLA:
            idx = cola_pair_indices(cfg.r, self.tp, self.rank)
        else:
            idx = np.arange(*col_shard_bounds(cfg.r, self.tp, self.rank))
        self._r_idx = idx
        B = {n: t.values[idx, :] for n, t in block.down_factors.items()}     # [r/tp, d_in]
        A = {n: t.values[:, idx] for n, t in block.up_factors.items()}       # [d_out, r/tp]
        self.W = {
            "d_qkv": self._dev(np.concatenate([B[n] for n in "qkv"])),      # [3rl, d]
            "u_qkv": [self._dev(A[n]) for n in "qkv"],                         # [d, rl] x3
            "d_o": self._dev(B["o"]), "u_o": self._dev(A["o"]),
            "d_gu": self._dev(np.concatenate([B["gate"], B["up"]])),           # [2rl, d]
            "u_gu": [self._dev(A["gate"]), self._dev(A["up"])],                # [d_ff, rl] x2
            "d_d": self._dev(B["down"]), "u_d": self._dev(A["down"]),          # [rl, d_ff], [d, rl]
        }
        self.gamma1 = self._dev(block.gamma1.values, F32)
        self.gamma2 = self._dev(block.gamma2.values, F32)
        self.grad = {
            k: ([torch.zeros(t.shape, device=self.dev, dtype=F32) for t in v] if isinstance(v, list)
                else torch.zeros(v.shape, device=self.dev, dtype=F32))
            for k, v in self.W.items()
        }
        self.grad["gamma1"] = torch.zeros(cfg.d, device=self.dev, dtype=F32)
        self.grad["gamma2"] = torch.zeros(cfg.d, device=self.dev, dtype=F32)
        self._flatten_params()

    # ------------------------------------------------------------------ lax bundle
    _CHUNK_NAMES = {"qkv": ("q", "k", "v"), "gate_up": ("gate", "up"), "o": ("o",), "down": ("down",),
                    "q": ("q",), "k": ("k",), "v": ("v",), "gate": ("gate",), "up": ("up",)}

    def set_h_prev(self, h_prev) -> None:
        """The logical bundle {projection: [T, r]} (replicated); each rank keeps its r-slice per
        chunk id, so the merge is one btp_add per chunk."""
        if h_prev is None:
            self.has_h_prev = False
            return
        if not self.lax:
            raise PlanError(f"h_prev is a lax input; this block is {self.pl.variant.value}")
        T, rl = self.T, self.rl
        idx = torch.as_tensor(self._r_idx)
        for cid, names in self._CHUNK_NAMES.items():
            hp = self.buf(f"hp_{cid}", (T, len(names) * rl))
            for i, n in enumerate(names):
                v = h_prev[n]
                v = torch.as_tensor(np.asarray(v).reshape(T, -1)) if not isinstance(v, torch.Tensor) else v.reshape(T, -1)
                hp[:, i * rl:(i + 1) * rl].copy_(v[:, idx].to(self.dev, self.act))
        self.has_h_prev = True

    # ------------------------------------------------------------------ one vanilla chunk group
    def _pair(self, names, inp, Wd, Wu, out_full, chunk_id):
        """down (col-parallel over r) -> local sigma -> up (row-parallel over r) -> AR of the
        full-width partial. Grouped: one down GEMM, one batched up launch, one AR."""
        T, rl, k = self.T, self.rl, len(names)
        z = self.buf(f"z_{chunk_id}", (T, k * rl))
        self._gemm(K.Gemm(inp, Wd, z))
        return z, self._pair_up(names, z, Wu, out_full, chunk_id)

    def _pair_up(self, names, z, Wu, out_full, chunk_id):
        """The chunk from its stored z on (also the checkpoint re-forward: it replays the AR)."""
        T, rl, k = self.T, self.rl, len(names)
        if self.var == 1:
            a = self.buf(f"a_{chunk_id}", (T, k * rl))
            K.fixup_sigma(z, r=rl, nproj=k, variant=1, z_out=z, a_out=a)
            self.stats.kernel_launches += 1
        elif self.lax and self.has_h_prev:
            a = self.buf(f"alax_{chunk_id}", (T, k * rl))
            K.add(z, self._buf[f"hp_{chunk_id}"], a)
            self.stats.kernel_launches += 1
        else:
            a = z
        if self.lax:  # h_cur = z: this rank's r-slice (the API gathers the full bundle)
            for i, n in enumerate(names):
                self.h_cur[n] = z[:, i * rl:(i + 1) * rl]
        widths = [w.shape[0] for w in Wu]
        offs = np.cumsum([0] + widths)
        probs = [K.Gemm(a[:, i * rl:(i + 1) * rl], Wu[i], out_full[:, offs[i]:offs[i + 1]]) for i in range(k)]
        if self.grouping or k == 1:
            self._gemm(*probs)
            self.comm.all_reduce(out_full, chunk_id)
        else:
            raise AssertionError("ungrouped path handled by caller")
        return a

    def _pairs(self, names, inp, Wd_all, Wu_list, chunk_grouped, widths, z_stored=None):
        """Grouped: one chunk. Ungrouped: one chunk per projection (separate buffers + ARs).
        z_stored (checkpoint re-forward): skip the down GEMMs, start from the kept z's."""
        T, rl = self.T, self.rl
        if self.grouping:
            full = self.buf(f"F_{chunk_grouped}", (T, sum(widths)))
            if z_stored is None:
                z, a = self._pair(names, inp, Wd_all, Wu_list, full, chunk_grouped)
            else:
                z = z_stored[0]
                a = self._pair_up(names, z, Wu_list, full, chunk_grouped)
            offs = np.cumsum([0] + widths)
            return [full[:, offs[i]:offs[i + 1]] for i in range(len(names))], [z], [a]
        outs, zs, as_ = [], [], []
        for i, n in enumerate(names):
            full = self.buf(f"F_{n}", (T, widths[i]))
            if z_stored is None:
                z, a = self._pair((n,), inp, Wd_all[i * rl:(i + 1) * rl], [Wu_list[i]], full, n)
            else:
                z = z_stored[i]
                a = self._pair_up((n,), z, [Wu_list[i]], full, n)
            outs.append(full)
            zs.append(z)
            as_.append(a)
        return outs, zs, as_

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        T, d, f = self.T, self.d, self.d_ff
        self.comm.pass_tag = "forward"
        self.h_cur = {}
        W = self.W
        n1, s1 = self._rnorm(x, self.gamma1, 1)
        (q, k, v), z_qkv, a_qkv = self._pairs(("q", "k", "v"), n1, W["d_qkv"], W["u_qkv"], "qkv", [d, d, d])
        attn, actx = self.attn.forward(q, k, v)
        o_full = self.buf("F_o", (T, d))
        z_o, a_o = self._pair(("o",), attn, W["d_o"], [W["u_o"]], o_full, "o")
        x_mid = self.buf("x_mid", (T, d))
        n2, s2 = self._rnorm(x, self.gamma2, 2, branch=o_full, x_out=x_mid)
        (g, u), z_gu, a_gu = self._pairs(("gate", "up"), n2, W["d_gu"], W["u_gu"], "gate_up", [f, f])
        act = self.buf("act", (T, f))
        K.swiglu(g, u, act)
        mlp = self.buf("F_down", (T, d))
        z_d, a_d = self._pair(("down",), act, W["d_d"], [W["u_d"]], mlp, "down")
        y = self.buf("y", (T, d))
        K.add(x_mid, mlp, y)
        self.stats.kernel_launches += 2
        if self.ckpt:
            # low-rank boundary checkpoint (reference checkpointing.py): keep x and the rank-local
            # z shards; backward re-forwards the rest, replaying the chunk all-reduces
            self.saved = dict(x=x, z_qkv=z_qkv, z_o=[z_o], z_gu=z_gu, z_d=[z_d])
        else:
            self.saved = dict(x=x, n1=n1, s1=s1, z_qkv=z_qkv, a_qkv=a_qkv, q=q, k=k, v=v, attn=attn, actx=actx,
                              z_o=[z_o], a_o=[a_o], x_mid=x_mid, n2=n2, s2=s2, z_gu=z_gu, a_gu=a_gu, g=g, u=u,
                              act=act, z_d=[z_d], a_d=[a_d])
        return y

    # names the checkpoint re-forward rebuilds (compared bitwise with the plain forward's)
    RECOMPUTED = ("n1", "q", "k", "v", "attn", "x_mid", "n2", "g", "u", "act", "a_qkv", "a_o", "a_gu", "a_d")

    def _reforward(self) -> None:
        """Everything backward needs, from x and the kept z shards: norms and sigma are local, but
        each up-projection output is a row-parallel PARTIAL over r, so its all-reduce is replayed
        (qkv, o, gate_up; the down chunk's output feeds nothing backward needs)."""
        S, W, T, d, f = self.saved, self.W, self.T, self.d, self.d_ff
        self.comm.pass_tag = "reforward"
        x = S["x"]
        n1, s1 = self._rnorm(x, self.gamma1, 1)
        (q, k, v), _, a_qkv = self._pairs(("q", "k", "v"), None, None, W["u_qkv"], "qkv", [d, d, d],
                                          z_stored=S["z_qkv"])
        attn, actx = self.attn.forward(q, k, v)
        o_full = self.buf("F_o", (T, d))
        a_o = self._pair_up(("o",), S["z_o"][0], [W["u_o"]], o_full, "o")
        x_mid = self.buf("x_mid", (T, d))
        n2, s2 = self._rnorm(x, self.gamma2, 2, branch=o_full, x_out=x_mid)
        (g, u), _, a_gu = self._pairs(("gate", "up"), None, None, W["u_gu"], "gate_up", [f, f], z_stored=S["z_gu"])
        act = self.buf("act", (T, f))
        K.swiglu(g, u, act)
        self.stats.kernel_launches += 1
        a_d = self._sigma_local(("down",), S["z_d"][0], "down")
        S.update(n1=n1, s1=s1, a_qkv=a_qkv, q=q, k=k, v=v, attn=attn, actx=actx, a_o=[a_o], x_mid=x_mid, n2=n2,
                 s2=s2, a_gu=a_gu, g=g, u=u, act=act, a_d=[a_d])

    def _sigma_local(self, names, z, chunk_id):
        T, rl, k = self.T, self.rl, len(names)
        if self.var == 1:
            a = self.buf(f"a_{chunk_id}", (T, k * rl))
            K.fixup_sigma(z, r=rl, nproj=k, variant=1, z_out=z, a_out=a)
        elif self.lax and self.has_h_prev:
            a = self.buf(f"alax_{chunk_id}", (T, k * rl))
            K.add(z, self._buf[f"hp_{chunk_id}"], a)
        else:
            return z
        self.stats.kernel_launches += 1
        return a

    # ------------------------------------------------------------------ backward
    def _pair_bwd(self, names, dout_list, zs, as_, Wd_all, Wu_list, inp, gkey_d, gkey_u, din_full, chunk_ids):
        """Backward of one vanilla chunk group. dout: grads of the full-width outputs (replicated).
        da = dout @ Wu (local, no AR); sigma-bwd; dWd = dz^T inp; din partial = dz @ Wd -> AR."""
        T, rl, k = self.T, self.rl, len(names)
        G = self.grad
        dz = self.buf(f"dz_{'_'.join(names)}", (T, k * rl))
        probs = [K.Gemm(dout_list[i], Wu_list[i], dz[:, i * rl:(i + 1) * rl], b_mn=True) for i in range(k)]
        z_all = zs[0] if len(zs) == 1 else None
        pairs = []
        for i in range(k):
            a_i = (as_[0] if len(as_) == 1 else as_[i])
            a_i = a_i[:, i * rl:(i + 1) * rl] if len(as_) == 1 else a_i
            gu = G[gkey_u][i] if isinstance(G[gkey_u], list) else G[gkey_u]
            pairs.append((dout_list[i], a_i, gu))
        if 2 * k <= 8:  # the dgrad and the up-factor weight gradients in one launch
            self._dgrad_wgrad(probs, pairs)
        else:
            self._gemm(*probs)
            for pr in pairs:
                self._wgrad([pr])
        if self.var == 1:
            if z_all is not None:
                K.fixup_sigma_bwd(z_all, dz, dz, r=rl, nproj=k, variant=1)
            else:
                for i in range(k):
                    K.fixup_sigma_bwd(zs[i], dz[:, i * rl:(i + 1) * rl], dz[:, i * rl:(i + 1) * rl], r=rl, nproj=1,
                                      variant=1)
            self.stats.kernel_launches += 1
        if self.lax and self.has_h_prev:  # the merge is an add: dL/dh_prev slice = dz (rank-local)
            if self.dh_prev is None:
                self.dh_prev = {}
            for i, n in enumerate(names):
                self.dh_prev[n] = dz[:, i * rl:(i + 1) * rl]
        self._dgrad_wgrad([K.Gemm(dz, Wd_all, din_full, b_mn=True)], [(dz, inp, G[gkey_d])])
        self.comm.all_reduce(din_full, chunk_ids[0])

    def backward(self, dy: torch.Tensor) -> torch.Tensor:
        if not self.saved:
            raise RuntimeError("backward called before forward")
        if self.ckpt:
            self._reforward()
        S, W, T, d, f = self.saved, self.W, self.T, self.d, self.d_ff
        self.comm.pass_tag = "backward"
        self.dh_prev = None
        dact = self.buf("dact", (T, f))
        self._pair_bwd(("down",), [dy], S["z_d"], S["a_d"], W["d_d"], [W["u_d"]], S["act"], "d_d", "u_d", dact,
                       ["down"])
        dgu = self.buf("dgu", (T, 2 * f))
        K.swiglu_bwd(S["g"], S["u"], dact, dgu[:, :f], dgu[:, f:])
        self.stats.kernel_launches += 1
        dn2 = self.buf("dn2", (T, d))
        self._pair_bwd(("gate", "up"), [dgu[:, :f], dgu[:, f:]], S["z_gu"], S["a_gu"], W["d_gu"], W["u_gu"], S["n2"],
                       "d_gu", "u_gu", dn2, ["gate_up"])
        dx_mid = self.buf("dx_mid", (T, d))
        self._rnorm_bwd(dn2, S["x_mid"], self.gamma2, S["s2"], dy, dx_mid, "gamma2")
        dattn = self.buf("dattn", (T, d))
        self._pair_bwd(("o",), [dx_mid], S["z_o"], S["a_o"], W["d_o"], [W["u_o"]], S["attn"], "d_o", "u_o", dattn,
                       ["o"])
        dq, dk, dv = self.attn.backward(dattn, S["actx"])
        dn1 = self.buf("dn1", (T, d))
        self._pair_bwd(("q", "k", "v"), [dq, dk, dv], S["z_qkv"], S["a_qkv"], W["d_qkv"], W["u_qkv"], S["n1"],
                       "d_qkv", "u_qkv", dn1, ["qkv"])
        dx = self.buf("dx", (T, d))
        self._rnorm_bwd(dn1, S["x"], self.gamma1, S["s1"], dx_mid, dx, "gamma1")
        self._join_side()
        return dx

    def weight_grads_by_name(self):
        g = {k: ([t.double().cpu().numpy() for t in v] if isinstance(v, list) else v.double().cpu().numpy())
             for k, v in self.grad.items()}
        rl = self.rl
        out = {"A": {}, "B": {}, "gamma1": g["gamma1"], "gamma2": g["gamma2"]}
        for i, n in enumerate("qkv"):
            out["B"][n] = g["d_qkv"][i * rl:(i + 1) * rl]
            out["A"][n] = g["u_qkv"][i]
        for i, n in enumerate(("gate", "up")):
            out["B"][n] = g["d_gu"][i * rl:(i + 1) * rl]
            out["A"][n] = g["u_gu"][i]
        out["B"]["o"], out["A"]["o"] = g["d_o"], g["u_o"]
        out["B"]["down"], out["A"]["down"] = g["d_d"], g["u_d"]
        return out


class FullRankExecutor(_ReplicatedNormMixin, ExecutorBase):
    residual_sharded = False

    def __init__(self, pl: ShardPlan, block: DecoderBlockWeights, comm: TPComm | None = None, device="cuda",
                 eps: float = 1e-6, attn_backend: str = "auto", precision: str = "bf16"):
        if pl.strategy is not Strategy.FULL_RANK or block.variant is not Variant.FULL_RANK:
            raise PlanError("FullRankExecutor needs a full-rank plan and block")
        self._setup(pl, comm, device, eps, precision)
        cfg, tp, rk = self.cfg, self.tp, self.rank
        self.grouping = pl.grouping
        self.d, self.d_ff = cfg.d, cfg.d_ff
        self.dl, self.fl, self.hl = cfg.d // tp, cfg.d_ff // tp, cfg.heads // tp
        self.attn = Attention(pl.shape.b, pl.shape.s, self.hl, cfg.head_dim,
                              "fp32" if precision == "fp32" else attn_backend)
        self.attn.stats = self.stats
        sl, fsl = slice(rk * self.dl, (rk + 1) * self.dl), slice(rk * self.fl, (rk + 1) * self.fl)
        Wf = {n: t.values for n, t in block.full.items()}
        # d_ff shard padded to a multiple of 8 for 16-byte TMA strides (exact: zero rows / columns)
        self.flp = -(-self.fl // 8) * 8
        pad = self.flp - self.fl
        rows = (lambda a: np.pad(a, ((0, pad), (0, 0)))) if pad else (lambda a: a)
        cols = (lambda a: np.pad(a, ((0, 0), (0, pad)))) if pad else (lambda a: a)
        self.W = {
            "qkv": self._dev(np.concatenate([Wf[n][sl, :] for n in "qkv"])),                   # [3dl, d] col-parallel
            "o": self._dev(Wf["o"][:, sl]),                                                     # [d, dl]  row-parallel
            "gu": self._dev(np.concatenate([rows(Wf["gate"][fsl, :]), rows(Wf["up"][fsl, :])])),  # [2flp, d]
            "down": self._dev(cols(Wf["down"][:, fsl])),                                        # [d, flp]
        }
        self.gamma1 = self._dev(block.gamma1.values, F32)
        self.gamma2 = self._dev(block.gamma2.values, F32)
        self.grad = {k: torch.zeros(v.shape, device=self.dev, dtype=F32) for k, v in self.W.items()}
        self.grad["gamma1"] = torch.zeros(cfg.d, device=self.dev, dtype=F32)
        self.grad["gamma2"] = torch.zeros(cfg.d, device=self.dev, dtype=F32)
        self._flatten_params()

    def _col(self, inp, Wcat, out, k):
        """Column-parallel GEMM(s): grouped = one launch over the concatenated weight."""
        n = Wcat.shape[0] // k
        if self.grouping:
            self._gemm(K.Gemm(inp, Wcat, out))
        else:
            for i in range(k):
                self._gemm(K.Gemm(inp, Wcat[i * n:(i + 1) * n], out[:, i * n:(i + 1) * n]))

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        T, d, dl, fl = self.T, self.d, self.dl, self.flp
        self.comm.pass_tag = "forward"
        W = self.W
        n1, s1 = self._rnorm(x, self.gamma1, 1)
        qkv = self.buf("qkv", (T, 3 * dl))
        self._col(n1, W["qkv"], qkv, 3)
        attn, actx = self.attn.forward(qkv[:, :dl], qkv[:, dl:2 * dl], qkv[:, 2 * dl:])
        o = self.buf("o", (T, d))
        self._gemm(K.Gemm(attn, W["o"], o))
        self.comm.all_reduce(o, "attn")
        x_mid = self.buf("x_mid", (T, d))
        n2, s2 = self._rnorm(x, self.gamma2, 2, branch=o, x_out=x_mid)
        gu = self.buf("gu", (T, 2 * fl))
        self._col(n2, W["gu"], gu, 2)
        act = self.buf("act", (T, fl))
        K.swiglu(gu[:, :fl], gu[:, fl:], act)
        mlp = self.buf("mlp", (T, d))
        self._gemm(K.Gemm(act, W["down"], mlp))
        self.comm.all_reduce(mlp, "mlp")
        y = self.buf("y", (T, d))
        K.add(x_mid, mlp, y)
        self.stats.kernel_launches += 2
        self.saved = dict(x=x, n1=n1, s1=s1, qkv=qkv, attn=attn, actx=actx, x_mid=x_mid, n2=n2, s2=s2, gu=gu, act=act)
        return y

    def backward(self, dy: torch.Tensor) -> torch.Tensor:
        S, W, G, T, d, dl, fl = self.saved, self.W, self.grad, self.T, self.d, self.dl, self.flp
        self.comm.pass_tag = "backward"
        dgu = self.buf("dgu", (T, 2 * fl))
        g, u = S["gu"][:, :fl], S["gu"][:, fl:]
        if self.fuse_swiglu_bwd:  # dact stays in the GEMM epilogue, which emits dg, du
            self._gemm(K.Gemm(dy, W["down"], dgu[:, :fl], b_mn=True, swiglu_bwd=(g, u, dgu[:, fl:])))
        else:
            dact = self.buf("dact", (T, fl))
            self._dgrad_wgrad([K.Gemm(dy, W["down"], dact, b_mn=True)], [(dy, S["act"], G["down"])])
            K.swiglu_bwd(g, u, dact, dgu[:, :fl], dgu[:, fl:])
            self.stats.kernel_launches += 1
        if self.fuse_swiglu_bwd:
            self._wgrad([(dy, S["act"], G["down"])])
        dn2 = self.buf("dn2", (T, d))
        self._dgrad_wgrad([K.Gemm(dgu, W["gu"], dn2, b_mn=True)], [(dgu, S["n2"], G["gu"])])
        self.comm.all_reduce(dn2, "mlp")
        dx_mid = self.buf("dx_mid", (T, d))
        self._rnorm_bwd(dn2, S["x_mid"], self.gamma2, S["s2"], dy, dx_mid, "gamma2")
        dattn = self.buf("dattn", (T, dl))
        self._dgrad_wgrad([K.Gemm(dx_mid, W["o"], dattn, b_mn=True)], [(dx_mid, S["attn"], G["o"])])
        dq, dk, dv = self.attn.backward(dattn, S["actx"])
        gq = G["qkv"]
        self._wgrad([(dq, S["n1"], gq[:dl]), (dk, S["n1"], gq[dl:2 * dl]), (dv, S["n1"], gq[2 * dl:])])
        dn1 = self.buf("dn1", (T, d))
        Wq = W["qkv"]
        self._gemm(K.Gemm(dq, Wq[:dl], dn1, b_mn=True))
        self._gemm(K.Gemm(dk, Wq[dl:2 * dl], dn1, b_mn=True, resid=dn1))
        self._gemm(K.Gemm(dv, Wq[2 * dl:], dn1, b_mn=True, resid=dn1))
        self.comm.all_reduce(dn1, "attn")
        dx = self.buf("dx", (T, d))
        self._rnorm_bwd(dn1, S["x"], self.gamma1, S["s1"], dx_mid, dx, "gamma1")
        self._join_side()
        return dx

    def weight_grads_by_name(self):
        g = {k: v.double().cpu().numpy() for k, v in self.grad.items()}
        dl, fl, flp = self.dl, self.fl, self.flp
        W = {"q": g["qkv"][:dl], "k": g["qkv"][dl:2 * dl], "v": g["qkv"][2 * dl:], "o": g["o"],
             "gate": g["gu"][:fl], "up": g["gu"][flp:flp + fl], "down": g["down"][:, :fl]}
        return {"W": W, "gamma1": g["gamma1"], "gamma2": g["gamma2"]}
