"""Torch-tensor front end of the C-ABI kernels (device memory and streams come from torch;
all arithmetic runs in libbtp.so).

Every wrapper takes 2-D row-major views (last stride 1), forwards data pointers, leading
dimensions and the current CUDA stream, and raises on a non-zero btp_status.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native
from ._native import GemmProblem

BF16 = torch.bfloat16
F32 = torch.float32


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _ld(t: torch.Tensor | None) -> int:
    if t is None:
        return 0
    if t.dim() == 1:
        return t.shape[0]
    if t.stride(-1) != 1:
        raise ValueError(f"tensor must be row-major in its last dim, strides {t.stride()}")
    return t.stride(-2)


def _fn(name: str, t: torch.Tensor) -> str:
    """bf16 entry point, or its fp32 parity-mode twin for fp32 activations."""
    if t.dtype == F32:
        return name + "_f32"
    if t.dtype != BF16:
        raise TypeError(f"{name}: activations must be bf16 or fp32, got {t.dtype}")
    return name


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check(t: torch.Tensor, dtype, name: str):
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")


@dataclass
class Gemm:
    """One problem of a (grouped) GEMM launch.

    a: [M, K] (a_mn False) or [K, M] (a_mn True);  b: [N, K] (b_mn False) or [K, N] (b_mn True)
    c: [M, N] bf16/fp32, or [splits, M, N] fp32 partials when splits > 1.
    """

    a: torch.Tensor
    b: torch.Tensor
    c: torch.Tensor | None    # None only for gemm_scatter (the output goes to the owners' buffers)
    a_mn: bool = False
    b_mn: bool = False
    row_scale: torch.Tensor | None = None
    col_scale: torch.Tensor | None = None
    resid: torch.Tensor | None = None
    splits: int = 1
    alpha: float = 1.0
    reduce_add: bool = False                # add into C (fp32, zeroed) via TMA reduce; needed for splits > 1
    swiglu_bwd: tuple | None = None         # (g, u, du): acc = dact -> C = dg, du written too
    sigma: tuple | None = None              # (a_out, r_half): C = z, a_out = crossgate(z) (TP = 1 boundary)

    def to_c(self) -> GemmProblem:
        op_dtype = F32 if self.a.dtype == F32 else BF16  # fp32 operands -> exact-fp32 parity GEMM
        _check(self.a, op_dtype, "A")
        _check(self.b, op_dtype, "B")
        M, K = (self.a.shape[1], self.a.shape[0]) if self.a_mn else (self.a.shape[0], self.a.shape[1])
        if self.b_mn:
            Kb, N = self.b.shape
        else:
            N, Kb = self.b.shape
        if Kb != K:
            raise ValueError(f"GEMM inner dims disagree: A {tuple(self.a.shape)} B {tuple(self.b.shape)}")
        if self.c is not None and tuple(self.c.shape) != (M, N):
            raise ValueError(f"GEMM output {tuple(self.c.shape)} != ({M}, {N})")
        c_fp32 = self.c is not None and self.c.dtype == F32
        if (self.splits > 1 or self.reduce_add) and not c_fp32:
            raise ValueError("split-K / reduce-add GEMMs need an fp32 output")
        split_stride = 0
        resid, epilogue, aux2, c2 = self.resid, 0, None, None
        sigma_half = 0
        if self.sigma is not None:
            a_out, sigma_half = self.sigma
            _check(a_out, BF16, "a_out")
            if tuple(a_out.shape) != (M, N):
                raise ValueError(f"sigma output {tuple(a_out.shape)} != ({M}, {N})")
            epilogue, c2 = 1, a_out
        if self.swiglu_bwd is not None:
            g, u, du = self.swiglu_bwd
            for t, nm in ((g, "g"), (u, "u"), (du, "du")):
                _check(t, BF16, nm)
                if tuple(t.shape) != (M, N):
                    raise ValueError(f"swiglu-bwd operand {nm} {tuple(t.shape)} != ({M}, {N})")
            resid, epilogue, aux2, c2 = g, 2, u, du
        return GemmProblem(
            a=self.a.data_ptr(), lda=_ld(self.a), a_mn=int(self.a_mn),
            b=self.b.data_ptr(), ldb=_ld(self.b), b_mn=int(self.b_mn),
            c=None if self.c is None else self.c.data_ptr(), ldc=N if self.c is None else _ld(self.c),
            c_fp32=int(c_fp32),
            M=M, N=N, K=K,
            row_scale=None if self.row_scale is None else self.row_scale.data_ptr(),
            col_scale=None if self.col_scale is None else self.col_scale.data_ptr(),
            resid=None if resid is None else resid.data_ptr(),
            ld_resid=_ld(resid),
            splits=self.splits, split_stride=split_stride, alpha=float(self.alpha),
            reduce_add=int(self.reduce_add or self.splits > 1),
            epilogue=epilogue,
            aux2=None if aux2 is None else aux2.data_ptr(), ld_aux2=_ld(aux2),
            c2=None if c2 is None else c2.data_ptr(), ldc2=_ld(c2),
            sigma_half=int(sigma_half),
        )


def gemm(*problems: Gemm, bn: int = 0) -> None:
    """One launch of the persistent tcgen05 GEMM over 1..8 problems (the fp32 SIMT GEMM: 1..4)."""
    arr = (GemmProblem * len(problems))(*[p.to_c() for p in problems])
    if problems[0].a.dtype == F32:
        _native.call("btp_gemm_f32", arr, len(problems), _stream())
    else:
        _native.call("btp_gemm", arr, len(problems), bn, _stream())


def gemm_scatter(*problems: Gemm, owners, rows_per_owner: int, width: int, ld: int, col0, bn: int = 0) -> None:
    """One tcgen05 GEMM launch whose epilogue reduce-adds each output row block into the owning
    rank's buffer (owners: tp device addresses, rank order) at columns col0[p] + n."""
    arr = (GemmProblem * len(problems))(*[p.to_c() for p in problems])
    own = (ctypes.c_void_p * len(owners))(*[int(o) for o in owners])
    cols = (ctypes.c_int * len(col0))(*[int(c) for c in col0])
    _native.call("btp_gemm_scatter", arr, len(problems), bn, own, len(owners), int(rows_per_owner), int(width),
                 int(ld), cols, _stream())


def adamw(master, m, v, g, work, *, lr, step=0, step_dev=None, b1=0.9, b2=0.95, eps=1e-8, wd=0.0):
    """Fused AdamW over flat fp32 buffers; rewrites the working copy `work` (bf16 or fp32).
    step_dev: int32 device counter read for the bias correction (graph-replay safe)."""
    n = master.numel()
    for t in (m, v, g, work):
        if t.numel() != n:
            raise ValueError("adamw buffers must all hold the same number of elements")
    _native.call(_fn("btp_adamw", work), _p(master), _p(m), _p(v), _p(g), _p(work), n, ctypes.c_float(lr),
                 ctypes.c_float(b1), ctypes.c_float(b2), ctypes.c_float(eps), ctypes.c_float(wd), int(step),
                 _p(step_dev), _stream())


def counter_add(ctr, delta: int = 1):
    _native.call("btp_counter_add", _p(ctr), int(delta), _stream())


def set_pair_mode(mode: int) -> int:
    """CTA-pair (cta_group::2) GEMM tiles: 0 off, 1 plain/sigma epilogues, 2 also residual
    epilogues (default); returns the previous setting."""
    return int(_native.load().btp_gemm_set_pair(int(mode)))


def set_res4(mode) -> int:
    """Residual GEMM epilogue layout: 3 (default) by width (pipeline + st.global for N <= 1024,
    whole-tile staging above), 2 pipelined residual slots fed by a producer warp (CTA pairs),
    1 whole-tile residual staging, 0 per-chunk prefetch; True/False map to 1/0. Returns the
    previous mode."""
    return int(_native.load().btp_gemm_set_res4(int(mode)))


def set_st_global(enable: bool) -> int:
    """GEMM epilogue stores via coalesced st.global, or TMA bulk stores (default); returns previous."""
    return int(_native.load().btp_gemm_set_st_global(int(bool(enable))))


def zero(t: torch.Tensor) -> None:
    _native.call("btp_zero", _p(t), t.numel() * t.element_size(), _stream())


def rmsnorm_residual(x, gamma, *, branch=None, x_out=None, n_out=None, ss_out=None, rl_out=None, eps=1e-6):
    rows, width = x.shape
    _native.call(
        _fn("btp_rmsnorm_residual", x), _p(x), _ld(x), _p(branch), _ld(branch), _p(x_out), _ld(x_out), _p(gamma),
        _p(n_out), _ld(n_out), _p(ss_out), _p(rl_out), rows, width, ctypes.c_float(eps), _stream(),
    )


def rmsnorm_apply(x, gamma, ss_total, d, n_out, *, rms_out=None, eps=1e-6):
    rows, width = x.shape
    _native.call(
        _fn("btp_rmsnorm_apply", x), _p(x), _ld(x), _p(gamma), _p(ss_total), d, ctypes.c_float(eps), _p(n_out),
        _ld(n_out), _p(rms_out), rows, width, _stream(),
    )


def fixup_sigma(P, *, r, nproj, variant, z_out=None, a_out=None, ss_total=None, d=1, s_out=None, eps=1e-6):
    """P fp32 with bf16 z_out: the fp32-reduced boundary (btp_fixup_sigma_f32in)."""
    rows = P.shape[0]
    mixed = P.dtype == F32 and z_out is not None and z_out.dtype == BF16
    _native.call(
        "btp_fixup_sigma_f32in" if mixed else _fn("btp_fixup_sigma", P), _p(P), _ld(P), _p(ss_total), d, ctypes.c_float(eps), _p(s_out), _p(z_out),
        _ld(z_out), _p(a_out), _ld(a_out), rows, r, nproj, variant, _stream(),
    )


def fixup_sigma_bwd(z, da, dP, *, r, nproj, variant, s=None, d=1, dss=None):
    rows = z.shape[0]
    _native.call(
        _fn("btp_fixup_sigma_bwd", z), _p(z), _ld(z), _p(da), _ld(da), _p(s), d, _p(dP), _ld(dP), _p(dss), rows, r,
        nproj, variant, _stream(),
    )


def swiglu(g, u, act):
    rows, cols = g.shape
    _native.call(_fn("btp_swiglu", g), _p(g), _ld(g), _p(u), _ld(u), _p(act), _ld(act), rows, cols, _stream())


def swiglu_bwd(g, u, dact, dg, du):
    rows, cols = g.shape
    _native.call(
        _fn("btp_swiglu_bwd", g), _p(g), _ld(g), _p(u), _ld(u), _p(dact), _ld(dact), _p(dg), _ld(dg), _p(du), _ld(du),
        rows, cols, _stream(),
    )


def rmsnorm_bwd(dh, x, gamma, dss, dx, dgamma_partial, *, dres=None) -> int:
    """dgamma_partial: fp32 [max_blocks, width]; returns the number of partial rows written."""
    rows, width = x.shape
    nblk = ctypes.c_int(0)
    _native.call(
        _fn("btp_rmsnorm_bwd", dh), _p(dh), _ld(dh), _p(x), _ld(x), _p(gamma), _p(dss), _p(dres), _ld(dres), _p(dx),
        _ld(dx), _p(dgamma_partial), dgamma_partial.shape[0], ctypes.byref(nblk), rows, width, _stream(),
    )
    return nblk.value


def reduce_rows(parts, out, *, splits=None, col_scale=None, accumulate=False):
    """out[r, c] = sum_s parts[s, r, c] (* col_scale[c]) (+ out); parts is [S, rows, cols] fp32."""
    S = parts.shape[0] if splits is None else splits
    rows, cols = out.shape if out.dim() == 2 else (1, out.shape[0])
    ldi = parts.stride(1) if parts.dim() == 3 else cols
    _native.call(
        "btp_reduce_rows", _p(parts), S, parts.stride(0), ldi, rows, cols, _p(col_scale), _p(out),
        _ld(out) if out.dim() == 2 else cols, int(accumulate), _stream(),
    )


def add(a, b, out):
    rows, cols = a.shape
    _native.call(_fn("btp_add", a), _p(a), _ld(a), _p(b), _ld(b), _p(out), _ld(out), rows, cols, _stream())


def rmsnorm_bwd_prep(dn, x, gamma, s, dh, dss):
    rows, width = x.shape
    _native.call(_fn("btp_rmsnorm_bwd_prep", dn), _p(dn), _ld(dn), _p(x), _ld(x), _p(gamma), _p(s), _p(dh), _ld(dh),
                 _p(dss), rows, width, _stream())


def dot(a, b, partial) -> int:
    """partial: fp32 [max_blocks]; returns the number of partials written (sum them with reduce_rows)."""
    rows, cols = a.shape
    nblk = ctypes.c_int(0)
    _native.call(_fn("btp_dot", a), _p(a), _ld(a), _p(b), _ld(b), rows, cols, _p(partial), partial.shape[0],
                 ctypes.byref(nblk), _stream())
    return nblk.value


def embedding_fwd(ids, table, out, *, col0=0, bad=None):
    """out[t, :] = table[ids[t], col0:col0+width] (this rank's d-shard); ids int32 [T]."""
    _check(ids, torch.int32, "ids")
    rows, width = out.shape
    _native.call(_fn("btp_embedding_fwd", out), _p(ids), _p(table), _ld(table), table.shape[0], int(col0), _p(out),
                 _ld(out), rows, width, _p(bad), _stream())


def embedding_bwd(ids, dx, dtable):
    """dtable[ids[t], :] += dx[t, :] (fp32, zeroed by the caller)."""
    _check(ids, torch.int32, "ids")
    _check(dtable, F32, "dtable")
    rows, width = dx.shape
    _native.call(_fn("btp_embedding_bwd", dx), _p(ids), _p(dx), _ld(dx), dtable.shape[0], _p(dtable), _ld(dtable),
                 rows, width, _stream())


def cross_entropy(logits, targets, loss_rows, *, dlogits=None, scale=1.0):
    """loss_rows[t] = lse(logits_t) - logits_t[target]; dlogits = scale*(softmax - onehot) (may alias)."""
    _check(targets, torch.int32, "targets")
    _check(loss_rows, F32, "loss_rows")
    rows, vocab = logits.shape
    _native.call(_fn("btp_cross_entropy", logits), _p(logits), _ld(logits), _p(targets), vocab, _p(loss_rows),
                 _p(dlogits), _ld(dlogits), rows, ctypes.c_float(scale), _stream())


def num_sms() -> int:
    return _native.load().btp_num_sms()


def attn_fwd(q, k, v, o, lse, *, b: int, s: int, heads: int, head_dim: int) -> None:
    """o = softmax(q k^T / sqrt(hd)) v per (batch, head) on [b*s, heads*hd] row-major bf16 views;
    lse fp32 [b, heads, s] gets the log2-domain log-sum-exp (btp_attn_fwd)."""
    for name, t in (("q", q), ("k", k), ("v", v), ("o", o)):
        _check(t, BF16, name)
    _check(lse, F32, "lse")
    _native.call("btp_attn_fwd", _p(q), _ld(q), _p(k), _ld(k), _p(v), _ld(v), _p(o), _ld(o), _p(lse),
                 b, s, heads, head_dim, _stream())


def attn_bwd(q, k, v, o, dO, lse, D, dq_acc, dq, dk, dv, *, b: int, s: int, heads: int, head_dim: int) -> None:
    """dq, dk, dv of attn_fwd's o for upstream dO (btp_attn_bwd); D fp32 [b, heads, s] and dq_acc fp32
    [b*s, heads*hd] are workspaces."""
    for name, t in (("q", q), ("k", k), ("v", v), ("o", o), ("dO", dO), ("dq", dq), ("dk", dk), ("dv", dv)):
        _check(t, BF16, name)
    for name, t in (("lse", lse), ("D", D), ("dq_acc", dq_acc)):
        _check(t, F32, name)
    _native.call("btp_attn_bwd", _p(q), _ld(q), _p(k), _ld(k), _p(v), _ld(v), _p(o), _ld(o), _p(dO), _ld(dO),
                 _p(lse), _p(D), _p(dq_acc), _ld(dq_acc), _p(dq), _ld(dq), _p(dk), _ld(dk), _p(dv), _ld(dv),
                 b, s, heads, head_dim, _stream())
