"""Unmasked multi-head attention on [T, heads*hd] feature-sliced inputs.

Attention is NOT one of the subsystems BTP changes: the reference runs an
unmasked softmax(q k^T / sqrt(hd)) v per head with heads as contiguous feature slices
(model.py:205-230, simulator.py:221-233). Two implementations behind one interface:

* "native": this package's tcgen05 / TMEM kernels (csrc/attn.cu, `btp_attn_fwd` / `btp_attn_bwd`)
  straight on the [T, width] buffers (head j = columns [j*hd, (j+1)*hd)), hd 64 / 128, s % 128 == 0;
  the forward keeps the log2-domain log-sum-exp for the backward.
* "cudnn" / "flash": torch's SDPA dispatcher (cuDNN's Blackwell kernels first), with q/k/v passed as
  strided [b, h, s, hd] views of the [T, d] buffers; the backward is one `torch.autograd.grad` over
  the recorded SDPA node.
* "hybrid": cuDNN's forward (the aten cuDNN SDPA op called directly, with its log-sum-exp, converted to
  the log2 domain) and this package's tcgen05 backward (faster than cuDNN's at hd 64:
  profiles/attention/README.md); same shape limits as "native".
"auto" picks "hybrid" at head_dim 64 (s % 128 == 0), where the own backward is the faster one (the
bench step: 4.41-4.51 vs 4.57-4.59 ms with cuDNN for both directions on one box), else cuDNN.
"fp32" is the parity mode (fp32 q/k/v through the exact SDPA kernels).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

from . import kernels as K

_BACKENDS = {
    "auto": [SDPBackend.CUDNN_ATTENTION, SDPBackend.FLASH_ATTENTION],
    "cudnn": [SDPBackend.CUDNN_ATTENTION],
    "flash": [SDPBackend.FLASH_ATTENTION],
    # parity mode: fp32 q/k/v (cuDNN / flash are 16-bit only); exact fp32 GEMM softmax path
    "fp32": [SDPBackend.EFFICIENT_ATTENTION, SDPBackend.MATH],
}


class _Timed:
    """CUDA events around one SDPA call when the owner's timer list is armed (bench breakdown;
    external events become record nodes inside a graph capture)."""

    def __init__(self, timer, kind):
        self.timer, self.kind = timer, kind

    def __enter__(self):
        if self.timer is not None:
            self.e0 = torch.cuda.Event(enable_timing=True, external=True)
            self.e0.record()

    def __exit__(self, *exc):
        if self.timer is not None:
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            e1.record()
            self.timer.append((self.e0, e1, self.kind))


def native_supported(s: int, head_dim: int) -> bool:
    return s % 128 == 0 and head_dim in (64, 128)


# "auto" resolution, from the measured A/B (scripts/microbench/gpu_attn_bench.py, bench.py's
# attention_ab, profiles/attention/README.md): the native forward is behind cuDNN's, the native hd-64
# backward ahead of it, the generic hd-128 backward behind it
AUTO_NATIVE = False
AUTO_HYBRID = True


def auto_backend(s: int, head_dim: int) -> str:
    if AUTO_NATIVE and native_supported(s, head_dim):
        return "native"
    if AUTO_HYBRID and native_supported(s, head_dim) and head_dim == 64:
        return "hybrid"
    return "auto"


class Attention:
    timer: list | None = None  # bench instrumentation: (start_event, end_event, "fwd"|"bwd")

    def __init__(self, b: int, s: int, heads: int, head_dim: int, backend: str = "auto"):
        self.b, self.s, self.h, self.hd = b, s, heads, head_dim
        self.scale = 1.0 / head_dim**0.5
        if backend == "auto":
            backend = auto_backend(s, head_dim)
        if backend in ("native", "hybrid") and not native_supported(s, head_dim):
            raise ValueError(f"{backend} attention needs s % 128 == 0 and head_dim in (64, 128); got s={s}, "
                             f"head_dim={head_dim}")
        self.hybrid = backend == "hybrid"
        self._hybrid_fallback = False
        self.native = backend == "native"
        self.backends = None if (self.native or self.hybrid) else _BACKENDS[backend]
        self.stats = None  # the owning executor's ExecStats: native launches are counted there

    def _view4(self, t2d: torch.Tensor) -> torch.Tensor:
        # [T, h*hd] -> [b, h, s, hd] view (heads are contiguous feature slices)
        return t2d.view(self.b, self.s, self.h, self.hd).transpose(1, 2)

    def _as2d(self, t4: torch.Tensor) -> torch.Tensor:
        t = t4.transpose(1, 2)
        if t.is_contiguous():
            return t.view(self.b * self.s, self.h * self.hd)
        return t.reshape(self.b * self.s, self.h * self.hd)

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, need_grad: bool = True):
        if self.native:
            T = self.b * self.s
            out = torch.empty(T, self.h * self.hd, device=q.device, dtype=torch.bfloat16)
            lse = torch.empty(self.b, self.h, self.s, device=q.device, dtype=torch.float32)
            with _Timed(self.timer, "fwd"):
                K.attn_fwd(q, k, v, out, lse, b=self.b, s=self.s, heads=self.h, head_dim=self.hd)
            if self.stats is not None:
                self.stats.kernel_launches += 1
            return out, (q, k, v, out, lse)
        if self.hybrid and not self._hybrid_fallback:
            try:
                with _Timed(self.timer, "fwd"):
                    res = torch.ops.aten._scaled_dot_product_cudnn_attention(
                        self._view4(q), self._view4(k), self._view4(v), None, True, 0.0, False, False,
                        scale=self.scale)
                    # cuDNN's natural-log lse of the scaled scores -> the native backward's log2 domain
                    lse = (res[1].reshape(self.b, self.h, self.s) * (1.0 / math.log(2.0))).contiguous()
                    out = self._as2d(res[0])
                return out, (q, k, v, out, lse)
            except RuntimeError as exc:  # no cuDNN SDPA for this build / device: our forward from now on
                import warnings

                warnings.warn(f"cuDNN SDPA forward unavailable ({exc}); hybrid attention uses btp_attn_fwd")
                self._hybrid_fallback = True
        if self.hybrid:  # fallback: the native forward (its lse is already in the backward's layout)
            T = self.b * self.s
            out = torch.empty(T, self.h * self.hd, device=q.device, dtype=torch.bfloat16)
            lse = torch.empty(self.b, self.h, self.s, device=q.device, dtype=torch.float32)
            with _Timed(self.timer, "fwd"):
                K.attn_fwd(q, k, v, out, lse, b=self.b, s=self.s, heads=self.h, head_dim=self.hd)
            if self.stats is not None:
                self.stats.kernel_launches += 1
            return out, (q, k, v, out, lse)
        q4, k4, v4 = (self._view4(t).detach().requires_grad_(need_grad) for t in (q, k, v))
        with torch.enable_grad() if need_grad else torch.no_grad(), sdpa_kernel(self.backends, set_priority=True), \
                _Timed(self.timer, "fwd"):
            out = F.scaled_dot_product_attention(q4, k4, v4, scale=self.scale)
        return self._as2d(out.detach()), (q4, k4, v4, out)

    def backward(self, dout: torch.Tensor, ctx):
        if self.native or self.hybrid:
            q, k, v, out, lse = ctx
            T, W = self.b * self.s, self.h * self.hd
            dq, dk, dv = (torch.empty(T, W, device=q.device, dtype=torch.bfloat16) for _ in range(3))
            D = torch.empty(self.b, self.h, self.s, device=q.device, dtype=torch.float32)
            acc = torch.empty(T, W, device=q.device, dtype=torch.float32)
            if dout.stride(-1) != 1:
                dout = dout.contiguous()
            with _Timed(self.timer, "bwd"):
                K.attn_bwd(q, k, v, out, dout, lse, D, acc, dq, dk, dv, b=self.b, s=self.s, heads=self.h,
                           head_dim=self.hd)
            if self.stats is not None:
                self.stats.kernel_launches += 3  # D / zero pass, the tcgen05 kernel, dq conversion
            return dq, dk, dv
        q4, k4, v4, out = ctx
        do4 = self._view4(dout)
        with sdpa_kernel(self.backends, set_priority=True), _Timed(self.timer, "bwd"):
            dq, dk, dv = torch.autograd.grad(out, (q4, k4, v4), do4)
        return self._as2d(dq), self._as2d(dk), self._as2d(dv)
