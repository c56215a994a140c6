"""Unmasked multi-head attention on [T, heads*hd] feature-sliced inputs.

Attention is NOT one of the subsystems BTP changes: the reference runs an
unmasked softmax(q k^T / sqrt(hd)) v per head with heads as contiguous feature slices
(model.py:205-230, simulator.py:221-233). Here it is delegated, like a cuBLAS GEMM, to the
cuDNN (Blackwell) or FlashAttention SDPA kernels through torch's SDPA dispatcher, with the
backend pinned by `sdpa_kernel` (cuDNN first). q/k/v are passed as strided [b, h, s, hd] views
of the [T, d] buffers, so no transposes are materialised; the backward is one
`torch.autograd.grad` over the recorded SDPA node (no Python autograd elsewhere in the block).
"""

from __future__ import annotations

import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

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


class Attention:
    timer: list | None = None  # bench instrumentation: (start_event, end_event, "fwd"|"bwd")

    def __init__(self, b: int, s: int, heads: int, head_dim: int, backend: str = "auto"):
        self.b, self.s, self.h, self.hd = b, s, heads, head_dim
        self.scale = 1.0 / head_dim**0.5
        self.backends = _BACKENDS[backend]

    def _view4(self, t2d: torch.Tensor) -> torch.Tensor:
        # [T, h*hd] -> [b, h, s, hd] view (heads are contiguous feature slices)
        return t2d.view(self.b, self.s, self.h, self.hd).transpose(1, 2)

    def _as2d(self, t4: torch.Tensor) -> torch.Tensor:
        t = t4.transpose(1, 2)
        if t.is_contiguous():
            return t.view(self.b * self.s, self.h * self.hd)
        return t.reshape(self.b * self.s, self.h * self.hd)

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, need_grad: bool = True):
        q4, k4, v4 = (self._view4(t).detach().requires_grad_(need_grad) for t in (q, k, v))
        with torch.enable_grad() if need_grad else torch.no_grad(), sdpa_kernel(self.backends, set_priority=True), \
                _Timed(self.timer, "fwd"):
            out = F.scaled_dot_product_attention(q4, k4, v4, scale=self.scale)
        return self._as2d(out.detach()), (q4, k4, v4, out)

    def backward(self, dout: torch.Tensor, ctx):
        q4, k4, v4, out = ctx
        do4 = self._view4(dout)
        with sdpa_kernel(self.backends, set_priority=True), _Timed(self.timer, "bwd"):
            dq, dk, dv = torch.autograd.grad(out, (q4, k4, v4), do4)
        return self._as2d(dq), self._as2d(dk), self._as2d(dv)
