"""Device versions of the reference's tensor-level operations (btpsim/tensor.py:86-139), with the
same signatures, return values and errors: `matmul(a, b) -> (Tensor, flops)`, `batched_matmul(
pairs) -> ([Tensor], flops)` (one grouped launch per <= 4 products, bitwise equal to sequential
calls), `swiglu(gate, up) -> Tensor`. Host `Tensor`s in, host `Tensor`s out; the arithmetic runs
in libbtp.so: precision="fp32" (default) on the exact-fp32 SIMT GEMM / fp32 row kernels (within
~1e-6 of the reference's float64), precision="bf16" on the tcgen05 GEMM (operands rounded to bf16,
fp32 accumulation)."""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import kernels as K
from .interop import as_tensor
from .tensor import DimensionError, Tensor

_MAX_GROUP = 4  # problems per grouped GEMM launch


def _dev(v: np.ndarray, dtype) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(v)).to("cuda", dtype)


def _pad_to(t: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    if tuple(t.shape) == (rows, cols):
        return t
    out = torch.zeros(rows, cols, device=t.device, dtype=t.dtype)
    out[: t.shape[0], : t.shape[1]] = t
    return out


def _check_pair(a: Tensor, b: Tensor) -> None:
    if a.values.ndim != 2 or b.values.ndim != 2:
        raise DimensionError(f"matmul needs 2-D operands, got {a.shape} and {b.shape}")
    if a.shape[1] != b.shape[0]:
        raise DimensionError(f"inner dimensions disagree: {a.shape} @ {b.shape}")


def _launch(pairs, precision: str) -> list[Tensor]:
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    probs, outs, shapes = [], [], []
    for a, b in pairs:
        m, k = a.shape
        n = b.shape[1]
        A, B = _dev(a.values, dt), _dev(b.values, dt)   # B stays [K, N]: an MN-major operand
        if precision == "bf16":  # 16-byte TMA rows: pad K and N to multiples of 8 (zeros are exact)
            kp, np_ = -(-k // 8) * 8, -(-n // 8) * 8
            A, B = _pad_to(A, m, kp), _pad_to(B, kp, np_)
            C = torch.empty(m, np_, device="cuda", dtype=torch.float32)
        else:
            C = torch.empty(m, n, device="cuda", dtype=torch.float32)
        probs.append(K.Gemm(A, B, C, b_mn=True))
        outs.append(C)
        shapes.append((m, n))
    for i in range(0, len(probs), _MAX_GROUP):
        K.gemm(*probs[i:i + _MAX_GROUP])
    torch.cuda.synchronize()
    return [Tensor(C[:, :n].double().cpu().numpy(), a.element_bytes)
            for C, (m, n), (a, _) in zip(outs, shapes, pairs)]


def matmul(a: Tensor, b: Tensor, *, precision: str = "fp32") -> tuple[Tensor, int]:
    """Dense 2-D product on the device; returns (result, flops) with flops = 2*M*N*K."""
    a, b = as_tensor(a), as_tensor(b)
    _check_pair(a, b)
    m, k = a.shape
    return _launch([(a, b)], precision)[0], 2 * m * b.shape[1] * k


def batched_matmul(pairs: Sequence[tuple[Tensor, Tensor]], *, precision: str = "fp32") -> tuple[list[Tensor], int]:
    """Independent 2-D products sharing grouped launches (<= 4 per launch). fp32: each output is
    bitwise the product matmul computes alone (per-problem CTA grid, same reduction order), as the
    reference requires of its batched kernel (tensor.py:97-112)."""
    if not pairs:
        raise DimensionError("batched_matmul needs at least one pair")
    pairs = [(as_tensor(a), as_tensor(b)) for a, b in pairs]
    for a, b in pairs:
        _check_pair(a, b)
    flops = sum(2 * a.shape[0] * b.shape[1] * a.shape[1] for a, b in pairs)
    return _launch(list(pairs), precision), flops


def swiglu(gate: Tensor, up: Tensor, *, precision: str = "fp32") -> Tensor:
    """Elementwise silu(gate) * up on the device; shapes must match exactly."""
    gate, up = as_tensor(gate), as_tensor(up)
    if gate.shape != up.shape:
        raise DimensionError(f"swiglu operands disagree: {gate.shape} vs {up.shape}")
    dt = torch.float32 if precision == "fp32" else torch.bfloat16
    n = int(np.prod(gate.shape)) if gate.values.ndim else 1
    npad = max(8, -(-n // 8) * 8)  # the row kernel works on 8-element vectors
    g = torch.zeros(npad, device="cuda", dtype=dt)
    u = torch.zeros(npad, device="cuda", dtype=dt)
    g[:n] = _dev(gate.values.reshape(-1), dt)
    u[:n] = _dev(up.values.reshape(-1), dt)
    out = torch.empty(npad, device="cuda", dtype=dt)
    K.swiglu(g.view(-1, 8), u.view(-1, 8), out.view(-1, 8))
    torch.cuda.synchronize()
    return Tensor(out[:n].double().cpu().numpy().reshape(gate.shape), gate.element_bytes)


__all__ = ["matmul", "batched_matmul", "swiglu"]
