"""ctypes binding of libbtp.so (the C-ABI in include/btp.h).

There is deliberately no fallback: if the library is missing or fails to load, every
kernel entry point raises NativeUnavailable, so a GPU run can never silently take a
CPU or PyTorch path.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libbtp.so"

BTP_OK = 0
BTP_ERR_DIM = 1
BTP_ERR_DIVISIBILITY = 2
BTP_ERR_ALIGNMENT = 3
BTP_ERR_CUDA = 4

_STATUS_NAMES = {
    BTP_ERR_DIM: "dimension mismatch",
    BTP_ERR_DIVISIBILITY: "divisibility",
    BTP_ERR_ALIGNMENT: "alignment (row strides / widths must be multiples of 8 elements, 16-byte pointers)",
    BTP_ERR_CUDA: "CUDA launch failure",
}

# Every symbol include/btp.h declares; tests check the library exports exactly these.
EXPORTED_SYMBOLS = (
    "btp_gemm",
    "btp_gemm_scatter",
    "btp_gemm_set_pair",
    "btp_gemm_set_res4",
    "btp_gemm_set_st_global",
    "btp_rmsnorm_residual",
    "btp_rmsnorm_apply",
    "btp_fixup_sigma",
    "btp_fixup_sigma_f32in",
    "btp_swiglu",
    "btp_swiglu_bwd",
    "btp_fixup_sigma_bwd",
    "btp_rmsnorm_bwd",
    "btp_reduce_rows",
    "btp_add",
    "btp_rmsnorm_bwd_prep",
    "btp_dot",
    "btp_zero",
    "btp_adamw",
    "btp_adamw_f32",
    "btp_counter_add",
    "btp_num_sms",
    "btp_version",
    # fp32 parity-mode twins
    "btp_gemm_f32",
    "btp_rmsnorm_residual_f32",
    "btp_rmsnorm_apply_f32",
    "btp_fixup_sigma_f32",
    "btp_swiglu_f32",
    "btp_swiglu_bwd_f32",
    "btp_fixup_sigma_bwd_f32",
    "btp_rmsnorm_bwd_f32",
    "btp_rmsnorm_bwd_prep_f32",
    "btp_add_f32",
    "btp_dot_f32",
    # model boundary (embedding shard, fused cross-entropy)
    "btp_embedding_fwd",
    "btp_embedding_fwd_f32",
    "btp_embedding_bwd",
    "btp_embedding_bwd_f32",
    "btp_cross_entropy",
    "btp_cross_entropy_f32",
    # chunk boundaries over peer memory
    "btp_peer_signal",
    "btp_peer_wait",
    "btp_peer_boundary_fwd",
    "btp_peer_boundary_bwd",
    "btp_peer_boundary_fwd_local",
    "btp_peer_boundary_bwd_local",
    "btp_peer_boundary_fwd_nvls",
    "btp_peer_boundary_bwd_nvls",
    # attention
    "btp_attn_fwd",
    "btp_attn_bwd",
    "btp_attn_bwd_trace",
    "btp_attn_tune",
    "btp_attn_fwd_trace",
)


class NativeUnavailable(RuntimeError):
    """libbtp.so is not built or cannot be loaded; there is no fallback path."""


class NativeError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} failed: {_STATUS_NAMES.get(code, 'status')} (code {code})")
        self.code = code


class GemmProblem(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p),
        ("lda", ctypes.c_longlong),
        ("a_mn", ctypes.c_int),
        ("b", ctypes.c_void_p),
        ("ldb", ctypes.c_longlong),
        ("b_mn", ctypes.c_int),
        ("c", ctypes.c_void_p),
        ("ldc", ctypes.c_longlong),
        ("c_fp32", ctypes.c_int),
        ("M", ctypes.c_int),
        ("N", ctypes.c_int),
        ("K", ctypes.c_int),
        ("row_scale", ctypes.c_void_p),
        ("col_scale", ctypes.c_void_p),
        ("resid", ctypes.c_void_p),
        ("ld_resid", ctypes.c_longlong),
        ("splits", ctypes.c_int),
        ("split_stride", ctypes.c_longlong),
        ("alpha", ctypes.c_float),
        ("reduce_add", ctypes.c_int),
        ("epilogue", ctypes.c_int),
        ("aux2", ctypes.c_void_p),
        ("ld_aux2", ctypes.c_longlong),
        ("c2", ctypes.c_void_p),
        ("ldc2", ctypes.c_longlong),
        ("sigma_half", ctypes.c_int),
    ]


_P = ctypes.c_void_p
_LL = ctypes.c_longlong
_I = ctypes.c_int
_F = ctypes.c_float

_SIGNATURES = {
    "btp_gemm": [ctypes.POINTER(GemmProblem), _I, _I, _P],
    "btp_gemm_scatter": [ctypes.POINTER(GemmProblem), _I, _I, ctypes.POINTER(_P), _I, _I, _I, _LL,
                         ctypes.POINTER(_I), _P],
    "btp_rmsnorm_residual": [_P, _LL, _P, _LL, _P, _LL, _P, _P, _LL, _P, _P, _I, _I, _F, _P],
    "btp_rmsnorm_apply": [_P, _LL, _P, _P, _I, _F, _P, _LL, _P, _I, _I, _P],
    "btp_fixup_sigma": [_P, _LL, _P, _I, _F, _P, _P, _LL, _P, _LL, _I, _I, _I, _I, _P],
    "btp_fixup_sigma_f32in": [_P, _LL, _P, _I, _F, _P, _P, _LL, _P, _LL, _I, _I, _I, _I, _P],
    "btp_swiglu": [_P, _LL, _P, _LL, _P, _LL, _I, _I, _P],
    "btp_swiglu_bwd": [_P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _LL, _I, _I, _P],
    "btp_fixup_sigma_bwd": [_P, _LL, _P, _LL, _P, _I, _P, _LL, _P, _I, _I, _I, _I, _P],
    "btp_rmsnorm_bwd": [_P, _LL, _P, _LL, _P, _P, _P, _LL, _P, _LL, _P, _I, ctypes.POINTER(_I), _I, _I, _P],
    "btp_reduce_rows": [_P, _I, _LL, _LL, _I, _I, _P, _P, _LL, _I, _P],
    "btp_add": [_P, _LL, _P, _LL, _P, _LL, _I, _I, _P],
    "btp_rmsnorm_bwd_prep": [_P, _LL, _P, _LL, _P, _P, _P, _LL, _P, _I, _I, _P],
    "btp_dot": [_P, _LL, _P, _LL, _I, _I, _P, _I, ctypes.POINTER(_I), _P],
    "btp_zero": [_P, _LL, _P],
    "btp_num_sms": [],
    "btp_version": [],
    "btp_gemm_f32": [ctypes.POINTER(GemmProblem), _I, _P],
    "btp_gemm_set_pair": [_I],
    "btp_gemm_set_res4": [_I],
    "btp_gemm_set_st_global": [_I],
    "btp_adamw": [_P, _P, _P, _P, _P, _LL, _F, _F, _F, _F, _F, _I, _P, _P],
    "btp_adamw_f32": [_P, _P, _P, _P, _P, _LL, _F, _F, _F, _F, _F, _I, _P, _P],
    "btp_counter_add": [_P, _I, _P],
    "btp_embedding_fwd": [_P, _P, _LL, _I, _I, _P, _LL, _I, _I, _P, _P],
    "btp_embedding_bwd": [_P, _P, _LL, _I, _P, _LL, _I, _I, _P],
    "btp_cross_entropy": [_P, _LL, _P, _I, _P, _P, _LL, _I, _F, _P],
    "btp_peer_signal": [_P, _P, _I, _I, _I, _P],
    "btp_peer_wait": [_P, _P, _I, _I, _P],
    "btp_peer_boundary_fwd": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _P, _P, _P],
    "btp_peer_boundary_bwd": [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "btp_peer_boundary_fwd_local": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _P, _P, _P],
    "btp_peer_boundary_bwd_local": [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "btp_peer_boundary_fwd_nvls": [_P, _P, _I, _I, _I, _I, _I, _I, _I, _F, _P, _P, _P, _P],
    "btp_peer_boundary_bwd_nvls": [_P, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P],
    "btp_attn_fwd": [_P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _I, _I, _I, _I, _P],
    "btp_attn_bwd": [_P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _P, _P, _LL, _P, _LL, _P, _LL, _P, _LL,
                     _I, _I, _I, _I, _P],
    "btp_attn_tune": [_I, _I],
    "btp_attn_fwd_trace": [_P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _I, _I, _I, _I, _P, _P],
    "btp_attn_bwd_trace": [_P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _LL, _P, _P, _P, _LL, _P, _LL, _P, _LL, _P, _LL,
                           _I, _I, _I, _I, _P, _P],
}
for _name in ("btp_rmsnorm_residual", "btp_rmsnorm_apply", "btp_fixup_sigma", "btp_swiglu", "btp_swiglu_bwd",
              "btp_fixup_sigma_bwd", "btp_rmsnorm_bwd", "btp_rmsnorm_bwd_prep", "btp_add", "btp_dot",
              "btp_embedding_fwd", "btp_embedding_bwd", "btp_cross_entropy"):
    _SIGNATURES[_name + "_f32"] = _SIGNATURES[_name]

_lib = None
_lock = threading.Lock()


def library_path() -> Path:
    return _LIB_PATH


def load(path: Path | None = None) -> ctypes.CDLL:
    """Load (once) and type the library. Raises NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        # BTP_LIB: an alternative build of the same library (in-process A/B of kernel versions)
        p = Path(path) if path else Path(os.environ.get("BTP_LIB", str(_LIB_PATH)))
        if not p.exists():
            raise NativeUnavailable(
                f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU or PyTorch fallback for the BTP kernels)"
            )
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeUnavailable(f"cannot load {p}: {exc}") from exc
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_char_p if name == "btp_version" else ctypes.c_int
        _lib = lib
        return lib


def call(name: str, *args) -> None:
    rc = getattr(load(), name)(*args)
    if rc != BTP_OK:
        raise NativeError(name, rc)
