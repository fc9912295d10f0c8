"""ctypes binding of the C ABI in include/fa3b.h.

This is the reference-side binding a Python caller would add (see
INTEGRATION.md): plain structs and pointers, no torch types cross the
boundary. ``load()`` fails loudly when the CUDA library has not been built;
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libfa3b.so"

F16, BF16, E4M3, F32 = 0, 1, 2, 3
SCHED_PINGPONG, SCHED_BASIC, SCHED_3STAGE, SCHED_2STAGE, SCHED_NO_WS = 0, 1, 2, 3, 4

OK = 0
ERR_EMPTY = -1
ERR_HEAD_DIM_MISMATCH = -2
ERR_SEQLEN_MISMATCH = -3
ERR_DTYPE = -8
ERR_DO_SHAPE = -10
ERR_FWD_SHAPE = -11
ERR_SCALES = -18
ERR_CUDA = -100


class Tensor4(ctypes.Structure):
    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("stride_batch", ctypes.c_int64),
        ("stride_seq", ctypes.c_int64),
        ("stride_head", ctypes.c_int64),
    ]


class FwdParams(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("batch", ctypes.c_int32),
        ("heads_q", ctypes.c_int32),
        ("heads_kv", ctypes.c_int32),
        ("seqlen", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("in_dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("q", Tensor4),
        ("k", Tensor4),
        ("v", Tensor4),
        ("o", Tensor4),
        ("lse", ctypes.c_void_p),
        ("alpha", ctypes.c_double),
        ("causal", ctypes.c_int32),
        ("schedule", ctypes.c_int32),
        ("q_scale", ctypes.c_void_p),
        ("k_scale", ctypes.c_void_p),
        ("v_scale", ctypes.c_void_p),
        ("q_block_rows", ctypes.c_int32),
        ("kv_block_rows", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
    ]


class Fp8PrepareParams(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("seqlen", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("src_dtype", ctypes.c_int32),
        ("src", Tensor4),
        ("dst", Tensor4),
        ("scales", ctypes.c_void_p),
        ("block_rows", ctypes.c_int32),
        ("hadamard", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("saturate", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("scale_pow2", ctypes.c_int32),
    ]


class BwdParams(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("batch", ctypes.c_int32),
        ("heads_q", ctypes.c_int32),
        ("heads_kv", ctypes.c_int32),
        ("seqlen", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("q", Tensor4),
        ("k", Tensor4),
        ("v", Tensor4),
        ("o", Tensor4),
        ("dout", Tensor4),
        ("dq", Tensor4),
        ("dk", Tensor4),
        ("dv", Tensor4),
        ("lse", ctypes.c_void_p),
        ("alpha", ctypes.c_double),
        ("causal", ctypes.c_int32),
        ("deterministic", ctypes.c_int32),
        ("workspace", ctypes.c_void_p),
        ("workspace_bytes", ctypes.c_size_t),
        ("stream", ctypes.c_void_p),
    ]


class BwdPreprocessParams(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("seqlen", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("o", Tensor4),
        ("dout", Tensor4),
        ("delta", ctypes.c_void_p),
        ("stream", ctypes.c_void_p),
    ]


# Every symbol include/fa3b.h declares; tests check the library exports them.
EXPORTED_SYMBOLS = (
    "fa3b_fwd",
    "fa3b_fp8_prepare",
    "fa3b_bwd_preprocess",
    "fa3b_bwd",
    "fa3b_bwd_workspace_bytes",
    "fa3b_flops_forward",
    "fa3b_flops_backward",
    "fa3b_error_string",
    "fa3b_last_cuda_error",
    "fa3b_abi_version",
    "fa3b_last_launch_count",
)

_lib = None


class Fa3bError(RuntimeError):
    """Raised for a nonzero fa3b status; ``status`` holds the code."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("FA3B_LIB", LIB_PATH)).resolve()
    if not path.exists():
        raise RuntimeError(
            f"fa3b CUDA library not found at {path}; run __graft_entry__.build() "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(path))
    for name, argt, rest in (
        ("fa3b_fwd", [ctypes.POINTER(FwdParams)], ctypes.c_int),
        ("fa3b_fp8_prepare", [ctypes.POINTER(Fp8PrepareParams)], ctypes.c_int),
        ("fa3b_bwd_preprocess", [ctypes.POINTER(BwdPreprocessParams)], ctypes.c_int),
        ("fa3b_bwd", [ctypes.POINTER(BwdParams)], ctypes.c_int),
        ("fa3b_bwd_workspace_bytes", [ctypes.c_int32] * 5, ctypes.c_size_t),
        ("fa3b_flops_forward", [ctypes.c_uint64] * 3 + [ctypes.c_int32], ctypes.c_uint64),
        ("fa3b_flops_backward", [ctypes.c_uint64] * 3 + [ctypes.c_int32], ctypes.c_uint64),
        ("fa3b_error_string", [ctypes.c_int], ctypes.c_char_p),
        ("fa3b_last_cuda_error", [], ctypes.c_int),
        ("fa3b_abi_version", [], ctypes.c_int),
        ("fa3b_last_launch_count", [], ctypes.c_int),
    ):
        fn = getattr(lib, name)
        fn.argtypes = argt
        fn.restype = rest
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != OK:
        lib = load()
        msg = lib.fa3b_error_string(status).decode()
        if status == ERR_CUDA:
            msg += f" (cudaError {lib.fa3b_last_cuda_error()})"
        raise Fa3bError(status, msg)
