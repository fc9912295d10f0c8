"""Device-tensor API over the C ABI (torch supplies device memory and streams).

Tensors are [batch, seqlen, heads, head_dim] with the head_dim axis
contiguous, f16/bf16 (or e4m3 codes for the FP8 path). Every function calls
exactly one C-ABI entry point of ``libfa3b.so``; nothing is computed in Python.
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib

_DT = {torch.float16: _lib.F16, torch.bfloat16: _lib.BF16, torch.float32: _lib.F32,
       torch.float8_e4m3fn: _lib.E4M3}
_SCHED = {"pingpong": _lib.SCHED_PINGPONG, "2stage": _lib.SCHED_PINGPONG,
          "basic": _lib.SCHED_BASIC, "3stage": _lib.SCHED_3STAGE}


def _t4(x: torch.Tensor | None) -> _lib.Tensor4:
    if x is None:
        return _lib.Tensor4(None, 0, 0, 0)
    if x.dim() != 4 or x.stride(3) != 1:
        raise ValueError("expected a [batch, seq, head, dim] tensor with contiguous dim")
    return _lib.Tensor4(x.data_ptr(), x.stride(0), x.stride(1), x.stride(2))


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(x):
    return None if x is None else x.data_ptr()


def fwd(q, k, v, *, causal: bool = False, alpha: float | None = None,
        schedule: str = "pingpong", out_dtype=None, out=None, lse=None,
        q_scale=None, k_scale=None, v_scale=None, q_block_rows: int = 128,
        kv_block_rows: int = 128, stream=None):
    """Attention forward; returns (O, LSE). LSE is natural-log, [B, H, N] fp32."""
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    fp8 = q.dtype == torch.float8_e4m3fn
    if out_dtype is None:
        out_dtype = torch.bfloat16 if fp8 else q.dtype
    if out is None:
        out = torch.empty((B, N, H, D), dtype=out_dtype, device=q.device)
    if lse is None:
        lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device)
    if alpha is None:
        alpha = 1.0 / math.sqrt(D)
    p = _lib.FwdParams()
    p.struct_size = ctypes.sizeof(_lib.FwdParams)
    p.batch, p.heads_q, p.heads_kv, p.seqlen, p.head_dim = B, H, Hkv, N, D
    p.in_dtype = _DT[q.dtype]
    p.out_dtype = _DT[out.dtype]
    p.q, p.k, p.v, p.o = _t4(q), _t4(k), _t4(v), _t4(out)
    p.lse = _ptr(lse)
    p.alpha = float(alpha)
    p.causal = int(bool(causal))
    p.schedule = _SCHED[schedule]
    p.q_scale, p.k_scale, p.v_scale = _ptr(q_scale), _ptr(k_scale), _ptr(v_scale)
    p.q_block_rows = q_block_rows
    p.kv_block_rows = kv_block_rows
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_fwd(ctypes.byref(p)))
    return out, lse


def fp8_prepare(x, *, block_rows: int = 128, hadamard: bool = True, seed: int = 0,
                saturate: bool = True, out=None, scales=None, stream=None):
    """Random-sign Hadamard (optional) + per-block e4m3 quantization.

    Returns (codes [B, N, H, D] float8_e4m3fn, scales [B, H, nblocks] fp32)."""
    B, N, H, D = x.shape
    nblk = 1 if block_rows == 0 else (N + block_rows - 1) // block_rows
    if out is None:
        out = torch.empty((B, N, H, D), dtype=torch.float8_e4m3fn, device=x.device)
    if scales is None:
        scales = torch.empty((B, H, nblk), dtype=torch.float32, device=x.device)
    p = _lib.Fp8PrepareParams()
    p.struct_size = ctypes.sizeof(_lib.Fp8PrepareParams)
    p.batch, p.heads, p.seqlen, p.head_dim = B, H, N, D
    p.src_dtype = _DT[x.dtype]
    p.src, p.dst = _t4(x), _t4(out)
    p.scales = _ptr(scales)
    p.block_rows = block_rows
    p.hadamard = int(bool(hadamard))
    p.seed = seed & 0xFFFFFFFFFFFFFFFF
    p.saturate = int(bool(saturate))
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_fp8_prepare(ctypes.byref(p)))
    return out, scales


def fp8_fwd(q, k, v, *, causal: bool = False, alpha: float | None = None,
            per_block: bool = True, incoherent: bool = True, seed: int = 0,
            schedule: str = "pingpong", out_dtype=None, stream=None):
    """The reference's fp8_flash_fwd (fp8_attention.cpp:77-181) on the device:
    K5 (Hadamard on Q and K with one seed, block or tensor quantization of Q,
    K, V) then K6. Inputs are 16-bit or fp32 [B, N, H, D]; returns (O, LSE)."""
    blk = 128 if per_block else 0
    q8, sq = fp8_prepare(q, block_rows=blk, hadamard=incoherent, seed=seed, stream=stream)
    k8, sk = fp8_prepare(k, block_rows=blk, hadamard=incoherent, seed=seed, stream=stream)
    v8, sv = fp8_prepare(v, block_rows=blk, hadamard=False, stream=stream)
    return fwd(q8, k8, v8, causal=causal, alpha=alpha, schedule=schedule, out_dtype=out_dtype,
               q_scale=sq, k_scale=sk, v_scale=sv, q_block_rows=blk, kv_block_rows=blk,
               stream=stream)


def bwd_preprocess(o, dout, *, delta=None, stream=None):
    """D = rowsum(dO * O) in fp32, [B, H, N]."""
    B, N, H, D = o.shape
    if delta is None:
        delta = torch.empty((B, H, N), dtype=torch.float32, device=o.device)
    p = _lib.BwdPreprocessParams()
    p.struct_size = ctypes.sizeof(_lib.BwdPreprocessParams)
    p.batch, p.heads, p.seqlen, p.head_dim = B, H, N, D
    p.dtype = _DT[o.dtype]
    p.o, p.dout = _t4(o), _t4(dout)
    p.delta = _ptr(delta)
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_bwd_preprocess(ctypes.byref(p)))
    return delta


def bwd_workspace_bytes(B, H, Hkv, N, D) -> int:
    return int(_lib.load().fa3b_bwd_workspace_bytes(B, H, Hkv, N, D))


def bwd(q, k, v, o, dout, lse, *, causal: bool = False, alpha: float | None = None,
        dq=None, dk=None, dv=None, workspace=None, stream=None):
    """Attention backward; returns (dQ, dK, dV) in the input dtype."""
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    if alpha is None:
        alpha = 1.0 / math.sqrt(D)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    ws = bwd_workspace_bytes(B, H, Hkv, N, D)
    if workspace is None:
        workspace = torch.empty(max(ws, 1), dtype=torch.uint8, device=q.device)
    p = _lib.BwdParams()
    p.struct_size = ctypes.sizeof(_lib.BwdParams)
    p.batch, p.heads_q, p.heads_kv, p.seqlen, p.head_dim = B, H, Hkv, N, D
    p.dtype = _DT[q.dtype]
    p.q, p.k, p.v, p.o, p.dout = _t4(q), _t4(k), _t4(v), _t4(o), _t4(dout)
    p.dq, p.dk, p.dv = _t4(dq), _t4(dk), _t4(dv)
    p.lse = _ptr(lse)
    p.alpha = float(alpha)
    p.causal = int(bool(causal))
    p.deterministic = 0
    p.workspace = _ptr(workspace)
    p.workspace_bytes = workspace.numel()
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_bwd(ctypes.byref(p)))
    return dq, dk, dv


def flops_forward(seqlen, headdim, heads, causal) -> int:
    return int(_lib.load().fa3b_flops_forward(seqlen, headdim, heads, int(bool(causal))))


def flops_backward(seqlen, headdim, heads, causal) -> int:
    return int(_lib.load().fa3b_flops_backward(seqlen, headdim, heads, int(bool(causal))))
