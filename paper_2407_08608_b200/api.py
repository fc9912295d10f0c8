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
_SCHED = {"pingpong": _lib.SCHED_PINGPONG, "basic": _lib.SCHED_BASIC,
          "3stage": _lib.SCHED_3STAGE, "2stage": _lib.SCHED_2STAGE, "no_ws": _lib.SCHED_NO_WS}


def _t4(x: torch.Tensor | None) -> _lib.Tensor4:
    if x is None:
        return _lib.Tensor4(None, 0, 0, 0)
    if x.dim() != 4 or x.stride(3) != 1:
        raise ValueError("expected a [batch, seq, head, dim] tensor with contiguous dim")
    return _lib.Tensor4(x.data_ptr(), x.stride(0), x.stride(1), x.stride(2))


def _fail(status: int, what: str):
    msg = _lib.load().fa3b_error_string(status).decode()
    raise _lib.Fa3bError(status, f"{msg} ({what})")


def _same_problem(q, k, v):
    """The C ABI carries one (batch, seqlen, head_dim) for Q, K and V; check
    that they agree before handing it the shapes of q (the reference's
    validate_inputs, attention_ref.cpp:20-29)."""
    for name, x in (("q", q), ("k", k), ("v", v)):
        if x.dim() != 4:
            raise ValueError(f"{name}: expected a [batch, seq, head, dim] tensor")
        if x.numel() == 0:
            _fail(_lib.ERR_EMPTY, f"{name} is empty")
    if k.shape[3] != q.shape[3] or v.shape[3] != q.shape[3]:
        _fail(_lib.ERR_HEAD_DIM_MISMATCH, f"q {tuple(q.shape)}, k {tuple(k.shape)}, v {tuple(v.shape)}")
    if k.shape[1] != q.shape[1] or v.shape[1] != q.shape[1]:
        _fail(_lib.ERR_SEQLEN_MISMATCH, f"q {tuple(q.shape)}, k {tuple(k.shape)}, v {tuple(v.shape)}")
    if k.shape[0] != q.shape[0] or v.shape[0] != q.shape[0] or v.shape[2] != k.shape[2]:
        _fail(_lib.ERR_EMPTY if 0 in (k.shape[0], v.shape[0]) else _lib.ERR_SEQLEN_MISMATCH,
              f"batch / kv heads differ: q {tuple(q.shape)}, k {tuple(k.shape)}, v {tuple(v.shape)}")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        _fail(_lib.ERR_DTYPE, f"q {q.dtype}, k {k.dtype}, v {v.dtype}")
    if q.dtype not in _DT:
        _fail(_lib.ERR_DTYPE, f"{q.dtype}")


def _like(x, shape, dtype, name, code):
    if x is None:
        return
    if tuple(x.shape) != tuple(shape):
        _fail(code, f"{name} has shape {tuple(x.shape)}, expected {tuple(shape)}")
    if x.dtype != dtype:
        _fail(_lib.ERR_DTYPE, f"{name} is {x.dtype}, expected {dtype}")


def _lse_ok(lse, B, H, N, code):
    if lse is None:
        return
    if tuple(lse.shape) != (B, H, N) or lse.dtype != torch.float32 or not lse.is_contiguous():
        _fail(code, f"lse must be a contiguous fp32 [{B}, {H}, {N}] tensor, got "
                    f"{lse.dtype} {tuple(lse.shape)}")


def _scales_ok(sc, B, H, N, name):
    """FP8 scales [B, H, nblocks] (nblocks = ceil(N / 128)) or per tensor [B, H] /
    [B, H, 1]; returns the block rows the C ABI takes (128 or 0)."""
    if sc is None:
        _fail(-9, f"{name} is required for e4m3 inputs")
    if sc.dtype != torch.float32 or not sc.is_contiguous():
        _fail(_lib.ERR_SCALES, f"{name} must be contiguous fp32")
    nb = (N + 127) // 128
    shp = tuple(sc.shape)
    if shp in ((B, H), (B, H, 1)) and not (nb == 1 and shp == (B, H, 1)):
        return 0
    if shp == (B, H, nb):
        return 128
    _fail(_lib.ERR_SCALES, f"{name} has shape {shp}; expected [{B}, {H}, {nb}] or [{B}, {H}]")


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(x):
    return None if x is None else x.data_ptr()


def fwd(q, k, v, *, causal: bool = False, alpha: float | None = None,
        schedule: str = "pingpong", out_dtype=None, out=None, lse=None,
        q_scale=None, k_scale=None, v_scale=None, q_block_rows: int = 128,
        kv_block_rows: int = 128, stream=None):
    """Attention forward; returns (O, LSE). LSE is natural-log, [B, H, N] fp32.

    e4m3 inputs need q/k/v_scale from fp8_prepare; the quantization block
    (128 rows or per tensor) is read from each scale tensor's shape
    (q_block_rows / kv_block_rows are accepted for compatibility and must agree)."""
    _same_problem(q, k, v)
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    fp8 = q.dtype == torch.float8_e4m3fn
    if out_dtype is None:
        out_dtype = out.dtype if out is not None else (torch.bfloat16 if fp8 else q.dtype)
    _like(out, (B, N, H, D), out_dtype, "out", _lib.ERR_FWD_SHAPE)
    _lse_ok(lse, B, H, N, _lib.ERR_FWD_SHAPE)
    if fp8:
        qb = _scales_ok(q_scale, B, H, N, "q_scale")
        kb = _scales_ok(k_scale, B, Hkv, N, "k_scale")
        vb = _scales_ok(v_scale, B, Hkv, N, "v_scale")
        if kb != vb:
            _fail(_lib.ERR_SCALES, "k_scale and v_scale must use the same block size")
        q_block_rows, kv_block_rows = qb, kb
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
                saturate: bool = True, scale_pow2: bool = False, out=None, scales=None,
                stream=None):
    """Random-sign Hadamard (optional) + per-block e4m3 quantization.

    scale_pow2: power-of-two block scales (the smallest 2^e >= amax / 448) instead
    of the reference's amax / 448; the FP8 forward quantizes V this way.
    Returns (codes [B, N, H, D] float8_e4m3fn, scales [B, H, nblocks] fp32)."""
    if x.dim() != 4 or x.numel() == 0:
        _fail(_lib.ERR_EMPTY, f"fp8_prepare input {tuple(x.shape)}")
    B, N, H, D = x.shape
    nblk = 1 if block_rows == 0 else (N + block_rows - 1) // block_rows
    _like(out, (B, N, H, D), torch.float8_e4m3fn, "out", _lib.ERR_FWD_SHAPE)
    if scales is not None and (tuple(scales.shape) != (B, H, nblk) or scales.dtype != torch.float32
                               or not scales.is_contiguous()):
        _fail(_lib.ERR_SCALES, f"scales must be contiguous fp32 [{B}, {H}, {nblk}]")
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
    p.scale_pow2 = int(bool(scale_pow2))
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_fp8_prepare(ctypes.byref(p)))
    return out, scales


def fp8_fwd(q, k, v, *, causal: bool = False, alpha: float | None = None,
            per_block: bool = True, incoherent: bool = True, seed: int = 0,
            schedule: str = "pingpong", out_dtype=None, stream=None):
    """The reference's fp8_flash_fwd (fp8_attention.cpp:77-181) on the device:
    K5 (Hadamard on Q and K with one seed, block or tensor quantization of Q,
    K, V) then K6. Inputs are 16-bit or fp32 [B, N, H, D]; returns (O, LSE).
    Per block, V gets power-of-two scales (a documented deviation from the
    reference's amax / 448: same e4m3 precision, and K6 applies each key block's
    V scale exactly as an exponent shift of the P codes)."""
    blk = 128 if per_block else 0
    q8, sq = fp8_prepare(q, block_rows=blk, hadamard=incoherent, seed=seed, stream=stream)
    k8, sk = fp8_prepare(k, block_rows=blk, hadamard=incoherent, seed=seed, stream=stream)
    v8, sv = fp8_prepare(v, block_rows=blk, hadamard=False, scale_pow2=per_block, stream=stream)
    return fwd(q8, k8, v8, causal=causal, alpha=alpha, schedule=schedule, out_dtype=out_dtype,
               q_scale=sq, k_scale=sk, v_scale=sv, q_block_rows=blk, kv_block_rows=blk,
               stream=stream)


def bwd_preprocess(o, dout, *, delta=None, stream=None):
    """D = rowsum(dO * O) in fp32, [B, H, N]."""
    B, N, H, D = o.shape
    _like(dout, (B, N, H, D), o.dtype, "dout", _lib.ERR_DO_SHAPE)
    _lse_ok(delta, B, H, N, _lib.ERR_FWD_SHAPE)
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
        dq=None, dk=None, dv=None, workspace=None, deterministic: bool = False, stream=None):
    """Attention backward; returns (dQ, dK, dV) in the input dtype.

    deterministic=True accumulates dQ in a fixed order (ascending KV block, the
    reference's order, flash_bwd.cpp:58-61) so reruns are bitwise identical."""
    _same_problem(q, k, v)
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    # the reference's flash_bwd shape checks (flash_bwd.cpp:44-52)
    _like(dout, (B, N, H, D), q.dtype, "dout", _lib.ERR_DO_SHAPE)
    _like(o, (B, N, H, D), q.dtype, "o", _lib.ERR_FWD_SHAPE)
    _lse_ok(lse, B, H, N, _lib.ERR_FWD_SHAPE)
    _like(dq, (B, N, H, D), q.dtype, "dq", _lib.ERR_FWD_SHAPE)
    _like(dk, (B, N, Hkv, D), q.dtype, "dk", _lib.ERR_FWD_SHAPE)
    _like(dv, (B, N, Hkv, D), q.dtype, "dv", _lib.ERR_FWD_SHAPE)
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
    p.deterministic = int(bool(deterministic))
    p.workspace = _ptr(workspace)
    p.workspace_bytes = workspace.numel()
    p.stream = _stream(stream)
    _lib.check(_lib.load().fa3b_bwd(ctypes.byref(p)))
    return dq, dk, dv


def flops_forward(seqlen, headdim, heads, causal) -> int:
    return int(_lib.load().fa3b_flops_forward(seqlen, headdim, heads, int(bool(causal))))


def flops_backward(seqlen, headdim, heads, causal) -> int:
    return int(_lib.load().fa3b_flops_backward(seqlen, headdim, heads, int(bool(causal))))
