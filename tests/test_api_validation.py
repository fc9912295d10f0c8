"""api.fwd / api.bwd / api.fp8_prepare validate every tensor against q before
the C ABI (which carries a single batch, seqlen, head_dim and dtype) sees
them, with the reference's error cases (attention_ref.cpp:20-29,
flash_bwd.cpp:44-52). Checked on CPU tensors: validation happens before any
device work, so no GPU is needed."""
from __future__ import annotations

import pytest
import torch

from paper_2407_08608_b200 import _lib, api


def _t(*shape, dtype=torch.bfloat16):
    return torch.zeros(*shape, dtype=dtype)


def _status(fn, *a, **kw):
    with pytest.raises(_lib.Fa3bError) as e:
        fn(*a, **kw)
    return e.value.status


def test_fwd_shape_mismatches(fa3b_lib):
    q = _t(2, 256, 4, 64)
    assert _status(api.fwd, q, _t(2, 256, 4, 128), _t(2, 256, 4, 64)) == _lib.ERR_HEAD_DIM_MISMATCH
    assert _status(api.fwd, q, _t(2, 200, 4, 64), _t(2, 200, 4, 64)) == _lib.ERR_SEQLEN_MISMATCH
    assert _status(api.fwd, q, _t(2, 256, 4, 64), _t(2, 250, 4, 64)) == _lib.ERR_SEQLEN_MISMATCH
    assert _status(api.fwd, q, _t(1, 256, 4, 64), _t(1, 256, 4, 64)) == _lib.ERR_SEQLEN_MISMATCH
    assert _status(api.fwd, q, _t(2, 256, 4, 64, dtype=torch.float16),
                   _t(2, 256, 4, 64)) == _lib.ERR_DTYPE
    assert _status(api.fwd, _t(2, 0, 4, 64), _t(2, 0, 4, 64), _t(2, 0, 4, 64)) == _lib.ERR_EMPTY
    # output / lse buffers must have q's shape and the requested dtype
    kv = _t(2, 256, 2, 64)
    assert _status(api.fwd, q, kv, kv, out=_t(2, 256, 4, 32)) == _lib.ERR_FWD_SHAPE
    assert _status(api.fwd, q, kv, kv, out=_t(2, 256, 4, 64, dtype=torch.float32),
                   out_dtype=torch.bfloat16) == _lib.ERR_DTYPE
    assert _status(api.fwd, q, kv, kv, lse=_t(2, 4, 255, dtype=torch.float32)) == _lib.ERR_FWD_SHAPE
    assert _status(api.fwd, q, kv, kv, lse=_t(2, 4, 256)) == _lib.ERR_FWD_SHAPE


def test_fp8_scale_shapes_decide_block_rows(fa3b_lib):
    e4 = torch.float8_e4m3fn
    q, k = _t(1, 300, 2, 128, dtype=e4), _t(1, 300, 1, 128, dtype=e4)
    f32 = torch.float32
    ok_q, ok_k = _t(1, 2, 3, dtype=f32), _t(1, 1, 3, dtype=f32)
    # [B, H, 1] with 3 blocks is per tensor; a wrong block count is an error
    assert _status(api.fwd, q, k, k, q_scale=_t(1, 2, 2, dtype=f32), k_scale=ok_k,
                   v_scale=ok_k) == _lib.ERR_SCALES
    assert _status(api.fwd, q, k, k, q_scale=ok_q, k_scale=ok_k,
                   v_scale=_t(1, 1, 1, dtype=f32)) == _lib.ERR_SCALES  # k blocked, v per tensor
    assert _status(api.fwd, q, k, k, q_scale=ok_q, k_scale=_t(1, 1, 3),
                   v_scale=ok_k) == _lib.ERR_SCALES  # not fp32
    assert api._scales_ok(_t(1, 2, 1, dtype=f32), 1, 2, 300, "q") == 0
    assert api._scales_ok(_t(1, 2, dtype=f32), 1, 2, 300, "q") == 0
    assert api._scales_ok(ok_q, 1, 2, 300, "q") == 128


def test_bwd_shape_mismatches(fa3b_lib):
    q, kv = _t(1, 256, 4, 64), _t(1, 256, 2, 64)
    lse = _t(1, 4, 256, dtype=torch.float32)
    assert _status(api.bwd, q, kv, kv, q, _t(1, 256, 4, 32), lse) == _lib.ERR_DO_SHAPE
    assert _status(api.bwd, q, kv, kv, _t(1, 256, 4, 64, dtype=torch.float32), q,
                   lse) == _lib.ERR_DTYPE
    assert _status(api.bwd, q, kv, kv, _t(1, 128, 4, 64), q, lse) == _lib.ERR_FWD_SHAPE
    assert _status(api.bwd, q, kv, kv, q, q, _t(1, 4, 128, dtype=torch.float32)) == _lib.ERR_FWD_SHAPE
    assert _status(api.bwd, q, kv, kv, q, q, lse, dk=_t(1, 256, 4, 64)) == _lib.ERR_FWD_SHAPE
    assert _status(api.bwd, q, kv, _t(1, 256, 2, 128), q, q, lse) == _lib.ERR_HEAD_DIM_MISMATCH


def test_prepare_buffers(fa3b_lib):
    x = _t(1, 300, 2, 128)
    assert _status(api.fp8_prepare, x, scales=_t(1, 2, 2, dtype=torch.float32)) == _lib.ERR_SCALES
    assert _status(api.fp8_prepare, x, out=_t(1, 300, 2, 128)) == _lib.ERR_DTYPE
    assert _status(api.fp8_prepare, _t(1, 0, 2, 128)) == _lib.ERR_EMPTY
