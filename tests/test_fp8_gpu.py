"""FP8 path on the device: K5 (fa3b_fp8_prepare) byte-exact against the
oracle's preprocess_incoherent + quantize (fp8_attention.cpp:33-42,94-96), and
K6 (e4m3 forward) against the FP64 reference with the reference's own FP8
emulation as the yardstick (fp8_attention.cpp:77-181).

K6 tolerance: RMSE(gpu - fp64) <= 1.3 * RMSE(ref_fp8 - fp64), where ref_fp8
is the reference's fp8_flash_fwd at the device's tile (128 x 128, per-block,
incoherent, same seed). The device deviates from the reference in documented
places (fixed P scale 2^thr/448 instead of the per-block amax, V's block
scale folded into P), so parity is by error band, not by value.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O
from _util import rmse

pytestmark = pytest.mark.gpu


def _outlier(port, B, N, H, D, seed):
    """fp32-exact outlier inputs (rng.cpp:50-71), [B, N, H, D] float64."""
    x = np.empty((B, N, H, D))
    for b in range(B):
        for h in range(H):
            x[b, :, h] = port.sample_outlier(N, D, port.substream(seed + 31 * b + h, 7)).astype(
                np.float32)
    return x


@pytest.mark.parametrize("D", [64, 128, 256])
@pytest.mark.parametrize("block_rows,hadamard", [(128, True), (128, False), (0, True), (0, False)])
def test_prepare_byte_exact(port, cuda, D, block_rows, hadamard):
    from paper_2407_08608_b200 import api
    import torch
    B, N, H = 2, 300, 2
    x = _outlier(port, B, N, H, D, seed=D + block_rows)
    xd = torch.from_numpy(x).float().cuda()
    codes, scales = api.fp8_prepare(xd, block_rows=block_rows, hadamard=hadamard, seed=1234)
    codes = codes.float().cpu().numpy()
    scales = scales.cpu().numpy()
    for b in range(B):
        for h in range(H):
            m = x[b, :, h]
            if hadamard:
                m, _ = port.preprocess_incoherent(m, m, 1234)
            want_c, want_s = port.quantize(m, block_rows)
            assert np.array_equal(codes[b, :, h], want_c), (b, h)
            assert np.array_equal(scales[b, h], want_s.astype(np.float32)), (b, h)


def test_prepare_from_bf16_and_saturation(port, cuda):
    from paper_2407_08608_b200 import api
    import torch
    x = torch.randn(1, 256, 1, 128, device="cuda", dtype=torch.bfloat16) * 3
    codes, scales = api.fp8_prepare(x, block_rows=128, hadamard=True, seed=9)
    xm = x[0, :, 0].double().cpu().numpy()
    qm, _ = port.preprocess_incoherent(xm, xm, 9)
    want_c, want_s = port.quantize(qm, 128)
    assert np.array_equal(codes[0, :, 0].float().cpu().numpy(), want_c)
    assert np.array_equal(scales[0, 0].cpu().numpy(), want_s.astype(np.float32))
    assert codes.float().abs().max().item() <= 448.0


def _fp8_case(port, ref, cuda, N, D, causal, seed, tile=128):
    from paper_2407_08608_b200 import api
    import torch
    q, k, v = (_outlier(port, 1, N, 1, D, seed + s)[0, :, 0] for s in (1, 2, 3))
    o_ref, l_ref = port.reference_attention(q, k, v, causal=causal)
    o_emu, l_emu = (ref or port).fp8_flash_fwd(q, k, v, causal=causal, seed=77,
                                               tile=(tile, tile))
    t = lambda a: torch.from_numpy(a[None, :, None, :]).float().cuda()  # noqa: E731
    o, lse = api.fp8_fwd(t(q), t(k), t(v), causal=causal, seed=77, out_dtype=torch.float32)
    return (o[0, :, 0].cpu().numpy(), lse[0, 0].cpu().numpy(), o_ref, l_ref, o_emu, l_emu, q, k,
            v)


@pytest.mark.parametrize("N,D,causal", [(1024, 128, False), (1024, 128, True), (640, 256, False),
                                        (1000, 256, True)])
def test_fp8_fwd_error_band(port, cuda, N, D, causal):
    o, lse, o_ref, l_ref, o_emu, l_emu, *_ = _fp8_case(port, None, cuda, N, D, causal,
                                                        seed=N + D)
    e_gpu, e_emu = rmse(o, o_ref), rmse(o_emu, o_ref)
    assert e_gpu <= 1.3 * e_emu, (e_gpu, e_emu)
    # scores come from e4m3 Q/K, so the LSE carries the same quantization error
    assert rmse(lse, l_ref) <= 1.3 * rmse(l_emu, l_ref) + 1e-4


def test_fp8_beats_per_tensor_baseline_at_8k(port, ref, cuda):
    """The paper's Table 2 claim at the reference's acceptance workload
    (acceptance_main.cpp:172-238: N 8192, d 128, outlier inputs): FA3-style
    FP8 (block quantization + incoherent processing) vs the per-tensor FP8
    standard-attention baseline, ratio >= 1.67, full-pipeline RMSE in the
    reference's band [6e-3, 1.3e-2]."""
    from paper_2407_08608_b200 import api
    import torch
    N, D = 8192, 128
    ratios = []
    for seed in (1, 2):
        q, k, v = (ref.sample_outlier(N, D, ref.substream(seed, s)) for s in (1, 2, 3))
        o_ref, _ = port.reference_attention(q, k, v)
        base, _ = ref.baseline_lowprec(q, k, v, O.E4M3)
        t = lambda a: torch.from_numpy(a[None, :, None, :]).float().cuda()  # noqa: E731
        o, _ = api.fp8_fwd(t(q), t(k), t(v), seed=ref.substream(seed, 9), out_dtype=torch.float32)
        e_full = rmse(o[0, :, 0].cpu().numpy(), o_ref)
        e_base = rmse(base, o_ref)
        assert 6e-3 <= e_full <= 1.3e-2, e_full
        ratios.append(e_base / e_full)
    assert min(ratios) >= 1.67, ratios


def test_fp8_gqa_and_batch(port, cuda):
    """Batched GQA through the fp8 path equals per-head calls bitwise."""
    from paper_2407_08608_b200 import api
    import torch
    q = torch.from_numpy(_outlier(port, 2, 384, 4, 128, 5)).float().cuda()
    k = torch.from_numpy(_outlier(port, 2, 384, 2, 128, 6)).float().cuda()
    v = torch.from_numpy(_outlier(port, 2, 384, 2, 128, 7)).float().cuda()
    o, lse = api.fp8_fwd(q, k, v, causal=True, seed=3)
    for b in range(2):
        for h in range(4):
            oo, ll = api.fp8_fwd(q[b:b + 1, :, h:h + 1].contiguous(),
                                 k[b:b + 1, :, h // 2:h // 2 + 1].contiguous(),
                                 v[b:b + 1, :, h // 2:h // 2 + 1].contiguous(), causal=True, seed=3)
            assert torch.equal(oo[0, :, 0], o[b, :, h]) and torch.equal(ll[0, 0], lse[b, h])


def test_fp8_rejects_bad_blocks(cuda):
    from paper_2407_08608_b200 import api
    from paper_2407_08608_b200._lib import Fa3bError
    import torch
    x = torch.randn(1, 256, 1, 128, device="cuda")
    q8, s = api.fp8_prepare(x, block_rows=64)
    with pytest.raises(Fa3bError, match="block"):
        api.fwd(q8, q8, q8, q_scale=s, k_scale=s, v_scale=s, q_block_rows=64, kv_block_rows=64)
    with pytest.raises(Fa3bError, match="power of two"):
        api.fp8_prepare(torch.randn(1, 8, 1, 96, device="cuda"))


@pytest.mark.parametrize("B,N,H,D,causal,per_block", [(1, 16384, 8, 256, False, True),
                                                      (2, 4173, 8, 256, True, True),
                                                      (1, 16384, 8, 256, False, False)])
def test_fp8_one_tile_many_items(cuda, B, N, H, D, causal, per_block):
    """K6 at d256 runs one query tile per CTA with a second S buffer in TMEM: many work
    items per persistent CTA, ragged causal blocks, both scale granularities (no
    Hadamard, so torch can emulate the quantization). Sampled rows against fp32 torch;
    yardstick: the same attention on e4m3-rounded Q/K/V (128-row block or tensor
    scales) and e4m3 P (scale 1/448), error within 1.3x of that emulation's."""
    from paper_2407_08608_b200 import api
    import torch
    e4m3 = torch.float8_e4m3fn
    gen = torch.Generator(device="cuda").manual_seed(N + H)
    q, k, v = (torch.randn(B, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
               for _ in range(3))
    o, lse = api.fp8_fwd(q, k, v, causal=causal, per_block=per_block, incoherent=False,
                         out_dtype=torch.float32)

    def quant(x):  # [N, D] fp32 -> e4m3-rounded values with the kernel's scales
        nb = (N + 127) // 128
        xp = torch.zeros(nb * 128, D, device="cuda")
        xp[:N] = x
        xb = xp.view(nb, 128, D) if per_block else xp.view(1, -1, D)
        sc = xb.abs().amax(dim=(1, 2), keepdim=True) / 448
        return ((xb / sc).to(e4m3).float() * sc).view(-1, D)[:N]

    rows = torch.unique(torch.cat([torch.tensor([0, 127, 128, N - 1]),
                                   torch.randint(0, N, (60,), generator=gen, device="cuda").cpu()])).cuda()
    alpha = 1 / math.sqrt(D)
    for b in sorted({0, B - 1}):
        for h in (0, H - 1):
            qf, kf, vf = (x[b, :, h].float() for x in (q, k, v))
            mask = torch.arange(N, device="cuda")[None, :] > rows[:, None]
            s = alpha * qf[rows] @ kf.T
            s8 = alpha * quant(qf)[rows] @ quant(kf).T
            if causal:
                s, s8 = s.masked_fill(mask, -math.inf), s8.masked_fill(mask, -math.inf)
            ref = torch.softmax(s, -1) @ vf
            p = torch.exp(s8 - s8.amax(-1, keepdim=True))
            emu = ((p * 448).to(e4m3).float() / 448) @ quant(vf) / p.sum(-1, keepdim=True)
            err, err_emu = (o[b, rows, h] - ref).norm().item(), (emu - ref).norm().item()
            assert err <= 1.3 * err_emu + 1e-3 * ref.norm().item(), (err, err_emu)
            assert (lse[b, h, rows] - torch.logsumexp(s, -1)).abs().max().item() < 0.05
