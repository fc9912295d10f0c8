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
                                        (1000, 256, True), (1024, 64, False), (1000, 64, True),
                                        (300, 64, False), (500, 128, False), (500, 128, True)])
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


@pytest.mark.parametrize("D,causal", [(128, False), (64, True), (256, True)])
def test_fp8_negative_alpha_equals_negated_keys(cuda, D, causal):
    """alpha < 0 (the reference accepts any finite nonzero alpha,
    attention_ref.cpp:27-28) flips the QK^T sign in the MMA instruction: with
    e4m3 codes symmetric and RNE accumulation, fp8_fwd(alpha = -a) equals
    fp8_fwd(-K, alpha = +a) bit for bit (Hadamard, block scales and all)."""
    from paper_2407_08608_b200 import api
    import torch
    g = torch.Generator(device="cuda").manual_seed(D + causal)
    q, k, v = (torch.randn(2, 300, 2, D, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    a = 0.7 / math.sqrt(D)
    o1, l1 = api.fp8_fwd(q, k, v, causal=causal, alpha=-a, seed=5)
    o2, l2 = api.fp8_fwd(q, -k, v, causal=causal, alpha=a, seed=5)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    # and against fp32 attention with the negative scale
    s = -a * q[0, :, 1].float() @ k[0, :, 1].float().T
    if causal:
        s = s.masked_fill(torch.arange(300, device="cuda")[None, :] > torch.arange(300, device="cuda")[:, None],
                          -math.inf)
    ref = torch.softmax(s, -1) @ v[0, :, 1].float()
    assert (o1[0, :, 1].float() - ref).norm().item() < 0.05 * ref.norm().item()


@pytest.mark.parametrize("N", [1, 127, 129, 300])
def test_fp8_zero_blocks_and_tiny_lengths(cuda, N):
    """Edge cases of the per-block path: an all-zero V block (scale 1 and zero
    codes, quantize.cpp:41-42 — the V-scale fold must not divide by it), an
    all-zero Q block (LSE = log N), single-row and ragged lengths:
    against fp32 attention."""
    from paper_2407_08608_b200 import api
    import torch
    g = torch.Generator(device="cuda").manual_seed(N)
    q, k, v = (torch.randn(1, N, 2, 128, device="cuda", generator=g, dtype=torch.bfloat16) for _ in range(3))
    v[:, 128:256] = 0
    q[:, 256:] = 0
    o, lse = api.fp8_fwd(q, k, v, seed=2, out_dtype=torch.float32)
    for h in range(2):
        s = q[0, :, h].float() @ k[0, :, h].float().T / math.sqrt(128)
        ref = torch.softmax(s, -1) @ v[0, :, h].float()
        assert torch.isfinite(o).all() and torch.isfinite(lse).all()
        # e4m3 Q/K/V/P: a few percent of the norm (N 127 gaussian measured 5.2 %)
        assert (o[0, :, h] - ref).norm().item() <= 0.08 * ref.norm().item() + 1e-6
        if N > 256:  # zero Q rows: S = 0 and LSE = log N up to the FP8 path's
            # degree-2 exp2 polynomial on 2 of 8 pairs (relative error <= 2e-3)
            assert (lse[0, h, 256:] - math.log(N)).abs().max().item() < 2e-3


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
                                                      (1, 16384, 8, 256, False, False),
                                                      (1, 8192, 16, 64, False, True),
                                                      (2, 4173, 4, 64, True, True),
                                                      (1, 8192, 16, 64, True, False)])
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
            # LSE: the kernel's scores are the e4m3 ones (tight), which differ from the
            # exact scores by the quantization error (loose: per tensor at d 64 a single
            # causal score moves by up to ~0.07)
            assert (lse[b, h, rows] - torch.logsumexp(s8, -1)).abs().max().item() < 0.01
            assert (lse[b, h, rows] - torch.logsumexp(s, -1)).abs().max().item() < 0.1


def _bf16_rows(kind, N, D, rng):
    """float32 matrices of bf16-exact values exercising the fast K5 path's cases:
    int32-exact rows, rows outside the int32 range (exponent spread, zeros mixed
    with non-zeros, subnormals), all-zero rows and blocks, extreme magnitudes."""
    import torch
    x = rng.standard_normal((N, D)).astype(np.float32) * 3
    if kind == "wide":  # every 7th row spans > 23 - log2(d) binades -> FP64 rows
        x[::7, 0] *= 2.0 ** 20
        x[3::11, 1] *= 2.0 ** -30
    elif kind == "zeros":
        x[::5, ::9] = 0.0          # zeros next to non-zeros
        x[1::13] = 0.0             # all-zero rows
        x[256:384] = 0.0           # an all-zero 128-row block
    elif kind == "tiny":
        x *= np.float32(2.0 ** -120)   # int path at the small end (k near 127)
        x[::6] *= np.float32(2.0 ** -12)  # subnormal bf16 values
    elif kind == "huge":
        x *= np.float32(2.0 ** 100)
    return torch.from_numpy(x).bfloat16().float().numpy()


@pytest.mark.parametrize("D", [64, 128, 256])
@pytest.mark.parametrize("hadamard", [True, False])
@pytest.mark.parametrize("kind", ["gauss", "wide", "zeros", "tiny", "huge"])
def test_prepare_bf16_fast_path_byte_exact(port, cuda, D, hadamard, kind):
    # the bf16 / 128-row-block kernel (int32 transform, FP32 encode with an exact
    # FP64 fallback) against the oracle's FP64 preprocess_incoherent + quantize
    from paper_2407_08608_b200 import api
    import torch
    rng = np.random.default_rng(D * 7 + hadamard + len(kind))
    B, N, H = 1, 1000, 2
    x = np.stack([_bf16_rows(kind, N, D, rng) for _ in range(H)], axis=1)[None]  # [1, N, H, D]
    xd = torch.from_numpy(x).cuda().bfloat16()
    codes, scales = api.fp8_prepare(xd, block_rows=128, hadamard=hadamard, seed=4321)
    codes = codes.float().cpu().numpy()
    scales = scales.cpu().numpy()
    for h in range(H):
        m = x[0, :, h].astype(np.float64)
        if hadamard:
            m, _ = port.preprocess_incoherent(m, m, 4321)
        want_c, want_s = port.quantize(m, 128)
        assert np.array_equal(scales[0, h], want_s.astype(np.float32)), h
        bad = np.argwhere(codes[0, :, h] != want_c)
        assert bad.size == 0, (h, bad[:5])


def test_prepare_bf16_fast_path_full_size(port, cuda):
    # C2 shape of one (batch, head) pair at N 8192, d 128: byte-exact at full size
    from paper_2407_08608_b200 import api
    import torch
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(1, 8192, 2, 128, device="cuda", generator=g, dtype=torch.bfloat16)
    for had in (True, False):
        codes, scales = api.fp8_prepare(x, block_rows=128, hadamard=had, seed=77)
        for h in range(2):
            m = x[0, :, h].double().cpu().numpy()
            if had:
                m, _ = port.preprocess_incoherent(m, m, 77)
            want_c, want_s = port.quantize(m, 128)
            assert np.array_equal(codes[0, :, h].float().cpu().numpy(), want_c), (had, h)
            assert np.array_equal(scales[0, h].cpu().numpy(), want_s.astype(np.float32)), (had, h)


@pytest.mark.parametrize("D", [64, 128, 256])
def test_prepare_bf16_fast_path_persistent_strided(port, cuda, D):
    # persistent CTAs walk several blocks each through the TMA ring (2 x 33 blocks x
    # H heads > CTAs), the last block ragged (N = 4100), the input a strided view of
    # a packed [B, N, 3, H, d] qkv tensor: sampled (batch, head) pairs byte-exact
    from paper_2407_08608_b200 import api
    import torch
    B, N, H = 2, 4100, 2048 // D
    g = torch.Generator(device="cuda").manual_seed(D)
    qkv = torch.randn(B, N, 3, H, D, device="cuda", generator=g, dtype=torch.bfloat16)
    x = qkv[:, :, 1]
    for had in (True, False):
        codes, scales = api.fp8_prepare(x, block_rows=128, hadamard=had, seed=9)
        for b, h in ((0, 0), (0, H - 1), (1, H // 2), (1, H - 1)):
            m = x[b, :, h].double().cpu().numpy()
            if had:
                m, _ = port.preprocess_incoherent(m, m, 9)
            want_c, want_s = port.quantize(m, 128)
            assert np.array_equal(codes[b, :, h].float().cpu().numpy(), want_c), (had, b, h)
            assert np.array_equal(scales[b, h].cpu().numpy(), want_s.astype(np.float32)), (had, b, h)


def test_prepare_bf16_nonfinite_block_reports_nan_scale(cuda):
    # the reference throws on non-finite input (quantize.cpp:15); the device marks
    # the block's scale NaN and leaves the other blocks intact
    from paper_2407_08608_b200 import api
    import torch
    x = torch.randn(1, 384, 1, 128, device="cuda", dtype=torch.bfloat16)
    x[0, 200, 0, 5] = float("inf")
    _, s = api.fp8_prepare(x, block_rows=128, hadamard=True, seed=3)
    s = s.cpu()
    assert torch.isnan(s[0, 0, 1]) and torch.isfinite(s[0, 0, 0]) and torch.isfinite(s[0, 0, 2])


def _quantize_pow2(port, m, block_rows=128):
    """quantize_per_block (quantize.cpp:47-60) with the scale raised to the
    smallest power of two >= amax / 448 (fa3b_fp8_prepare_params.scale_pow2)."""
    codes, scales = np.empty_like(m), []
    for r0 in range(0, m.shape[0], block_rows):
        blk = m[r0:r0 + block_rows]
        amax = float(np.abs(blk).max())
        s = amax / 448.0 if amax != 0.0 else 1.0
        mant, ex = np.frexp(s)
        if mant != 0.5:
            s = 2.0 ** ex
        codes[r0:r0 + block_rows] = port.round_array(blk * (1.0 / s), O.E4M3)
        scales.append(s)
    return codes, np.array(scales)


@pytest.mark.parametrize("D", [64, 128, 256])
@pytest.mark.parametrize("src", ["bf16", "f32"])
@pytest.mark.parametrize("hadamard", [True, False])
def test_prepare_pow2_scales_byte_exact(port, cuda, D, src, hadamard):
    from paper_2407_08608_b200 import api
    import torch
    rng = np.random.default_rng(D + hadamard)
    x = np.stack([_bf16_rows("gauss", 700, D, rng) for _ in range(2)], axis=1)[None]
    xd = torch.from_numpy(x).cuda()
    xd = xd.bfloat16() if src == "bf16" else xd.float()
    codes, scales = api.fp8_prepare(xd, block_rows=128, hadamard=hadamard, seed=99, scale_pow2=True)
    codes, scales = codes.float().cpu().numpy(), scales.cpu().numpy()
    for h in range(2):
        m = x[0, :, h].astype(np.float64)
        if hadamard:
            m, _ = port.preprocess_incoherent(m, m, 99)
        want_c, want_s = _quantize_pow2(port, m)
        assert np.array_equal(scales[0, h], want_s.astype(np.float32)), h
        assert np.array_equal(codes[0, :, h], want_c), h
        assert np.all(np.log2(scales[0, h]) == np.round(np.log2(scales[0, h])))


def test_fp8_p2_pair_variant_matches_default(tmp_path, cuda):
    """The P2 pair (FA3B_FWD_P2=1: 64-key blocks, one softmax warpgroup per tile,
    per-tile double S buffers; an A/B alternative, profiles/r02/r02u_p2_pair_ab.log)
    computes the same FP8 attention as the default ping-pong pair: run in a child
    process (the switch is read once per process), outputs within FP8 noise."""
    import subprocess
    import sys
    import textwrap
    import torch
    from paper_2407_08608_b200 import api
    script = textwrap.dedent('''
        import sys, torch
        sys.path.insert(0, sys.argv[2])
        from paper_2407_08608_b200 import api
        g = torch.Generator(device="cuda").manual_seed(11)
        q, k, v = (torch.randn(2, 1000, 4, 128, device="cuda", generator=g).bfloat16() for _ in range(3))
        outs = [api.fp8_fwd(q, k, v, causal=c, seed=5, out_dtype=torch.float32) for c in (False, True)]
        torch.save([(o.cpu(), l.cpu()) for o, l in outs], sys.argv[1])
    ''')
    from pathlib import Path
    root = str(Path(__file__).resolve().parents[1])
    f = tmp_path / "p2.pt"
    env = dict(__import__("os").environ, FA3B_FWD_P2="1")
    subprocess.run([sys.executable, "-c", script, str(f), root], env=env, check=True, timeout=300)
    p2 = torch.load(f)
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v = (torch.randn(2, 1000, 4, 128, device="cuda", generator=g).bfloat16() for _ in range(3))
    for (o2, l2), c in zip(p2, (False, True)):
        o, l = api.fp8_fwd(q, k, v, causal=c, seed=5, out_dtype=torch.float32)
        o, l = o.cpu(), l.cpu()
        # both against fp32 attention on the bf16 inputs: P2 quantizes P per 64-key
        # block with its own lazy-max timing, so it matches the default's error, not
        # its bits
        qf, kf, vf = (x.float().cpu() for x in (q, k, v))
        s_ = torch.einsum("bnhd,bmhd->bhnm", qf, kf) / 128 ** 0.5
        if c:
            s_ = s_.masked_fill(torch.ones(1000, 1000, dtype=torch.bool).triu(1), float("-inf"))
        ref = torch.einsum("bhnm,bmhd->bnhd", torch.softmax(s_, -1), vf)
        assert torch.isfinite(o2).all()
        e2, e1 = (o2 - ref).norm().item(), (o - ref).norm().item()
        assert e2 <= 1.25 * e1 + 1e-3 * ref.norm().item(), (c, e2, e1)
        assert (l2 - l).abs().max() < 0.05, c
