"""K1 forward on the device against the CPU oracle.

Tolerance (stated per SURVEY.md §8(c)): with both sides fed the same
bf16/fp16-rounded inputs,
    RMSE(gpu - fp64)   <= 2 * RMSE(emu - fp64) + 1e-6
    max|gpu - fp64|    <= 8 * max|emu - fp64| + 1e-6
    max|LSE_gpu - LSE| <= 1e-3
where fp64 is the reference's exact attention (reference_attention_o) and
emu is the oracle's tiled low-precision forward (lowprec.cpp:166-240 in the
input format: fp32 scores/softmax/accumulator, P rounded to the format,
output rounded to the format).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from _util import FMT, make_inputs, maxabs, rmse, to_dev

pytestmark = pytest.mark.gpu


def _api():
    from paper_2407_08608_b200 import api
    return api


def _torch():
    import torch
    return torch


def _dtype(fmt):
    torch = _torch()
    return torch.bfloat16 if fmt == "bf16" else torch.float16


def _oracle_fwd(port, q, k, v, alpha, causal, fmt):
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    g = H // Hkv
    ref_o = np.empty_like(q)
    ref_l = np.empty((B, H, N))
    emu_o = np.empty_like(q)
    for b in range(B):
        for h in range(H):
            args = (q[b, :, h], k[b, :, h // g], v[b, :, h // g])
            ref_o[b, :, h], ref_l[b, h] = port.reference_attention(*args, alpha=alpha,
                                                                   causal=causal)
            emu_o[b, :, h], _ = port.lowprec_flash_fwd(*args, alpha=alpha, causal=causal,
                                                       tile=(128, 128), fmt=FMT[fmt])
    return ref_o, ref_l, emu_o


CASES = [
    # B, H, Hkv, N, D, causal, fmt, schedule, alpha
    pytest.param(2, 8, 8, 512, 64, False, "fp16", "pingpong", None, id="C1-B2H8N512d64-fp16"),
    pytest.param(1, 2, 2, 1000, 128, True, "bf16", "pingpong", None, id="ragged-causal-d128"),
    pytest.param(1, 2, 1, 777, 256, True, "bf16", "basic", None, id="d256-gqa-causal"),
    pytest.param(1, 4, 2, 384, 128, False, "bf16", "basic", -0.09, id="negative-alpha"),
    pytest.param(2, 2, 2, 130, 64, True, "fp16", "pingpong", 0.3, id="tile1-partial"),
    pytest.param(1, 2, 2, 100, 64, False, "bf16", "pingpong", None, id="N-lt-128"),
    pytest.param(1, 1, 1, 1, 64, False, "bf16", "pingpong", None, id="N1"),
    pytest.param(1, 2, 2, 640, 128, True, "fp16", "3stage", None, id="3stage-d128"),
    pytest.param(1, 2, 2, 512, 256, False, "fp16", "basic", 0.02, id="d256-fp16-serial"),
    pytest.param(1, 2, 1, 700, 64, True, "bf16", "2stage", None, id="2stage-d64-gqa"),
    pytest.param(1, 2, 2, 513, 256, True, "bf16", "2stage", None, id="2stage-d256"),
    pytest.param(2, 2, 2, 1000, 128, False, "fp16", "no_ws", None, id="nows-d128"),
    pytest.param(1, 4, 2, 300, 64, True, "bf16", "no_ws", -0.2, id="nows-d64-causal"),
    pytest.param(1, 2, 2, 257, 128, True, "bf16", "basic", None, id="serial-d128"),
]


@pytest.mark.parametrize("B,H,Hkv,N,D,causal,fmt,sched,alpha", CASES)
def test_fwd_matches_oracle(port, cuda, B, H, Hkv, N, D, causal, fmt, sched, alpha):
    api = _api()
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    q, k, v = make_inputs(port, B, H, Hkv, N, D, seed=1000 + N + D, fmt=fmt)
    dt = _dtype(fmt)
    o, lse = api.fwd(to_dev(q, dt), to_dev(k, dt), to_dev(v, dt), causal=causal, alpha=alpha,
                     schedule=sched)
    o = o.float().cpu().numpy()
    lse = lse.cpu().numpy()
    ref_o, ref_l, emu_o = _oracle_fwd(port, q, k, v, alpha, causal, fmt)
    e_gpu, e_emu = rmse(o, ref_o), rmse(emu_o, ref_o)
    m_gpu, m_emu = maxabs(o, ref_o), maxabs(emu_o, ref_o)
    assert e_gpu <= 2 * e_emu + 1e-6, (e_gpu, e_emu)
    assert m_gpu <= 8 * m_emu + 1e-6, (m_gpu, m_emu)
    assert maxabs(lse, ref_l) <= 1e-3


def test_fwd_fp32_output_is_tighter(port, cuda):
    api = _api()
    torch = _torch()
    q, k, v = make_inputs(port, 1, 2, 2, 300, 128, seed=77)
    o, lse = api.fwd(to_dev(q, torch.bfloat16), to_dev(k, torch.bfloat16),
                     to_dev(v, torch.bfloat16), causal=True, out_dtype=torch.float32)
    ref_o, ref_l, emu_o = _oracle_fwd(port, q, k, v, 1 / math.sqrt(128), True, "bf16")
    # no output rounding: only P's bf16 rounding and fp32 accumulation remain
    assert rmse(o.cpu().numpy(), ref_o) <= 0.75 * rmse(emu_o, ref_o)
    assert maxabs(lse.cpu().numpy(), ref_l) <= 1e-4


@pytest.mark.parametrize("name", ["dev_n200_d64_causal", "dev_n160_d128"])
def test_fwd_against_reference_golden(golden, cuda, name):
    """Straight against outputs of the reference library (tests/golden)."""
    api = _api()
    torch = _torch()
    n, d, causal, a = golden[f"{name}_meta"]
    q, k, v = (golden[f"{name}_{x}"][None, :, None, :] for x in ("q", "k", "v"))
    o, lse = api.fwd(to_dev(q, torch.bfloat16), to_dev(k, torch.bfloat16),
                     to_dev(v, torch.bfloat16), causal=bool(causal), alpha=float(a),
                     out_dtype=torch.float32)
    assert maxabs(o.cpu().numpy()[0, :, 0], golden[f"{name}_o"]) < 2e-2
    assert rmse(o.cpu().numpy()[0, :, 0], golden[f"{name}_o"]) < 2e-3
    assert maxabs(lse.cpu().numpy()[0, 0], golden[f"{name}_lse"]) < 1e-4


def test_gqa_mapping_equals_duplication_bitwise(port, cuda):
    """acceptance criterion 10 (acceptance_main.cpp:357-383): bit-exact."""
    api = _api()
    torch = _torch()
    for hkv in (4, 2, 1):
        q, k, v = make_inputs(port, 1, 4, hkv, 256, 64, seed=500 + hkv)
        qd, kd, vd = (to_dev(x, torch.bfloat16) for x in (q, k, v))
        o1, l1 = api.fwd(qd, kd, vd)
        g = 4 // hkv
        o2, l2 = api.fwd(qd, kd.repeat_interleave(g, 2).contiguous(),
                         vd.repeat_interleave(g, 2).contiguous())
        assert torch.equal(o1, o2) and torch.equal(l1, l2)


SCHEDULES = ("pingpong", "basic", "3stage", "2stage", "no_ws")


@pytest.mark.parametrize("D", [64, 128, 256])
def test_schedules_and_reruns_bit_identical(port, cuda, D):
    """The reference demands bit-identical schedules (test_flash_fwd.cpp:152-196)
    and deterministic reruns; every device schedule (ping-pong, serial basic,
    3-stage, 2-stage, no warp specialization) runs the same per-tile arithmetic
    in another order, so all agree bitwise in 16-bit."""
    api = _api()
    torch = _torch()
    from paper_2407_08608_b200._lib import Fa3bError
    for causal in (False, True):
        q, k, v = (to_dev(x, torch.bfloat16) for x in make_inputs(port, 1, 2, 2, 700, D, 9))
        a = api.fwd(q, k, v, causal=causal, schedule="pingpong")
        c = api.fwd(q, k, v, causal=causal, schedule="pingpong")
        assert torch.equal(a[0], c[0]) and torch.equal(a[1], c[1])
        for sched in SCHEDULES[1:]:
            if D == 256 and sched == "no_ws":
                with pytest.raises(Fa3bError, match="schedule"):
                    api.fwd(q, k, v, causal=causal, schedule=sched)
                continue
            b = api.fwd(q, k, v, causal=causal, schedule=sched)
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), sched


@pytest.mark.parametrize("sched", ["basic", "2stage", "3stage", "no_ws"])
def test_schedule_variants_many_items(cuda, sched):
    """The one-tile variants over many persistent work items (several rounds of the
    148-CTA grid, ragged last block, GQA): sampled rows against fp32 torch."""
    api = _api()
    torch = _torch()
    B, N, H, Hkv, D = 2, 4100, 24, 8, 128
    gen = torch.Generator(device="cuda").manual_seed(11)
    q = torch.randn(B, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
    k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen, dtype=torch.bfloat16)
            for _ in range(2))
    for causal in (False, True):
        o, lse = api.fwd(q, k, v, causal=causal, schedule=sched)
        o_ref, lse_ref = api.fwd(q, k, v, causal=causal)
        assert torch.equal(o, o_ref) and torch.equal(lse, lse_ref)
        rows = torch.tensor([0, 1, 127, 128, 2049, N - 1], device="cuda")
        for b, h in ((0, 0), (1, 23)):
            s = q[b, rows, h].float() @ k[b, :, h // 3].float().T / math.sqrt(D)
            if causal:
                s = s.masked_fill(torch.arange(N, device="cuda")[None, :] > rows[:, None], -math.inf)
            ref = torch.softmax(s, -1) @ v[b, :, h // 3].float()
            assert (o[b, rows, h].float() - ref).abs().max().item() < 2e-2


def test_strided_inputs(port, cuda):
    """Q/K/V as views into a packed [B, N, 3, H, D] buffer."""
    api = _api()
    torch = _torch()
    q, k, v = make_inputs(port, 2, 4, 4, 300, 64, seed=3)
    qkv = torch.stack([to_dev(x, torch.bfloat16) for x in (q, k, v)], dim=2)
    o1, l1 = api.fwd(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2], causal=True)
    o2, l2 = api.fwd(*(qkv[:, :, i].contiguous() for i in range(3)), causal=True)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("D", [64, 128, 256])
def test_output_rows_16_byte_aligned(cuda, D):
    """O (and dK / dV) rows only 16-byte aligned (head stride D + 8 elements): the
    epilogues fall back from 256-bit to 128-bit stores; results bitwise equal to
    the contiguous, 32-byte aligned outputs."""
    api = _api()
    torch = _torch()
    B, N, H = 2, 300, 2
    g = torch.Generator(device="cuda").manual_seed(D)
    q, k, v, do = (torch.randn(B, N, H, D, device="cuda", generator=g, dtype=torch.bfloat16)
                   for _ in range(4))
    o1, l1 = api.fwd(q, k, v, causal=True)
    wide = torch.zeros(B, N, H, D + 8, device="cuda", dtype=torch.bfloat16)
    o2, l2 = api.fwd(q, k, v, causal=True, out=wide[..., :D])
    assert o2.data_ptr() == wide.data_ptr() and torch.equal(o1, o2) and torch.equal(l1, l2)
    assert torch.count_nonzero(wide[..., D:]) == 0  # nothing written past the view
    if D <= 128:
        g1 = api.bwd(q, k, v, o1, do, l1, causal=True, deterministic=True)
        dkw, dvw = (torch.zeros(B, N, H, D + 8, device="cuda", dtype=torch.bfloat16) for _ in range(2))
        g2 = api.bwd(q, k, v, o1, do, l1, causal=True, deterministic=True, dk=dkw[..., :D], dv=dvw[..., :D])
        for a, b_ in zip(g1, g2):
            assert torch.equal(a, b_)
        assert torch.count_nonzero(dkw[..., D:]) == 0 and torch.count_nonzero(dvw[..., D:]) == 0


@pytest.mark.parametrize("D,causal", [(128, False), (128, True), (64, True), (256, False)])
def test_full_size_against_torch_rows(cuda, D, causal):
    """C2 at N = 16k (B = 1, H = 2048 / D): a sample of query rows checked
    against fp32 torch attention over all 16k keys."""
    api = _api()
    torch = _torch()
    N, H = 16384, 2048 // D
    gen = torch.Generator(device="cuda").manual_seed(D + causal)
    q, k, v = (torch.randn(1, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
               for _ in range(3))
    o, lse = api.fwd(q, k, v, causal=causal)
    rows = torch.cat([torch.arange(0, 64), torch.randint(64, N, (192,), generator=gen,
                                                          device="cuda").cpu()]).cuda()
    alpha = 1 / math.sqrt(D)
    for h in range(0, H, max(1, H // 4)):
        s = alpha * q[0, rows, h].float() @ k[0, :, h].float().T
        if causal:
            s = s.masked_fill(torch.arange(N, device="cuda")[None, :] > rows[:, None], -math.inf)
        ref_l = torch.logsumexp(s, -1)
        ref_o = torch.softmax(s, -1) @ v[0, :, h].float()
        assert (o[0, rows, h].float() - ref_o).abs().max().item() < 2e-2
        assert (lse[0, h, rows] - ref_l).abs().max().item() < 1e-3


@pytest.mark.parametrize("B,N,H,Hkv,causal", [(1, 65536, 1, 1, True), (1, 8192, 64, 8, False),
                                              (64, 256, 8, 8, True), (1, 256, 149, 149, True),
                                              (3, 512, 99, 33, True)])
def test_extreme_shapes_against_torch_rows(cuda, B, N, H, Hkv, causal):
    """64k keys, C5's 64/8 GQA, a 4096-item grid, and item counts one past one and
    two rounds of the 148-CTA persistent grid (causal boustrophedon rounds):
    sampled rows against fp32 torch."""
    api = _api()
    torch = _torch()
    D = 128
    gen = torch.Generator(device="cuda").manual_seed(N + H)
    q = torch.randn(B, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
    k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen, dtype=torch.bfloat16)
            for _ in range(2))
    o, lse = api.fwd(q, k, v, causal=causal)
    alpha = 1 / math.sqrt(D)
    rows = torch.unique(torch.cat([torch.tensor([0, 1, N - 1]),
                                   torch.randint(0, N, (61,), generator=gen, device="cuda").cpu()])).cuda()
    for b in sorted({0, B - 1}):
        for h in sorted({0, H // 2, H - 1}):
            kh = h // (H // Hkv)
            s = alpha * q[b, rows, h].float() @ k[b, :, kh].float().T
            if causal:
                s = s.masked_fill(torch.arange(N, device="cuda")[None, :] > rows[:, None], -math.inf)
            assert (o[b, rows, h].float() - torch.softmax(s, -1) @ v[b, :, kh].float()).abs().max().item() < 2e-2
            assert (lse[b, h, rows] - torch.logsumexp(s, -1)).abs().max().item() < 1e-3


def test_fwd_rejects_bad_arguments(cuda):
    api = _api()
    torch = _torch()
    from paper_2407_08608_b200._lib import Fa3bError
    q = torch.zeros(1, 128, 2, 96, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Fa3bError, match="head dimension"):
        api.fwd(q, q, q)
    q = torch.zeros(1, 128, 2, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Fa3bError, match="alpha"):
        api.fwd(q, q, q, alpha=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("B,N,H,Hkv,D,causal,sched", [
    (1, 16384, 8, 8, 256, False, "pingpong"),   # 1024 items: ~7 per CTA (the S2 hang case)
    (2, 4173, 8, 2, 256, True, "pingpong"),     # ragged causal GQA, one-tile S2 path
    (1, 16384, 16, 16, 128, True, "basic"),     # one-tile S2 at d128, causal
    (3, 1000, 32, 8, 64, False, "basic"),       # one-tile S2 at d64, ragged
])
def test_one_tile_double_buffered_s(cuda, B, N, H, Hkv, D, causal, sched):
    """One-tile CTAs keep two S buffers in TMEM and load K/V in MMA order (K_0, K_1,
    {V_j, K_{j+2}}); many work items per persistent CTA, ragged and causal blocks,
    GQA: sampled rows of every checked head against fp32 torch."""
    api = _api()
    torch = _torch()
    gen = torch.Generator(device="cuda").manual_seed(N + D)
    q = torch.randn(B, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
    k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen, dtype=torch.bfloat16)
            for _ in range(2))
    o, lse = api.fwd(q, k, v, causal=causal, schedule=sched)
    alpha = 1 / math.sqrt(D)
    rows = torch.unique(torch.cat([torch.tensor([0, 127, 128, N - 1]),
                                   torch.randint(0, N, (60,), generator=gen, device="cuda").cpu()])).cuda()
    for b in sorted({0, B - 1}):
        for h in sorted({0, H // 3, H - 1}):
            kh = h // (H // Hkv)
            s = alpha * q[b, rows, h].float() @ k[b, :, kh].float().T
            if causal:
                s = s.masked_fill(torch.arange(N, device="cuda")[None, :] > rows[:, None], -math.inf)
            assert (o[b, rows, h].float() - torch.softmax(s, -1) @ v[b, :, kh].float()).abs().max().item() < 2e-2
            assert (lse[b, h, rows] - torch.logsumexp(s, -1)).abs().max().item() < 1e-3


@pytest.mark.gpu
@pytest.mark.parametrize("D", [64, 128, 256])
@pytest.mark.parametrize("causal", [False, True])
def test_tiny_and_ragged_lengths_buffer_rotation(cuda, D, causal):
    """The S-buffer schedules (three rotating buffers at d64, two at d256) at every
    block-count edge: N = 1, partial first block, exactly one / two blocks, one past.
    All heads and rows against fp32 torch."""
    api = _api()
    torch = _torch()
    for N in (1, 5, 127, 128, 129, 255, 256, 257, 383, 640):
        gen = torch.Generator(device="cuda").manual_seed(N * 7 + D)
        B, H = 2, 3
        q, k, v = (torch.randn(B, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16)
                   for _ in range(3))
        o, lse = api.fwd(q, k, v, causal=causal)
        s = (q.float().permute(0, 2, 1, 3) @ k.float().permute(0, 2, 3, 1)) / math.sqrt(D)
        if causal:
            s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), -math.inf)
        ref = (torch.softmax(s, -1) @ v.float().permute(0, 2, 1, 3)).permute(0, 2, 1, 3)
        assert (o.float() - ref).abs().max().item() < 2e-2, N
        assert (lse - torch.logsumexp(s, -1)).abs().max().item() < 1e-3, N
