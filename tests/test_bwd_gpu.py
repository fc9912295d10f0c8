"""K2-K4 backward on the device against the CPU oracle (reference flash_bwd,
core/src/flash_bwd.cpp:29-126).

Tolerance: per gradient tensor, with the same 16-bit
inputs and the FP64 forward's O (rounded to the input format) and LSE,
    relRMS(gpu) <= 2 * relRMS(emu) + 1e-5
where relRMS(x) = rms(x - exact) / rms(exact), exact is the reference's
FP64 flash_bwd and emu the oracle's tensor-core emulation of it
(orc_lowprec_flash_bwd: P and dS rounded to the format, fp32 accumulation).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O
from _util import FMT, make_inputs, rmse, to_dev

pytestmark = pytest.mark.gpu


def _dt(fmt):
    import torch
    return torch.bfloat16 if fmt == "bf16" else torch.float16


def _oracle(port, q, k, v, do, alpha, causal, fmt):
    """Exact FP64 grads, the emulated grads, and the (O, LSE) both sides use."""
    B, N, H, D = q.shape
    Hkv = k.shape[2]
    g = H // Hkv
    o = np.empty_like(q)
    lse = np.empty((B, H, N))
    ex = [np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)]
    em = [np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)]
    for b in range(B):
        for h in range(H):
            kh, vh = k[b, :, h // g], v[b, :, h // g]
            oo, ll, _ = port.flash_fwd(q[b, :, h], kh, vh, alpha=alpha, causal=causal,
                                       tile=(128, 128))
            o[b, :, h] = port.round_array(oo, FMT[fmt])
            lse[b, h] = ll
            e = port.flash_bwd(q[b, :, h], kh, vh, do[b, :, h], oo, ll, alpha=alpha,
                               causal=causal, tile=(128, 128))
            m = port.flash_bwd(q[b, :, h], kh, vh, do[b, :, h], o[b, :, h], ll, alpha=alpha,
                               causal=causal, tile=(128, 128), fmt=FMT[fmt])
            ex[0][b, :, h] = e[0]
            em[0][b, :, h] = m[0]
            for t in (1, 2):
                ex[t][b, :, h // g] += e[t]
                em[t][b, :, h // g] += m[t]
    return o, lse, ex, em


def _rel(x, ref):
    return rmse(x, ref) / max(float(np.sqrt(np.mean(ref ** 2))), 1e-30)


CASES = [
    # B, H, Hkv, N, D, causal, fmt, alpha
    pytest.param(1, 2, 2, 512, 64, False, "bf16", None, id="d64"),
    pytest.param(1, 2, 2, 512, 128, True, "bf16", None, id="d128-causal"),
    pytest.param(2, 2, 1, 300, 128, False, "fp16", None, id="gqa-ragged-fp16"),
    pytest.param(1, 4, 2, 200, 64, True, "bf16", -0.11, id="neg-alpha-causal-gqa"),
    pytest.param(1, 1, 1, 1000, 128, True, "bf16", None, id="ragged-1000"),
    # long GQA groups: the Q/dO ring and the LSE/D buffers wrap many times within a CTA
    pytest.param(1, 8, 1, 640, 128, True, "bf16", None, id="gqa8-ring-d128"),
    pytest.param(1, 4, 1, 520, 64, False, "fp16", None, id="gqa4-ring-d64"),
    # tiny and ragged lengths: one valid row / one row past a tile boundary
    pytest.param(2, 2, 2, 1, 128, True, "bf16", None, id="n1-d128"),
    pytest.param(1, 2, 1, 1, 64, False, "bf16", None, id="n1-d64-gqa"),
    pytest.param(1, 2, 2, 129, 128, True, "bf16", None, id="n129-causal"),
]


@pytest.mark.parametrize("B,H,Hkv,N,D,causal,fmt,alpha", CASES)
def test_bwd_matches_oracle(port, cuda, B, H, Hkv, N, D, causal, fmt, alpha):
    from paper_2407_08608_b200 import api
    import torch
    alpha = 1.0 / math.sqrt(D) if alpha is None else alpha
    q, k, v, do = make_inputs(port, B, H, Hkv, N, D, seed=2000 + N + D, fmt=fmt, with_do=True)
    o, lse, ex, em = _oracle(port, q, k, v, do, alpha, causal, fmt)
    dt = _dt(fmt)
    dq, dk, dv = api.bwd(to_dev(q, dt), to_dev(k, dt), to_dev(v, dt), to_dev(o, dt),
                         to_dev(do, dt), torch.from_numpy(lse).float().cuda(), causal=causal,
                         alpha=alpha)
    scale = float(np.sqrt(np.mean(ex[2] ** 2)))  # dV's RMS: the gradients' natural size
    for name, got, e, m in zip(("dq", "dk", "dv"), (dq, dk, dv), ex, em):
        got = got.float().cpu().numpy()
        if float(np.sqrt(np.mean(e ** 2))) < 1e-6 * scale:
            # N = 1: dS = P (dP - D) is exactly 0 (one key, P = 1, O = V), so dQ and dK
            # are rounding noise of the 16-bit O: absolute, against the emulation's
            assert rmse(got, e) <= 2 * rmse(m, e) + 1e-3 * scale, (name, rmse(got, e), rmse(m, e))
            continue
        r_gpu, r_emu = _rel(got, e), _rel(m, e)
        # + the rounding of the 16-bit gradient outputs (the emulation keeps FP64
        # outputs: at N = 1 with GQA its dV is exact, the device's is one RN away)
        out_rn = 2.0 ** -8 if fmt == "bf16" else 2.0 ** -11
        assert r_gpu <= 2 * r_emu + out_rn, (name, r_gpu, r_emu)


def test_bwd_end_to_end_with_device_forward(port, cuda):
    """fa3b_fwd -> fa3b_bwd, as a training step would chain them."""
    from paper_2407_08608_b200 import api
    import torch
    q, k, v, do = make_inputs(port, 1, 2, 2, 384, 128, seed=55, with_do=True)
    o_ref, lse_ref, ex, em = _oracle(port, q, k, v, do, 1 / math.sqrt(128), True, "bf16")
    qd, kd, vd, dod = (to_dev(x, torch.bfloat16) for x in (q, k, v, do))
    o, lse = api.fwd(qd, kd, vd, causal=True)
    grads = api.bwd(qd, kd, vd, o, dod, lse, causal=True)
    for got, e, m in zip(grads, ex, em):
        assert _rel(got.float().cpu().numpy(), e) <= 2 * _rel(m, e) + 1e-5


def test_bwd_zero_upstream_gives_zero(port, cuda):
    """test_flash_bwd.cpp:56-66."""
    from paper_2407_08608_b200 import api
    import torch
    q, k, v = (to_dev(x, torch.bfloat16) for x in make_inputs(port, 1, 2, 2, 256, 64, seed=930))
    o, lse = api.fwd(q, k, v, causal=True)
    dq, dk, dv = api.bwd(q, k, v, o, torch.zeros_like(o), lse, causal=True)
    assert not dq.any() and not dk.any() and not dv.any()


def test_bwd_corrupted_lse_is_quiet_but_wrong(port, cuda):
    """test_flash_bwd.cpp:105-119: no error, finite, visibly different."""
    from paper_2407_08608_b200 import api
    import torch
    q, k, v, do = (to_dev(x, torch.bfloat16)
                   for x in make_inputs(port, 1, 1, 1, 256, 64, seed=935, with_do=True))
    o, lse = api.fwd(q, k, v)
    good = api.bwd(q, k, v, o, do, lse)
    bad_lse = lse.clone()
    bad_lse[0, 0, 0] += 0.05
    bad = api.bwd(q, k, v, o, do, bad_lse)
    assert all(torch.isfinite(x.float()).all() for x in bad)
    assert max((a.float() - b.float()).abs().max().item() for a, b in zip(good, bad)) > 1e-4


def test_bwd_dkdv_deterministic(port, cuda):
    """dK/dV accumulate in TMEM in a fixed order -> bitwise repeatable even in the
    default (arrival-order dQ) mode."""
    from paper_2407_08608_b200 import api
    import torch
    q, k, v, do = (to_dev(x, torch.bfloat16)
                   for x in make_inputs(port, 1, 4, 2, 640, 128, seed=937, with_do=True))
    o, lse = api.fwd(q, k, v, causal=True)
    a = api.bwd(q, k, v, o, do, lse, causal=True)
    b = api.bwd(q, k, v, o, do, lse, causal=True)
    assert torch.equal(a[1], b[1]) and torch.equal(a[2], b[2])
    assert (a[0].float() - b[0].float()).abs().max().item() < 1e-2


@pytest.mark.parametrize("B,H,Hkv,N,D,causal", [
    (1, 4, 2, 640, 128, True), (2, 8, 8, 2048, 128, False), (1, 16, 4, 3000, 64, True),
    (2, 16, 16, 8192, 64, False), (1, 32, 32, 4096, 128, True)])
def test_bwd_deterministic_mode_bitwise(port, cuda, B, H, Hkv, N, D, causal):
    """deterministic=True: every dQ tile takes its KV tiles' contributions in
    ascending order (flash_bwd.cpp:58-61), so dQ, dK and dV are bitwise equal
    across reruns (test_flash_bwd.cpp:121-131) — on shapes with many KV tiles
    per dQ tile and several persistent rounds — and within the usual tolerance
    of the arrival-order result."""
    from paper_2407_08608_b200 import api
    import torch
    gen = torch.Generator(device="cuda").manual_seed(N + D + H)
    q, do = (torch.randn(B, N, H, D, device="cuda", generator=gen).bfloat16() for _ in range(2))
    k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen).bfloat16() for _ in range(2))
    o, lse = api.fwd(q, k, v, causal=causal)
    runs = [api.bwd(q, k, v, o, do, lse, causal=causal, deterministic=True) for _ in range(3)]
    for r in runs[1:]:
        for x, y in zip(runs[0], r):
            assert torch.equal(x, y)
    fast = api.bwd(q, k, v, o, do, lse, causal=causal)
    scale = fast[0].float().abs().max().item()
    assert (runs[0][0].float() - fast[0].float()).abs().max().item() <= 1e-2 * scale
    assert torch.equal(runs[0][1], fast[1]) and torch.equal(runs[0][2], fast[2])


def test_bwd_preprocess_matches_numpy(port, cuda):
    from paper_2407_08608_b200 import api
    import torch
    o = torch.randn(2, 300, 3, 128, device="cuda", dtype=torch.bfloat16)
    do = torch.randn_like(o)
    delta = api.bwd_preprocess(o, do)
    want = (o.float() * do.float()).sum(-1).permute(0, 2, 1)
    assert (delta - want).abs().max().item() < 1e-3


@pytest.mark.parametrize("D,causal", [(128, True), (64, False)])
def test_bwd_full_size_against_torch_autograd(cuda, D, causal):
    """C4 at N = 16k for one head against fp32 torch autograd."""
    from paper_2407_08608_b200 import api
    import torch
    N = 16384
    gen = torch.Generator(device="cuda").manual_seed(7 + D)
    q, k, v, do = (torch.randn(1, N, 1, D, device="cuda", generator=gen, dtype=torch.bfloat16)
                   for _ in range(4))
    o, lse = api.fwd(q, k, v, causal=causal)
    dq, dk, dv = api.bwd(q, k, v, o, do, lse, causal=causal)
    qf, kf, vf = (x[0, :, 0].float().requires_grad_(True) for x in (q, k, v))
    s = (qf @ kf.T) / math.sqrt(D)
    if causal:
        s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), -math.inf)
    out = torch.softmax(s, -1) @ vf
    out.backward(do[0, :, 0].float())
    for got, ref in ((dq, qf.grad), (dk, kf.grad), (dv, vf.grad)):
        rel = ((got[0, :, 0].float() - ref).norm() / ref.norm()).item()
        assert rel < 1e-2, rel


def test_bwd_rejects_bad_arguments(cuda):
    from paper_2407_08608_b200 import api
    from paper_2407_08608_b200._lib import Fa3bError
    import torch
    q = torch.zeros(1, 128, 2, 256, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(1, 2, 128, device="cuda")
    with pytest.raises(Fa3bError, match="head dimension"):
        api.bwd(q, q, q, q, q, lse)
    q = torch.zeros(1, 128, 2, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(Fa3bError, match="workspace"):
        api.bwd(q, q, q, q, q, lse, workspace=torch.empty(16, dtype=torch.uint8, device="cuda"))


@pytest.mark.gpu
@pytest.mark.parametrize("H,Hkv,N,D,causal", [(75, 75, 256, 64, True), (150, 75, 256, 128, False),
                                             (3, 1, 4500, 128, True)])
def test_bwd_persistent_rounds_against_torch(cuda, H, Hkv, N, D, causal):
    """Work-item counts just past one and two rounds of the persistent grid (150 and 300
    items on 148 SMs, causal boustrophedon rounds) and a long ragged causal GQA case,
    every head checked against fp32 torch autograd."""
    from paper_2407_08608_b200 import api
    import torch
    gen = torch.Generator(device="cuda").manual_seed(H + N)
    q, do = (torch.randn(1, N, H, D, device="cuda", generator=gen, dtype=torch.bfloat16) for _ in range(2))
    k, v = (torch.randn(1, N, Hkv, D, device="cuda", generator=gen, dtype=torch.bfloat16) for _ in range(2))
    o, lse = api.fwd(q, k, v, causal=causal)
    dq, dk, dv = api.bwd(q, k, v, o, do, lse, causal=causal)
    g = H // Hkv
    qf = q[0].float().transpose(0, 1).requires_grad_(True)                 # [H, N, D]
    kf = k[0].float().transpose(0, 1).requires_grad_(True)                 # [Hkv, N, D]
    vf = v[0].float().transpose(0, 1).requires_grad_(True)
    s = qf @ kf.repeat_interleave(g, 0).transpose(1, 2) / math.sqrt(D)
    if causal:
        s = s.masked_fill(torch.ones(N, N, device="cuda", dtype=torch.bool).triu(1), -math.inf)
    out = torch.softmax(s, -1) @ vf.repeat_interleave(g, 0)
    out.backward(do[0].float().transpose(0, 1))
    for got, ref in ((dq, qf.grad), (dk, kf.grad), (dv, vf.grad)):
        rel = ((got[0].float().transpose(0, 1) - ref).norm() / ref.norm()).item()
        assert rel < 1e-2, rel
