"""The BASELINE configs at full size pinned to the CPU oracle (not to fp32
torch): the device runs the whole workload, and two sampled (batch, head)
units of each are recomputed by the oracle on the same 16-bit inputs.

    C2 fwd N 8192 d128 (B2 H16), non-causal and causal; N 16384 d64 (B1 H32)
    C5 fwd Llama-3-70B N 8192, 64 query / 8 KV heads (units of one KV group)
    C4 bwd N 8192 d128 (B2 H16) and d64 (B2 H32), non-causal and causal

"exact" is the oracle's FP64 tiled forward (flash_fwd.cpp:18-232; the reference
pins it to the dense FP64 attention at 1e-12, test_flash_fwd.cpp:106-118) or
FP64 flash_bwd (flash_bwd.cpp:43-126); "emu" is the oracle's tensor-core
emulation of the same path in bf16 (lowprec.cpp:166-240 forward, P and dS
rounded to bf16 with fp32 accumulation backward). Tolerances, as in
test_fwd_gpu.py / test_bwd_gpu.py:
    fwd  RMSE(gpu - exact) <= 2 RMSE(emu - exact) + 1e-6, max-abs <= 8x, LSE <= 1e-3
    bwd  relRMS(gpu) <= 2 relRMS(emu) + 1e-5 for dQ, dK, dV
The backward sides share the device forward's O and LSE as inputs. All oracle
jobs of the module run at once in a thread pool (ctypes releases the GIL), so
the wall time is about that of the longest single job (~1 min).
"""
from __future__ import annotations

import math
import os
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from _util import maxabs, rmse

pytestmark = pytest.mark.gpu

FWD = {
    # name: (B, H, Hkv, N, D, causal, sampled (b, h) units)
    "c2-n8192-d128": (2, 16, 16, 8192, 128, False, [(0, 3), (1, 12)]),
    "c2-n8192-d128-causal": (2, 16, 16, 8192, 128, True, [(0, 0), (1, 15)]),
    "c2-n16384-d64": (1, 32, 32, 16384, 64, False, [(0, 5), (0, 31)]),
    "c5-gqa64-8-n8192-causal": (1, 64, 8, 8192, 128, True, [(0, 8), (0, 15)]),
}
BWD = {
    "c4-n8192-d128": (2, 16, 16, 8192, 128, False, [(0, 2), (1, 9)]),
    "c4-n8192-d128-causal": (2, 16, 16, 8192, 128, True, [(1, 0), (0, 14)]),
    "c4-n8192-d64": (2, 32, 32, 8192, 64, False, [(0, 7), (1, 30)]),
    "c4-n8192-d64-causal": (2, 32, 32, 8192, 64, True, [(0, 0), (1, 21)]),
}


def _np(x):
    return x.double().cpu().numpy()


@pytest.fixture(scope="module")
def runs(port, cuda):
    """Run every config on the device, then queue all oracle jobs."""
    import torch

    from paper_2407_08608_b200 import api
    pool = ThreadPoolExecutor(max_workers=max(4, len(os.sched_getaffinity(0))))
    out = {}
    for name, (B, H, Hkv, N, D, causal, units) in FWD.items():
        gen = torch.Generator(device="cuda").manual_seed(zlib.crc32(name.encode()))
        q = torch.randn(B, N, H, D, device="cuda", generator=gen).bfloat16()
        k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen).bfloat16()
                for _ in range(2))
        o, lse = api.fwd(q, k, v, causal=causal)
        g, a = H // Hkv, 1 / math.sqrt(D)
        res = []
        for b, h in units:
            qu, ku, vu = _np(q[b, :, h]), _np(k[b, :, h // g]), _np(v[b, :, h // g])
            ex = pool.submit(port.flash_fwd, qu, ku, vu, alpha=a, causal=causal, tile=(128, 128))
            em = pool.submit(port.lowprec_flash_fwd, qu, ku, vu, alpha=a, causal=causal,
                             tile=(128, 128), fmt=O.BF16)
            res.append((b, h, _np(o[b, :, h]), _np(lse[b, h]), ex, em))
        out[name] = res
        del q, k, v, o, lse
    for name, (B, H, Hkv, N, D, causal, units) in BWD.items():
        gen = torch.Generator(device="cuda").manual_seed(zlib.crc32(name.encode()))
        q, do = (torch.randn(B, N, H, D, device="cuda", generator=gen).bfloat16()
                 for _ in range(2))
        k, v = (torch.randn(B, N, Hkv, D, device="cuda", generator=gen).bfloat16()
                for _ in range(2))
        o, lse = api.fwd(q, k, v, causal=causal)
        dq, dk, dv = api.bwd(q, k, v, o, do, lse, causal=causal)
        a = 1 / math.sqrt(D)
        res = []
        for b, h in units:  # Hkv == H here: the unit's K/V head is h
            args = [_np(x[b, :, h]) for x in (q, k, v, do, o)] + [_np(lse[b, h])]
            ex = pool.submit(port.flash_bwd, *args, alpha=a, causal=causal, tile=(128, 128))
            em = pool.submit(port.flash_bwd, *args, alpha=a, causal=causal, tile=(128, 128),
                             fmt=O.BF16)
            res.append((b, h, [_np(x[b, :, h]) for x in (dq, dk, dv)], ex, em))
        out[name] = res
        del q, k, v, do, o, lse, dq, dk, dv
    torch.cuda.empty_cache()
    yield out
    pool.shutdown(wait=True)


@pytest.mark.parametrize("name", list(FWD))
def test_fwd_full_size_against_oracle(runs, name):
    for b, h, o, lse, ex, em in runs[name]:
        ex_o, ex_l, _ = ex.result()
        em_o, _ = em.result()
        e_gpu, e_emu = rmse(o, ex_o), rmse(em_o, ex_o)
        m_gpu, m_emu = maxabs(o, ex_o), maxabs(em_o, ex_o)
        assert e_gpu <= 2 * e_emu + 1e-6, (name, b, h, e_gpu, e_emu)
        assert m_gpu <= 8 * m_emu + 1e-6, (name, b, h, m_gpu, m_emu)
        assert maxabs(lse, ex_l) <= 1e-3, (name, b, h, maxabs(lse, ex_l))


def _rel(x, ref):
    return rmse(x, ref) / max(float(np.sqrt(np.mean(ref ** 2))), 1e-30)


@pytest.mark.parametrize("name", list(BWD))
def test_bwd_full_size_against_oracle(runs, name):
    for b, h, got, ex, em in runs[name]:
        exact, emu = ex.result(), em.result()
        for t, g, e, m in zip(("dq", "dk", "dv"), got, exact, emu):
            r_gpu, r_emu = _rel(g, e), _rel(m, e)
            assert r_gpu <= 2 * r_emu + 1e-5, (name, b, h, t, r_gpu, r_emu)


def test_gpu_baselines_match_reference_lowprec(ref, cuda):
    """report.py's device restatements of the reference's standard-attention
    comparators (lowprec.cpp:46-152) against the reference library itself
    (Ref.baseline_lowprec) on identical inputs, N 1024 d128, outlier inputs.
    Both round O to fp16; the device's fp32 GEMMs and row sums use another
    summation order, so entries may differ by an fp16 ulp: the difference must
    be negligible next to each baseline's own error."""
    import torch

    from paper_2407_08608_b200 import report
    n, d = 1024, 128
    alpha = 1 / math.sqrt(d)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for causal in (False, True):
            q, k, v = (ref.sample_outlier(n, d, ref.substream(17, s)) for s in (1, 2, 3))
            exact, _ = ref.reference_attention(q, k, v, alpha=alpha, causal=causal)
            qd, kd, vd = (torch.from_numpy(x).cuda() for x in (q, k, v))
            for fmt, fn in ((O.FP16, report._fp16_baseline), (O.E4M3, report._fp8_baseline)):
                want, _ = ref.baseline_lowprec(q, k, v, fmt, alpha=alpha, causal=causal)
                got = fn(torch, qd, kd, vd, alpha, causal).cpu().numpy()
                err = rmse(want, exact)
                # (measured on CPU torch: 0.052 / 96-97 % equal for fp16, 0.0007 / 99.8 % e4m3)
                assert rmse(got, want) <= 0.1 * err, (fmt, causal, rmse(got, want), err)
                assert np.mean(got == want) >= 0.9, (fmt, causal, np.mean(got == want))
                assert abs(rmse(got, exact) - err) <= 0.01 * err
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
