"""Pin the CPU oracle (oracle/fa3b_oracle.c) before trusting it.

Three anchors, in order of authority:
  1. the reference library itself run here (oracle/_ref, built from
     /root/reference) — bit-exact agreement on random inputs;
  2. tests/golden/golden_ref.npz, outputs of that same library committed so the
     check also runs where /root/reference is absent — bit-exact;
  3. the known-answer values the reference's own unit tests assert
     (proj/tests/test_*.cpp), restated here with their file:line.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O

LN2 = math.log(2.0)


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


# ------------------------------------------------------------------ golden
def test_rng_matches_golden(port, golden):
    assert port.substream(902, 1) == int(golden["rng_substream_902_1"][0])
    assert [port.word(7, c) for c in range(16)] == [int(x) for x in golden["rng_words_seed7"]]
    assert _eq(port.sample_gaussian(4, 4, 11), golden["rng_gauss_4x4_seed11"])
    assert _eq(port.sample_outlier(8, 8, 12), golden["rng_outlier_8x8_seed12"])
    assert _eq(port.sign_vector(16, 5), golden["rng_signs_16_seed5"])


@pytest.mark.parametrize("name,fmt", [("fp32", O.FP32), ("fp16", O.FP16), ("bf16", O.BF16),
                                      ("e4m3", O.E4M3)])
def test_round_to_matches_golden(port, golden, name, fmt):
    assert _eq(port.round_array(golden["round_x"], fmt), golden[f"round_{name}"])


def test_quantize_matches_golden(port, golden):
    c, s = port.quantize(golden["quant_in"], 8)
    assert _eq(c, golden["quant_b8_codes"]) and _eq(s, golden["quant_b8_scales"])
    c, s = port.quantize(golden["quant_in"], 0)
    assert _eq(c, golden["quant_pt_codes"]) and _eq(s, golden["quant_pt_scales"])


def test_hadamard_matches_golden(port, golden):
    qo, ko = port.preprocess_incoherent(golden["had_q"], golden["had_k"], 23)
    assert _eq(qo, golden["had_qo"]) and _eq(ko, golden["had_ko"])


@pytest.mark.parametrize("name", ["fwd_n100_d16_causal", "fwd_n64_d32"])
def test_fwd_bwd_match_golden(port, golden, name):
    n, d, causal, br, bc = (int(x) for x in golden[f"{name}_meta"])
    q, k, v, do = (golden[f"{name}_{x}"] for x in ("q", "k", "v", "do"))
    o, lse, st = port.flash_fwd(q, k, v, causal=bool(causal), tile=(br, bc))
    assert _eq(o, golden[f"{name}_o"]) and _eq(lse, golden[f"{name}_lse"])
    assert [st["blocks_visited"], st["blocks_skipped"]] == list(golden[f"{name}_stats"])
    dq, dk, dv = port.flash_bwd(q, k, v, do, o, lse, causal=bool(causal), tile=(br, bc))
    assert _eq(dq, golden[f"{name}_dq"]) and _eq(dk, golden[f"{name}_dk"])
    assert _eq(dv, golden[f"{name}_dv"])


def test_fp8_matches_golden(port, golden):
    q, k, v = golden["fp8_q"], golden["fp8_k"], golden["fp8_v"]
    for pb in (0, 1):
        for inc in (0, 1):
            for c in (0, 1):
                o, lse = port.fp8_flash_fwd(q, k, v, causal=bool(c), per_block=bool(pb),
                                            incoherent=bool(inc), seed=77, tile=(32, 32))
                assert _eq(o, golden[f"fp8_o_pb{pb}_inc{inc}_c{c}"]), (pb, inc, c)
                assert _eq(lse, golden[f"fp8_lse_pb{pb}_inc{inc}_c{c}"]), (pb, inc, c)


def test_lowprec_fp16_matches_golden(port, golden):
    o, lse = port.lowprec_flash_fwd(golden["fp8_q"], golden["fp8_k"], golden["fp8_v"],
                                    tile=(32, 32), fmt=O.FP16)
    assert _eq(o, golden["fp16_flash_o"]) and _eq(lse, golden["fp16_flash_lse"])


def test_device_cases_consistent(port, golden):
    # The device-shaped golden cases (fp32-stored) agree with the port.
    for name in ("dev_n200_d64_causal", "dev_n160_d128"):
        n, d, causal, a = golden[f"{name}_meta"]
        q, k, v = (golden[f"{name}_{x}"].astype(np.float64) for x in ("q", "k", "v"))
        o, lse, _ = port.flash_fwd(q, k, v, alpha=float(a), causal=bool(causal), tile=(64, 64))
        assert np.abs(o - golden[f"{name}_o"]).max() < 1e-6
        assert np.abs(lse - golden[f"{name}_lse"]).max() < 1e-5


# ------------------------------------------------------- live reference
@pytest.mark.parametrize("seed", range(6))
def test_port_equals_reference_random_sweep(port, ref, seed):
    """Acceptance criterion 1's generator (acceptance_main.cpp:79-110), shortened."""
    w = ref.word(20260801, seed)
    n = 8 + w % 160
    d = (16, 32, 64)[(w >> 16) % 3]
    tile = ((16, 32, 64)[(w >> 24) % 3], (16, 32, 64)[(w >> 32) % 3])
    causal = seed % 2 == 1
    q, k, v = (ref.sample_gaussian(n, d, ref.substream(40000 + seed, s)) for s in (1, 2, 3))
    do = ref.sample_gaussian(n, d, ref.substream(40000 + seed, 4))
    for sched in (0, 1, 2):
        a = ref.flash_fwd(q, k, v, causal=causal, tile=tile, schedule=sched)
        b = port.flash_fwd(q, k, v, causal=causal, tile=tile)
        assert _eq(a[0], b[0]) and _eq(a[1], b[1])
    ga = ref.flash_bwd(q, k, v, do, a[0], a[1], causal=causal, tile=tile)
    gb = port.flash_bwd(q, k, v, do, a[0], a[1], causal=causal, tile=tile)
    assert all(_eq(x, y) for x, y in zip(ga, gb))
    ra = ref.reference_attention(q, k, v, causal=causal)
    rb = port.reference_attention(q, k, v, causal=causal)
    assert _eq(ra[0], rb[0]) and _eq(ra[1], rb[1])


def test_port_equals_reference_fp8_and_lowprec(port, ref):
    q, k, v = (ref.sample_outlier(130, 64, ref.substream(5, s)) for s in (1, 2, 3))
    for pb in (0, 1):
        a = ref.fp8_flash_fwd(q, k, v, causal=True, per_block=pb, seed=3, tile=(64, 48))
        b = port.fp8_flash_fwd(q, k, v, causal=True, per_block=pb, seed=3, tile=(64, 48))
        assert _eq(a[0], b[0]) and _eq(a[1], b[1])
    a = ref.fp16_flash_fwd(q, k, v, causal=True, tile=(64, 64))
    b = port.lowprec_flash_fwd(q, k, v, causal=True, tile=(64, 64), fmt=O.FP16)
    assert _eq(a[0], b[0]) and _eq(a[1], b[1])


# -------------------------------------------- reference unit-test KATs
def test_online_softmax_hand_values(port):
    """test_flash_fwd.cpp:58-78: [0, ln2] then [ln4]; l = 1.5 then 1.75.

    Expressed as a 1-query attention with alpha = 1, q = [1], keys = the
    scores: block 1 gives LSE ln2 + ln1.5 = ln3, adding block 2 gives ln7."""
    q = np.ones((2, 1))
    k2 = np.array([[0.0], [LN2]])
    v2 = np.array([[1.0], [3.0]])
    o, lse, _ = port.flash_fwd(q, k2, v2, alpha=1.0, tile=(1, 2))
    assert abs(lse[0] - math.log(3.0)) < 1e-15
    assert abs(o[0, 0] - (0.5 * 1 + 1.0 * 3) / 1.5) < 1e-15
    # 3 keys need 3 query rows (N_q = N_k); row 0 sees all keys (non-causal)
    q3 = np.ones((3, 1))
    k3 = np.array([[0.0], [LN2], [math.log(4.0)]])
    v3 = np.array([[1.0], [3.0], [5.0]])
    o, lse, _ = port.flash_fwd(q3, k3, v3, alpha=1.0, tile=(3, 2))
    assert abs(lse[0] - math.log(7.0)) < 1e-15
    assert abs(o[0, 0] - (0.25 * 1 + 0.5 * 3 + 1.0 * 5) / 1.75) < 1e-14


def test_causal_block_skipping_counts(port):
    """test_flash_fwd.cpp:139-150: N128, 32x32 tiles -> 10 visited / 6 skipped."""
    q, k, v = (port.sample_gaussian(128, 16, port.substream(906, s)) for s in (0, 1, 2))
    _, _, st = port.flash_fwd(q, k, v, causal=True, tile=(32, 32))
    assert (st["blocks_visited"], st["blocks_skipped"]) == (10, 6)
    _, _, st = port.flash_fwd(q, k, v, causal=False, tile=(32, 32))
    assert (st["blocks_visited"], st["blocks_skipped"]) == (16, 0)


def test_tiled_matches_dense_and_ragged(port):
    """test_flash_fwd.cpp:106-118: 1e-12 to the dense forward, ragged N=100."""
    for n, d, causal, tile, seed in ((128, 32, False, (32, 32), 902), (128, 32, True, (32, 32), 902),
                                     (100, 16, True, (16, 24), 903)):
        q, k, v = (port.sample_gaussian(n, d, port.substream(seed, s)) for s in (0, 1, 2))
        o, lse, _ = port.flash_fwd(q, k, v, causal=causal, tile=tile)
        ro, rl = port.reference_attention(q, k, v, causal=causal)
        assert np.abs(o - ro).max() <= 1e-12 and np.abs(lse - rl).max() <= 1e-12


def test_flop_counts(golden):
    """test_flash_fwd.cpp:224-230."""
    assert [int(x) for x in golden["flops"]] == [2147483648, 1073741824, 2147483648 * 5 // 2, 4]


def test_bwd_preprocess_hand_values(port):
    """test_flash_bwd.cpp:45-54: D = [32, 3]."""
    d = port.bwd_preprocess(np.array([[1.0, 2, 3], [-1, 0.5, 2]]),
                            np.array([[4.0, 5, 6], [2, 2, 2]]))
    assert list(d) == [32.0, 3.0]


def test_bwd_zero_upstream_and_corrupted_lse(port):
    """test_flash_bwd.cpp:56-66 (zero dO -> zero grads) and :105-119."""
    q, k, v = (port.sample_gaussian(32, 8, port.substream(930, s)) for s in (0, 1, 2))
    o, lse, _ = port.flash_fwd(q, k, v, causal=True, tile=(16, 16))
    g = port.flash_bwd(q, k, v, np.zeros((32, 8)), o, lse, causal=True, tile=(16, 16))
    assert all(not x.any() for x in g)
    do = port.sample_gaussian(32, 8, 936)
    good = port.flash_bwd(q, k, v, do, o, lse, tile=(16, 16))
    bad_lse = lse.copy()
    bad_lse[0] += 0.05
    bad = port.flash_bwd(q, k, v, do, o, bad_lse, tile=(16, 16))
    assert all(np.isfinite(x).all() for x in bad)
    assert max(np.abs(a - b).max() for a, b in zip(good, bad)) > 1e-4


def test_bwd_matches_finite_differences(port):
    """test_flash_bwd.cpp:82-103: central differences, h = 1e-5, tol 1e-6."""
    h = 1e-5
    q, k, v = (port.sample_gaussian(12, 4, port.substream(933, s)) for s in (0, 1, 2))
    w = port.sample_gaussian(12, 4, 934)
    o, lse, _ = port.flash_fwd(q, k, v, causal=True, tile=(4, 8))
    g = port.flash_bwd(q, k, v, w, o, lse, causal=True, tile=(4, 8))

    def loss(qq, kk, vv):
        return float((port.reference_attention(qq, kk, vv, causal=True)[0] * w).sum())

    for which in range(3):
        base = [q, k, v]
        for idx in ((0, 0), (5, 2), (11, 3)):
            up = [x.copy() for x in base]
            dn = [x.copy() for x in base]
            up[which][idx] += h
            dn[which][idx] -= h
            fd = (loss(*up) - loss(*dn)) / (2 * h)
            assert abs(fd - g[which][idx]) < 1e-6


def test_e4m3_spot_values(port):
    """test_formats.cpp:50-68 and :40-48 (ties to even)."""
    r = lambda x: port.round_to(x, O.E4M3)  # noqa: E731
    assert r(1.06) == 1.0 and r(1.07) == 1.125
    assert r(500.0) == 448.0 and r(-500.0) == -448.0 and r(470.0) == 448.0
    assert r(2.0 ** -10) == 0.0 and r(1.2 * 2.0 ** -9) == 2.0 ** -9
    assert r(1.0625) == 1.0 and r(1.1875) == 1.25
    assert math.isnan(r(float("nan")))
    assert port.round_to(500.0, O.E4M3, overflow_infinite=True) == math.inf
    assert port.round_to(460.0, O.E4M3, overflow_infinite=True) == 448.0


def test_fp16_bf16_spot_values(port):
    """test_formats.cpp:80-98."""
    f = lambda x: port.round_to(x, O.FP16)  # noqa: E731
    assert f(65519.0) == 65504.0 and f(65520.0) == 65504.0
    assert f(1.0 + 2.0 ** -11) == 1.0 and f(2.0 ** -25) == 0.0 and f(2.0 ** -24) == 2.0 ** -24
    b = lambda x: port.round_to(x, O.BF16)  # noqa: E731
    assert b(1.0 + 2.0 ** -7) == 1.0 + 2.0 ** -7 and b(1.0 + 2.0 ** -8) == 1.0


def test_quantize_scale_kat(port):
    """test_quantize.cpp:38-44: amax 896 -> scale 2, code -448; zero -> scale 1."""
    c, s = port.quantize(np.array([[1.0, -896.0], [0.25, 3.0]]), 0)
    assert s[0] == 2.0 and c[0, 1] == -448.0
    c, s = port.quantize(np.zeros((3, 3)), 0)
    assert s[0] == 1.0 and not c.any()


def test_hadamard_preserves_scores(port):
    """test_fp8_attention.cpp:46-55: QK^T preserved to 1e-10; odd widths rejected."""
    for d in (64, 128, 256):
        q, k = port.sample_gaussian(32, d, 701 + d), port.sample_gaussian(32, d, 801 + d)
        qp, kp = port.preprocess_incoherent(q, k, 11)
        assert np.abs(q @ k.T - qp @ kp.T).max() <= 1e-10
    with pytest.raises(O.OracleError, match="power of two"):
        port.preprocess_incoherent(np.ones((2, 24)), np.ones((2, 24)), 5)


def test_fp8_outlier_error_bands(port):
    """test_fp8_attention.cpp:118-132: N1024 d128 tile 64, seed 31."""
    q, k, v = (port.sample_outlier(1024, 128, port.substream(718, s)) for s in (1, 2, 3))
    ref_o, _ = port.reference_attention(q, k, v)
    full, _ = port.fp8_flash_fwd(q, k, v, seed=31, tile=(64, 64))
    plain, _ = port.fp8_flash_fwd(q, k, v, seed=31, incoherent=False, tile=(64, 64))
    e_full = np.sqrt(np.mean((full - ref_o) ** 2))
    e_plain = np.sqrt(np.mean((plain - ref_o) ** 2))
    assert e_full < e_plain and 1e-3 < e_full < 2e-2 and e_plain < 6e-2


def test_validation_messages_match_reference(port, ref):
    """attention_ref.cpp:20-29 and flash_fwd.cpp:127-129 wording."""
    one = np.ones((4, 4))
    for call, msg in ((lambda m: m.flash_fwd(one, one, one, alpha=0.0), "alpha must be finite"),
                      (lambda m: m.flash_fwd(one, one, one, alpha=float("inf")), "alpha must be finite"),
                      (lambda m: m.flash_fwd(one, one, one, tile=(0, 4)), "block sizes must be positive")):
        for m in (port, ref):
            with pytest.raises(O.OracleError, match=msg):
                call(m)
    with pytest.raises(O.OracleError, match="sequence length mismatch"):
        port.flash_fwd(one, np.ones((3, 4)), np.ones((3, 4)))
    with pytest.raises(O.OracleError, match="head dimension mismatch"):
        port.flash_fwd(one, np.ones((4, 2)), one)
