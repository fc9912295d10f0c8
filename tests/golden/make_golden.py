"""Generate tests/golden/golden_ref.npz by running the reference library itself
(oracle/_ref, compiled from /root/reference) on small seeded inputs.

Run from the repo root:  python tests/golden/make_golden.py
The fixture is committed; the GPU box (no /root/reference) reads it to pin
the oracle port and to check the CUDA path against the reference directly.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent / "golden_ref.npz"


def main() -> None:
    R = O.Ref()
    g: dict[str, np.ndarray] = {}
    # RNG words and draws (rng.cpp)
    g["rng_substream_902_1"] = np.array([R.substream(902, 1)], dtype=np.uint64)
    g["rng_words_seed7"] = np.array([R.word(7, c) for c in range(16)], dtype=np.uint64)
    g["rng_gauss_4x4_seed11"] = R.sample_gaussian(4, 4, 11)
    g["rng_outlier_8x8_seed12"] = R.sample_outlier(8, 8, 12)
    g["rng_signs_16_seed5"] = R.sign_vector(16, 5)
    # Rounding of a wide sweep (formats.cpp)
    xs = np.concatenate([R.sample_outlier(1, 512, 3)[0] * 37.0,
                         [1.06, 1.07, 500.0, -500.0, 470.0, 2.0 ** -10, 65520.0, 1.0625]])
    g["round_x"] = xs
    for name, f in (("fp32", O.FP32), ("fp16", O.FP16), ("bf16", O.BF16), ("e4m3", O.E4M3)):
        g[f"round_{name}"] = R.round_array(xs, f)
    # Quantization (quantize.cpp)
    m = R.sample_outlier(20, 8, 93)
    g["quant_in"] = m
    g["quant_b8_codes"], g["quant_b8_scales"] = R.quantize(m, 8)
    g["quant_pt_codes"], g["quant_pt_scales"] = R.quantize(m, 0)
    # Hadamard preprocessing (hadamard.cpp, fp8_attention.cpp:33-42)
    qh, kh = R.sample_gaussian(8, 64, 21), R.sample_gaussian(8, 64, 22)
    g["had_q"], g["had_k"] = qh, kh
    g["had_qo"], g["had_ko"] = R.preprocess_incoherent(qh, kh, 23)
    # Forward / backward on small shapes, several tilings (flash_fwd.cpp, flash_bwd.cpp)
    cases = [("fwd_n100_d16_causal", 100, 16, True, (16, 24), 903),
             ("fwd_n64_d32", 64, 32, False, (32, 32), 904)]
    for name, n, d, causal, tile, seed in cases:
        q = R.sample_gaussian(n, d, R.substream(seed, 0))
        k = R.sample_gaussian(n, d, R.substream(seed, 1))
        v = R.sample_gaussian(n, d, R.substream(seed, 2))
        do = R.sample_gaussian(n, d, R.substream(seed, 4))
        o, lse, st = R.flash_fwd(q, k, v, causal=causal, tile=tile)
        dq, dk, dv = R.flash_bwd(q, k, v, do, o, lse, causal=causal, tile=tile)
        g[f"{name}_q"], g[f"{name}_k"], g[f"{name}_v"], g[f"{name}_do"] = q, k, v, do
        g[f"{name}_o"], g[f"{name}_lse"] = o, lse
        g[f"{name}_dq"], g[f"{name}_dk"], g[f"{name}_dv"] = dq, dk, dv
        g[f"{name}_stats"] = np.array([st["blocks_visited"], st["blocks_skipped"]])
        g[f"{name}_meta"] = np.array([n, d, int(causal), tile[0], tile[1]])
    # Device-shaped cases (bf16-rounded inputs, d in {64, 128}): the CUDA path
    # is compared against these reference outputs directly.
    for name, n, d, causal, alpha, seed in (("dev_n200_d64_causal", 200, 64, True, None, 31),
                                            ("dev_n160_d128", 160, 128, False, -0.07, 32)):
        q = R.round_array(R.sample_gaussian(n, d, R.substream(seed, 1)), O.BF16)
        k = R.round_array(R.sample_gaussian(n, d, R.substream(seed, 2)), O.BF16)
        v = R.round_array(R.sample_gaussian(n, d, R.substream(seed, 3)), O.BF16)
        do = R.round_array(R.sample_gaussian(n, d, R.substream(seed, 4)), O.BF16)
        a = (1.0 / np.sqrt(d)) if alpha is None else alpha
        o, lse, _ = R.flash_fwd(q, k, v, alpha=a, causal=causal, tile=(64, 64))
        dq, dk, dv = R.flash_bwd(q, k, v, do, o, lse, alpha=a, causal=causal, tile=(64, 64))
        for key, val in (("q", q), ("k", k), ("v", v), ("do", do), ("o", o), ("lse", lse),
                         ("dq", dq), ("dk", dk), ("dv", dv)):
            # bf16-exact inputs are exact in fp32; outputs are compared with tolerances
            g[f"{name}_{key}"] = np.asarray(val, dtype=np.float32)
        g[f"{name}_meta"] = np.array([n, d, int(causal), a])
    # FP8 forward variants (fp8_attention.cpp), outlier inputs
    q8, k8, v8 = (R.sample_outlier(96, 64, R.substream(720, s)) for s in (1, 2, 3))
    g["fp8_q"], g["fp8_k"], g["fp8_v"] = q8, k8, v8
    for pb in (0, 1):
        for inc in (0, 1):
            for causal in (0, 1):
                o, lse = R.fp8_flash_fwd(q8, k8, v8, causal=causal, per_block=pb, incoherent=inc,
                                         seed=77, tile=(32, 32))
                g[f"fp8_o_pb{pb}_inc{inc}_c{causal}"] = o
                g[f"fp8_lse_pb{pb}_inc{inc}_c{causal}"] = lse
    # Low-precision comparators (lowprec.cpp)
    g["fp16_flash_o"], g["fp16_flash_lse"] = R.fp16_flash_fwd(q8, k8, v8, tile=(32, 32))
    g["base_fp16_o"], _ = R.baseline_lowprec(q8, k8, v8, O.FP16)
    g["base_fp8_o"], _ = R.baseline_lowprec(q8, k8, v8, O.E4M3)
    g["flops"] = np.array([R.flops_forward(512, 64, 32, False), R.flops_forward(512, 64, 32, True),
                           R.flops_backward(512, 64, 32, False), R.flops_forward(1, 1, 1, False)],
                          dtype=np.uint64)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
