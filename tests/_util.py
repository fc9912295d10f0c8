"""Helpers shared by the GPU parity tests: seeded inputs from the reference's
counter RNG (rng.cpp), laid out [batch, seq, head, dim], and per-unit oracle
runs. The oracle is the checker here, never the thing measured."""
from __future__ import annotations

import numpy as np

import oracle as O

FMT = {"bf16": O.BF16, "fp16": O.FP16}


def unit_seed(seed: int, b: int, h: int, heads: int) -> int:
    return seed + b * heads + h


def make_inputs(port, B, H, Hkv, N, D, seed, fmt="bf16", outlier=False, with_do=False):
    """FP64 arrays [B, N, H(kv), D] already rounded to fmt (exact in fmt)."""
    sample = port.sample_outlier if outlier else port.sample_gaussian
    f = FMT[fmt]
    q = np.empty((B, N, H, D))
    k = np.empty((B, N, Hkv, D))
    v = np.empty((B, N, Hkv, D))
    do = np.empty((B, N, H, D)) if with_do else None
    for b in range(B):
        for h in range(H):
            s = unit_seed(seed, b, h, H)
            q[b, :, h] = port.round_array(sample(N, D, port.substream(s, 1)), f)
            if with_do:
                do[b, :, h] = port.round_array(sample(N, D, port.substream(s, 4)), f)
        for h in range(Hkv):
            s = unit_seed(seed, b, h, Hkv) + 7919
            k[b, :, h] = port.round_array(sample(N, D, port.substream(s, 2)), f)
            v[b, :, h] = port.round_array(sample(N, D, port.substream(s, 3)), f)
    return (q, k, v, do) if with_do else (q, k, v)


def to_dev(x, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda").to(dtype)


def rmse(a, b):
    return float(np.sqrt(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2)))


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))
