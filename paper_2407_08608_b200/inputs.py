"""Synthetic workloads of the reference, vectorised with numpy.

The reference draws every input from a counter-based splitmix64 stream
(proj/core/src/rng.cpp): ``word(seed, c) = mix64(seed + (c + 1) * gamma)``
(:25-27), ``substream(seed, salt) = mix64(seed ^ mix64(salt + gamma))``
(:21-23), Box-Muller Gaussians from words 2c, 2c+1 (:37-48) and the outlier
mixture N(0,1) + 10 N(0,1) Bern(p) from five words per entry (:50-71). These
are pure functions of (seed, index), so the device tools here regenerate the
reference's own Q/K/V/dO (bench.v1 and rmse.v1 reports) instead of random
tensors. Integer arithmetic is exact (uint64 wrap-around); log/cos come from
numpy, so values agree with libm to the last ulp or so (pinned against the
oracle in tests/test_inputs.py).
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_PI = 2.0 * np.pi


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def substream(seed: int, salt: int) -> int:
    """rng.cpp:21-23"""
    with np.errstate(over="ignore"):
        inner = _mix64(np.uint64(salt) + _GAMMA)
    return int(_mix64(np.uint64(seed) ^ inner))


def _words(seed: int, c):
    with np.errstate(over="ignore"):
        return _mix64(np.uint64(seed) + (c + np.uint64(1)) * _GAMMA)


def _uniform(seed, c):      # rng.cpp:29-31, [0, 1)
    return (_words(seed, c) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def _uniform_pos(seed, c):  # rng.cpp:33-35, (0, 1]
    return ((_words(seed, c) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def sample_gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """rng.cpp:43-48: entry e = Box-Muller of words 2e, 2e+1; FP64 [rows, cols]."""
    c = np.arange(rows * cols, dtype=np.uint64)
    u1 = _uniform_pos(seed, np.uint64(2) * c)
    u2 = _uniform(seed, np.uint64(2) * c + np.uint64(1))
    return (np.sqrt(-2.0 * np.log(u1)) * np.cos(_TWO_PI * u2)).reshape(rows, cols)


def sample_outlier_matrix(rows: int, cols: int, seed: int, p: float = 0.001) -> np.ndarray:
    """rng.cpp:50-71: N(0,1) + 10 N(0,1) Bern(p), five words per entry."""
    if not 0.0 <= p <= 1.0:
        raise ValueError("sample_outlier_matrix: probability out of range")
    base = np.uint64(5) * np.arange(rows * cols, dtype=np.uint64)
    v = np.sqrt(-2.0 * np.log(_uniform_pos(seed, base))) * np.cos(
        _TWO_PI * _uniform(seed, base + np.uint64(1)))
    hit = _uniform(seed, base + np.uint64(2)) < p
    if hit.any():
        b = base[hit]
        v[hit] += 10.0 * (np.sqrt(-2.0 * np.log(_uniform_pos(seed, b + np.uint64(3)))) *
                          np.cos(_TWO_PI * _uniform(seed, b + np.uint64(4))))
    return v.reshape(rows, cols)


def sample_sign_vector(n: int, seed: int) -> np.ndarray:
    """rng.cpp:73-78: +1 where word(i) is odd, else -1."""
    return np.where(_words(seed, np.arange(n, dtype=np.uint64)) & np.uint64(1), 1.0, -1.0)
