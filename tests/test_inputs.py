"""The device tools' workload generator (paper_2407_08608_b200/inputs.py) against
the oracle's restatement of the reference RNG (rng.cpp) and the reference itself."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2407_08608_b200 import inputs


import oracle as O


def _impls(port):
    out = [port]
    if O.Ref.available():
        out.append(O.Ref())
    return out


def test_counter_streams_bit_exact(port):
    for impl in _impls(port):
        for seed, salt in [(0, 1), (7, 9), (2**63 + 5, 4), (123456789, 0)]:
            assert inputs.substream(seed, salt) == impl.substream(seed, salt)
        s = impl.substream(3, 9)
        assert np.array_equal(inputs.sample_sign_vector(257, s), impl.sign_vector(257, s))


@pytest.mark.parametrize("rows,cols,salt", [(1, 1, 1), (37, 64, 2), (128, 128, 3)])
def test_gaussian_and_outlier_match(port, rows, cols, salt):
    for impl in _impls(port):
        seed = impl.substream(11, salt)
        g = inputs.sample_gaussian_matrix(rows, cols, seed)
        np.testing.assert_allclose(g, impl.sample_gaussian(rows, cols, seed), rtol=1e-13, atol=1e-13)
        o = inputs.sample_outlier_matrix(rows, cols, seed, p=0.05)
        np.testing.assert_allclose(o, impl.sample_outlier(rows, cols, seed, p=0.05), rtol=1e-13, atol=1e-13)
    with pytest.raises(ValueError, match="probability out of range"):
        inputs.sample_outlier_matrix(2, 2, 1, p=1.5)
