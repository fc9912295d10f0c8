"""Shared fixtures. ``-m gpu`` tests need an sm_100 device and the built
libfa3b.so; everything else runs on CPU (oracle, host logic, ABI surface)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU oracle work")


@pytest.fixture(scope="session")
def port():
    if not O.PORT_LIB.exists():
        O.build()
    return O.Port()


@pytest.fixture(scope="session")
def ref():
    if not O.Ref.available():
        pytest.skip("reference library (oracle/_ref) not built")
    return O.Ref()


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(ROOT / "tests" / "golden" / "golden_ref.npz"))


@pytest.fixture(scope="session")
def fa3b_lib():
    from paper_2407_08608_b200 import _lib, build
    if not _lib.LIB_PATH.exists():
        build.build()
    return _lib.load()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test requested but no CUDA device is visible")
    major, minor = torch.cuda.get_device_capability()
    if (major, minor) != (10, 0):
        pytest.fail(f"fa3b needs sm_100, found sm_{major}{minor}")
    from paper_2407_08608_b200 import build
    build.build()
    return torch.device("cuda:0")
