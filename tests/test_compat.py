"""The C++ mirror of the reference API (include/fa3b/flashlab_compat.hpp),
exercised by a C++ test program in the style of the reference's suites."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_2407_08608_b200"


@pytest.fixture(scope="module")
def compat_exe(tmp_path_factory, fa3b_lib):
    exe = tmp_path_factory.mktemp("compat") / "test_flashlab_compat"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cpp" / "test_flashlab_compat.cpp"), "-o", str(exe),
                    f"-L{PKG}", "-lfa3b_flashlab", "-lfa3b", f"-Wl,-rpath,{PKG}"], check=True)
    return exe


def test_compat_validation_without_device(compat_exe):
    r = subprocess.run([str(compat_exe), "--validation-only"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_compat_on_device(compat_exe, cuda):
    r = subprocess.run([str(compat_exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
