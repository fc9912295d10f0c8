"""Build the in-tree native libraries.

  libfa3b.so           CUDA kernels + C ABI (include/fa3b.h), sm_100a only
  libfa3b_flashlab.so  C++ host mirror of the reference's flashlab API
                       (include/fa3b/flashlab_compat.hpp) over the C ABI
  dropin/              link-level drop-in of flashlab::core built against the
                       reference's own headers, plus the reference's unmodified
                       acceptance_main.cpp linked to it (only where
                       /root/reference exists; the outputs travel)

Both are compiled with nvcc/g++ directly (no JIT cache), so the .so files
travel with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.environ.get("NVCC", f"{CUDA_HOME}/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CUDA_SOURCES = ["fa3b_capi.cu", "fwd16_d64.cu", "fwd16_d128.cu", "fwd16_d256.cu",
                "fwd16_sched_bf16_c0.cu", "fwd16_sched_bf16_c1.cu", "fwd16_sched_f16_c0.cu",
                "fwd16_sched_f16_c1.cu", "fwd_fp8.cu", "fwd_fp8_d64.cu", "fp8_prepare.cu", "bwd.cu"]
COMPAT_SOURCES = ["flashlab_compat.cpp"]


def _digest(paths) -> str:
    h = hashlib.sha256()
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def _inputs():
    files = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.cpp"))
    files += list(CSRC.glob("*.inc"))
    files += list((ROOT / "include").rglob("*.h*"))
    return files


def _run(cmd):
    print("[fa3b build]", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose_ptxas: bool = False) -> Path:
    out = PKG / "libfa3b.so"
    compat = PKG / "libfa3b_flashlab.so"
    stamp = PKG / ".build_stamp"
    digest = _digest(_inputs())
    if (not force and out.exists() and compat.exists() and stamp.exists()
            and stamp.read_text() == digest):
        return out
    # one nvcc per translation unit, in parallel, then one link
    objdir = ROOT / "build" / "obj"
    objdir.mkdir(parents=True, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xcompiler", "-fvisibility=hidden", "-I", str(ROOT / "include")]
    if verbose_ptxas:
        flags.insert(0, "-Xptxas=-v")
    jobs = []
    for name in CUDA_SOURCES:
        src = CSRC / name
        if src.exists():
            jobs.append((src, objdir / (src.stem + ".o")))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        list(ex.map(lambda j: _run([NVCC, *flags, "-c", "-o", str(j[1]), str(j[0])]), jobs))
    _run([NVCC, *ARCH, "-shared", "-Xlinker", "--no-undefined", "-o", str(out),
          *[str(o) for _, o in jobs], "-lcuda"])
    csrcs = [str(CSRC / s) for s in COMPAT_SOURCES if (CSRC / s).exists()]
    if csrcs:
        _run(["g++", "-O2", "-std=c++20", "-Wall", "-fPIC", "-shared", "-I", str(ROOT / "include"),
              "-I", f"{CUDA_HOME}/include", "-o", str(compat), *csrcs, f"-L{PKG}", "-lfa3b",
              f"-L{CUDA_HOME}/lib64", "-lcudart", "-Wl,--no-undefined",
              f"-Wl,-rpath,$ORIGIN:{CUDA_HOME}/lib64"])
    stamp.write_text(digest)
    build_dropin()
    return out


def build_dropin() -> Path | None:
    """The link-level drop-in of flashlab::core (dropin/Makefile): needs the
    reference tree, so it is built here and its outputs travel with the
    snapshot; on a box without /root/reference the prebuilt files are used."""
    root = Path(os.environ.get("FLASHLAB_ROOT", "/root/reference/proj"))
    if not (root / "core" / "include" / "flashlab" / "flash_fwd.hpp").exists():
        return None
    _run(["make", "-s", "-C", str(PKG / "dropin"), f"FLASHLAB_ROOT={root}", "-j8"])
    return PKG / "dropin" / "libflashlab_core_fa3b.so"


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
