"""TEST INFRASTRUCTURE ONLY — numpy front end for the CPU oracle.

Two implementations of the reference algorithms, one head per call, FP64
row-major [n, d] arrays:

  ``Port``  the C restatement in fa3b_oracle.c (always built by build())
  ``Ref``   the reference library itself, compiled from its own sources into
            _ref/libflashlab_ref.so (present when /root/reference was
            available at build time; the .so travels to the GPU box)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this module. The product (paper_2407_08608_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "_build" / "libfa3b_oracle.so"
REF_LIB = HERE / "_ref" / "libflashlab_ref.so"
REF_SIM = HERE / "_ref" / "flashlab_sim"
REF_SRC = Path(os.environ.get("FLASHLAB_REF_DIR", "/root/reference/proj/core"))

FP64, FP32, FP16, BF16, E4M3 = 0, 1, 2, 3, 4

_D = ctypes.POINTER(ctypes.c_double)
_U64P = ctypes.POINTER(ctypes.c_uint64)
_SZ = ctypes.c_size_t
_U64 = ctypes.c_uint64
_I = ctypes.c_int
_DBL = ctypes.c_double


def build(quiet: bool = True) -> None:
    """make the port (always) and the reference (when its sources exist)."""
    targets = ["oracle"]
    if (REF_SRC / "src" / "flash_fwd.cpp").exists():
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), f"-j{os.cpu_count() or 4}", *targets],
                   check=True, stdout=subprocess.DEVNULL if quiet else None)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _shapes(q, k, v):
    """validate_inputs (attention_ref.cpp:20-29) for the shape cases the C
    entry points cannot see (they take a single n and d)."""
    q, k, v = _c(q), _c(k), _c(v)
    if q.ndim != 2 or q.size == 0:
        raise OracleError("attention: empty inputs")
    if q.shape[1] != k.shape[1] or k.shape[1] != v.shape[1]:
        raise OracleError("attention: head dimension mismatch")
    if q.shape[0] != k.shape[0] or k.shape[0] != v.shape[0]:
        raise OracleError("attention: sequence length mismatch")
    return q, k, v


class OracleError(ValueError):
    pass


class _Base:
    prefix = ""

    def __init__(self, path: Path, err_fn: str):
        if not path.exists():
            build()
        if not path.exists():
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(str(path))
        self._err = getattr(self.lib, err_fn)
        self._err.restype = ctypes.c_char_p

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(self._err().decode())

    def fn(self, name, argtypes, restype=_I):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f


class Port(_Base):
    """The C restatement (oracle/fa3b_oracle.c)."""

    prefix = "orc_"

    def __init__(self):
        super().__init__(PORT_LIB, "fa3b_oracle_last_error")

    def substream(self, seed, salt):
        return int(self.fn("substream", [_U64, _U64], _U64)(seed, salt))

    def word(self, seed, c):
        return int(self.fn("word", [_U64, _U64], _U64)(seed, c))

    def sample_gaussian(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self.fn("sample_gaussian", [_SZ, _SZ, _U64, _D], None)(rows, cols, seed, _dp(out))
        return out

    def sample_outlier(self, rows, cols, seed, p=0.001):
        out = np.empty((rows, cols))
        self._check(self.fn("sample_outlier", [_SZ, _SZ, _U64, _DBL, _D])(rows, cols, seed, p,
                                                                          _dp(out)))
        return out

    def sign_vector(self, n, seed):
        out = np.empty(n)
        self.fn("sign_vector", [_SZ, _U64, _D], None)(n, seed, _dp(out))
        return out

    def round_to(self, x, fmt, overflow_infinite=False):
        f = self.fn("round_to", [_DBL, _I, _I], _DBL)
        return float(f(float(x), fmt, int(overflow_infinite)))

    def round_array(self, a, fmt):
        a = _c(a)
        out = np.empty_like(a)
        self.fn("round_array", [_D, _SZ, _I, _D], None)(_dp(a), a.size, fmt, _dp(out))
        return out

    def fwht(self, v):
        v = _c(v).copy()
        self._check(self.fn("fwht", [_D, _SZ])(_dp(v), v.size))
        return v

    def preprocess_incoherent(self, q, k, seed):
        q, k = _c(q), _c(k)
        qo, ko = np.empty_like(q), np.empty_like(k)
        n, d = q.shape
        self._check(self.fn("preprocess_incoherent", [_D, _D, _SZ, _SZ, _U64, _D, _D])(
            _dp(q), _dp(k), n, d, seed, _dp(qo), _dp(ko)))
        return qo, ko

    def quantize(self, m, block_rows=0, overflow_infinite=False):
        m = _c(m)
        rows, cols = m.shape
        nb = 1 if block_rows == 0 else -(-rows // block_rows)
        codes, scales = np.empty_like(m), np.empty(nb)
        self._check(self.fn("quantize", [_D, _SZ, _SZ, _SZ, _I, _D, _D])(
            _dp(m), rows, cols, block_rows, int(overflow_infinite), _dp(codes), _dp(scales)))
        return codes, scales

    def flash_fwd(self, q, k, v, alpha=None, causal=False, tile=(64, 64)):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        vis, skip = _U64(0), _U64(0)
        self._check(self.fn("flash_fwd", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _SZ, _SZ, _D, _D,
                                          _U64P, _U64P])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), tile[0], tile[1], _dp(o),
            _dp(lse), ctypes.byref(vis), ctypes.byref(skip)))
        return o, lse, {"blocks_visited": vis.value, "blocks_skipped": skip.value}

    def reference_attention(self, q, k, v, alpha=None, causal=False):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("reference_attention", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _D, _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), _dp(o), _dp(lse)))
        return o, lse

    def bwd_preprocess(self, dO, o):
        dO, o = _c(dO), _c(o)
        out = np.empty(dO.shape[0])
        self._check(self.fn("bwd_preprocess", [_D, _D, _SZ, _SZ, _D])(
            _dp(dO), _dp(o), dO.shape[0], dO.shape[1], _dp(out)))
        return out

    def flash_bwd(self, q, k, v, dO, o, lse, alpha=None, causal=False, tile=(64, 64), fmt=FP64):
        q, k, v, dO, o, lse = map(_c, (q, k, v, dO, o, lse))
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        dq, dk, dv = np.empty_like(q), np.empty_like(q), np.empty_like(q)
        args = [_dp(q), _dp(k), _dp(v), _dp(dO), _dp(o), _dp(lse), n, d, alpha, int(causal),
                tile[0], tile[1]]
        types = [_D] * 6 + [_SZ, _SZ, _DBL, _I, _SZ, _SZ]
        if fmt == FP64:
            f = self.fn("flash_bwd", types + [_D, _D, _D])
            self._check(f(*args, _dp(dq), _dp(dk), _dp(dv)))
        else:
            f = self.fn("lowprec_flash_bwd", types + [_I, _D, _D, _D])
            self._check(f(*args, fmt, _dp(dq), _dp(dk), _dp(dv)))
        return dq, dk, dv

    def lowprec_flash_fwd(self, q, k, v, alpha=None, causal=False, tile=(128, 128), fmt=BF16):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("lowprec_flash_fwd", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _SZ, _SZ, _I,
                                                  _D, _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), tile[0], tile[1], fmt, _dp(o),
            _dp(lse)))
        return o, lse

    def fp8_flash_fwd(self, q, k, v, alpha=None, causal=False, per_block=True, incoherent=True,
                      seed=0, tile=(64, 64)):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("fp8_flash_fwd", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _I, _I, _U64, _SZ,
                                              _SZ, _D, _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), int(per_block), int(incoherent),
            seed, tile[0], tile[1], _dp(o), _dp(lse)))
        return o, lse


class Ref(_Base):
    """The reference library itself (oracle/_ref/libflashlab_ref.so)."""

    prefix = "flref_"

    def __init__(self):
        super().__init__(REF_LIB, "flref_last_error")

    @staticmethod
    def available() -> bool:
        if not REF_LIB.exists() and (REF_SRC / "src" / "flash_fwd.cpp").exists():
            build()
        return REF_LIB.exists()

    def substream(self, seed, salt):
        return int(self.fn("substream", [_U64, _U64], _U64)(seed, salt))

    def word(self, seed, c):
        return int(self.fn("word", [_U64, _U64], _U64)(seed, c))

    def sample_gaussian(self, rows, cols, seed):
        out = np.empty((rows, cols))
        self._check(self.fn("sample_gaussian", [_SZ, _SZ, _U64, _D])(rows, cols, seed, _dp(out)))
        return out

    def sample_outlier(self, rows, cols, seed, p=0.001):
        out = np.empty((rows, cols))
        self._check(self.fn("sample_outlier", [_SZ, _SZ, _U64, _DBL, _D])(rows, cols, seed, p,
                                                                          _dp(out)))
        return out

    def sign_vector(self, n, seed):
        out = np.empty(n)
        self._check(self.fn("sign_vector", [_SZ, _U64, _D])(n, seed, _dp(out)))
        return out


    def round_to(self, x, fmt, overflow_infinite=False):
        return float(self.fn("round_to", [_DBL, _I, _I], _DBL)(float(x), fmt,
                                                              int(overflow_infinite)))

    def round_array(self, a, fmt):
        a = _c(a)
        out = np.empty_like(a)
        self.fn("round_array", [_D, _SZ, _I, _D])(_dp(a), a.size, fmt, _dp(out))
        return out

    def flops_forward(self, n, d, h, causal):
        return int(self.fn("flops_forward", [_U64, _U64, _U64, _I], _U64)(n, d, h, int(causal)))

    def flops_backward(self, n, d, h, causal):
        return int(self.fn("flops_backward", [_U64, _U64, _U64, _I], _U64)(n, d, h, int(causal)))

    def gqa_head_map(self, heads, kv_heads):
        out = (ctypes.c_uint64 * max(heads, 1))()
        self._check(self.fn("gqa_head_map", [_SZ, _SZ, _U64P])(heads, kv_heads, out))
        return [int(x) for x in out[:heads]]

    def fwht(self, v):
        v = _c(v).copy()
        self._check(self.fn("fwht", [_D, _SZ])(_dp(v), v.size))
        return v

    def preprocess_incoherent(self, q, k, seed):
        q, k = _c(q), _c(k)
        qo, ko = np.empty_like(q), np.empty_like(k)
        self._check(self.fn("preprocess_incoherent", [_D, _D, _SZ, _SZ, _U64, _D, _D])(
            _dp(q), _dp(k), q.shape[0], q.shape[1], seed, _dp(qo), _dp(ko)))
        return qo, ko

    def quantize(self, m, block_rows=0, overflow_infinite=False):
        m = _c(m)
        rows, cols = m.shape
        nb = 1 if block_rows == 0 else -(-rows // block_rows)
        codes, scales = np.empty_like(m), np.empty(nb)
        self._check(self.fn("quantize", [_D, _SZ, _SZ, _SZ, _I, _D, _D])(
            _dp(m), rows, cols, block_rows, int(overflow_infinite), _dp(codes), _dp(scales)))
        return codes, scales

    def flash_fwd(self, q, k, v, alpha=None, causal=False, tile=(64, 64), schedule=0):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        st = (ctypes.c_uint64 * 6)()
        self._check(self.fn("flash_fwd", [_I, _D, _D, _D, _SZ, _SZ, _DBL, _I, _SZ, _SZ, _D, _D,
                                          _U64P])(
            schedule, _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), tile[0], tile[1], _dp(o),
            _dp(lse), st))
        keys = ("blocks_visited", "blocks_skipped", "max_pending_scores", "max_live_probs",
                "deferred_output_scale", "fell_back_to_basic")
        return o, lse, dict(zip(keys, (int(x) for x in st)))

    def reference_attention(self, q, k, v, alpha=None, causal=False):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("reference_attention", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _D, _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), _dp(o), _dp(lse)))
        return o, lse

    def std_attention_bwd(self, q, k, v, dO, alpha=None, causal=False):
        q, k, v, dO = map(_c, (q, k, v, dO))
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        dq, dk, dv = np.empty_like(q), np.empty_like(q), np.empty_like(q)
        self._check(self.fn("std_attention_bwd", [_D, _D, _D, _D, _SZ, _SZ, _DBL, _I, _D, _D,
                                                  _D])(
            _dp(q), _dp(k), _dp(v), _dp(dO), n, d, alpha, int(causal), _dp(dq), _dp(dk),
            _dp(dv)))
        return dq, dk, dv

    def bwd_preprocess(self, dO, o):
        dO, o = _c(dO), _c(o)
        out = np.empty(dO.shape[0])
        self._check(self.fn("bwd_preprocess", [_D, _D, _SZ, _SZ, _D])(
            _dp(dO), _dp(o), dO.shape[0], dO.shape[1], _dp(out)))
        return out

    def flash_bwd(self, q, k, v, dO, o, lse, alpha=None, causal=False, tile=(64, 64)):
        q, k, v, dO, o, lse = map(_c, (q, k, v, dO, o, lse))
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        dq, dk, dv = np.empty_like(q), np.empty_like(q), np.empty_like(q)
        self._check(self.fn("flash_bwd", [_D] * 6 + [_SZ, _SZ, _DBL, _I, _SZ, _SZ, _D, _D, _D])(
            _dp(q), _dp(k), _dp(v), _dp(dO), _dp(o), _dp(lse), n, d, alpha, int(causal),
            tile[0], tile[1], _dp(dq), _dp(dk), _dp(dv)))
        return dq, dk, dv

    def fp8_flash_fwd(self, q, k, v, alpha=None, causal=False, per_block=True, incoherent=True,
                      seed=0, tile=(64, 64), permuted=False):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("fp8_flash_fwd", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _I, _I, _U64, _SZ,
                                              _SZ, _I, _D, _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), int(per_block), int(incoherent),
            seed, tile[0], tile[1], int(permuted), _dp(o), _dp(lse)))
        return o, lse

    def baseline_lowprec(self, q, k, v, fmt, alpha=None, causal=False, block_rows=128):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("baseline_lowprec", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _I, _SZ, _D,
                                                 _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), fmt, block_rows, _dp(o), _dp(lse)))
        return o, lse

    def fp16_flash_fwd(self, q, k, v, alpha=None, causal=False, tile=(128, 128)):
        q, k, v = _shapes(q, k, v)
        n, d = q.shape
        alpha = 1.0 / np.sqrt(d) if alpha is None else alpha
        o, lse = np.empty_like(q), np.empty(n)
        self._check(self.fn("fp16_flash_fwd", [_D, _D, _D, _SZ, _SZ, _DBL, _I, _SZ, _SZ, _D,
                                               _D])(
            _dp(q), _dp(k), _dp(v), n, d, alpha, int(causal), tile[0], tile[1], _dp(o),
            _dp(lse)))
        return o, lse

    def accumulator_permutation(self, width):
        out = (ctypes.c_uint64 * max(width, 1))()
        self._check(self.fn("accumulator_permutation", [_SZ, _U64P])(width, out))
        return [int(x) for x in out[:width]]


def simulate(model_path, *, seqlen=8192, headdim=128, block_rows=128, block_cols=128,
             backward=False, fp8=False, schedule="pingpong+2stage") -> dict:
    """The reference's discrete-event schedule model (pipeline_sim.hpp) run by
    _ref/flashlab_sim (a subprocess: the simulator's iostream code and numpy's
    runtime libraries do not share one process)."""
    if not REF_SIM.exists():
        build()
    args = [str(REF_SIM), str(model_path), str(seqlen), str(headdim), str(block_rows),
            str(block_cols), str(int(backward)), str(int(fp8)), schedule]
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        raise OracleError(r.stderr.strip() or r.stdout.strip())
    import json
    return json.loads(r.stdout)
