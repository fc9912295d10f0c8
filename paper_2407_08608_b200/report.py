"""Reference-compatible reports from the device path.

  python -m paper_2407_08608_b200.report bench [--seqlen N] [--headdim D] [--heads H]
         [--batch B] [--causal] [--backward] [--seed S] [--out FILE]
  python -m paper_2407_08608_b200.report rmse [--seqlen N] [--headdim D] [--trials T]
         [--seed S] [--causal] [--out FILE]

``bench`` writes the reference's ``flashlab.bench.v1`` CSV (proj/tools/cmd_bench.cpp:20-85,
docs/formats.md): the same workload (per (batch, head) unit ``u``, Q/K/V =
sample_gaussian_matrix(N, d, substream(seed + u, 1/2/3)), dO from salt 4), the
same exact closed-form ``flops`` column, and ``wall_seconds`` / ``emulation_gflops``
measured on the fa3b kernels (device time, CUDA events, median of the
repetitions) instead of the FP64 emulation. Two columns are appended:
``tflops`` and ``pct_of_peak`` (of the measured bf16 peak, MEASURED_PEAKS.json).

``rmse`` writes ``flashlab.rmse.v1`` (proj/tools/cmd_rmse.cpp:34-80): per trial the
outlier workload (sample_outlier_matrix, substream(seed + t, 1/2/3)), an FP64
dense forward as ground truth, and the six variants. ``fp16-flash`` and the
three ``fp8-*`` rows run the fa3b kernels (K1 on f16 operands; K5 + K6 with the
Hadamard seed substream(seed + t, 9), 128-row quantization blocks). The
``fp16-baseline`` / ``fp8-baseline`` rows restate the reference's standard
attention comparators (proj/core/src/lowprec.cpp:46-152) as device tensor code
with the same rounding points (fp32 GEMM accumulation, fp16 softmax
intermediates, per-tensor e4m3 operands, global-amax P requantization); the
ground truth is torch float64 on the device. These comparators and the truth
are measurement infrastructure, not the product path.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

from . import inputs

E4M3_MAX = 448.0


def format_double(x: float) -> str:
    """report.cpp:13-17 (%.17g)."""
    return "%.17g" % x


def csv_text(schema: str, columns, rows) -> str:
    """CsvReport::text (report.cpp:27-41)."""
    out = [f"# schema={schema}", ",".join(columns)]
    for r in rows:
        if len(r) != len(columns):
            raise ValueError("csv row width mismatch")
        out.append(",".join(r))
    return "\n".join(out) + "\n"


def resolve_output_path(name: str) -> Path:
    """config.cpp:54-69: relative paths land under $FLASHLAB_OUT_DIR."""
    p = Path(name)
    if not p.is_absolute() and os.environ.get("FLASHLAB_OUT_DIR"):
        p = Path(os.environ["FLASHLAB_OUT_DIR"]) / p
    p.parent.mkdir(parents=True, exist_ok=True)
    return p


def write_report(path: str | None, text: str) -> None:
    if not path:
        sys.stdout.write(text)
        return
    p = resolve_output_path(path)
    p.write_text(text)
    print(f"wrote {p}", file=sys.stderr)


def flops_forward(n, d, h, causal) -> int:
    """flash_fwd.hpp:69-73 (integer halving for causal)."""
    f = 4 * n * n * d * h
    return f // 2 if causal else f


def flops_backward(n, d, h, causal) -> int:
    """flash_fwd.hpp:74-77: 2.5 x forward."""
    return flops_forward(n, d, h, causal) * 5 // 2


def _peak_bf16() -> float:
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["bf16_tflops"])
    except (OSError, ValueError, KeyError):
        return 1590.0


# ------------------------------------------------------------------ bench.v1
def _unit_inputs(seqlen, headdim, batch, heads, seed, salts):
    """[batch, seqlen, heads, headdim] arrays, unit u = b * heads + h (cmd_bench.cpp:29-39)."""
    out = []
    for salt in salts:
        a = np.empty((batch, seqlen, heads, headdim))
        for b in range(batch):
            for h in range(heads):
                u = b * heads + h
                a[b, :, h, :] = inputs.sample_gaussian_matrix(seqlen, headdim,
                                                              inputs.substream(seed + u, salt))
        out.append(a)
    return out


def _device_ms(fn, torch, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def bench_report(seqlen=512, headdim=64, heads=32, batch=1, causal=False, backward=False,
                 seed=1, dtype="bf16", reps=10) -> str:
    import torch

    from . import api
    dev = torch.device("cuda")
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    salts = (1, 2, 3, 4) if backward else (1, 2, 3)
    arrs = _unit_inputs(seqlen, headdim, batch, heads, seed, salts)
    q, k, v, *rest = (torch.from_numpy(a).to(dev).to(tdt) for a in arrs)
    peak = _peak_bf16()
    rows = []

    def emit(pas, flops, seconds):
        rows.append([pas, str(seqlen), str(headdim), str(heads), str(batch), "1" if causal else "0",
                     str(flops), format_double(seconds),
                     format_double(flops / seconds / 1e9 if seconds > 0 else 0.0),
                     format_double(flops / seconds / 1e12), format_double(100 * flops / seconds / 1e12 / peak)])

    o, lse = api.fwd(q, k, v, causal=causal)
    ms = _device_ms(lambda: api.fwd(q, k, v, causal=causal, out=o, lse=lse), torch, reps)
    emit("forward", flops_forward(seqlen, headdim, heads, causal) * batch, ms * 1e-3)
    if backward:
        do = rest[0]
        ws = torch.empty(api.bwd_workspace_bytes(batch, heads, heads, seqlen, headdim),
                         dtype=torch.uint8, device=dev)
        g = [torch.empty_like(x) for x in (q, k, v)]
        ms = _device_ms(lambda: api.bwd(q, k, v, o, do, lse, causal=causal, dq=g[0], dk=g[1],
                                        dv=g[2], workspace=ws), torch, reps)
        emit("backward", flops_backward(seqlen, headdim, heads, causal) * batch, ms * 1e-3)
    cols = ["pass", "seqlen", "headdim", "heads", "batch", "causal", "flops", "wall_seconds",
            "emulation_gflops", "tflops", "pct_of_peak"]
    return csv_text("flashlab.bench.v1", cols, rows)


# ------------------------------------------------------------------- rmse.v1
def _causal_mask(torch, n, dev):
    return torch.ones(n, n, dtype=torch.bool, device=dev).triu(1)


def _truth(torch, q, k, v, alpha, causal):
    """reference_attention_o (attention_ref.cpp:78-89) in float64 on the device."""
    s = (q @ k.T) * alpha
    if causal:
        s = s.masked_fill(_causal_mask(torch, s.shape[0], s.device), -math.inf)
    return torch.softmax(s, -1) @ v


def _round(torch, x, dt):
    return x.to(dt).to(x.dtype)


def _quant_tensor(torch, x):
    """quantize_per_tensor (quantize.cpp:35-60): scale = amax/448 (1 if 0), RNE saturating codes."""
    amax = float(x.abs().max())
    scale = 1.0 if amax == 0.0 else amax / E4M3_MAX
    codes = (x * (1.0 / scale)).clamp(-E4M3_MAX, E4M3_MAX)
    return _round(torch, codes, torch.float8_e4m3fn), scale


def _fp16_baseline(torch, q, k, v, alpha, causal):
    """lowprec.cpp:46-85: fp16 operands, fp32 GEMMs, every softmax intermediate in fp16."""
    f32, f16 = torch.float32, torch.float16
    q16, k16, v16 = (_round(torch, x, f16).to(f32) for x in (q, k, v))
    s = _round(torch, (q16 @ k16.T).double() * alpha, f16)
    if causal:
        s = s.masked_fill(_causal_mask(torch, s.shape[0], s.device), -math.inf)
    p = _round(torch, torch.exp(s - s.max(-1, keepdim=True).values), f16)
    ell = p.to(f32).sum(-1, keepdim=True).double()
    p = _round(torch, p / ell, f16)
    return _round(torch, (p.to(f32) @ v16).double(), f16)


def _fp8_baseline(torch, q, k, v, alpha, causal):
    """lowprec.cpp:92-152: per-tensor e4m3 operands, fp32 S, fp16 softmax, P requantized
    with one global-amax scale, O rounded to fp16."""
    f32, f16 = torch.float32, torch.float16
    qc, sq = _quant_tensor(torch, q)
    kc, sk = _quant_tensor(torch, k)
    vc, sv = _quant_tensor(torch, v)
    s = ((qc.to(f32) @ kc.to(f32).T).double() * (alpha * sq * sk)).to(f32).double()
    if causal:
        s = s.masked_fill(_causal_mask(torch, s.shape[0], s.device), -math.inf)
    p = _round(torch, torch.exp(s - s.max(-1, keepdim=True).values), f16)
    ell = p.to(f32).sum(-1, keepdim=True).double()
    p = _round(torch, p / ell, f16)
    amax = float(p.max())
    sp = 1.0 if amax == 0.0 else amax / E4M3_MAX
    pc = _round(torch, (p / sp).clamp(-E4M3_MAX, E4M3_MAX), torch.float8_e4m3fn)
    return _round(torch, (pc.to(f32) @ vc.to(f32)).double() * (sp * sv), f16)


VARIANTS = ("fp16-baseline", "fp16-flash", "fp8-baseline", "fp8-full", "fp8-no-block",
            "fp8-no-incoherent")


def rmse_rows(seqlen=8192, headdim=128, trials=10, seed=1, causal=False):
    """Per-trial RMSE of every variant against the FP64 truth: {variant: [rmse per trial]}."""
    import torch

    from . import api
    dev = torch.device("cuda")
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    alpha = 1.0 / math.sqrt(headdim)
    series = {v: [] for v in VARIANTS}
    try:
        for t in range(trials):
            base = seed + t
            q, k, v = (torch.from_numpy(inputs.sample_outlier_matrix(
                seqlen, headdim, inputs.substream(base, salt))).to(dev) for salt in (1, 2, 3))
            truth = _truth(torch, q, k, v, alpha, causal)
            q4, k4, v4 = (x[None, :, None, :] for x in (q, k, v))
            outs = {"fp16-baseline": _fp16_baseline(torch, q, k, v, alpha, causal)}
            o16, _ = api.fwd(*(x.half() for x in (q4, k4, v4)), causal=causal, alpha=alpha,
                             out_dtype=torch.float32)
            outs["fp16-flash"] = o16[0, :, 0].double()
            outs["fp8-baseline"] = _fp8_baseline(torch, q, k, v, alpha, causal)
            hseed = inputs.substream(base, 9)
            f32 = [x.float() for x in (q4, k4, v4)]
            for name, pb, inc in (("fp8-full", True, True), ("fp8-no-block", False, True),
                                  ("fp8-no-incoherent", True, False)):
                o8, _ = api.fp8_fwd(*f32, causal=causal, alpha=alpha, per_block=pb, incoherent=inc,
                                    seed=hseed, out_dtype=torch.float32)
                outs[name] = o8[0, :, 0].double()
            for name in VARIANTS:
                series[name].append(float(((outs[name] - truth) ** 2).mean().sqrt()))
            torch.cuda.synchronize()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    return series


def rmse_report(seqlen=8192, headdim=128, trials=10, seed=1, causal=False) -> str:
    series = rmse_rows(seqlen, headdim, trials, seed, causal)
    rows = [[str(t), v, format_double(series[v][t])] for t in range(trials) for v in VARIANTS]
    rows += [["median", v, format_double(float(np.median(series[v])))] for v in VARIANTS]
    return csv_text("flashlab.rmse.v1", ["trial", "variant", "rmse"], rows)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2407_08608_b200.report")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--seqlen", type=int, default=512)
    b.add_argument("--headdim", type=int, default=64)
    b.add_argument("--heads", type=int, default=32)
    b.add_argument("--batch", type=int, default=1)
    b.add_argument("--causal", action="store_true")
    b.add_argument("--backward", action="store_true")
    b.add_argument("--dtype", choices=("bf16", "f16"), default="bf16")
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--out", default="")
    r = sub.add_parser("rmse")
    r.add_argument("--seqlen", type=int, default=8192)
    r.add_argument("--headdim", type=int, default=128)
    r.add_argument("--trials", type=int, default=10)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--causal", action="store_true")
    r.add_argument("--out", default="")
    a = ap.parse_args(argv)
    if a.cmd == "bench":
        text = bench_report(a.seqlen, a.headdim, a.heads, a.batch, a.causal, a.backward, a.seed,
                            a.dtype)
    else:
        text = rmse_report(a.seqlen, a.headdim, a.trials, a.seed, a.causal)
    write_report(a.out, text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
