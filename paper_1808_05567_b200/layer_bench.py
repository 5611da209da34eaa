"""Per-layer benchmark with the reference's CLI, report schema and layer-CSV
ingestion, on the sm_100a engine.

Mirrors `tools/bench.cpp` (flags), `run_benchmark` / `print_report` /
`write_report_json` / `write_report_csv` (`core/src/harness.cpp:100-506`),
`builtin_resnet50` / `parse_layer_csv` (`core/src/layer_table.cpp:11-124`) and
the CFT1 failure dumps (`core/src/tensor_io.cpp:42-61`), so a user of the
reference's `bench` finds the same switches and the same JSON / CSV columns:

    python -m paper_1808_05567_b200.layer_bench --layers resnet50 --minibatch 32 \\
        --iters 10 --pass F --check --fuse relu --out report.json --csv report.csv

Times are device time per execute call (CUDA events on the launch stream,
inputs resident in HBM, plan built outside the timed region as in
`bench_layer`). `--check` compares against PyTorch float64 convolutions of the
same seeded tensors on the GPU (conv2d / conv2d_input / conv2d_weight) with
the reference's own gates (`harness.cpp:30-43`: F/B linf_rel <= 1e-4 and
l2_rel <= 1e-5, U linf_rel <= 1e-4 for fp32; bf16 runs use linf_rel <= 2e-2,
l2_rel <= 1e-2). `--chain` runs the layer list as a fused forward chain
(`run_chain`, `harness.cpp:311-358`).
"""
from __future__ import annotations

import argparse
import csv
import dataclasses
import io
import json
import math
import os
import struct
import sys
from typing import List, Optional

import torch

from . import api as d
from .api import ParseError

# ResNet-50 Table I (layer_table.cpp:11-33): id, C, K, H, W, R, S, stride
RESNET50 = [
    (1, 3, 64, 224, 224, 7, 7, 2), (2, 64, 256, 56, 56, 1, 1, 1), (3, 64, 64, 56, 56, 1, 1, 1),
    (4, 64, 64, 56, 56, 3, 3, 1), (5, 256, 64, 56, 56, 1, 1, 1), (6, 256, 512, 56, 56, 1, 1, 2),
    (7, 256, 128, 56, 56, 1, 1, 2), (8, 128, 128, 28, 28, 3, 3, 1), (9, 128, 512, 28, 28, 1, 1, 1),
    (10, 512, 128, 28, 28, 1, 1, 1), (11, 512, 1024, 28, 28, 1, 1, 2), (12, 512, 256, 28, 28, 1, 1, 2),
    (13, 256, 256, 14, 14, 3, 3, 1), (14, 256, 1024, 14, 14, 1, 1, 1), (15, 1024, 256, 14, 14, 1, 1, 1),
    (16, 1024, 2048, 14, 14, 1, 1, 2), (17, 1024, 512, 14, 14, 1, 1, 2), (18, 512, 512, 7, 7, 3, 3, 1),
    (19, 512, 2048, 7, 7, 1, 1, 1), (20, 2048, 512, 7, 7, 1, 1, 1),
]


@dataclasses.dataclass
class LayerEntry:
    id: int
    spec: d.ConvLayerSpec


def builtin_resnet50(minibatch: int, vlen: int = 16) -> List[LayerEntry]:
    """builtin_resnet50 (layer_table.cpp:62-73)."""
    return [LayerEntry(r[0], d.make_layer_spec(minibatch, *r[1:], vlen)) for r in RESNET50]


def parse_layer_csv(text: str, minibatch: int, vlen: int = 16) -> List[LayerEntry]:
    """parse_layer_csv (layer_table.cpp:76-119): header row starting with 'id',
    rows `id,C,K,H,W,R,S,stride[,pad_h,pad_w]`, '#' comments, blank lines."""
    layers, have_header, line_no = [], False, 0
    for line_no, line in enumerate(io.StringIO(text), start=1):
        if not line.strip() or line.strip().startswith("#"):
            continue
        fields = [f.strip() for f in next(csv.reader([line]))]
        if not have_header:
            if not fields or fields[0] != "id":
                raise ParseError(f"line {line_no}: expected header starting with 'id'")
            have_header = True
            continue
        if len(fields) not in (8, 10):
            raise ParseError(f"line {line_no}: expected 8 or 10 fields, got {len(fields)}")
        try:
            vals = [int(f) for f in fields]
        except ValueError:
            raise ParseError(f"line {line_no}: non-integer field") from None
        try:
            spec = (d.make_layer_spec(minibatch, *vals[1:8], vals[8], vals[9], vlen) if len(vals) == 10
                    else d.make_layer_spec(minibatch, *vals[1:8], vlen))
        except d.Error as e:
            raise ParseError(f"line {line_no}: {e}") from None
        layers.append(LayerEntry(vals[0], spec))
    if not layers:
        raise ParseError(f"line {max(line_no, 1)}: no layer rows found")
    return layers


@dataclasses.dataclass
class LayerReport:
    """LayerReport (harness.hpp:38-56); `blocking` is the sm_100a tile plan."""
    id: int
    spec: d.ConvLayerSpec
    flops: int = 0
    best_ms: float = 0.0
    avg_ms: float = 0.0
    gflops: float = 0.0
    samples: int = 0
    checked: bool = False
    check_ok: bool = True
    norms: Optional[dict] = None
    blocking: Optional[dict] = None
    strategy: Optional[str] = None
    copies: int = 0
    route: Optional[str] = None


@dataclasses.dataclass
class BenchReport:
    layers_source: str
    minibatch: int
    iterations: int
    pass_: str
    dtype: str
    impl: str = "direct"
    threads: int = 1
    seed: int = 42
    per_layer: List[LayerReport] = dataclasses.field(default_factory=list)
    all_ok: bool = True


def error_norms(ref: torch.Tensor, got: torch.Tensor) -> dict:
    """compute_error_norms (norms.cpp:7-25), in float64."""
    r, g = ref.double().flatten(), got.double().flatten()
    diff = (r - g).abs()
    linf_abs, l2_abs = float(diff.max()) if diff.numel() else 0.0, float(diff.norm())
    rmax, rl2 = float(r.abs().max()) if r.numel() else 0.0, float(r.norm())
    return {"linf_abs": linf_abs, "l2_abs": l2_abs, "linf_rel": linf_abs / rmax if rmax > 0 else linf_abs,
            "l2_rel": l2_abs / rl2 if rl2 > 0 else l2_abs}


def write_cft(path: str, t: torch.Tensor) -> None:
    """CFT1 writer (tensor_io.cpp:42-51): magic, u32 dtype (1 = f32), 4 x u64 dims, payload."""
    t = t.detach().float().cpu().contiguous()
    dims = list(t.shape) + [1] * (4 - t.dim())
    with open(path, "wb") as f:
        f.write(b"CFT1" + struct.pack("<I", 1) + struct.pack("<4Q", *dims))
        f.write(t.numpy().tobytes())


def _gates(pass_: str, dtype: str):
    if dtype == "bf16":
        return 2e-2, 1e-2
    return (1e-4, math.inf) if pass_ == "U" else (1e-4, 1e-5)


def _seeded(shape, seed, scale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.rand(shape, generator=g) * 2 - 1) * scale).cuda()


def _timed(fn, iterations: int):
    fn()  # warm-up (also materialises the checked result), time_runs semantics
    torch.cuda.synchronize()
    times = []
    for _ in range(iterations):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    return min(times), sum(times) / len(times)


def bench_layer(entry: LayerEntry, pass_: str, dtype: str, iterations: int, check: bool, fuse: Optional[str],
                seed: int, dump_dir: str = "") -> LayerReport:
    """bench_layer (harness.cpp:100-265) for one pass of one layer."""
    s = entry.spec
    math_ = d.Math.BF16 if dtype == "bf16" else d.Math.F32
    P, Q = d.derive_output_shape(s)
    lseed = seed ^ (entry.id << 32)  # harness.cpp:108
    x = _seeded((s.N, s.C, s.H, s.W), lseed)
    w = _seeded((s.K, s.C, s.R, s.S), lseed + 1, math.sqrt(2.0 / (s.C * s.R * s.S)))
    g = _seeded((s.N, s.K, P, Q), lseed + 2)
    rep = LayerReport(entry.id, s, flops=d.pass_flops(s))
    xb, wb = d.to_blocked_activation(x, s), d.to_blocked_weight(w, s)
    if pass_ == "F":
        op = None
        if fuse == "relu":
            op = d.FusedOp(d.FusedOpKind.RELU)
        elif fuse == "bias_relu":
            op = d.FusedOp(d.FusedOpKind.BIAS_RELU, [0.01 * ((i % 7) - 3) for i in range(s.K)])
        plan = d.make_forward_plan(s, 1, op, None, math_)
        out = d.BlockedActivation(s.N, s.K, P, Q, s.vlen, 0, 0)
        rep.best_ms, rep.avg_ms = _timed(lambda: plan.execute(xb, wb, out), iterations)
        rep.blocking = plan.blocking
        got = d.from_blocked_activation(out)
        if check:
            ref = torch.nn.functional.conv2d(x.double(), w.double(), stride=s.stride, padding=(s.pad_h, s.pad_w))
            if op is not None and op.kind in (d.FusedOpKind.BIAS_ADD, d.FusedOpKind.BIAS_RELU):
                ref = ref + torch.tensor(op.bias, dtype=torch.float64, device=ref.device).view(1, -1, 1, 1)
            if op is not None and op.kind in (d.FusedOpKind.RELU, d.FusedOpKind.BIAS_RELU):
                ref = ref.clamp_min(0)
    elif pass_ == "B":
        ctx = d.prepare_backward(s, wb, 1, None, math_)
        gb = d.to_blocked_activation(g, s.vlen, 0, 0)
        gi = d.BlockedActivation(s.N, s.C, s.H, s.W, s.vlen, 0, 0)
        rep.best_ms, rep.avg_ms = _timed(lambda: ctx.execute(wb, gb, gi), iterations)
        rep.blocking, rep.route = ctx.blocking, d.choose_backward_route(s).name.lower()
        got = d.from_blocked_activation(gi)
        if check:
            ref = torch.nn.grad.conv2d_input((s.N, s.C, s.H, s.W), w.double(), g.double(), stride=s.stride,
                                             padding=(s.pad_h, s.pad_w))
    else:
        plan = d.UpdatePlan(s, None, math_)
        gb = d.to_blocked_activation(g, s.vlen, 0, 0)
        dw = d.BlockedWeight(s.K, s.C, s.R, s.S, s.vlen)
        rep.best_ms, rep.avg_ms = _timed(lambda: plan.execute(xb, gb, dw), iterations)
        rep.blocking = plan.blocking
        rep.copies = plan.splits
        rep.strategy = "copy_reduce" if rep.copies > 1 else "task_parallel"
        got = d.from_blocked_weight(dw)
        if check:
            ref = torch.nn.grad.conv2d_weight(x.double(), (s.K, s.C, s.R, s.S), g.double(), stride=s.stride,
                                              padding=(s.pad_h, s.pad_w))
    rep.samples = iterations
    rep.gflops = rep.flops / (rep.best_ms * 1e-3) / 1e9 if rep.best_ms > 0 else 0.0
    if check:
        rep.checked = True
        rep.norms = error_norms(ref, got)
        lin, l2 = _gates(pass_, dtype)
        rep.check_ok = rep.norms["linf_rel"] <= lin and rep.norms["l2_rel"] <= l2
        if not rep.check_ok and dump_dir:
            os.makedirs(dump_dir, exist_ok=True)
            stem = os.path.join(dump_dir, f"layer{entry.id}_{pass_}")
            write_cft(stem + "_ref.cft", ref)
            write_cft(stem + "_got.cft", got)
    return rep


def run_benchmark(layers: List[LayerEntry], source: str, pass_: str = "F", dtype: str = "f32", iterations: int = 1,
                  check: bool = False, fuse: Optional[str] = None, seed: int = 42, dump_dir: str = "") -> BenchReport:
    """run_benchmark (harness.cpp:280-309)."""
    rep = BenchReport(source, layers[0].spec.N if layers else 0, iterations, pass_, dtype, seed=seed)
    for e in layers:
        lr = bench_layer(e, pass_, dtype, iterations, check, fuse, seed, dump_dir)
        rep.per_layer.append(lr)
        rep.all_ok = rep.all_ok and lr.check_ok
    return rep


def print_report(report: BenchReport, out=sys.stdout) -> None:
    """print_report (harness.cpp:400-432)."""
    out.write(f"# pass={report.pass_} impl={report.impl} dtype={report.dtype} N={report.minibatch} "
              f"threads={report.threads} iters={report.iterations} seed={report.seed}\n")
    out.write(f"{'id':>4}{'C':>6}{'K':>6}{'H':>5}{'W':>5}{'R':>3}{'S':>3}{'str':>4}{'MFLOP':>13}{'best ms':>11}"
              f"{'avg ms':>11}{'GFLOPS':>9}{'check':>8}{'linf_rel':>12}\n")
    for lr in report.per_layer:
        s = lr.spec
        chk = (f"{'ok' if lr.check_ok else 'FAIL':>8}{lr.norms['linf_rel']:>12.2e}" if lr.checked
               else f"{'-':>8}{'-':>12}")
        out.write(f"{lr.id:>4}{s.C:>6}{s.K:>6}{s.H:>5}{s.W:>5}{s.R:>3}{s.S:>3}{s.stride:>4}{lr.flops / 1e6:>13.1f}"
                  f"{lr.best_ms:>11.3f}{lr.avg_ms:>11.3f}{lr.gflops:>9.2f}{chk}\n")


def report_json(report: BenchReport) -> dict:
    """write_report_json (harness.cpp:434-483) field for field, plus the GPU plan."""
    j = {"layers": report.layers_source, "minibatch": report.minibatch, "iterations": report.iterations,
         "pass": report.pass_, "impl": report.impl, "dtype": report.dtype, "threads": report.threads,
         "seed": report.seed, "all_ok": report.all_ok, "results": []}
    for lr in report.per_layer:
        s = lr.spec
        r = {"id": lr.id, "C": s.C, "K": s.K, "H": s.H, "W": s.W, "R": s.R, "S": s.S, "stride": s.stride,
             "pad_h": s.pad_h, "pad_w": s.pad_w, "flops": lr.flops, "best_ms": lr.best_ms, "avg_ms": lr.avg_ms,
             "gflops": lr.gflops, "samples": lr.samples}
        if lr.checked:
            r["check_ok"] = lr.check_ok
            r.update({k: lr.norms[k] for k in ("linf_abs", "l2_abs", "linf_rel", "l2_rel")})
        r["blocking"] = lr.blocking or {}
        if lr.strategy:
            r["strategy"], r["copies"] = lr.strategy, lr.copies
        if lr.route:
            r["route"] = lr.route
        j["results"].append(r)
    return j


def write_report_csv(report: BenchReport, out) -> None:
    """write_report_csv (harness.cpp:485-504)."""
    out.write("id,C,K,H,W,R,S,stride,pad_h,pad_w,flops,best_ms,avg_ms,gflops,check_ok,linf_abs,l2_abs,linf_rel,l2_rel\n")
    for lr in report.per_layer:
        s = lr.spec
        row = [lr.id, s.C, s.K, s.H, s.W, s.R, s.S, s.stride, s.pad_h, s.pad_w, lr.flops, lr.best_ms, lr.avg_ms,
               lr.gflops]
        tail = ([int(lr.check_ok)] + [lr.norms[k] for k in ("linf_abs", "l2_abs", "linf_rel", "l2_rel")]
                if lr.checked else ["", "", "", "", ""])
        out.write(",".join(str(v) for v in row + tail) + "\n")


def run_chain_mode(layers: List[LayerEntry], dtype: str, seed: int, check: bool) -> int:
    """run_chain (harness.cpp:311-358): forward only, each layer's output (ReLU
    fused) feeds the next; checks K_i = C_{i+1} and the spatial chaining."""
    math_ = d.Math.BF16 if dtype == "bf16" else d.Math.F32
    for a, b in zip(layers, layers[1:]):
        P, Q = d.derive_output_shape(a.spec)
        if a.spec.K != b.spec.C or (P, Q) != (b.spec.H, b.spec.W):
            raise d.ChainShapeMismatch(f"layer {a.id} -> {b.id}: output {a.spec.K}x{P}x{Q} does not feed "
                                       f"{b.spec.C}x{b.spec.H}x{b.spec.W}")
    s0 = layers[0].spec
    x = _seeded((s0.N, s0.C, s0.H, s0.W), seed)
    ws = [_seeded((e.spec.K, e.spec.C, e.spec.R, e.spec.S), seed + 1 + i,
                  math.sqrt(2.0 / (e.spec.C * e.spec.R * e.spec.S))) for i, e in enumerate(layers)]
    cur = d.to_blocked_activation(x, s0)
    relu = d.FusedOp(d.FusedOpKind.RELU)
    for i, e in enumerate(layers):
        nxt = layers[i + 1].spec if i + 1 < len(layers) else None
        plan = d.make_forward_plan(e.spec, 1, relu, None, math_, nxt.pad_h if nxt else 0, nxt.pad_w if nxt else 0)
        cur = d.forward(e.spec, cur, d.to_blocked_weight(ws[i], e.spec), plan)
    out = d.from_blocked_activation(cur)
    print(f"chain of {len(layers)} layers -> output {list(out.shape)}")
    if check:
        ref = x.double()
        for e, w in zip(layers, ws):
            ref = torch.nn.functional.conv2d(ref, w.double(), stride=e.spec.stride,
                                             padding=(e.spec.pad_h, e.spec.pad_w)).clamp_min(0)
        n = error_norms(ref, out)
        lin, _ = _gates("F", dtype)
        print(f"chain check linf_rel={n['linf_rel']:.3e} l2_rel={n['l2_rel']:.3e}")
        if n["linf_rel"] > lin:
            print("chain check FAILED", file=sys.stderr)
            return 1
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="direct convolution layer benchmark (sm_100a engine)")
    ap.add_argument("--layers", default="resnet50", help="builtin table name (resnet50) or layer CSV path")
    ap.add_argument("--minibatch", type=int, default=1)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--pass", dest="pass_", default="F", choices=["F", "B", "U"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"],
                    help="f32 = fp32-accurate tensor-core math; bf16 = bf16 operands (i16 is not on sm_100a)")
    ap.add_argument("--impl", default="direct", choices=["direct"])
    ap.add_argument("--threads", type=int, default=1, help="accepted for compatibility; the GPU ignores it")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--fuse", default="none", choices=["none", "relu", "bias_relu"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--vlen", type=int, default=16)
    ap.add_argument("--out", default="")
    ap.add_argument("--csv", default="")
    ap.add_argument("--dump-dir", default="")
    ap.add_argument("--chain", action="store_true")
    a = ap.parse_args(argv)
    if a.minibatch < 1 or a.iters < 1:
        ap.error("--minibatch and --iters must be positive")
    if a.layers == "resnet50":
        layers = builtin_resnet50(a.minibatch, a.vlen)
    else:
        with open(a.layers) as f:
            layers = parse_layer_csv(f.read(), a.minibatch, a.vlen)
    if a.chain:
        return run_chain_mode(layers, a.dtype, a.seed, a.check)
    rep = run_benchmark(layers, a.layers, a.pass_, a.dtype, a.iters, a.check, None if a.fuse == "none" else a.fuse,
                        a.seed, a.dump_dir)
    rep.threads = a.threads
    print_report(rep)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(report_json(rep), f, indent=2)
    if a.csv:
        with open(a.csv, "w") as f:
            write_report_csv(rep, f)
    return 0 if rep.all_ok else 1


if __name__ == "__main__":
    sys.exit(main())
