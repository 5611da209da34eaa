#!/usr/bin/env python3
"""bench.py — the driver's benchmark contract for dconv-b200.

Default workload (BASELINE.json configs[3], the config the metric's images/s at
1/2/4/8 GPUs is quoted on, and the largest single-GPU configuration): the
ResNet-50 v1 conv stack, 53 convs, forward + backward-data + weight-update with
ReLU / residual adds fused, stem max-pool, SGD, bf16 activations and weights
(fp32 master weights and gradients, fp32 accumulate), global minibatch 256
sharded over the ranks, NCCL all-reduce of the weight gradients inside the
step. Seeded synthetic inputs (splitmix64 uniform images and top
gradient, He-normal weights). One step = one training step of the whole
global minibatch; the step runs as ONE CUDA graph (native executor capture).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload resnet50|layer]

value  : whole-job images/s = global batch / max-over-ranks device time per step.
e2e    : the same through the executor's public calls with the images copied
         H2D from pinned host memory every step and the loss read back.
Extra objects on rank 0 at N=1: `layers` (per-conv F/B/U device times and the
roofline of the dominant kernel), `cfg2` (BASELINE configs[1]: the 1x1
bottleneck F+B+U in fp32-accurate math, GFLOP/s and HBM roofline) and `cfg5`
(BASELINE configs[4]: the Inception-v3 layer mix at N=128, bf16).
--gpus N with no torchrun environment re-launches itself as N NCCL ranks.
--impl reference: the reference's own CPU direct engine (oracle/_ref, built
from /root/reference sources with its Release flags) on all host cores, same
metric, on a bounded sample (2 images through every distinct conv).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv GFLOP/s per layer (fwd/bwd/upd) and conv-stack images/s at 1/2/4/8 B200"
CFG2 = dict(N=32, C=256, K=64, H=56, W=56, R=1, S=1, stride=1, pad_h=0, pad_w=0)
# BASELINE configs[4]: (C, K, H, W, R, S, stride, pad_h, pad_w), N = 128
CFG5 = [
    (192, 64, 35, 35, 1, 1, 1, 0, 0), (768, 192, 17, 17, 1, 1, 1, 0, 0), (1280, 320, 8, 8, 1, 1, 1, 0, 0),
    (160, 160, 17, 17, 1, 7, 1, 0, 3), (160, 160, 17, 17, 7, 1, 1, 3, 0), (192, 192, 17, 17, 1, 7, 1, 0, 3),
    (192, 192, 17, 17, 7, 1, 1, 3, 0), (288, 384, 35, 35, 3, 3, 2, 0, 0), (384, 384, 8, 8, 1, 3, 1, 0, 1),
    (384, 384, 8, 8, 3, 1, 1, 1, 0),
]


def measured_peaks():
    """(HBM GB/s, bf16 dense TF/s burst, sustained, source)"""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), \
            "measured (MEASURED_PEAKS.json)"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, 1590.0, "fallback (B200_PROFILING.md)"


def out_shape(w):
    P = (w["H"] + 2 * w["pad_h"] - w["R"]) // w["stride"] + 1
    Q = (w["W"] + 2 * w["pad_w"] - w["S"]) // w["stride"] + 1
    return P, Q


def pass_flops(w):
    """harness.cpp:269-272, logical C"""
    P, Q = out_shape(w)
    return 2 * w["N"] * w["K"] * w["C"] * P * Q * w["R"] * w["S"]


def alg_bytes(w, e_in=4, e_out=4):
    """SURVEY.md 8(d) compulsory bytes per pass (halos not counted; stored channels)."""
    N, C, K, H, W, R, S = (w[k] for k in ("N", "C", "K", "H", "W", "R", "S"))
    st = w["stride"]
    P, Q = out_shape(w)
    Cp = -(-C // 16) * 16
    Kp = -(-K // 16) * 16
    touched = N * Cp * P * Q if (R == 1 and S == 1 and st > 1) else N * Cp * H * W
    fwd = e_in * (touched + Kp * Cp * R * S) + e_out * N * Kp * P * Q
    bwd = e_in * (N * Kp * P * Q + Kp * Cp * R * S) + e_out * N * Cp * H * W
    upd = e_in * (touched + N * Kp * P * Q) + 4 * Kp * Cp * R * S
    return {"F": fwd, "B": bwd, "U": upd}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the GPU is busy."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x80: "hw_power_brake",
               0x100: "display_clocks_setting"}

    def __init__(self, index=0):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001  (no NVML: report nothing rather than guess)
            self.nv = None

    def _sample(self):
        try:
            mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append(mhz)
            for bit, name in self.REASONS.items():
                if mask & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self._stop.clear()
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()
            self._t = None

    def report(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def ncu_traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch from the committed
    ncu --set full capture of the benchmarked commit (profiles/r02_ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
            d = json.load(f)
        v = d.get(key)
        return (int(v), "profiles/r02_ncu_traffic.json") if v else (None, None)
    except (OSError, ValueError):
        return None, None


def stack_config(world):
    """the config dict both arms print (identical keys and values)"""
    return {"workload": "resnet50_conv_stack (BASELINE configs[3]): 53 convs F+B+U (stem backward-data skipped), "
                        "ReLU / residual fused, stem max-pool, SGD, dW all-reduce",
            "global_batch": 256, "image": 224, "parallelism": f"dp{world}"}


# ---------------------------------------------------------------------- relaunch (--gpus N)


def relaunch(args) -> int:
    """bench.py --gpus N without a torchrun environment: run N NCCL ranks of this
    script on this node (rank 0 prints the line)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------- CPU (reference) legs


def _ref_builds():
    """the reference builds to time: the portable parity build and, when this host runs
    it, the reference's own Release flags (-O3 -march=native). g++ 13.3 vectorises the
    FWD / BWD microkernel with gathers under -march=native (5-6x slower there) but the
    weight update gains, so each pass is timed with both and the FASTER one counts."""
    from oracle import oracle as orc

    builds = [False]
    if orc.native_usable():
        builds.append(True)
    return builds


def _ref_pass_best(orc, s, pss, threads, k, a, b, builds, per_build):
    best = mean = float("inf")
    for nat in builds:
        _, bt, av = orc.ref_direct_pass(s, pss, threads, k, a, b, native=nat)
        per_build[nat] = per_build.get(nat, 0.0) + bt / 1e3
        if bt < best:
            best, mean = bt, av
    return best / 1e3, mean / 1e3


def _build_note(orc, builds, per_build, unit_fn):
    return "; ".join(f"{orc.ref_build_info(nat)}: {unit_fn(per_build[nat])}" for nat in builds) + \
        " -- per pass the faster build is counted"


def stack_cpu_reference(threads, n_img=2, k=5):
    """Reference direct engine on every distinct conv of the stack (F + B + U, plan
    setup excluded, one warm-up + best of k per pass, harness.cpp:55-72), N = n_img
    images, summed with the stack multiplicities; the stem's backward-data skipped.
    Returns (images/s from best times, images/s from mean times, sample, build)."""
    from oracle import oracle as orc
    from paper_1808_05567_b200 import executor as ex

    builds = _ref_builds()
    nodes = ex.resnet50_conv_stack()
    shapes = ex.tensor_shapes(nodes)
    mult = {}
    for nd in nodes:
        if isinstance(nd, ex.ConvNode):
            c, h, w = shapes[nd.src]
            key = (nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, nd.pad, nd.src == "x")
            mult[key] = mult.get(key, 0) + 1
    best_t = mean_t = 0.0
    per_build = {}
    for (C, K, H, W, R, S, st, pad, stem), m in mult.items():
        s = orc.spec(n_img, C, K, H, W, R, S, st, pad, pad, 16)
        P, Q = orc.output_shape(s)
        x = orc.uniform(0, (n_img, C, H, W))
        wt = orc.he_normal(1, (K, C, R, S), C * R * S)
        g = orc.uniform(2, (n_img, K, P, Q))
        for pss, (a, b) in enumerate(((x, wt), (g, wt), (x, g))):
            if pss == 1 and stem:
                continue
            pb = {}
            bt, av = _ref_pass_best(orc, s, pss, threads, k, a, b, builds, pb)
            best_t += m * bt
            mean_t += m * av
            for kk, v in pb.items():
                per_build[kk] = per_build.get(kk, 0.0) + m * v
    sample = f"reference direct engine, {n_img} images x {len(mult)} distinct convs (x multiplicity), F+B+U, " \
             f"plan setup excluded, 1 warm-up + best of {k}"
    note = _build_note(orc, builds, per_build, lambda t: f"{n_img / t:.3f} images/s")
    return n_img / best_t, n_img / mean_t, sample, note


def cfg2_cpu_reference(threads, k=3):
    from oracle import oracle as orc

    builds = _ref_builds()
    w = CFG2
    s = orc.spec(w["N"], w["C"], w["K"], w["H"], w["W"], w["R"], w["S"], w["stride"], w["pad_h"], w["pad_w"], 16)
    P, Q = orc.output_shape(s)
    x = orc.uniform(0, (w["N"], w["C"], w["H"], w["W"]))
    wt = orc.he_normal(1, (w["K"], w["C"], w["R"], w["S"]), w["C"] * w["R"] * w["S"])
    g = orc.uniform(2, (w["N"], w["K"], P, Q))
    best = mean = 0.0
    per_build = {}
    for pss, (a, b) in enumerate(((x, wt), (g, wt), (x, g))):
        bt, av = _ref_pass_best(orc, s, pss, threads, k, a, b, builds, per_build)
        best += bt
        mean += av
    fl = 3 * orc.pass_flops(s)
    note = _build_note(orc, builds, per_build, lambda t: f"{fl / t / 1e9:.1f} GFLOP/s")
    return fl / best / 1e9, fl / mean / 1e9, note


# ---------------------------------------------------------------------- GPU helpers


def _timed(torch, fn, reps=5, trials=3):
    """device ms per call: `reps` back-to-back calls queued behind a spin, best of `trials`"""
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(trials):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


def roof_ms(flops, byts, tflops, gbs):
    return max(flops / (tflops * 1e12), byts / (gbs * 1e9)) * 1e3


def measure_cfg2(torch, d, dev, steps, warmup, math_f32=True):
    """BASELINE configs[1]: 1x1 N32 C256 K64 56^2, one step = F, then B || U
    (side stream), fp32-accurate, L2 flushed between timed steps. Also each pass's
    conv kernel timed alone (roofline) through the library's event hooks."""
    from paper_1808_05567_b200 import _lib

    lib = _lib.lib()
    w = CFG2
    math = d.Math.F32 if math_f32 else d.Math.BF16
    spec = d.make_layer_spec(w["N"], w["C"], w["K"], w["H"], w["W"], w["R"], w["S"], w["stride"], w["pad_h"],
                             w["pad_w"], 16)
    P, Q = d.derive_output_shape(spec)
    import numpy as np

    def host(shape, seed, kind, fan_in=1):
        a = np.empty(int(np.prod(shape)), np.float32)
        if kind == "u":
            lib.dconv_fill_uniform_host(seed, -1.0, 1.0, a.ctypes.data, a.size)
        else:
            lib.dconv_fill_he_normal_host(seed, float(np.sqrt(2.0 / fan_in)), a.ctypes.data, a.size)
        return torch.from_numpy(a.reshape(shape))

    ib = d.to_blocked_activation(host((spec.N, spec.C, spec.H, spec.W), 0, "u").to(dev), spec)
    wb = d.to_blocked_weight(host((spec.K, spec.C, spec.R, spec.S), 1, "n", spec.C).to(dev), spec)
    gb = d.to_blocked_activation(host((spec.N, spec.K, P, Q), 2, "u").to(dev), 16, 0, 0)
    fplan = d.make_forward_plan(spec, 1, None, None, math)
    bctx = d.prepare_backward(spec, wb, 1, None, math)
    uplan = d.UpdatePlan(spec, None, math)
    out = d.BlockedActivation(spec.N, spec.K, P, Q, 16, 0, 0, torch.float32, dev)
    gi = d.BlockedActivation(spec.N, spec.C, spec.H, spec.W, 16, 0, 0, torch.float32, dev)
    dw = d.BlockedWeight(spec.K, spec.C, spec.R, spec.S, 16, torch.float32, dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    upd_stream = torch.cuda.Stream(dev)
    ev_fork = torch.cuda.Event()

    def step():
        fplan.execute(ib, wb, out)
        ev_fork.record(stream)
        upd_stream.wait_event(ev_fork)
        with torch.cuda.stream(upd_stream):
            uplan.execute(ib, gb, dw)
        bctx.execute(wb, gb, gi)
        stream.wait_stream(upd_stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.fill_(i & 0xFF)
        flush.view(torch.int32).sum()
        torch.cuda._sleep(4_000_000)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    lib.dconv_profile(1)
    kern = {"F": [], "B": [], "U": []}
    for i in range(min(steps, 10)):
        flush.fill_(i & 0xFF)
        flush.view(torch.int32).sum()
        torch.cuda._sleep(4_000_000)
        fplan.execute(ib, wb, out)
        bctx.execute(wb, gb, gi)
        uplan.execute(ib, gb, dw)
        torch.cuda.synchronize()
        for k, idx in (("F", 0), ("B", 1), ("U", 2)):
            kern[k].append(lib.dconv_profile_last_ms(idx))
    lib.dconv_profile(0)
    # layout kernels on the same tensor (to_/from_blocked_activation, blocked.hpp:133-178):
    # NCHW fp32 <-> NCHW16c fp32, bytes = read + write
    import ctypes as C

    x_nchw = torch.empty(spec.N, spec.C, spec.H, spec.W, dtype=torch.float32, device=dev).uniform_(-1, 1)
    blk = d.BlockedActivation(spec.N, spec.C, spec.H, spec.W, 16, 0, 0, torch.float32, dev)
    st = stream.cuda_stream
    t_pack = _timed(torch, lambda: lib.dconv_pack_act(x_nchw.data_ptr(), 0, C.byref(blk.to_c()), st), reps=10)
    t_unpack = _timed(torch, lambda: lib.dconv_unpack_act(C.byref(blk.to_c()), x_nchw.data_ptr(), 0, st), reps=10)
    layout_bytes = 2 * x_nchw.numel() * 4
    hbm, _, _, src = measured_peaks()
    layout = {"tensor": f"NCHW fp32 [{spec.N},{spec.C},{spec.H},{spec.W}] <-> NCHW16c", "bytes": layout_bytes,
              "pack_gbs": round(layout_bytes / (t_pack * 1e-3) / 1e9, 1),
              "unpack_gbs": round(layout_bytes / (t_unpack * 1e-3) / 1e9, 1),
              "pack_frac": round(layout_bytes / (t_pack * 1e-3) / 1e9 / hbm, 3),
              "unpack_frac": round(layout_bytes / (t_unpack * 1e-3) / 1e9 / hbm, 3)}
    byts = alg_bytes(w)
    avg = {k: sum(v) / len(v) for k, v in kern.items()}
    dom = max(avg, key=avg.get)
    achieved = byts[dom] / (avg[dom] * 1e-3) / 1e9
    fl = pass_flops(w)
    traffic, tsrc = ncu_traffic("cfg2_" + dom)
    res = {
        "value": round(3 * fl / (ms * 1e-3) / 1e9, 1), "unit": "GFLOP/s", "ms_per_step": round(ms, 4),
        "math": "fp32-accurate (exact bf16x3 split, 6 products, fp32 accumulate)" if math_f32 else "bf16",
        "pass_gflops": {k: round(fl / (v * 1e-3) / 1e9, 1) for k, v in avg.items()},
        "kernel_ms": {k: round(v, 4) for k, v in avg.items()},
        "tiles": {"fwd": fplan.blocking, "bwd": bctx.blocking, "upd": uplan.blocking},
        "roofline": {"bound": "hbm", "pass": dom, "kernel": {"F": "conv_fwd_kernel (TS)", "B": "conv_fwd_kernel (dual)",
                                                           "U": "conv_upd_ts_kernel"}[dom],
                     "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "alg_bytes_per_launch": byts[dom], "traffic": traffic, "traffic_source": tsrc,
                     "peak_source": src},
        "l2": "flushed between timed steps (256 MiB write + read-back, untimed)",
        "launches_per_step": fplan.launches() + bctx.launches() + uplan.launches(ib, gb),
        "layout_kernels": layout,
    }
    return res, (fplan, bctx, uplan, spec, ib, wb, gb, out, gi, dw)


def measure_cfg5(torch, d, dev):
    """BASELINE configs[4]: each Inception-v3 layer at N = 128, bf16 storage and math,
    F / B / U device time (each pass alone, best of 3 x 5 calls)."""
    hbm, peak, _, _ = measured_peaks()
    rows, tot_ms, tot_roof = [], 0.0, 0.0
    for (C_, K, H, W, R, S, st, ph, pw) in CFG5:
        N = 128
        spec = d.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
        P, Q = d.derive_output_shape(spec)
        g = torch.Generator(device="cpu").manual_seed(7)
        ib = d.to_blocked_activation((torch.rand(N, C_, H, W, generator=g) * 2 - 1).to(dev), 16, 0, 0,
                                     dtype=torch.bfloat16)
        wb = d.to_blocked_weight((torch.randn(K, C_, R, S, generator=g) * (2.0 / (C_ * R * S)) ** 0.5).to(dev), spec)
        gb = d.to_blocked_activation((torch.rand(N, K, P, Q, generator=g) * 2 - 1).to(dev), 16, 0, 0,
                                     dtype=torch.bfloat16)
        out = d.BlockedActivation(N, K, P, Q, 16, 0, 0, torch.bfloat16, dev)
        gi = d.BlockedActivation(N, C_, H, W, 16, 0, 0, torch.bfloat16, dev)
        dw = d.BlockedWeight(K, C_, R, S, 16, torch.float32, dev)
        fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
        bp = d.prepare_backward(spec, wb, 1, None, d.Math.BF16)
        up = d.UpdatePlan(spec, None, d.Math.BF16)
        t = {"F": _timed(torch, lambda: fp.execute(ib, wb, out)), "B": _timed(torch, lambda: bp.execute(wb, gb, gi)),
             "U": _timed(torch, lambda: up.execute(ib, gb, dw))}
        w = dict(N=N, C=C_, K=K, H=H, W=W, R=R, S=S, stride=st, pad_h=ph, pad_w=pw)
        fl = pass_flops(w)
        byts = alg_bytes(w, 2, 2)
        roof = {k: roof_ms(fl, byts[k], peak, hbm) for k in t}
        tot_ms += sum(t.values())
        tot_roof += sum(roof.values())
        rows.append({"layer": f"{C_}->{K} {R}x{S}/s{st} @{H}x{W}", "tflops": {k: round(fl / (v * 1e-3) / 1e12, 1)
                                                                           for k, v in t.items()},
                     "ms": {k: round(v, 4) for k, v in t.items()},
                     "roof_frac": {k: round(roof[k] / t[k], 3) for k in t}})
    return {"N": 128, "dtype": "bf16", "layers": rows, "sum_ms": round(tot_ms, 3),
            "roof_frac_of_sum": round(tot_roof / tot_ms, 3), "peaks": "bf16 burst TF/s and HBM GB/s (MEASURED_PEAKS)"}


def fused_operand_bytes(e, n):
    """extra compulsory bytes of each conv's fused graph epilogue (bf16): the forward's
    residual add reads the shortcut tensor; the backward-data's ReLU mask reads the
    input activation and its branch sum reads the other branch's gradient."""
    from paper_1808_05567_b200 import executor as ex

    convs = [nd for nd in e.nodes if isinstance(nd, ex.ConvNode)]
    ident = {nd.add for nd in convs if nd.add is not None}
    n_conv_consumers = {}
    for nd in convs:
        n_conv_consumers[nd.src] = n_conv_consumers.get(nd.src, 0) + 1
    out = {}
    for nd in convs:
        c, h, w = e.shapes[nd.src]
        k, p, q = e.shapes[nd.out]
        f = 2 * n * k * p * q if nd.add else 0
        b = 0
        # strided 1x1 backward-data touches only its stride lattice of dI with the mask / sum
        pix = p * q if (nd.R == 1 and nd.S == 1 and nd.stride > 1) else h * w
        if nd.src != "x":
            if nd.src in e.relu_out:
                b += 2 * n * c * pix  # mask
            if nd.src in ident or n_conv_consumers.get(nd.src, 0) > 1:
                b += 2 * n * c * pix  # branch-gradient sum
        out[nd.name] = {"F": f, "B": b, "U": 0}
    return out


def stack_layer_roofline(e, prof, n):
    """the dominant (layer shape, pass) group of the step: largest total device time"""
    from paper_1808_05567_b200 import executor as ex

    hbm, peak, _, src = measured_peaks()
    groups = {}
    step_roof = 0.0
    fused = fused_operand_bytes(e, n)
    for nd in e.convs:
        c, h, w = e.shapes[nd.src]
        wl = dict(N=n, C=nd.C, K=nd.K, H=h, W=w, R=nd.R, S=nd.S, stride=nd.stride, pad_h=nd.pad, pad_w=nd.pad)
        fl = pass_flops(wl)
        byts = alg_bytes(wl, 2, 2)
        for k in byts:  # the executor's fused epilogue operands are compulsory traffic of that kernel
            byts[k] += fused[nd.name][k]
        for k in ("F", "B", "U"):
            ms = prof[nd.name][k]
            if ms <= 0:
                continue
            key = (nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, k, byts[k])  # same shape AND same fused operands
            gdat = groups.setdefault(key, {"ms": 0.0, "count": 0, "flops": fl, "bytes": byts[k],
                                           "layers": []})
            gdat["ms"] += ms
            gdat["count"] += 1
            gdat["layers"].append(nd.name)
            step_roof += roof_ms(fl, byts[k], peak, hbm)
    key, g = max(groups.items(), key=lambda kv: kv[1]["ms"])
    C_, K, H, W, R, S, st, pss, _ = key
    avg = g["ms"] / g["count"]
    ai = g["flops"] / g["bytes"]
    ridge = peak * 1e12 / (hbm * 1e9)
    kern = {"F": "conv_fwd_kernel<bf16>", "B": "conv_fwd_kernel<bf16> (backward-data)",
            "U": "conv_upd_kernel<1,1> (bf16 SW32)"}[pss]
    tkey = f"r50_{C_}_{K}_{H}_{R}x{S}s{st}_{pss}"
    traffic, tsrc = ncu_traffic(tkey)
    if ai >= ridge:
        achieved, unit, pk, bound = g["flops"] / (avg * 1e-3) / 1e12, "TFLOP/s", peak, "tensor"
    else:
        achieved, unit, pk, bound = g["bytes"] / (avg * 1e-3) / 1e9, "GB/s", hbm, "hbm"
    total = sum(v["F"] + v["B"] + v["U"] for v in prof.values())
    return {"bound": bound, "kernel": kern, "layer": f"{C_}->{K} {R}x{S}/s{st} @{H}x{W} {pss}",
            "layers": g["layers"],
            "instances": g["count"], "achieved": round(achieved, 1), "peak": pk, "unit": unit,
            "frac": round(achieved / pk, 4), "traffic": traffic, "traffic_key": tkey, "traffic_source": tsrc,
            "alg_flops_per_launch": g["flops"], "alg_bytes_per_launch": g["bytes"], "kernel_ms": round(avg, 4),
            "share_of_step_kernels": round(g["ms"] / total, 3), "peak_source": src + " (burst; kernel timed alone)",
            "per_layer_roof_step_ms": round(step_roof, 3), "kernels_sum_ms": round(total, 3)}


# ---------------------------------------------------------------------- the stack (default)


def run_stack(args):
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_stack_reference(args, world, rank)
    import torch

    import paper_1808_05567_b200 as d
    from paper_1808_05567_b200 import _lib
    from paper_1808_05567_b200 import executor as ex

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    global_batch = args.global_batch
    n = global_batch // world
    nodes = ex.resnet50_conv_stack(224)
    lib = _lib.lib()
    if args.sm_budget:  # leave SMs for NCCL's kernels (persistent conv grids use the rest)
        d.api._check(lib.dconv_set_sm_budget(args.sm_budget))
    e = ex.ConvStackExecutor(nodes, n, 224, d.Math.BF16, "cuda", group=pg, lr=1e-6)
    # seeded synthetic images (this rank's shard) and top gradient
    x_h = torch.empty(n, 3, 224, 224, dtype=torch.float32)
    lib.dconv_fill_uniform_host(1000 * rank, -1.0, 1.0, x_h.data_ptr(), x_h.numel())
    x_pin = x_h.pin_memory()
    x_dev = torch.empty_like(x_h, device=dev)
    c, h, w = e.shapes[nodes[-1].out]
    g_h = torch.empty(n, c, h, w, dtype=torch.float32)
    lib.dconv_fill_uniform_host(2 + 1000 * rank, -1.0, 1.0, g_h.data_ptr(), g_h.numel())
    dtop = d.to_blocked_activation(g_h.to(dev), 16, 0, 0, dtype=torch.bfloat16)
    loss_dev = torch.zeros(1, dtype=torch.float32, device=dev)
    loss_pin = torch.zeros(1, dtype=torch.float32).pin_memory()
    stream = torch.cuda.Stream(dev)  # the step's stream (a captured graph needs a non-default stream)
    torch.cuda.set_stream(stream)
    x_dev.copy_(x_pin)
    e.load_input_nchw(x_dev)

    for _ in range(args.warmup):
        e.step(dtop)
    torch.cuda.synchronize()
    graph = not args.no_graph
    if graph:
        e.capture(dtop)  # one CUDA graph per step, the NCCL all-reduces inside it
        torch.cuda.synchronize()
        run = e.replay
        for _ in range(2):
            run()
        torch.cuda.synchronize()
    else:
        def run():
            e.step(dtop)
    launches = e.launches_per_step()

    def barrier():
        if pg is not None:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def maxred(v):
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if pg is not None:
            import torch.distributed as dist

            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            run()
        e1.record(stream)
        barrier()
    ms_per_step = maxred(e0.elapsed_time(e1) / args.steps)
    value = global_batch / (ms_per_step * 1e-3)

    # ---------------- end to end: the next step's images copied H2D (pinned) on a side
    # stream during this step (a training loop's input pipeline), packed, step, loss D2H
    h2d = x_pin.numel() * 4
    x_bufs = [x_dev, torch.empty_like(x_dev)]
    copy_stream = torch.cuda.Stream(dev)
    copied = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def issue_copy(i):
        b = i % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[b])
            x_bufs[b].copy_(x_pin, non_blocking=True)
            copied[b].record(copy_stream)

    def e2e_step(i, last):
        b = i % 2
        stream.wait_event(copied[b])
        e.load_input_nchw(x_bufs[b])
        consumed[b].record(stream)
        if not last:
            issue_copy(i + 1)
        run()
        top = e.act[nodes[-1].out].data
        loss_dev.copy_((top.float() * dtop.data.float()).sum().reshape(1))
        loss_pin.copy_(loss_dev, non_blocking=True)

    for b in range(2):
        consumed[b].record(stream)
    issue_copy(0)
    for i in range(2):
        e2e_step(i, i == 1)
    barrier()
    with sampler:
        e0.record(stream)
        copy_stream.wait_event(e0)  # the first copy starts inside the timed region
        issue_copy(0)
        for i in range(args.steps):
            e2e_step(i, i == args.steps - 1)
        e1.record(stream)
        barrier()
    e2e_ms = maxred(e0.elapsed_time(e1) / args.steps)
    e2e_value = global_batch / (e2e_ms * 1e-3)

    hbm, peak, sustained, peak_src = measured_peaks()
    flops_img = ex.step_flops_per_image(nodes)
    achieved = flops_img * global_batch / (ms_per_step * 1e-3) / 1e12

    # ---------------- per-layer times and the dominant kernel's roofline (rank 0)
    roof, layers = None, None
    if rank == 0 and not args.no_layers:
        prof = e.profile(dtop)
        roof = stack_layer_roofline(e, prof, n)
        tot = {k: round(sum(v[k] for v in prof.values()), 3) for k in ("F", "B", "U")}
        layers = {"per_gpu_batch": n, "pass_ms_sum": tot,
                  "roof_img_s_per_gpu": round(n / (roof["per_layer_roof_step_ms"] * 1e-3), 1),
                  "frac_of_per_layer_roof": round(roof["per_layer_roof_step_ms"] / ms_per_step, 4) if world == 1
                  else None}
    cfg2 = cfg5 = cpu = None
    if world == 1 and not args.no_layers:
        try:
            cfg2, _ = measure_cfg2(torch, d, dev, 10, 3)
        except Exception as ex_:  # noqa: BLE001
            cfg2 = {"error": str(ex_)}
        try:
            cfg5 = measure_cfg5(torch, d, dev)
        except Exception as ex_:  # noqa: BLE001
            cfg5 = {"error": str(ex_)}
    if world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as orc

            if orc.ref_available():
                stack_cpu_reference(os.cpu_count() or 1, k=1)  # warm-up sweep (untimed)
                ips, ips_mean, sample, build = stack_cpu_reference(os.cpu_count() or 1)
                cpu = {"value": round(ips, 4), "unit": "images/s", "cores": os.cpu_count(), "kind": "reference",
                       "sample": sample, "mean_value": round(ips_mean, 4), "build": build}
        except Exception as ex_:  # noqa: BLE001
            cpu = {"value": None, "unit": "images/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex_}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded splitmix64 images 3x224x224 and top gradient; He-normal weights)",
            "config": stack_config(world),
            "details": {"per_gpu_batch": n, "cuda_graph": graph, "sm_budget": args.sm_budget or None, "math": "bf16 operands, fp32 accumulate; fp32 "
                        "master weights / gradients", "l2": "not flushed: the step's working set (activations "
                        "and gradients, GBs) is far larger than the 126 MB L2",
                        "exchange": "NCCL all-reduce of fp32 dW in backward-order buckets inside the step"
                        if world > 1 else "none (1 rank)",
                        "step_tflops": round(achieved, 1), "step_frac_of_sustained_bf16": round(achieved / sustained, 4),
                        "flops_per_image": flops_img},
            "e2e": {"value": round(e2e_value, 2), "unit": "images/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": 4 * world,
                    "pipeline": "step i+1's images copied H2D (pinned) on a side stream during step i; pack, step, "
                                "loss D2H every step", "ms_per_step": round(e2e_ms, 3)},
            "gpu_launches": launches * args.steps,
            "roofline": roof,
            "layers": layers,
            "cfg2": cfg2,
            "cfg5": cfg5,
            "cpu_baseline": cpu,
            "clocks": sampler.report(),
        }
        print(json.dumps(line), flush=True)
    del e
    if pg is not None:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_stack_reference(args, world, rank):
    """--impl reference: the reference CPU direct engine on rank 0, same metric / config."""
    if rank != 0:
        return 0
    from oracle import oracle as orc

    threads = os.cpu_count() or 1
    if not orc.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (needs /root/reference)"}))
        return 0
    for _ in range(args.warmup and 1):
        stack_cpu_reference(threads, k=1)
    vals = []
    for _ in range(max(1, min(args.steps, 3))):
        ips, ips_mean, sample, build = stack_cpu_reference(threads)
        vals.append(ips)
    value = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "images/s", "n_gpus": world,
            "steps": len(vals), "warmup": 1, "ms_per_step": round(256 / value * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded splitmix64)", "config": stack_config(world),
            "cpu_baseline": {"value": round(value, 4), "unit": "images/s", "cores": threads, "kind": "reference",
                             "sample": sample + "; each step = one such sweep, extrapolated to the 256-image step",
                             "build": build, "mean_value": round(ips_mean, 4)},
            "e2e": {"value": round(value, 4), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- cfg2 line (--workload layer)


def run_layer(args):
    world, rank, local = dist_env()
    w = CFG2
    cfg = {"workload": "resnet50_id5_1x1_bottleneck_fwd_bwd_upd (BASELINE configs[1])", **w,
           "parallelism": f"dp{world}"}
    if args.impl == "reference":
        if rank != 0:
            return 0
        threads = os.cpu_count() or 1
        from oracle import oracle as orc

        cfg2_cpu_reference(threads, k=1)
        v, vm, build = cfg2_cpu_reference(threads, k=max(1, min(args.steps, 5)))
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "GFLOP/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(3 * pass_flops(w) / v / 1e6, 3), "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64)",
                          "config": cfg,
                          "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads,
                                           "kind": "reference" if orc.ref_available() else "port",
                                           "sample": "reference direct engine, full N=32 F+B+U, best of k",
                                           "build": build, "mean_value": round(vm, 3)},
                          "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    import torch

    import paper_1808_05567_b200 as d

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    sampler = ClockSampler(local)
    with sampler:
        res, objs = measure_cfg2(torch, d, dev, args.steps, args.warmup)
    fplan, bctx, uplan, spec, ib, wb, gb, out, gi, dw = objs
    ms = res["ms_per_step"]
    if pg is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    flops_step = 3 * pass_flops(w)
    value = world * flops_step / (ms * 1e-3) / 1e9
    # e2e through the host-buffer execute contract (dconv_host_step_run)
    B = d.BlockedActivation

    def pinned(t):
        return t.data.cpu().pin_memory()

    x_hb = B(ib.n, ib.c, ib.h, ib.w, 16, ib.halo_h, ib.halo_w, device="cpu", data=pinned(ib))
    g_hb = B(gb.n, gb.c, gb.h, gb.w, 16, 0, 0, device="cpu", data=pinned(gb))
    w_hb = d.BlockedWeight(wb.k, wb.c, wb.r, wb.s, 16, device="cpu", data=pinned(wb))
    y_hb = B(out.n, out.c, out.h, out.w, 16, 0, 0, device="cpu", data=pinned(out))
    dx_hb = B(gi.n, gi.c, gi.h, gi.w, 16, 0, 0, device="cpu", data=pinned(gi))
    dw_hb = d.BlockedWeight(dw.k, dw.c, dw.r, dw.s, 16, device="cpu", data=pinned(dw))
    h2d = (x_hb.data.numel() + g_hb.data.numel() + w_hb.data.numel()) * 4
    d2h = (y_hb.data.numel() + dx_hb.data.numel() + dw_hb.data.numel()) * 4
    hstep = d.HostStep(spec, d.Math.F32, args.chunk)
    stream = torch.cuda.current_stream()
    for _ in range(max(1, args.warmup // 2)):
        hstep.run(x_hb, w_hb, g_hb, y_hb, dx_hb, dw_hb, sync=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        e0.record(stream)
        for _ in range(args.steps):
            hstep.run(x_hb, w_hb, g_hb, y_hb, dx_hb, dw_hb, sync=False)
        e1.record(stream)
        torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            cfg2_cpu_reference(os.cpu_count() or 1, k=1)
            v, vm, build = cfg2_cpu_reference(os.cpu_count() or 1)
            cpu = {"value": round(v, 3), "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "reference direct engine, full N=32 F+B+U, best of 3", "build": build,
                   "mean_value": round(vm, 3)}
        except Exception as ex_:  # noqa: BLE001
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex_}"}
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64: uniform(-1,1) x/dO, "
                "He-normal W)", "config": cfg,
                "details": {"math": res["math"], "l2": res["l2"], "tiles": res["tiles"], "pass_gflops": res["pass_gflops"],
                            "step_order": "forward, then backward-data || weight update (side stream, joined)"},
                "e2e": {"value": round(flops_step / (e2e_ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                        "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                        "api": "dconv_host_step_run (pinned host blocked tensors)", "chunk_images": hstep.chunk,
                        "ms_per_step": round(e2e_ms, 4)},
                "gpu_launches": res["launches_per_step"] * args.steps, "roofline": res["roofline"],
                "cpu_baseline": cpu, "clocks": sampler.report()}
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


# ---------------------------------------------------------------------- cfg5 (--workload cfg5)


def cfg5_config(world):
    return {"workload": "inception_v3_layer_mix (BASELINE configs[4]): 10 layers F+B+U, bf16, dW all-reduce",
            "global_batch": 128, "parallelism": f"dp{world}"}


def run_cfg5(args):
    """BASELINE configs[4] as a data-parallel step: every layer of the Inception-v3 mix
    forward, then backward-data || weight update, at 128 / world images per rank; the
    fp32 dW of all layers live in one flat buffer, all-reduced with NCCL at the end of
    the step (the COPY_REDUCE exchange); the step is one CUDA graph."""
    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as orc

        threads = os.cpu_count() or 1
        builds = _ref_builds()
        n_img, tot = 2, 0.0
        for (C_, K, H, W, R, S, st, ph, pw) in CFG5:
            sp = orc.spec(n_img, C_, K, H, W, R, S, st, ph, pw, 16)
            P, Q = orc.output_shape(sp)
            x = orc.uniform(0, (n_img, C_, H, W))
            wt = orc.he_normal(1, (K, C_, R, S), C_ * R * S)
            g = orc.uniform(2, (n_img, K, P, Q))
            for pss, (a, b) in enumerate(((x, wt), (g, wt), (x, g))):
                tot += _ref_pass_best(orc, sp, pss, threads, 3, a, b, builds, {})[0]
        value = n_img / tot
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "images/s",
                          "n_gpus": world, "steps": 1, "warmup": 1, "ms_per_step": round(128 / value * 1e3, 1),
                          "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic (seeded splitmix64)", "config": cfg5_config(world),
                          "cpu_baseline": {"value": round(value, 3), "unit": "images/s", "cores": threads,
                                           "kind": "reference", "sample": "2 images through the 10 layers, F+B+U, "
                                           "best of 3 per pass, faster build per pass"},
                          "e2e": {"value": round(value, 3), "unit": "images/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    import torch

    import paper_1808_05567_b200 as d

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    n = 128 // world
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    side = torch.cuda.Stream(dev)
    layers, sizes = [], []
    gen = torch.Generator(device="cpu").manual_seed(7 + rank)
    for (C_, K, H, W, R, S, st, ph, pw) in CFG5:
        spec = d.make_layer_spec(n, C_, K, H, W, R, S, st, ph, pw, 16)
        P, Q = d.derive_output_shape(spec)
        ib = d.to_blocked_activation((torch.rand(n, C_, H, W, generator=gen) * 2 - 1).to(dev), 16, 0, 0,
                                     dtype=torch.bfloat16)
        wb = d.to_blocked_weight((torch.randn(K, C_, R, S, generator=gen) * (2.0 / (C_ * R * S)) ** 0.5).to(dev), spec)
        gb = d.to_blocked_activation((torch.rand(n, K, P, Q, generator=gen) * 2 - 1).to(dev), 16, 0, 0,
                                     dtype=torch.bfloat16)
        layers.append(dict(spec=spec, ib=ib, wb=wb, gb=gb,
                           out=d.BlockedActivation(n, K, P, Q, 16, 0, 0, torch.bfloat16, dev),
                           gi=d.BlockedActivation(n, C_, H, W, 16, 0, 0, torch.bfloat16, dev),
                           fp=d.make_forward_plan(spec, 1, None, None, d.Math.BF16),
                           bp=d.prepare_backward(spec, wb, 1, None, d.Math.BF16),
                           up=d.UpdatePlan(spec, None, d.Math.BF16)))
        sizes.append(wb.data.numel())
    flat = torch.zeros(sum(sizes), dtype=torch.float32, device=dev)
    off = 0
    for L, sz in zip(layers, sizes):
        L["dw"] = d.BlockedWeight(L["spec"].K, L["spec"].C, L["spec"].R, L["spec"].S, 16, torch.float32, dev,
                                  data=flat[off:off + sz])
        off += sz
    ev = [torch.cuda.Event() for _ in layers]

    def step():
        for i, L in enumerate(layers):
            L["fp"].execute(L["ib"], L["wb"], L["out"])
            ev[i].record(stream)
            side.wait_event(ev[i])
            with torch.cuda.stream(side):
                L["up"].execute(L["ib"], L["gb"], L["dw"])
            L["bp"].execute(L["wb"], L["gb"], L["gi"])
        stream.wait_stream(side)
        if pg is not None:
            pg.all_reduce(flat)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else step
    launches = sum(L["fp"].launches() + L["bp"].launches() + L["up"].launches(L["ib"], L["gb"]) for L in layers)
    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            run()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if pg is not None:
        pg.all_reduce(ms, op=pg.ReduceOp.MAX)
    ms = float(ms.item())
    # end to end: every layer's input activations and output gradients copied H2D
    # (pinned) each step, the flat dW read back
    host_in = [(L["ib"].data.cpu().pin_memory(), L["gb"].data.cpu().pin_memory()) for L in layers]
    dw_host = torch.empty_like(flat, device="cpu").pin_memory()
    h2d = sum(a.numel() * 2 + b.numel() * 2 for a, b in host_in)

    def e2e_step():
        for L, (a, b) in zip(layers, host_in):
            L["ib"].data.copy_(a, non_blocking=True)
            L["gb"].data.copy_(b, non_blocking=True)
        run()
        dw_host.copy_(flat, non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if pg is not None:
        pg.all_reduce(e2e, op=pg.ReduceOp.MAX)
    e2e = float(e2e.item())
    hbm, peak, _, src = measured_peaks()
    fl = sum(3 * pass_flops(dict(N=128, C=c, K=k, H=h, W=w, R=r, S=s_, stride=st, pad_h=ph, pad_w=pw))
             for (c, k, h, w, r, s_, st, ph, pw) in CFG5)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": round(128 / (ms * 1e-3), 1), "unit": "images/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded uniform / He-normal)",
            "config": cfg5_config(world),
            "details": {"per_gpu_batch": n, "cuda_graph": graph is not None, "step_tflops": round(fl / (ms * 1e-3) / 1e12, 1),
                        "step_frac_of_burst_bf16": round(fl / (ms * 1e-3) / 1e12 / peak, 4),
                        "l2": "not flushed (the step's 10 layers move ~1.3 GB)"},
            "e2e": {"value": round(128 / (e2e * 1e-3), 1), "unit": "images/s", "h2d_bytes_per_step": h2d * world,
                    "d2h_bytes_per_step": flat.numel() * 4 * world, "ms_per_step": round(e2e, 4)},
            "gpu_launches": launches * args.steps, "clocks": sampler.report()}), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=["resnet50", "layer", "cfg5"])
    ap.add_argument("--global-batch", type=int, default=256)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-graph", action="store_true", help="eager steps instead of the captured CUDA graph")
    ap.add_argument("--no-layers", action="store_true", help="skip the per-layer / cfg2 / cfg5 sub-objects")
    ap.add_argument("--chunk", type=int, default=8, help="images per host-step chunk (layer e2e); 0 = N/4")
    ap.add_argument("--sm-budget", type=int, default=0, help="cap the persistent conv kernels at this many SMs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.workload == "layer":
        return run_layer(args)
    if args.workload == "cfg5":
        return run_cfg5(args)
    return run_stack(args)


if __name__ == "__main__":
    sys.exit(main())
