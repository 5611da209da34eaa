#!/usr/bin/env python3
"""bench.py — the driver's benchmark contract for dconv-b200.

Default workload (BASELINE.json configs[1], the config the per-layer metric
is quoted on): ResNet-50 Table I layer 5, the 1x1 bottleneck conv
N=32, C=256 -> K=64, 56x56, stride 1, pad 0; one step = forward +
backward-data + weight-update, fp32-accurate (exact bf16x3 split, fp32
accumulate), seeded synthetic inputs (uniform(-1,1) seed 0 activations,
He-normal seed 1 weights, uniform(-1,1) seed 2 output gradients).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value  : whole-job GFLOP/s (pass_flops x 3 passes x ranks / max-over-ranks
         device time), inputs resident in HBM, L2 flushed between steps.
e2e    : same metric through the reference-facing call with HOST buffers:
         pinned blocked tensors copied H2D, the three passes, outputs D2H.
Multi-GPU (torchrun): weak scaling, each rank runs its own N=32 shard and the
fp32 weight gradient is summed across ranks with NCCL all-reduce (the
COPY_REDUCE exchange promoted to GPUs); max-over-ranks device time.
--impl reference: the reference's own CPU direct engine (oracle/_ref, built
from /root/reference sources) on all host cores, same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "conv GFLOP/s per layer (fwd/bwd/upd) and conv-stack images/s at 1/2/4/8 B200"
WORKLOAD = dict(N=32, C=256, K=64, H=56, W=56, R=1, S=1, stride=1, pad_h=0, pad_w=0)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def alg_bytes(w, e_in=4, e_out=4):
    """SURVEY.md 8(d) compulsory bytes per pass (halos not counted)."""
    N, C, K, H, W, R, S = (w[k] for k in ("N", "C", "K", "H", "W", "R", "S"))
    st = w["stride"]
    P = (H + 2 * w["pad_h"] - R) // st + 1
    Q = (W + 2 * w["pad_w"] - S) // st + 1
    Cp = -(-C // 16) * 16
    Kp = -(-K // 16) * 16
    touched = N * Cp * P * Q if (R == 1 and S == 1 and st > 1) else N * Cp * H * W
    fwd = e_in * (touched + Kp * Cp * R * S) + e_out * N * Kp * P * Q
    bwd = e_in * (N * Kp * P * Q + Kp * Cp * R * S) + e_out * N * Cp * H * W
    upd = e_in * (touched + N * Kp * P * Q) + 4 * Kp * Cp * R * S
    return {"fwd": fwd, "bwd": bwd, "upd": upd}


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
        # may be entered once per timed region; samples accumulate
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


def ncu_traffic(pass_name):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) of the pass's kernel
    from the committed ncu --set full capture, or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_ncu_full_cfg2.json")
    try:
        with open(path) as f:
            ks = json.load(f)["kernels"]
    except (OSError, ValueError, KeyError):
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for k in ks:
        if k.get("pass", "").startswith(pass_name):
            tot = 0.0
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                val, unit = k[key].split()
                tot += float(val) * scale[unit]
            return int(tot)
    return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------- reference arm


def cpu_inputs(w):
    from oracle import oracle as orc

    N, C, K, H, W, R, S = (w[k] for k in ("N", "C", "K", "H", "W", "R", "S"))
    s = orc.spec(N, C, K, H, W, R, S, w["stride"], w["pad_h"], w["pad_w"], 16)
    P, Q = orc.output_shape(s)
    x = orc.uniform(0, (N, C, H, W))
    wt = orc.he_normal(1, (K, C, R, S), C * R * S)
    g = orc.uniform(2, (N, K, P, Q))
    return orc, s, x, wt, g


def cpu_step_reference(orc, s, x, wt, g, threads):
    """One F+B+U step of the reference direct engine; returns seconds (sum of the
    three timed execute calls, setup excluded as in bench_layer)."""
    t = 0.0
    for p, (a, b) in enumerate(((x, wt), (g, wt), (x, g))):
        _, best, _ = orc.ref_direct_pass(s, p, threads, 1, a, b)
        t += best / 1e3
    return t


def cpu_step_port(orc, s, x, wt, g, threads):
    t0 = time.perf_counter()
    orc.conv_forward(s, x, wt, threads)
    orc.conv_backward(s, g, wt, threads)
    orc.conv_update(s, x, g, threads)
    return time.perf_counter() - t0


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    orc, s, x, wt, g = cpu_inputs(WORKLOAD)
    threads = os.cpu_count() or 1
    flops = 3 * orc.pass_flops(s)
    kind = "reference" if orc.ref_available() else "port"
    if kind == "port":
        # the f64 naive port is ~100x slower: bounded sample of 2 images
        s2 = orc.spec(2, s.C, s.K, s.H, s.W, s.R, s.S, s.stride, s.pad_h, s.pad_w, 16)
        x, g = x[:2].copy(), g[:2].copy()
        s, flops = s2, 3 * orc.pass_flops(s2)
        step = lambda: cpu_step_port(orc, s, x, wt, g, threads)  # noqa: E731
        sample = "naive f64 oracle port, 2 of 32 images, F+B+U"
    else:
        step = lambda: cpu_step_reference(orc, s, x, wt, g, threads)  # noqa: E731
        sample = "reference direct engine (oracle/_ref), full N=32 F+B+U, plan setup excluded"
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    sec = sum(times) / len(times)
    value = flops / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded splitmix64)",
        "config": {"workload": "resnet50_id5_1x1_bottleneck_fwd_bwd_upd", **WORKLOAD,
                   "parallelism": "cpu threads"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- our arm


def run_ours(args):
    import numpy as np
    import torch

    import paper_1808_05567_b200 as d
    from paper_1808_05567_b200 import _lib

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        pg = dist
    w = WORKLOAD
    math = d.Math.BF16 if args.math == "bf16" else d.Math.F32
    spec = d.make_layer_spec(w["N"], w["C"], w["K"], w["H"], w["W"], w["R"], w["S"], w["stride"], w["pad_h"],
                             w["pad_w"], 16)
    P, Q = d.derive_output_shape(spec)
    # seeded synthetic inputs (host generator in the product library; rank-dependent shards)
    lib = _lib.lib()

    def host(shape, seed, kind, fan_in=1):
        a = np.empty(int(np.prod(shape)), np.float32)
        if kind == "u":
            lib.dconv_fill_uniform_host(seed + 1000 * rank, -1.0, 1.0, a.ctypes.data, a.size)
        else:
            lib.dconv_fill_he_normal_host(seed, float(np.sqrt(2.0 / fan_in)), a.ctypes.data, a.size)
        return torch.from_numpy(a.reshape(shape))

    x_h = host((spec.N, spec.C, spec.H, spec.W), 0, "u")
    w_h = host((spec.K, spec.C, spec.R, spec.S), 1, "n", spec.C * spec.R * spec.S)
    g_h = host((spec.N, spec.K, P, Q), 2, "u")
    ib = d.to_blocked_activation(x_h.to(dev), spec)
    wb = d.to_blocked_weight(w_h.to(dev), spec)
    gb = d.to_blocked_activation(g_h.to(dev), 16, 0, 0)
    fplan = d.make_forward_plan(spec, 1, None, None, math)
    bctx = d.prepare_backward(spec, wb, 1, None, math)
    uplan = d.UpdatePlan(spec, None, math)
    out = d.BlockedActivation(spec.N, spec.K, P, Q, 16, 0, 0, torch.float32, dev)
    gi = d.BlockedActivation(spec.N, spec.C, spec.H, spec.W, 16, 0, 0, torch.float32, dev)
    dw = d.BlockedWeight(spec.K, spec.C, spec.R, spec.S, 16, torch.float32, dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def flush_l2(i):
        # write a buffer larger than L2, then read it back: the step's inputs are
        # evicted and the flush's own dirty lines are written back here (untimed)
        # rather than during the timed kernels
        flush.fill_(i & 0xFF)
        flush.view(torch.int32).sum()

    # a training step's order: forward, then backward-data and weight update -- the
    # latter two concurrently (the update on a side stream joined before the gradient
    # exchange), exactly as the graph executor runs them
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
        if pg is not None:
            pg.all_reduce(dw.data)

    def step_serial():  # the per-kernel roofline pass: one kernel at a time
        fplan.execute(ib, wb, out)
        bctx.execute(wb, gb, gi)
        uplan.execute(ib, gb, dw)

    launches = fplan.launches() + bctx.launches() + uplan.launches(ib, gb)

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    # ---------------- device-resident timing (value)
    for _ in range(args.warmup):
        step()
    barrier()
    sampler = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with sampler:
        barrier()
        for i in range(args.steps):
            flush_l2(i)  # evict L2 between steps (untimed)
            # untimed spin so the whole step is queued before its first kernel
            # runs: the events then bracket device work, not host launch gaps
            torch.cuda._sleep(4_000_000)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            if sampler.nv is not None:
                sampler._sample()  # one reading per step while the GPU is busy
            torch.cuda.synchronize()
        barrier()
    # per-pass conv-kernel times for the roofline: a separate pass of the same
    # steps with the library's event brackets on (brackets serialise the
    # programmatic launch overlap, so they stay out of the timed loop above)
    lib.dconv_profile(1)
    kern_ms = {"fwd": [], "bwd": [], "upd": []}
    for i in range(min(args.steps, 10)):
        flush_l2(i)
        torch.cuda._sleep(4_000_000)
        step_serial()
        torch.cuda.synchronize()
        for k, idx in (("fwd", 0), ("bwd", 1), ("upd", 2)):
            kern_ms[k].append(lib.dconv_profile_last_ms(idx))
    lib.dconv_profile(0)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if pg is not None:
        pg.all_reduce(t_local, op=pg.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    flops_step = 3 * d.pass_flops(spec)
    value = world * flops_step / (ms_per_step * 1e-3) / 1e9

    # ---------------- end to end through the host-buffer API (e2e)
    # dconv_host_step_run: the reference's host-memory execute contract; the batch
    # streams through the GPU in image chunks with H2D / kernels / D2H overlapped
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
    hstep = d.HostStep(spec, math, args.chunk)

    def e2e_step():
        hstep.run(x_hb, w_hb, g_hb, y_hb, dx_hb, dw_hb, sync=False)
        if pg is not None:  # data-parallel dW sum (64 KiB) through the device
            dw.data.copy_(dw_hb.data, non_blocking=True)
            pg.all_reduce(dw.data)
            dw_hb.data.copy_(dw.data, non_blocking=True)

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    barrier()
    with sampler:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if pg is not None:
        pg.all_reduce(e2e_ms, op=pg.ReduceOp.MAX)
    e2e_value = world * flops_step / (float(e2e_ms.item()) * 1e-3) / 1e9

    # ---------------- roofline of the dominant kernel
    hbm_peak, bf16_peak, peak_src = measured_peaks()
    byts = alg_bytes(w)
    avg = {k: sum(v) / len(v) for k, v in kern_ms.items() if v and min(v) > 0}
    dom = max(avg, key=avg.get) if avg else "fwd"
    achieved = byts[dom] / (avg.get(dom, float("nan")) * 1e-3) / 1e9
    traffic = ncu_traffic(dom) if math == d.Math.F32 else None
    upd_kernel = "conv_upd_ts_kernel" if uplan.blocking.get("a_in_tmem") else "conv_upd_raw_kernel"
    roofline = {"bound": "hbm", "kernel": {"fwd": "conv_fwd_kernel", "bwd": "conv_fwd_kernel (dual)",
                                           "upd": upd_kernel}[dom],
                "pass": dom, "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "peak_source": peak_src,
                "traffic_source": "profiles/r01_ncu_full_cfg2.json (dram read+write bytes of one ncu --set full launch)"
                if traffic else None,
                "alg_bytes_per_launch": byts[dom], "kernel_ms": {k: round(v, 4) for k, v in avg.items()},
                "share_of_step": round(avg.get(dom, 0) / ms_per_step, 3)}

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            orc, s_c, x_c, w_c, g_c = cpu_inputs(w)
            threads = os.cpu_count() or 1
            if orc.ref_available():
                sec = cpu_step_reference(orc, s_c, x_c, w_c, g_c, threads)
                cpu = {"value": round(3 * orc.pass_flops(s_c) / sec / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
                       "kind": "reference",
                       "sample": "reference direct engine (oracle/_ref), full N=32 F+B+U, one step"}
            else:
                s2 = orc.spec(2, s_c.C, s_c.K, s_c.H, s_c.W, s_c.R, s_c.S, 1, 0, 0, 16)
                sec = cpu_step_port(orc, s2, x_c[:2].copy(), w_c, g_c[:2].copy(), threads)
                cpu = {"value": round(3 * orc.pass_flops(s2) / sec / 1e9, 3), "unit": "GFLOP/s", "cores": threads,
                       "kind": "port", "sample": "naive f64 oracle port, 2 of 32 images, F+B+U"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if math == d.Math.F32 else "bf16",
            "data": "synthetic (seeded splitmix64: uniform(-1,1) x/dO, He-normal W)",
            "config": {"workload": "resnet50_id5_1x1_bottleneck_fwd_bwd_upd (BASELINE configs[1])", **w,
                       "global_batch": w["N"] * world, "parallelism": f"dp{world}",
                       "math": "fp32-accurate bf16x3 split (6 products, fp32 accumulate)" if math == d.Math.F32
                       else "bf16 operands, fp32 accumulate",
                       "l2": "flushed between timed steps (256 MiB write + read-back, untimed)",
                       "step_order": "forward, then backward-data || weight update (side stream, joined)",
                       "tiles": {"fwd": fplan.blocking, "bwd": bctx.blocking, "upd": uplan.blocking}},
            "e2e": {"value": round(e2e_value, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "dconv_host_step_run (pinned host blocked tensors)",
                    "chunk_images": hstep.chunk, "ms_per_step": round(float(e2e_ms.item()), 4),
                    "gpu_launches_per_step": hstep.launches()},
            "gpu_launches": launches * args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": sampler.report(),
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


# ---------------------------------------------------------------------- ResNet-50 conv stack (cfg4)


def stack_cpu_reference(threads, n_img=2):
    """Reference direct engine on every distinct conv of the stack (F + B + U,
    one timed call each, plan setup excluded), N = n_img images, summed with
    the stack multiplicities; the stem's backward-data is skipped."""
    from oracle import oracle as orc
    from paper_1808_05567_b200 import executor as ex

    nodes = ex.resnet50_conv_stack()
    shapes = ex.tensor_shapes(nodes)
    mult = {}
    for nd in nodes:
        if isinstance(nd, ex.ConvNode):
            c, h, w = shapes[nd.src]
            key = (nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, nd.pad, nd.src == "x")
            mult[key] = mult.get(key, 0) + 1
    total = 0.0
    for (C, K, H, W, R, S, st, pad, stem), m in mult.items():
        s = orc.spec(n_img, C, K, H, W, R, S, st, pad, pad, 16)
        P, Q = orc.output_shape(s)
        x = orc.uniform(0, (n_img, C, H, W))
        wt = orc.he_normal(1, (K, C, R, S), C * R * S)
        g = orc.uniform(2, (n_img, K, P, Q))
        t = 0.0
        for pss, (a, b) in enumerate(((x, wt), (g, wt), (x, g))):
            if pss == 1 and stem:
                continue
            _, best, _ = orc.ref_direct_pass(s, pss, threads, 1, a, b)
            t += best / 1e3
        total += m * t
    return n_img / total, f"reference direct engine (oracle/_ref), {n_img} images x {len(mult)} distinct convs, F+B+U"


def run_stack(args):
    import numpy as np
    import torch

    import paper_1808_05567_b200 as d
    from paper_1808_05567_b200 import _lib
    from paper_1808_05567_b200 import executor as ex

    world, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as orc

        threads = os.cpu_count() or 1
        if not orc.ref_available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}), flush=True)
            return 0
        times = []
        for _ in range(max(1, args.steps // 10)):
            ips, sample = stack_cpu_reference(threads)
            times.append(ips)
        value = sum(times) / len(times)
        line = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "images/s", "n_gpus": world,
                "steps": len(times), "warmup": 0, "ms_per_step": round(256 / value * 1e3, 1),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded splitmix64)",
                "config": {"workload": "resnet50_conv_stack (BASELINE configs[3])", "global_batch": 256,
                           "parallelism": "cpu threads"},
                "cpu_baseline": {"value": round(value, 4), "unit": "images/s", "cores": threads, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": round(value, 4), "unit": "images/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

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
    e = ex.ConvStackExecutor(nodes, n, 224, d.Math.BF16, "cuda", group=pg, lr=1e-5)
    lib = _lib.lib()
    # seeded synthetic images (rank shard) and top gradient
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
    stream = torch.cuda.current_stream()

    def pack_input():
        e.load_input_nchw(x_dev)

    x_dev.copy_(x_pin)
    pack_input()

    def step():
        e.step(dtop)

    def loss_of_step():
        top = e.act[nodes[-1].out].data
        loss_dev.copy_((top.float() * dtop.data.float()).sum().reshape(1))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    graph = None
    if world == 1 and not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        torch.cuda.synchronize()
        run = graph.replay
    else:
        run = step
    launches = e.launches_per_step()

    def barrier():
        if pg is not None:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with sampler:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            run()
        e1.record(stream)
        barrier()
    ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if pg is not None:
        import torch.distributed as dist

        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_per_step = float(ms.item())
    value = global_batch / (ms_per_step * 1e-3)
    # end to end: H2D of this step's images (pinned), pack, step, loss D2H
    h2d = x_pin.numel() * 4

    # input pipeline as a training loop runs it: the NEXT step's images are copied
    # H2D on a side stream into the other of two device buffers while this step
    # computes (every step's copy is inside the timed region; the first one is
    # issued after the start event)
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
        loss_of_step()
        loss_pin.copy_(loss_dev, non_blocking=True)

    for b in range(2):
        consumed[b].record(stream)
    issue_copy(0)
    for i in range(2):
        e2e_step(i, i == 1)
    barrier()
    e0.record(stream)
    copy_stream.wait_event(e0)  # the first copy starts inside the timed region
    issue_copy(0)
    for i in range(args.steps):
        e2e_step(i, i == args.steps - 1)
    e1.record(stream)
    barrier()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if pg is not None:
        import torch.distributed as dist

        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = global_batch / (float(e2e_ms.item()) * 1e-3)
    hbm_peak, bf16_peak, peak_src = measured_peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sustained = float(json.load(f).get("bf16_tflops_sustained", bf16_peak))
    except (OSError, ValueError):
        sustained = bf16_peak
    flops_img = ex.step_flops_per_image(nodes)
    achieved = flops_img * n / (ms_per_step * 1e-3) / 1e12
    cpu = None
    if world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as orc

            if orc.ref_available():
                ips, sample = stack_cpu_reference(os.cpu_count() or 1)
                cpu = {"value": round(ips, 4), "unit": "images/s", "cores": os.cpu_count(), "kind": "reference",
                       "sample": sample}
        except Exception as ex_:  # noqa: BLE001
            cpu = {"value": None, "unit": "images/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex_}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "images/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded splitmix64 images 3x224x224 and top gradient; He-normal weights)",
            "config": {"workload": "resnet50_conv_stack (BASELINE configs[3]): 53 convs F+B+U, ReLU/residual fused,"
                                   " stem max-pool, SGD, NCCL dW all-reduce", "global_batch": global_batch,
                       "per_gpu_batch": n, "image": 224, "parallelism": f"dp{world}",
                       "cuda_graph": graph is not None, "l2": "working set >> L2 (activations ~GBs)"},
            "e2e": {"value": round(e2e_value, 2), "unit": "images/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 4,
                    "pipeline": "step i+1's images copied H2D (pinned) on a side stream during step i; pack, step, "
                                "loss D2H every step"},
            "gpu_launches": launches * args.steps,
            "roofline": {"bound": "tensor", "kernel": "whole step (53 convs x F/B/U)", "achieved": round(achieved, 1),
                         "peak": sustained, "unit": "TFLOP/s", "frac": round(achieved / sustained, 4),
                         "traffic": None, "peak_source": peak_src + " bf16_tflops_sustained",
                         "flops_per_image": flops_img},
            "cpu_baseline": cpu,
            "clocks": sampler.report(),
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--math", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--workload", default="layer", choices=["layer", "resnet50"])
    ap.add_argument("--global-batch", type=int, default=256)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--chunk", type=int, default=8, help="images per host-step chunk (e2e); 0 = N/4")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.workload == "resnet50":
        return run_stack(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
