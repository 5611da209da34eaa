"""Dev tool: plan descriptions and device time of each bf16 pass for a list of layer shapes.
Usage: layer_plans.py "C,K,H,R[,N]" ..."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for arg in sys.argv[1:]:
    v = [int(t) for t in arg.split(",")]
    C, K, H, R = v[:4]
    N = v[4] if len(v) > 4 else 256
    pad = (R - 1) // 2
    spec = d.make_layer_spec(N, C, K, H, H, R, R, 1, pad, pad, 16)
    x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    x.data.uniform_(-1, 1)
    y = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    g = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    g.data.uniform_(-1, 1)
    dx = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    w = d.BlockedWeight(K, C, R, R)
    w.data.normal_()
    dw = d.BlockedWeight(K, C, R, R)
    fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
    bc = d.prepare_backward(spec, w, 1, None, d.Math.BF16)
    up = d.UpdatePlan(spec, None, d.Math.BF16)
    tf = timed(lambda: fp.execute(x, w, y))
    tb = timed(lambda: bc.execute(w, g, dx))
    tu = timed(lambda: up.execute(x, g, dw))
    fl = 2.0 * N * H * H * C * K * R * R
    print(f"== {C}->{K} @{H} {R}x{R} N={N}: F {tf*1e3:.1f} us ({fl/tf/1e9:.0f} TF)  B {tb*1e3:.1f} us  U {tu*1e3:.1f} us")
    for nm, pl in (("F", fp), ("B", bc), ("U", up)):
        try:
            print("  ", nm, json.dumps(pl.blocking))
        except Exception as exc:  # noqa: BLE001
            print("  ", nm, "describe failed:", exc)
