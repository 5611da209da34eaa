"""Dev tool: bf16 1x1 forward / backward-data of small-plane layers against a float32 torch
convolution of the same bf16-rounded operands, with device times and the chosen plans.
Usage: mimg_check.py "C,K,H[,N]" ...   (plan env knobs apply: DCONV_DEV=1 DCONV_MIMG_MB1=1 ...)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

if os.environ.get("DCONV_DEV"):
    _lib.lib().dconv_set_dev_mode(1)  # DCONV_* overrides act only in developer mode


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
    C, K, H = v[:3]
    N = v[3] if len(v) > 3 else 256
    torch.manual_seed(C + K + H)
    spec = d.make_layer_spec(N, C, K, H, H, 1, 1, 1, 0, 0, 16)
    xt = torch.empty(N, C, H, H, device="cuda").uniform_(-1, 1).bfloat16().float()
    wt = (torch.randn(K, C, 1, 1, device="cuda") * (2.0 / C) ** 0.5).bfloat16().float()
    gt = torch.empty(N, K, H, H, device="cuda").uniform_(-1, 1).bfloat16().float()
    x = d.to_blocked_activation(xt, 16, 0, 0, torch.bfloat16)
    g = d.to_blocked_activation(gt, 16, 0, 0, torch.bfloat16)
    w = d.to_blocked_weight(wt, spec)
    y = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    dx = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
    bc = d.prepare_backward(spec, w, 1, None, d.Math.BF16)
    fp.execute(x, w, y)
    bc.execute(w, g, dx)
    ry = torch.nn.functional.conv2d(xt, wt)
    rdx = torch.nn.functional.conv_transpose2d(gt, wt)
    ey = (d.from_blocked_activation(y).float() - ry).abs().max().item() / ry.pow(2).mean().sqrt().item()
    edx = (d.from_blocked_activation(dx).float() - rdx).abs().max().item() / rdx.pow(2).mean().sqrt().item()
    tf = timed(lambda: fp.execute(x, w, y))
    tb = timed(lambda: bc.execute(w, g, dx))
    print(f"== {C}->{K} @{H} N={N}: F {tf*1e3:.1f} us err {ey:.2e}   B {tb*1e3:.1f} us err {edx:.2e}")
    print("   F", json.dumps(fp.blocking))
