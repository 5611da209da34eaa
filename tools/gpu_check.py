"""Quick GPU parity sweep (dev tool): FWD / BWD / UPD vs the CPU oracle."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from oracle import oracle as orc  # noqa: E402

CASES = [
    # N, C, K, H, W, R, S, stride, pad_h, pad_w
    (2, 24, 16, 12, 12, 3, 3, 1, 1, 1),
    (2, 32, 48, 10, 10, 1, 1, 1, 0, 0),
    (2, 32, 32, 12, 12, 1, 1, 2, 0, 0),
    (2, 16, 16, 11, 11, 3, 3, 2, 0, 0),
    (1, 16, 32, 9, 9, 3, 3, 2, 1, 1),
    (2, 3, 16, 20, 20, 7, 7, 2, 3, 3),
    (2, 160, 160, 17, 17, 1, 7, 1, 0, 3),
    (2, 64, 64, 56, 56, 3, 3, 1, 1, 1),
    (2, 256, 64, 56, 56, 1, 1, 1, 0, 0),
]

which = sys.argv[1] if len(sys.argv) > 1 else "FBU"
maths = [d.Math.F32, d.Math.BF16]
worst = {}
for case in CASES:
    N, C_, K, H, W, R, S, st, ph, pw = case
    s = orc.spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    ds = d.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    P, Q = orc.output_shape(s)
    x = orc.uniform(0, (N, C_, H, W))
    w = orc.he_normal(1, (K, C_, R, S), C_ * R * S)
    g = orc.uniform(2, (N, K, P, Q))
    xt, wt, gt = (torch.from_numpy(a).cuda() for a in (x, w, g))
    for math in maths:
        tol = 1e-4 if math == d.Math.F32 else 2e-2
        if "F" in which:
            ref = orc.conv_forward(s, x, w)
            ib = d.to_blocked_activation(xt, ds)
            wb = d.to_blocked_weight(wt, ds)
            plan = d.make_forward_plan(ds, 1, None, None, math)
            t0 = time.time()
            out = d.forward(ds, ib, wb, plan)
            got = d.from_blocked_activation(out).cpu().numpy()
            n = orc.error_norms(ref, got)
            print(f"F {case} {math.name}: e={n['max_over_rms']:.2e} l2rel={n['l2_rel']:.2e} "
                  f"{'PASS' if n['max_over_rms'] <= tol else 'FAIL'} {plan.blocking}", flush=True)
        if "B" in which:
            ref = orc.conv_backward(s, g, w)
            gb = d.to_blocked_activation(gt, 16, 0, 0)
            wb = d.to_blocked_weight(wt, ds)
            ctx = d.prepare_backward(ds, wb, 1, None, math)
            gi = d.backward_with(ctx, gb)
            got = d.from_blocked_activation(gi).cpu().numpy()
            n = orc.error_norms(ref, got)
            print(f"B {case} {math.name} route={ctx.route.name}: e={n['max_over_rms']:.2e} l2rel={n['l2_rel']:.2e} "
                  f"{'PASS' if n['max_over_rms'] <= tol else 'FAIL'}", flush=True)
        if "U" in which:
            ref = orc.conv_update(s, x, g)
            ib = d.to_blocked_activation(xt, ds)
            gb = d.to_blocked_activation(gt, 16, 0, 0)
            dw = d.weight_update(ds, ib, gb, None, dtype=math)
            got = d.from_blocked_weight(dw).cpu().numpy()
            n = orc.error_norms(ref, got)
            print(f"U {case} {math.name}: e={n['max_over_rms']:.2e} l2rel={n['l2_rel']:.2e} "
                  f"{'PASS' if n['max_over_rms'] <= tol else 'FAIL'}", flush=True)
