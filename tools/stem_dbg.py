import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_1808_05567_b200 as d
from oracle import oracle as orc
for H, K in [(20, 16), (56, 16), (112, 16), (224, 16), (224, 64), (112, 64)]:
    for M in (d.Math.F32, d.Math.BF16):
        s = orc.spec(1, 3, K, H, H, 7, 7, 2, 3, 3, 16)
        ds = d.make_layer_spec(1, 3, K, H, H, 7, 7, 2, 3, 3, 16)
        x = orc.uniform(0, (1, 3, H, H)); w = orc.he_normal(1, (K, 3, 7, 7), 147)
        ib = d.to_blocked_activation(torch.from_numpy(x).cuda(), ds); wb = d.to_blocked_weight(torch.from_numpy(w).cuda(), ds)
        plan = d.make_forward_plan(ds, 1, None, None, M)
        out = d.from_blocked_activation(d.forward(ds, ib, wb, plan)).cpu().numpy()
        n = orc.error_norms(orc.conv_forward(s, x, w), out)
        print(H, K, M.name, f"{n['max_over_rms']:.2e}", plan.blocking, flush=True)
