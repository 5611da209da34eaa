"""Dev tool: per ResNet-50 layer shape (executor view: strided 1x1 run at stride 1 on
the lattice copy), the bf16 UPD plan's split count, partial bytes, and the UPD
kernel vs whole-call (kernel + split reduce) time."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402
from paper_1808_05567_b200 import executor as ex  # noqa: E402

lib = _lib.lib()
N = int(os.environ.get("N", "256"))
nodes = [nd for nd in ex.resnet50_conv_stack() if isinstance(nd, ex.ConvNode)]
shapes = ex.tensor_shapes(ex.resnet50_conv_stack())
seen = {}
for nd in nodes:
    c, h, w = shapes[nd.src]
    st, R = nd.stride, nd.R
    if R == 1 and st == 2:
        h, w, st = (h + 1) // 2, (w + 1) // 2, 1
    key = (nd.C, nd.K, h, R, st)
    seen.setdefault(key, []).append(nd.name)
lib.dconv_profile(1)
tot_k = tot_c = 0.0
for (C, K, H, R, st), names in seen.items():
    if C < 16:
        continue
    pad = (R - 1) // 2 if R > 1 else 0
    spec = d.make_layer_spec(N, C, K, H, H, R, R, st, pad, pad, 16)
    P = (H + 2 * pad - R) // st + 1
    x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    x.data.uniform_(-1, 1)
    g = d.BlockedActivation(N, K, P, P, 16, 0, 0, torch.bfloat16)
    g.data.uniform_(-1, 1)
    dw = d.BlockedWeight(K, C, R, R)
    up = d.UpdatePlan(spec, None, d.Math.BF16)
    up.execute(x, g, dw)
    b = up.blocking
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks, cs = [], []
    for i in range(7):
        torch.cuda.synchronize()
        e0.record()
        up.execute(x, g, dw)
        e1.record()
        torch.cuda.synchronize()
        ks.append(lib.dconv_profile_last_ms(2) * 1e3)
        cs.append(e0.elapsed_time(e1) * 1e3)
    ks.sort()
    cs.sort()
    part_mb = b["splits"] * R * R * C * K * 4 / 1e6
    n = len(names)
    tot_k += n * ks[3]
    tot_c += n * cs[3]
    print(f"{C:5d}->{K:5d} {R}x{R} @{H:3d} x{n}: splits {b['splits']:3d} grid {b['grid']} partial {part_mb:7.1f} MB "
          f"kernel {ks[3]:6.1f} us call {cs[3]:6.1f} us (reduce ~{cs[3] - ks[3]:5.1f})")
print(f"sum over the stack: kernels {tot_k / 1e3:.3f} ms, calls {tot_c / 1e3:.3f} ms")
