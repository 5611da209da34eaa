"""Dev tool: bf16 weight-update kernel time (library event brackets) of LAYERS under
ablation bits MODES (dev build: 8 no MMAs, 256 no operand loads, 512 no input
loads, 1024 no dO loads) and plan overrides from the environment."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
N = int(os.environ.get("N", "256"))
lib.dconv_profile(1)
for lay in os.environ.get("LAYERS", "64,64,56,3 128,128,28,3 256,256,14,3 512,512,7,3").split():
    C, K, H, R = (int(v) for v in lay.split(","))
    pad = (R - 1) // 2
    spec = d.make_layer_spec(N, C, K, H, H, R, R, 1, pad, pad, 16)
    x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    x.data.uniform_(-1, 1)
    g = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    g.data.uniform_(-1, 1)
    dw = d.BlockedWeight(K, C, R, R)
    up = d.UpdatePlan(spec, None, d.Math.BF16)
    up.execute(x, g, dw)
    b = up.blocking
    print(lay, {k: b[k] for k in ("mode", "wsub", "rows_ps", "vs", "a_px", "nb", "tap_groups", "tg", "splits",
                                  "stages", "smem", "grid", "xs", "pimg", "sw32") if k in b})
    res = []
    for mode in [int(m) for m in os.environ.get("MODES", "0 8 256 264 512 1024 2048 4096 4360").split()]:
        lib.dconv_debug_mode(mode)
        ts = []
        for i in range(7):
            up.execute(x, g, dw)
            torch.cuda.synchronize()
            ts.append(lib.dconv_profile_last_ms(2) * 1e3)
        ts.sort()
        res.append("%d:%.1f" % (mode, ts[len(ts) // 2]))
    lib.dconv_debug_mode(0)
    print("   upd kernel us", " ".join(res))
