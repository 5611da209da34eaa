"""Dev tool: cfg2 UPD kernel time (library event brackets, L2 flushed) under ablation bits."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
N = 32
spec = d.make_layer_spec(N, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, 256, 56, 56)
x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, 64, 56, 56)
g.data.uniform_(-1, 1)
dw = d.BlockedWeight(64, 256, 1, 1)
up = d.UpdatePlan(spec, None, d.Math.F32)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
lib.dconv_profile(1)
for mode in [int(m) for m in os.environ.get("MODES", "0 4 8 12").split()]:
    lib.dconv_debug_mode(mode)
    ts = []
    for i in range(8):
        flush.fill_(i)
        flush.view(torch.int32).sum()
        torch.cuda._sleep(2_000_000)
        up.execute(x, g, dw)
        torch.cuda.synchronize()
        ts.append(lib.dconv_profile_last_ms(2) * 1e3)
    ts.sort()
    print("mode", mode, "upd kernel us", round(ts[len(ts) // 2], 1))
lib.dconv_debug_mode(0)
print(up.blocking)
