"""Dev tool: one bf16 pass (F, B or U) of one layer shape, launched a few times (for ncu captures).
Usage: one_layer.py C K H R [passes] [N]"""
import sys
import os

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402

C, K, H, R = (int(v) for v in sys.argv[1:5])
passes = sys.argv[5] if len(sys.argv) > 5 else "f"
N = int(sys.argv[6]) if len(sys.argv) > 6 else 256
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
for _ in range(3):
    if "f" in passes:
        fp.execute(x, w, y)
    if "b" in passes:
        bc.execute(w, g, dx)
    if "u" in passes:
        up.execute(x, g, dw)
torch.cuda.synchronize()
print("done", fp.blocking if "f" in passes else "")
