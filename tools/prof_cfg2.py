"""Profiling driver: cfg2 (N=32 1x1 256->64 @56^2) F, B, U once each after warm-up."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402

math = d.Math.BF16 if (len(sys.argv) > 1 and sys.argv[1] == "bf16") else d.Math.F32
spec = d.make_layer_spec(32, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = torch.rand(32, 256, 56, 56, device="cuda") * 2 - 1
w = torch.randn(64, 256, 1, 1, device="cuda") * 0.088
g = torch.rand(32, 64, 56, 56, device="cuda") * 2 - 1
ib, wb, gb = d.to_blocked_activation(x, spec), d.to_blocked_weight(w, spec), d.to_blocked_activation(g, 16, 0, 0)
fp = d.make_forward_plan(spec, 1, None, None, math)
bc = d.prepare_backward(spec, wb, 1, None, math)
up = d.UpdatePlan(spec, None, math)
out = d.BlockedActivation(32, 64, 56, 56, 16, 0, 0)
gi = d.BlockedActivation(32, 256, 56, 56, 16, 0, 0)
dw = d.BlockedWeight(64, 256, 1, 1, 16)
for _ in range(int(os.environ.get("ITERS", "3"))):
    fp.execute(ib, wb, out)
    bc.execute(wb, gb, gi)
    up.execute(ib, gb, dw)
torch.cuda.synchronize()
print("ok")
