"""Dev tool: CUPTI kernel trace (torch.profiler) of the cfg2 F+B+U step, L2
flushed between steps as in bench.py: per-kernel device time and the step's
critical path (first kernel start -> last kernel end)."""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402

math = d.Math.BF16 if "bf16" in sys.argv else d.Math.F32
N = 32
spec = d.make_layer_spec(N, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, 256, 56, 56)
x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, 64, 56, 56)
g.data.uniform_(-1, 1)
w = d.BlockedWeight(64, 256, 1, 1)
w.data.normal_()
y, dx, dw = d.BlockedActivation(N, 64, 56, 56), d.BlockedActivation(N, 256, 56, 56), d.BlockedWeight(64, 256, 1, 1)
fp = d.make_forward_plan(spec, 1, None, None, math)
bc = d.prepare_backward(spec, w, 1, None, math)
up = d.UpdatePlan(spec, None, math)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


def step():
    fp.execute(x, w, y)
    bc.execute(w, g, dx)
    up.execute(x, g, dw)


for _ in range(3):
    step()
torch.cuda.synchronize()
STEPS = 10
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(STEPS):
        flush.fill_(i)
        torch.cuda._sleep(1_000_000)
        step()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = [e for e in evs if "dconv" in e.name or "conv_" in e.name]
agg = collections.defaultdict(list)
for e in kern:
    agg[e.name[:70]].append(e.device_time)  # us
tot = 0.0
for k, v in agg.items():
    tot += sum(v) / STEPS
    print(f"{sum(v) / len(v):8.2f} us x{len(v) // STEPS}  {k}")
print("sum of kernels per step (us):", round(tot, 2))
# critical path per step: kernels between flush fills
kern.sort(key=lambda e: e.time_range.start)
per = len(kern) // STEPS
spans = [kern[i * per + per - 1].time_range.end - kern[i * per].time_range.start for i in range(STEPS)]
print("span first->last kernel per step (us):", [round(s, 1) for s in spans])
print("last step, kernel by kernel (start offset us, duration us):")
t0 = kern[(STEPS - 1) * per].time_range.start
for e in kern[(STEPS - 1) * per:]:
    print(f"  {e.time_range.start - t0:8.1f} {e.device_time:8.2f}  {e.name[:60]}")
