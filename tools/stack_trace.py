"""Dev tool: CUPTI kernel trace of one ResNet-50 conv-stack step (bf16, N from env),
aggregated by kernel name: where the non-conv time goes."""
import collections
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import executor as ex  # noqa: E402

N = int(os.environ.get("N", "256"))
nodes = ex.resnet50_conv_stack()
e = ex.ConvStackExecutor(nodes, N, 224, d.Math.BF16, "cuda", lr=0.0)
c, h, w = e.shapes[nodes[-1].out]
dtop = d.BlockedActivation(N, c, h, w, 16, 0, 0, torch.bfloat16)
dtop.data.uniform_(-1, 1)
e.act["x"].data.uniform_(-1, 1)
for _ in range(2):
    e.step(dtop)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e.step(dtop)
    torch.cuda.synchronize()
evs = [x for x in prof.events() if x.device_type == torch.autograd.DeviceType.CUDA]
agg = collections.defaultdict(lambda: [0, 0.0])
for x in evs:
    k = x.name.split("(")[0][:70]
    agg[k][0] += 1
    agg[k][1] += x.device_time
tot = sum(v[1] for v in agg.values())
span = max(x.time_range.end for x in evs) - min(x.time_range.start for x in evs)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / 1e3:8.2f} ms  x{v[0]:4d}  {k}")
print(f"sum {tot / 1e3:.2f} ms, span {span / 1e3:.2f} ms")

if os.environ.get("PER_LAUNCH"):
    seq = sorted([x for x in evs if "conv_fwd_kernel" in x.name or "conv_upd" in x.name], key=lambda x: x.time_range.start)
    names = [nd.name for nd in e.convs]
    # forward: one conv_fwd launch per conv in order; backward: reverse order, BWD (if any) then UPD
    i = 0
    print("FWD")
    for nm in names:
        print(f"  {nm:8s} {seq[i].device_time:8.1f} us")
        i += 1
    print("BWD/UPD (reverse)")
    for nm in reversed(names):
        row = []
        while i < len(seq) and len(row) < 2:
            row.append(f"{seq[i].name.split('<')[0][-12:]} {seq[i].device_time:7.1f}")
            i += 1
            if "conv_upd" in row[-1]:
                break
        print(f"  {nm:8s} " + " | ".join(row))
