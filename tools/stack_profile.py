"""Dev tool: per-layer / per-pass device time of the ResNet-50 conv stack (bf16),
each pass alone (native dconv_graph_profile), against its per-layer roof."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import executor as ex  # noqa: E402

N = int(os.environ.get("N", "256"))
if os.environ.get("DBG"):  # dev lib: ablation / issue-loop bits (before any plan is built)
    from paper_1808_05567_b200 import _lib
    _lib.lib().dconv_debug_mode(int(os.environ["DBG"]))
nodes = ex.resnet50_conv_stack()
e = ex.ConvStackExecutor(nodes, N, 224, d.Math.BF16, "cuda", lr=0.0)
c, h, w = e.shapes[nodes[-1].out]
dtop = d.BlockedActivation(N, c, h, w, 16, 0, 0, torch.bfloat16)
dtop.data.uniform_(-1, 1)
x = torch.empty(N, 3, 224, 224, device="cuda").uniform_(-1, 1)
e.load_input_nchw(x)
prof = e.profile(dtop)
hbm, peak, _, _ = bench.measured_peaks()
fused = bench.fused_operand_bytes(e, N)
tot = {"F": 0.0, "B": 0.0, "U": 0.0}
troof = {"F": 0.0, "B": 0.0, "U": 0.0}
print(f"{'layer':7s} {'C':>5s} {'K':>5s} {'H':>4s} R s  " + "  ".join(f"{p}_ms  roof  frac" for p in "FBU"))
for nd in e.convs:
    cc, hh, ww = e.shapes[nd.src]
    wl = dict(N=N, C=nd.C, K=nd.K, H=hh, W=ww, R=nd.R, S=nd.S, stride=nd.stride, pad_h=nd.pad, pad_w=nd.pad)
    fl = bench.pass_flops(wl)
    byts = bench.alg_bytes(wl, 2, 2)
    byts = {k: v + fused[nd.name][k] for k, v in byts.items()}
    cols = []
    for p in "FBU":
        ms = prof[nd.name][p]
        r = bench.roof_ms(fl, byts[p], peak, hbm) if ms > 0 else 0.0
        tot[p] += ms
        troof[p] += r
        cols.append(f"{ms:5.3f} {r:5.3f} {(r / ms if ms else 0):4.2f}")
    print(f"{nd.name:7s} {nd.C:5d} {nd.K:5d} {hh:4d} {nd.R} {nd.stride}  " + "  ".join(cols))
print("totals ms", {k: round(v, 3) for k, v in tot.items()}, "sum", round(sum(tot.values()), 3))
print("roof ms  ", {k: round(v, 3) for k, v in troof.items()}, "sum", round(sum(troof.values()), 3))
