"""Dev tool: per-layer / per-pass device time of the ResNet-50 conv stack (bf16)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200.api import _check as _chk  # noqa: E402
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
lib = e.lib
lib.dconv_profile(1)
rows = []
# re-run pass by pass, timing each library call with events
st = torch.cuda.current_stream()


def timed(fn, reps=3, trials=3):
    """device time per call: mean of `reps` back-to-back calls queued behind a spin
    (host launch gaps not timed), best of `trials` (a host stall longer than the
    spin would otherwise be timed as device idle)"""
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(trials):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)
        a.record(st)
        for _ in range(reps):
            fn()
        b.record(st)
        b.synchronize()
        best = min(best, a.elapsed_time(b) / reps)
    return best


peak = 1332.6
tot = {"F": 0.0, "B": 0.0, "U": 0.0}
for nd in e.convs:
    s = e.specs[nd.name]
    fl = 2 * s.N * s.K * s.C * s.P() * s.Q() * s.R * s.S
    tf = timed(lambda: e.conv_forward(nd))
    tu = timed(lambda: e.conv_update(nd))
    tb = 0.0
    if nd.name in e.bplan:
        bp = e.bplan[nd.name]
        wsb = bp._ws.get(lib.dconv_bwd_workspace_bytes(bp._h), e.dev)
        tb = timed(lambda: _chk(lib.dconv_backward_data(bp._h, C.byref(e.w[nd.name].to_c()),
                                                            C.byref(e.grad[nd.out].to_c()),
                                                            C.byref(e.grad[nd.src].to_c()), wsb, st.cuda_stream)))
    tot["F"] += tf
    tot["B"] += tb
    tot["U"] += tu
    rows.append((nd.name, s.C, s.K, s.H, s.R, s.stride, fl, tf, tb, tu))
print(f"{'layer':8s} {'C':>5s} {'K':>5s} {'H':>4s} R st  {'GF':>6s}  F_ms  F_TF  B_ms  B_TF  U_ms  U_TF")
for r in rows:
    name, C_, K, H, R, st_, fl, tf, tb, tu = r
    print(f"{name:8s} {C_:5d} {K:5d} {H:4d} {R} {st_}  {fl/1e9:6.1f} {tf:5.2f} {fl/tf/1e9:5.0f} {tb:5.2f} "
          f"{(fl/tb/1e9 if tb else 0):5.0f} {tu:5.2f} {fl/tu/1e9:5.0f}")
print("totals ms", {k: round(v, 2) for k, v in tot.items()}, "sum", round(sum(tot.values()), 2))
