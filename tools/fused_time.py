"""Dev tool: forward / backward-data of the ResNet-50 stack's convs WITH their
graph epilogues (residual add, ReLU mask), as the executor runs them, timed per
layer (N=256, bf16). Env DBG = ablation bits."""
import os, sys, ctypes as C, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import executor as ex  # noqa: E402
N = int(os.environ.get("N", "256"))
nodes = ex.resnet50_conv_stack()
e = ex.ConvStackExecutor(nodes, N, 224, d.Math.BF16, "cuda", lr=0.0)
e.act["x"].data.uniform_(-1, 1)
c, h, w = e.shapes[nodes[-1].out]
dtop = d.BlockedActivation(N, c, h, w, 16, 0, 0, torch.bfloat16)
dtop.data.uniform_(-1, 1)
e.step(dtop)
torch.cuda.synchronize()
e.lib.dconv_debug_mode(int(os.environ.get("DBG", "0")))
st = torch.cuda.current_stream()
def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(2_000_000)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps * 1e3
tot = 0.0
for nd in e.convs:
    if nd.add is None and not os.environ.get("ALL"):
        continue
    t = timed(lambda: e.conv_forward(nd))
    tot += t
    print(f"{nd.name:6s} F(fused) {t:7.1f} us")
print("total", round(tot, 1))
tf = timed(lambda: e.forward())
tb = timed(lambda: e.backward(dtop))
print(f"whole forward {tf:.1f} us, whole backward (incl. side-stream updates) {tb:.1f} us")
