import os, sys, ctypes as C, torch
sys.path.insert(0, "/root/repo")
import paper_1808_05567_b200 as d
from paper_1808_05567_b200 import executor as ex
N = 256
nodes = ex.resnet50_conv_stack()
e = ex.ConvStackExecutor(nodes, N, 224, d.Math.BF16, "cuda", lr=0.0)
e.act["x"].data.uniform_(-1, 1)
nd = e.convs[0]
sd = e.s2d[nd.name]
st = torch.cuda.current_stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps): fn()
    b.record(st); b.synchronize()
    return a.elapsed_time(b) / reps * 1e3
lib = e.lib
print("s2d_act us", timed(lambda: lib.dconv_s2d_act(C.byref(e.act["x"].to_c()), C.byref(sd["x"].to_c()), 3, st.cuda_stream)))
print("s2d_wt us", timed(lambda: lib.dconv_s2d_wt(C.byref(e.w["stem"].to_c()), C.byref(sd["w"].to_c()), 0, st.cuda_stream)))
print("conv_forward (all) us", timed(lambda: e.conv_forward(nd)))
print("conv_update (all) us", timed(lambda: e.conv_update(nd)))
print("fwd plan", e.fplan["stem"].blocking)
print("upd plan", e.uplan["stem"].blocking)
