"""Dev tool: cfg2 kernel time of one pass (F, B or U; library event brackets,
L2 flushed) under ablation bits of dconv_debug_mode. Usage: pass_ablate.py F 0 4 8"""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
which = sys.argv[1]
modes = [int(m) for m in sys.argv[2:]] or [0]
math = d.Math.BF16 if os.environ.get("MATH") == "bf16" else d.Math.F32
N = 32
spec = d.make_layer_spec(N, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, 256, 56, 56)
x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, 64, 56, 56)
g.data.uniform_(-1, 1)
w = d.BlockedWeight(64, 256, 1, 1)
w.data.normal_()
y, dx, dw = d.BlockedActivation(N, 64, 56, 56), d.BlockedActivation(N, 256, 56, 56), d.BlockedWeight(64, 256, 1, 1)
cfg = None
if os.environ.get("NB") or os.environ.get("STAGES"):
    cfg = d.EngineConfig(tile_nb=int(os.environ.get("NB", "0")), stages=int(os.environ.get("STAGES", "0")))
fp = d.make_forward_plan(spec, 1, None, cfg, math)
bc = d.prepare_backward(spec, w, 1, cfg, math)
up = d.UpdatePlan(spec, None, math)
run, slot, plan = {"F": (lambda: fp.execute(x, w, y), 0, fp), "B": (lambda: bc.execute(w, g, dx), 1, bc),
                   "U": (lambda: up.execute(x, g, dw), 2, up)}[which]
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
lib.dconv_profile(1)
for mode in modes:
    lib.dconv_debug_mode(mode)
    ts = []
    for i in range(10):
        flush.fill_(i)
        flush.view(torch.int32).sum()
        torch.cuda._sleep(2_000_000)
        run()
        torch.cuda.synchronize()
        ts.append(lib.dconv_profile_last_ms(slot) * 1e3)
    ts.sort()
    print(which, "mode", mode, "kernel us", round(ts[len(ts) // 2], 2), "min", round(ts[0], 2))
lib.dconv_debug_mode(0)
print(plan.blocking)
if os.environ.get("PROBE"):
    import ctypes as C
    pl = C.CDLL(os.path.join(os.path.dirname(__file__), "probe_lib", "libprobe_reader.so"))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for ring, variant in ((3, 0), (3, 1), (3, 2)):
        ts = []
        for i in range(10):
            flush.fill_(i)
            flush.view(torch.int32).sum()
            torch.cuda._sleep(2_000_000)
            s.record()
            pl.probe_read(C.c_void_p(x.data.data_ptr()), N, 16, 56 * 56, ring, 4, variant,
                          C.c_void_p(torch.cuda.current_stream().cuda_stream))
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) * 1e3)
        ts.sort()
        print("probe reader on x, ring", ring, "variant", variant, "us", round(ts[len(ts) // 2], 2), "min", round(ts[0], 2))
