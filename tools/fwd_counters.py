"""Dev tool: per-role cycle counters of the forward kernel (cfg2 FWD / BWD)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
lib.dconv_debug_counters.argtypes = [C.c_void_p]
lib.dconv_debug_mode(int(os.environ.get("DBG_MODE", "0")))
math = d.Math.BF16 if (len(sys.argv) > 1 and sys.argv[1] == "bf16") else d.Math.F32
Nn, Cc, Kk, Hh, Rr = (int(v) for v in os.environ.get("LAYER", "32,256,64,56,1").split(","))
pad = (Rr - 1) // 2
spec = d.make_layer_spec(Nn, Cc, Kk, Hh, Hh, Rr, Rr, 1, pad, pad, 16)
x = torch.rand(Nn, Cc, Hh, Hh, device="cuda") * 2 - 1
w = torch.randn(Kk, Cc, Rr, Rr, device="cuda") * 0.088
g = torch.rand(Nn, Kk, Hh, Hh, device="cuda") * 2 - 1
ib, wb, gb = d.to_blocked_activation(x, spec), d.to_blocked_weight(w, spec), d.to_blocked_activation(g, 16, 0, 0)
if math == d.Math.BF16:
    ib = d.BlockedActivation(Nn, Cc, Hh, Hh, 16, 0, 0, torch.bfloat16)
    ib.data.uniform_(-1, 1)
    gb = d.BlockedActivation(Nn, Kk, Hh, Hh, 16, 0, 0, torch.bfloat16)
    gb.data.uniform_(-1, 1)
fp = d.make_forward_plan(spec, 1, None, None, math)
bc = d.prepare_backward(spec, wb, 1, None, math)
out = d.BlockedActivation(Nn, Kk, Hh, Hh, 16, 0, 0, *( [torch.bfloat16] if math == d.Math.BF16 else []))
gi = d.BlockedActivation(Nn, Cc, Hh, Hh, 16, 0, 0, *( [torch.bfloat16] if math == d.Math.BF16 else []))
buf = torch.zeros(148 * 16 + 8 * 256 + 2 * 148 + 5 * 148, dtype=torch.int64, device="cuda")
names = ["prod_wait", "cvt_wait_raw", "cvt_wait_slot", "cvt_busy", "mma_wait_ops", "mma_wait_acc", "epi_wait",
         "epi_busy", "total"]
for label, run in (("fwd", lambda: fp.execute(ib, wb, out)), ("bwd", lambda: bc.execute(wb, gb, gi))):
    run()
    torch.cuda.synchronize()
    lib.dconv_debug_counters(buf.data_ptr())
    buf.zero_()
    if os.environ.get("FLUSH"):
        flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
        flush.fill_(1)
    run()
    torch.cuda.synchronize()
    lib.dconv_debug_counters(None)
    v = buf[:148 * 16].view(148, 16)[:, :9].double().mean(0).tolist()
    per = buf[:148 * 16].view(148, 16)
    g0 = per[:, 9].min().item()
    starts = (per[:, 9] - g0).double() / 1e3
    ends = (per[:, 10] - g0).double() / 1e3
    print(label, "CTA start us: min %.2f max %.2f | end us: min %.2f max %.2f | total kcyc max %.1f" % (
        starts.min().item(), starts.max().item(), ends.min().item(), ends.max().item(), per[:, 8].max().item() / 1e3),
        "epi bodies kcyc %.1f (tmem ld %.1f slab-wait %.1f fence %.1f tma %.1f)" % tuple(per[:, i].double().mean().item() / 1e3 for i in (11, 12, 13, 14, 15)))
    if os.environ.get("ENDS"):
        e = ends.tolist()
        order = sorted(range(148), key=lambda i: e[i])
        print(label, "fastest CTAs", [(i, round(e[i], 1)) for i in order[:8]])
        print(label, "slowest CTAs", [(i, round(e[i], 1)) for i in order[-12:]])
        print(label, "ends by CTA id (x10):", [round(sum(e[i:i + 10]) / len(e[i:i + 10]), 1) for i in range(0, 148, 10)])
    ex = buf[148 * 16 + 2048:148 * 16 + 2048 + 296].view(148, 2).double().mean(0) / 1e3
    mm = buf[148 * 16 + 2048 + 296:].view(148, 5).double().mean(0) / 1e3
    print(label, "MMA warp kcyc: wait %.1f misc %.1f fence %.1f issue %.1f commit %.1f" % tuple(mm.tolist()))
    print(label, "vals..relu kcyc %.1f staging kcyc %.1f" % (ex[0].item(), ex[1].item()))
    print(label, getattr(fp if label == "fwd" else bc, "blocking", None))
    if os.environ.get("TRACE") and label == "fwd":
        tr = buf[148 * 16:148 * 16 + 2048].view(256, 8).tolist()
        print("stage: prod_issue wprod_issue | cvt: raw_seen slot_free done | mma: conv_seen w_seen issued")
        for i in range(0, 100):
            t = tr[i]
            print(i, t[6], t[7], "|", t[3], t[4], t[5], "|", t[0], t[1], t[2])
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        run()
    e.record()
    torch.cuda.synchronize()
    print(label, math.name, "us/launch", round(s.elapsed_time(e) * 200, 1), {n: round(x / 1e3, 1) for n, x in zip(names, v)}, "(kcycles, mean over CTAs)")
