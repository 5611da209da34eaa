"""Dev tool: per-stage timestamps (CTA 0) and per-role cycle counters of one bf16
forward launch of a given layer. Env: LAYER="C,K,H,R" (default 128,128,28,3), N,
DBG (ablation bits), plus any plan override env (DCONV_WCAP ...)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import ctypes as Ct  # noqa: E402

import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
lib.dconv_debug_counters.argtypes = [Ct.c_void_p]
C, K, H, R = (int(v) for v in os.environ.get("LAYER", "128,128,28,3").split(","))
N = int(os.environ.get("N", "256"))
pad = int(os.environ.get("PAD", (R - 1) // 2))
spec = d.make_layer_spec(N, C, K, H, H, R, R, 1, pad, pad, 16)
x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
x.data.uniform_(-1, 1)
P_ = H + 2 * pad - R + 1
y = d.BlockedActivation(N, K, P_, P_, 16, 0, 0, torch.bfloat16)
w = d.BlockedWeight(K, C, R, R)
w.data.normal_()
fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
if os.environ.get("ADD"):  # the executor's fused residual-add + ReLU epilogue
    from paper_1808_05567_b200._lib import Epilogue
    res = d.BlockedActivation(N, K, P_, P_, 16, 0, 0, torch.bfloat16)
    res.data.uniform_(-1, 1)
    ep = Epilogue(res.data.data_ptr(), None, 1)
    ws = fp._ws.get(lib.dconv_fwd_workspace_bytes(fp._h), torch.device("cuda"))

    def _fwd(a, b, c):
        d.api._check(lib.dconv_forward_ex(fp._h, Ct.byref(a.to_c()), Ct.byref(b.to_c()), Ct.byref(c.to_c()), Ct.byref(ep),
                                      ws, torch.cuda.current_stream().cuda_stream))
    fp.execute = _fwd
print(fp.blocking)
buf = torch.zeros(148 * 16 + 8 * 256 + 2 * 148 + 5 * 148, dtype=torch.int64, device="cuda")
lib.dconv_debug_mode(int(os.environ.get("DBG", "0")))
fp.execute(x, w, y)
torch.cuda.synchronize()
lib.dconv_debug_counters(buf.data_ptr())
fp.execute(x, w, y)
torch.cuda.synchronize()
lib.dconv_debug_counters(None)
per = buf[:148 * 16].view(148, 16)
g0 = per[:, 9].min().item()
starts = (per[:, 9] - g0).double() / 1e3
ends = (per[:, 10] - g0).double() / 1e3
print("CTA start us min %.2f max %.2f | end us min %.2f max %.2f | total kcyc max %.1f" % (
    starts.min().item(), starts.max().item(), ends.min().item(), ends.max().item(), per[:, 8].max().item() / 1e3))
names = {0: "prod_wait", 4: "mma_wait_ops", 5: "mma_wait_acc", 6: "epi_wait", 7: "epi_busy", 8: "total"}
print({n: round(per[:, i].double().mean().item() / 1e3, 1) for i, n in names.items()}, "(kcyc, mean over CTAs)")
tr = buf[148 * 16:148 * 16 + 2048].view(256, 8).tolist()
print("stage: prod_issue wprod_issue | mma: a_seen w_seen issued   (cycles from CTA start)")
for i in range(0, int(os.environ.get("STAGES", "48"))):
    t = tr[i]
    print(i, t[6], t[7], "|", t[0], t[1], "loop_end", t[3], "commit1", t[4], "issued", t[2])
