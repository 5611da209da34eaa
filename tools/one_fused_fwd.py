"""Dev tool: the executor's fused forward of one bf16 layer (residual add + ReLU in the
epilogue), launched three times (for ncu captures). Usage: one_fused_fwd.py C K H [N]"""
import ctypes as Ct
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402
from paper_1808_05567_b200._lib import Epilogue  # noqa: E402

C, K, H = (int(v) for v in sys.argv[1:4])
N = int(sys.argv[4]) if len(sys.argv) > 4 else 256
lib = _lib.lib()
spec = d.make_layer_spec(N, C, K, H, H, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
x.data.uniform_(-1, 1)
res = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
res.data.uniform_(-1, 1)
y = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
w = d.BlockedWeight(K, C, 1, 1)
w.data.normal_()
fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
ep = Epilogue(res.data.data_ptr(), None, 1, 0)
ws = fp._ws.get(lib.dconv_fwd_workspace_bytes(fp._h), torch.device("cuda"))
for _ in range(3):
    d.api._check(lib.dconv_forward_ex(fp._h, Ct.byref(x.to_c()), Ct.byref(w.to_c()), Ct.byref(y.to_c()), Ct.byref(ep),
                                      ws, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print(fp.blocking)
