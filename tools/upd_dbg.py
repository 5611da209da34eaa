import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_1808_05567_b200 as d
from paper_1808_05567_b200 import _lib
lib = _lib.lib()
N = int(os.environ.get("N", "4"))
mode = int(sys.argv[1])
spec = d.make_layer_spec(N, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, 256, 56, 56); x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, 64, 56, 56); g.data.uniform_(-1, 1)
dw = d.BlockedWeight(64, 256, 1, 1)
up = d.UpdatePlan(spec, None, d.Math.F32)
lib.dconv_debug_mode(mode)
up.execute(x, g, dw)
torch.cuda.synchronize()
print("mode", mode, up.blocking)
