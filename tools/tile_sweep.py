"""Dev tool: cfg2 pass times (CUDA events, L2 flushed) under tile overrides."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402

N = 32
spec = d.make_layer_spec(N, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
x = d.BlockedActivation(N, 256, 56, 56)
x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, 64, 56, 56)
g.data.uniform_(-1, 1)
w = d.BlockedWeight(64, 256, 1, 1)
w.data.normal_()
y, dx, dw = d.BlockedActivation(N, 64, 56, 56), d.BlockedActivation(N, 256, 56, 56), d.BlockedWeight(64, 256, 1, 1)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")


from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
lib.dconv_profile(1)
SLOT = {"fwd": 0, "bwd": 1, "upd": 2}


def timeit(fn, which, reps=10):
    """median conv-kernel device time (library event brackets), L2 flushed"""
    ts = []
    for i in range(reps):
        flush.fill_(i)
        flush.view(torch.int32).sum()
        torch.cuda._sleep(2_000_000)
        fn()
        torch.cuda.synchronize()
        ts.append(lib.dconv_profile_last_ms(SLOT[which]) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for nb in (0, 4, 6, 8, 16):
    for st in (0,):
        cfg = d.EngineConfig(tile_nb=nb, stages=st)
        try:
            bc = d.prepare_backward(spec, w, 1, cfg, d.Math.F32)
            t = timeit(lambda: bc.execute(w, g, dx), "bwd")
            print("bwd nb", nb, "stages", st, round(t, 1), "us", bc.blocking["phases"][0])
        except d.Error as e:
            print("bwd nb", nb, "error", e)
for nb in (0, 2, 4):
    cfg = d.EngineConfig(tile_nb=nb)
    fp = d.make_forward_plan(spec, 1, None, cfg, d.Math.F32)
    t = timeit(lambda: fp.execute(x, w, y), "fwd")
    print("fwd nb", nb, round(t, 1), "us", fp.blocking)
