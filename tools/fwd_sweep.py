"""Dev tool: bf16 FWD / BWD kernel times of the ResNet-50 3x3 (and selected 1x1)
layers at N=256 under debug plan overrides (env DCONV_WST / DCONV_WCAP /
anything in SWEEP), L2 flushed, library event brackets around the conv kernel."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import _lib  # noqa: E402

lib = _lib.lib()
lib.dconv_profile(1)
lib.dconv_set_dev_mode(1)  # DCONV_* overrides act only in developer mode
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
N = int(os.environ.get("N", "256"))
LAYERS = [(64, 64, 56, 3), (128, 128, 28, 3), (256, 256, 14, 3), (512, 512, 7, 3)]
if os.environ.get("LAYERS"):
    LAYERS = [tuple(int(v) for v in s.split(",")) for s in os.environ["LAYERS"].split(";")]
SWEEP = [s for s in os.environ.get("SWEEP", "").split(";")] or [""]
PASSES = os.environ.get("PASSES", "fb")


def timeit(fn, slot, reps=7):
    ts = []
    for i in range(reps):
        if not os.environ.get("NOFLUSH"):
            flush.fill_(i)
        torch.cuda._sleep(1_000_000)
        fn()
        torch.cuda.synchronize()
        ts.append(lib.dconv_profile_last_ms(slot) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


for (C, K, H, R) in LAYERS:
    pad = (R - 1) // 2
    spec = d.make_layer_spec(N, C, K, H, H, R, R, 1, pad, pad, 16)
    fl = d.pass_flops(spec)
    x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    x.data.uniform_(-1, 1)
    y = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    g = d.BlockedActivation(N, K, H, H, 16, 0, 0, torch.bfloat16)
    g.data.uniform_(-1, 1)
    dx = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
    w = d.BlockedWeight(K, C, R, R)
    w.data.normal_()
    for sw in SWEEP:
        env = dict(kv.split("=") for kv in sw.split(",") if kv)
        saved = {k: os.environ.get(k) for k in env}
        dbg = int(env.pop("DBG", "0"))
        os.environ.update(env)
        lib.dconv_debug_mode(dbg)
        try:
            out = []
            if "f" in PASSES:
                fp = d.make_forward_plan(spec, 1, None, None, d.Math.BF16)
                t = timeit(lambda: fp.execute(x, w, y), 0)
                out.append(f"F {t:7.1f} us {fl / t / 1e6:6.0f} TF")
            if "b" in PASSES:
                bc = d.prepare_backward(spec, w, 1, None, d.Math.BF16)
                t = timeit(lambda: bc.execute(w, g, dx), 1)
                out.append(f"B {t:7.1f} us {fl / t / 1e6:6.0f} TF")
            if "u" in PASSES:
                up = d.UpdatePlan(spec, None, d.Math.BF16)
                dw = d.BlockedWeight(K, C, R, R)
                t = timeit(lambda: up.execute(x, g, dw), 2)
                out.append(f"U {t:7.1f} us {fl / t / 1e6:6.0f} TF")
            if "u" in PASSES and os.environ.get("SHOWU"):
                print("   upd plan", up.blocking)
            if os.environ.get("FULL"):
                if "f" in PASSES:
                    print("   fwd plan", fp.blocking)
                if "b" in PASSES:
                    print("   bwd plan", bc.blocking)
            blk = fp.blocking if "f" in PASSES else {}
            print(f"C{C} K{K} H{H} R{R} [{sw or 'default'}] " + " | ".join(out) +
                  f"  wst={blk.get('w_stages')} pcst={blk.get('pc_stages')} mb={blk.get('mb')} nb={blk.get('nb')}",
                  flush=True)
        except d.Error as e:
            print(f"C{C} K{K} H{H} [{sw}] error {e}", flush=True)
        finally:
            lib.dconv_debug_mode(0)
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
