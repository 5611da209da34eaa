"""Dev tool: one bf16 weight-update launch of LAYER="C,K,H,R[,pad[,stride]]" at N (for ncu)."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
v = [int(t) for t in os.environ.get("LAYER", "256,256,14,3").split(",")]
C, K, H, R = v[:4]
pad = v[4] if len(v) > 4 else (R - 1) // 2
st = v[5] if len(v) > 5 else 1
N = int(os.environ.get("N", "256"))
spec = d.make_layer_spec(N, C, K, H, H, R, R, st, pad, pad, 16)
P = (H + 2 * pad - R) // st + 1
x = d.BlockedActivation(N, C, H, H, 16, 0, 0, torch.bfloat16)
x.data.uniform_(-1, 1)
g = d.BlockedActivation(N, K, P, P, 16, 0, 0, torch.bfloat16)
g.data.uniform_(-1, 1)
dw = d.BlockedWeight(K, C, R, R)
up = d.UpdatePlan(spec, None, d.Math.BF16)
for _ in range(3):
    up.execute(x, g, dw)
torch.cuda.synchronize()
print(up.blocking)
