"""Dev tool: fp32-accurate multi-tap forward kernel times (cfg1 and friends), L2 flushed."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
lib = d._lib.lib()
lib.dconv_profile(1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (N, C, K, H, R, st) in [(32, 64, 64, 56, 3, 1), (32, 256, 256, 14, 3, 1), (32, 128, 128, 28, 3, 1), (32, 3, 64, 224, 7, 2)]:
    pad = (R - 1) // 2
    spec = d.make_layer_spec(N, C, K, H, H, R, R, st, pad, pad, 16)
    P = (H + 2 * pad - R) // st + 1
    x = d.to_blocked_activation(torch.rand(N, C, H, H, device="cuda") * 2 - 1, spec)
    w = d.to_blocked_weight(torch.randn(K, C, R, R, device="cuda") * 0.05, spec)
    y = d.BlockedActivation(N, K, P, P)
    fp = d.make_forward_plan(spec, 1, None, None, d.Math.F32)
    ts = []
    for i in range(7):
        flush.fill_(i)
        torch.cuda._sleep(1_000_000)
        fp.execute(x, w, y)
        torch.cuda.synchronize()
        ts.append(lib.dconv_profile_last_ms(0) * 1e3)
    ts.sort()
    fl = d.pass_flops(spec)
    print(f"N{N} C{C} K{K} H{H} R{R} s{st}: {ts[3]:.1f} us  {fl / ts[3] / 1e6:.0f} TF")
