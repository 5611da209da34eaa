"""GPU parity of the bf16 staging modes added in round 2 (weight update, and the packed
multi-tap forward / backward-data tiles), each pinned
to the plan it is meant to run (plan describe) and checked against the oracle on
the same bf16-rounded operands (tolerance 2e-2, BASELINE north_star):

* cross-stacking (UpdParams::xs): narrow stride-1 multi-tap layers, N holding xs
  column-shifted dO copies -- the 64-channel 3x3 (xs = 3: tap groups of 2 + 1 A
  slots) and a 12-channel 4x4 (the space-to-depth stem's shape, xs = 2);
* packed images (UpdParams::pimg): small stride-1 planes, whole images along K with
  shared padding rows -- the 7x7 3x3 at an odd image count (the last stage's second
  image is past the batch: zero fill);
* SWIZZLE_128B staging of linear 1x1 updates (UpdParams::sw32 = 2), plane sizes
  divisible by 4.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


CASES = [
    # (N, C, K, H, W, R, S, pad_h, pad_w, expect) -- expect: predicate on the plan describe
    (3, 64, 64, 20, 20, 3, 3, 1, 1, ("tg", 3)),
    (2, 12, 64, 18, 18, 4, 4, 1, 2, ("tg", 2)),
    (3, 512, 256, 7, 7, 3, 3, 1, 1, ("rows_ps", 8)),
    (5, 128, 128, 7, 7, 3, 3, 1, 1, ("rows_ps", 8)),
    (2, 256, 512, 14, 14, 1, 1, 0, 0, None),
]


@pytest.mark.parametrize("case", CASES, ids=[f"N{c[0]}_{c[1]}to{c[2]}_{c[5]}x{c[6]}_{c[3]}" for c in CASES])
def test_bf16_update_modes(dconv, orc, case):
    N, C_, K, H, W, R, S, ph, pw, expect = case
    s = orc.spec(N, C_, K, H, W, R, S, 1, ph, pw, 16)
    spec = dconv.make_layer_spec(N, C_, K, H, W, R, S, 1, ph, pw, 16)
    P, Q = orc.output_shape(s)
    rnd = lambda a: torch.from_numpy(a).bfloat16().float().numpy()  # noqa: E731
    x = rnd(orc.uniform(21, (N, C_, H, W)))
    g = rnd(orc.uniform(22, (N, K, P, Q)))
    bf = torch.bfloat16
    ib = dconv.to_blocked_activation(dev(x), 16, 0, 0, dtype=bf)
    gb = dconv.to_blocked_activation(dev(g), 16, 0, 0, dtype=bf)
    up = dconv.UpdatePlan(spec, None, dconv.Math.BF16)
    dw = dconv.BlockedWeight(K, C_, R, S)
    up.execute(ib, gb, dw)
    torch.cuda.synchronize()
    blk = up.blocking
    if expect is not None:
        key, val = expect
        assert blk[key] == val, blk
    n = orc.error_norms(orc.conv_update(s, x, g), dconv.from_blocked_weight(dw).cpu().numpy())
    assert n["max_over_rms"] <= 2e-2, (n, blk)
    # bitwise reproducible (fixed-order split reduction)
    dw2 = dconv.BlockedWeight(K, C_, R, S)
    up.execute(ib, gb, dw2)
    torch.cuda.synchronize()
    assert torch.equal(dw.data, dw2.data)
    # the plan validator accepts the launch (tap coverage, stage coverage, limits)
    assert up.validate(ib, gb)["ok"]


@pytest.mark.parametrize("N", [4, 5])
def test_packed_image_forward_backward(dconv, orc, N):
    """Packed multi-tap tiles (FwdParams::img_pitch): three 7x7 images per 256-row tile,
    forward and the dual backward-data, batch not a multiple of three (a tile's last
    images past the batch), against the oracle on the same bf16-rounded operands."""
    C_, K, H = 128, 256, 7
    s = orc.spec(N, C_, K, H, H, 3, 3, 1, 1, 1, 16)
    spec = dconv.make_layer_spec(N, C_, K, H, H, 3, 3, 1, 1, 1, 16)
    rnd = lambda a: torch.from_numpy(a).bfloat16().float().numpy()  # noqa: E731
    x = rnd(orc.uniform(31, (N, C_, H, H)))
    w = rnd(orc.he_normal(32, (K, C_, 3, 3), C_ * 9))
    g = rnd(orc.uniform(33, (N, K, H, H)))
    bf = torch.bfloat16
    ib = dconv.to_blocked_activation(dev(x), 16, 0, 0, dtype=bf)
    gb = dconv.to_blocked_activation(dev(g), 16, 0, 0, dtype=bf)
    wb = dconv.to_blocked_weight(dev(w), spec)
    M = dconv.Math.BF16
    fp = dconv.make_forward_plan(spec, 1, None, None, M)
    y = dconv.BlockedActivation(N, K, H, H, 16, 0, 0, bf)
    fp.execute(ib, wb, y)
    torch.cuda.synchronize()
    assert fp.blocking["mimg"] == 3 and fp.blocking["mode"] == "rows", fp.blocking
    n = orc.error_norms(orc.conv_forward(s, x, w), dconv.from_blocked_activation(y, dtype=torch.float32).cpu().numpy())
    assert n["max_over_rms"] <= 2e-2, n
    assert fp.validate(ib, y)["ok"]
    bc = dconv.prepare_backward(spec, wb, 1, None, M)
    dx = dconv.BlockedActivation(N, C_, H, H, 16, 0, 0, bf)
    bc.execute(wb, gb, dx)
    torch.cuda.synchronize()
    assert bc.blocking["phases"][0]["mimg"] == 3, bc.blocking
    n = orc.error_norms(orc.conv_backward(s, g, w), dconv.from_blocked_activation(dx, dtype=torch.float32).cpu().numpy())
    assert n["max_over_rms"] <= 2e-2, n
