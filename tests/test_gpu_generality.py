"""Descriptor generality (VERDICT r1 missing #6): every layer the reference accepts.

* vlen != 16 (the reference runs vlen 4 and 5, test_propagation.cpp:64-76): the
  plans re-block around a 16-lane twin; results in the caller's vlen layout;
* strides 3 and 4 (s^2 stride phases; the generic backward route);
* filters with more than 64 taps (9x9, 11x11, 11x11/s4);
each F / B / U against the CPU oracle in both math modes, plus the plan
validator on each plan. Gates: max|d|/rms(ref) <= 1e-4 (fp32-accurate), 2e-2 (bf16).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = {0: 1e-4, 1: 2e-2}

CASES = [
    # N, C, K, H, W, R, S, stride, pad_h, pad_w, vlen
    (2, 20, 24, 9, 9, 3, 3, 1, 1, 1, 4),
    (2, 20, 24, 9, 9, 3, 3, 1, 1, 1, 5),
    (2, 13, 19, 10, 10, 1, 1, 2, 0, 0, 8),
    (2, 6, 10, 15, 15, 7, 7, 2, 3, 3, 4),
    (2, 16, 32, 17, 17, 3, 3, 3, 1, 1, 16),
    (2, 24, 16, 23, 23, 5, 5, 3, 2, 2, 16),
    (2, 8, 32, 35, 35, 7, 7, 4, 3, 3, 16),
    (2, 3, 48, 63, 63, 11, 11, 4, 2, 2, 16),
    (2, 16, 16, 20, 20, 9, 9, 1, 4, 4, 16),
    (2, 8, 24, 19, 19, 11, 11, 1, 5, 5, 16),
    (2, 12, 20, 11, 11, 5, 5, 1, 2, 2, 5),
]


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("case", CASES, ids=[f"{c[5]}x{c[6]}s{c[7]}_v{c[10]}_C{c[1]}" for c in CASES])
@pytest.mark.parametrize("math", [0, 1])
def test_general_descriptors(dconv, orc, case, math):
    N, C_, K, H, W, R, S, st, ph, pw, v = case
    M = dconv.Math(math)
    s = orc.spec(N, C_, K, H, W, R, S, st, ph, pw, v)
    spec = dconv.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, v)
    P, Q = orc.output_shape(s)
    x = orc.uniform(31, (N, C_, H, W))
    w = orc.he_normal(32, (K, C_, R, S), C_ * R * S)
    g = orc.uniform(33, (N, K, P, Q))
    ib = dconv.to_blocked_activation(_dev(x), spec)
    wb = dconv.to_blocked_weight(_dev(w), spec)
    gb = dconv.to_blocked_activation(_dev(g), v, 0, 0)
    assert ib.vlen == v and wb.vlen == v
    plan = dconv.make_forward_plan(spec, 1, None, None, M)
    out = dconv.forward(spec, ib, wb, plan)
    assert out.vlen == v
    plan.validate(ib, out)
    for name, ref, got in (
            ("forward", orc.conv_forward(s, x, w), dconv.from_blocked_activation(out)),
            ("backward", orc.conv_backward(s, g, w),
             dconv.from_blocked_activation(dconv.backward_with(dconv.prepare_backward(spec, wb, 1, None, M), gb))),
            ("update", orc.conv_update(s, x, g), dconv.from_blocked_weight(dconv.weight_update(spec, ib, gb, None,
                                                                                              dtype=M)))):
        got = got.cpu().numpy()
        n = orc.error_norms(ref, got)
        assert n["max_over_rms"] <= TOL[math], (name, case, n)
    if v != 16:
        # tail lanes of the caller's vlen-v layout stay exactly zero (test_propagation.cpp:90-102)
        blk = out.data.view(N, -(-K // v), P, Q, v).cpu()
        if K % v:
            assert not blk[:, -1, :, :, K % v:].any()
