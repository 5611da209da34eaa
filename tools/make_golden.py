"""Generate tests/golden/ fixtures from the REFERENCE itself.

Runs the unmodified reference core (oracle/_ref/libdconv_ref.so, built from
/root/reference/proj sources by `make -C oracle ref`) on small seeded cases
and stores inputs + outputs, so parity tests can pin both the C oracle and
the GPU engine to the reference's own results on machines without
/root/reference (the GPU box). Re-run: python tools/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as orc  # noqa: E402

# (N, C, K, H, W, R, S, stride, pad_h, pad_w): the reference's own test shapes
# (test_propagation.cpp:52-195, test_reference.cpp:118-124) at vlen 16
CASES = [
    (2, 24, 16, 12, 12, 3, 3, 1, 1, 1),   # forward matches the naive oracle
    (2, 16, 24, 10, 10, 3, 3, 1, 1, 1),   # stride-1 duality route
    (2, 16, 24, 12, 12, 1, 1, 2, 0, 0),   # 1x1 stride-2 lattice route
    (2, 16, 16, 11, 11, 3, 3, 2, 0, 0),   # generic route
    (1, 8, 8, 9, 9, 3, 3, 2, 1, 1),       # generic route, padded strided
    (2, 5, 7, 8, 9, 3, 3, 1, 1, 1),       # adjoint spec 1 (tails)
    (2, 8, 4, 6, 6, 1, 1, 2, 0, 0),       # adjoint spec 3
    (1, 3, 5, 10, 10, 5, 5, 1, 2, 2),     # adjoint spec 4 (5x5)
    (2, 3, 16, 20, 20, 7, 7, 2, 3, 3),    # stem-like 7x7/s2/p3, C=3
    (2, 32, 32, 9, 9, 1, 7, 1, 0, 3),     # Inception 1x7
    (2, 32, 32, 9, 9, 7, 1, 1, 3, 0),     # Inception 7x1
]


def main():
    r = orc.ref()
    if r is None:
        sys.exit("oracle/_ref/libdconv_ref.so missing: make -C oracle ref (needs /root/reference)")
    out = {}
    meta = []
    for i, cs in enumerate(CASES):
        N, C, K, H, W, R, S, st, ph, pw = cs
        s = orc.spec(N, C, K, H, W, R, S, st, ph, pw, 16)
        P, Q = orc.output_shape(s)
        x = np.empty(N * C * H * W, np.float32)
        r.ref_random_f32(1000 + i, x, x.size)  # Rng(seed).next_f32 stream (harness.cpp:274-278)
        w = np.empty(K * C * R * S, np.float32)
        r.ref_random_f32(2000 + i, w, w.size)
        g = np.empty(N * K * P * Q, np.float32)
        r.ref_random_f32(3000 + i, g, g.size)
        x, w, g = x.reshape(N, C, H, W), w.reshape(K, C, R, S), g.reshape(N, K, P, Q)
        sa = orc.spec_array(s)
        fo = np.empty((N, K, P, Q), np.float32)
        bo = np.empty((N, C, H, W), np.float32)
        uo = np.empty((K, C, R, S), np.float32)
        assert r.ref_conv_forward_naive(sa, x, w, fo) == 0
        assert r.ref_conv_backward_naive(sa, g, w, bo) == 0
        assert r.ref_conv_update_naive(sa, x, g, uo) == 0
        # the reference direct engine too (its own f32 path)
        fd, _, _ = orc.ref_direct_pass(s, 0, 2, 0, x, w)
        bd, _, _ = orc.ref_direct_pass(s, 1, 2, 0, g, w)
        ud, _, _ = orc.ref_direct_pass(s, 2, 2, 0, x, g)
        xb = np.empty(orc.lib().orc_act_elems(N, C, H, W, 16, ph, pw), np.float32)
        assert r.ref_to_blocked_act(x, N, C, H, W, 16, ph, pw, xb) == 0
        wb = np.empty(orc.lib().orc_wt_elems(K, C, R, S, 16), np.float32)
        assert r.ref_to_blocked_wt(w.reshape(-1), K, C, R, S, 16, wb) == 0
        wd = np.empty(orc.lib().orc_wt_elems(C, K, R, S, 16), np.float32)
        assert r.ref_transform_weight_stride1(w.reshape(-1), K, C, R, S, 16, wd) == 0
        for k, v in dict(x=x, w=w, g=g, fwd=fo, bwd=bo, upd=uo, fwd_direct=fd, bwd_direct=bd, upd_direct=ud,
                         x_blocked=xb, w_blocked=wb, w_dual=wd).items():
            out[f"c{i}_{k}"] = v
        meta.append({"case": i, "spec": dict(zip(["N", "C", "K", "H", "W", "R", "S", "stride", "pad_h", "pad_w"], cs)),
                     "seeds": {"x": 1000 + i, "w": 2000 + i, "g": 3000 + i}, "P": P, "Q": Q,
                     "flops": int(r.ref_pass_flops(sa))})
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    np.savez_compressed(os.path.join(ROOT, "tests", "golden", "ref_cases.npz"), **out)
    with open(os.path.join(ROOT, "tests", "golden", "ref_cases.json"), "w") as f:
        json.dump({"generator": "tools/make_golden.py", "source": "oracle/_ref (reference core @ /root/reference/proj)",
                   "compiler": open(os.path.join(ROOT, "oracle", "_ref", "COMPILER")).read().strip().splitlines(),
                   "cases": meta}, f, indent=1)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()
