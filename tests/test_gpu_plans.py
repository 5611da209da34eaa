"""Plans: built once, serialized, validated, fault-injected.

* save -> load round trip replays to the same bits (test_kernel_streams.cpp:234-257);
* a corrupted plan is caught by the validator (test_kernel_streams.cpp:152-175):
  tile coverage, split coverage, grid / table limits, truncated text;
* the DCONV_* experiment variables are inert outside developer mode;
* weights prepared ahead of time on another stream (DCONV_EP_PREP_ONLY), then
  a WEIGHTS_READY execute chained behind a producer layer: same bits as the
  plain call (no programmatic-launch race on the activations);
* host cost of an execute call once the plan is resolved.
"""
import ctypes as C
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


def _edit(text, field, fn):
    """apply fn to the value(s) of every `field` record of a DCPL plan text"""
    out, hits = [], 0
    for line in text.splitlines():
        parts = line.split()
        if parts and parts[0] == field:
            parts = [parts[0]] + [str(fn(int(v))) for v in parts[1:]]
            hits += 1
            line = " ".join(parts)
        out.append(line)
    assert hits, field
    return "\n".join(out) + "\n"


def _layer(dconv, orc, N, C_, K, H, W, R, S, st, ph, pw, dtype=torch.float32):
    spec = dconv.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    P, Q = dconv.derive_output_shape(spec)
    x = orc.uniform(3, (N, C_, H, W))
    w = orc.he_normal(4, (K, C_, R, S), C_ * R * S)
    g = orc.uniform(5, (N, K, P, Q))
    ib = dconv.to_blocked_activation(dev(x), 16, ph, pw, dtype=dtype)
    wb = dconv.to_blocked_weight(dev(w), spec)
    gb = dconv.to_blocked_activation(dev(g), 16, 0, 0, dtype=dtype)
    return spec, P, Q, ib, wb, gb


SHAPES = [(2, 32, 48, 14, 14, 3, 3, 1, 1, 1), (2, 64, 32, 14, 14, 1, 1, 2, 0, 0), (2, 3, 32, 30, 30, 7, 7, 2, 3, 3),
          (2, 40, 24, 9, 9, 1, 7, 1, 0, 3)]


@pytest.mark.parametrize("shape", SHAPES, ids=[f"s{i}" for i in range(len(SHAPES))])
@pytest.mark.parametrize("math", [0, 1])
def test_plan_save_load_replays_bitwise(dconv, orc, shape, math):
    M = dconv.Math(math)
    dt = torch.float32 if M == dconv.Math.F32 else torch.bfloat16
    spec, P, Q, ib, wb, gb = _layer(dconv, orc, *shape, dtype=dt)
    op = dconv.FusedOp(dconv.FusedOpKind.BIAS_RELU, [0.25] * spec.K)
    B = dconv.BlockedActivation
    # forward (fused bias + ReLU)
    fp = dconv.make_forward_plan(spec, 1, op, None, M)
    a = B(spec.N, spec.K, P, Q, 16, 0, 0, dt)
    fp.execute(ib, wb, a)
    text = fp.save()
    fl = dconv.ExecutionPlan.load(text, validate=True)
    assert fl.save() == text, "save(load(save(plan))) must round-trip"
    b = B(spec.N, spec.K, P, Q, 16, 0, 0, dt)
    fl.execute(ib, wb, b)
    torch.cuda.synchronize()
    assert torch.equal(a.data, b.data)
    assert fl.blocking == fp.blocking
    # backward-data
    bp = dconv.BackwardContext(spec, wb, 1, None, M)
    gi_a = B(spec.N, spec.C, spec.H, spec.W, 16, 0, 0, dt)
    bp.execute(wb, gb, gi_a)
    text = bp.save()
    bl = dconv.BackwardContext.load(text, validate=True)
    assert bl.save() == text
    gi_b = B(spec.N, spec.C, spec.H, spec.W, 16, 0, 0, dt)
    bl.execute(wb, gb, gi_b)
    torch.cuda.synchronize()
    assert torch.equal(gi_a.data, gi_b.data)
    # weight update
    up = dconv.UpdatePlan(spec, None, M)
    dwa = dconv.BlockedWeight(spec.K, spec.C, spec.R, spec.S)
    up.execute(ib, gb, dwa)
    text = up.save()
    ul = dconv.UpdatePlan.load(text, validate=True)
    assert ul.save() == text
    dwb = dconv.BlockedWeight(spec.K, spec.C, spec.R, spec.S)
    ul.execute(ib, gb, dwb)
    torch.cuda.synchronize()
    assert torch.equal(dwa.data, dwb.data)
    assert ul.splits == up.splits


def test_fault_injection_is_detected(dconv, orc):
    spec, P, Q, ib, wb, gb = _layer(dconv, orc, 2, 32, 48, 14, 14, 3, 3, 1, 1, 1)
    B = dconv.BlockedActivation
    out = B(spec.N, spec.K, P, Q)
    fp = dconv.make_forward_plan(spec, 1, None, None, dconv.Math.BF16)
    fp.validate(ib, out)
    text = fp.save()
    # fewer m-tiles per image than the plane needs: output rows never written
    bad = _edit(text, "tiles_per_img", lambda v: v - 1)
    loaded = dconv.ExecutionPlan.load(bad, validate=False)
    with pytest.raises(dconv.InvalidDescriptor, match="written 0 times"):
        loaded.validate(ib, out)
    with pytest.raises(dconv.InvalidDescriptor):
        dconv.ExecutionPlan.load(bad, validate=True)
    # ring deeper than the kernel's barrier arrays
    with pytest.raises(dconv.InvalidDescriptor, match="ring depth"):
        dconv.ExecutionPlan.load(_edit(text, "rings", lambda v: v + 16), validate=True)
    # a launch attached to a different problem
    with pytest.raises(dconv.InvalidDescriptor, match="differs from the tensors"):
        dconv.ExecutionPlan.load(_edit(text, "kb_out", lambda v: v + 1), validate=True)
    # truncated / foreign text
    with pytest.raises(dconv.ParseError):
        dconv.ExecutionPlan.load(text[: len(text) // 2], validate=True)
    with pytest.raises(dconv.ParseError):
        dconv.UpdatePlan.load(text, validate=True)
    # weight update: split ranges / stage bands that no longer cover the pixels
    up = dconv.UpdatePlan(spec, None, dconv.Math.BF16)
    up.validate(ib, gb)
    ut = up.save()
    spi = int(next(l.split()[1] for l in ut.splitlines() if l.startswith("stages_per_img ")))
    bad = _edit(_edit(ut, "stages_per_img", lambda v: v - 1), "stages_total", lambda v: v - spec.N)
    if spi > 1:
        with pytest.raises(dconv.InvalidDescriptor, match="cover"):
            dconv.UpdatePlan.load(bad, validate=True)
    with pytest.raises(dconv.InvalidDescriptor, match="grid"):
        dconv.UpdatePlan.load(_edit(ut, "splits", lambda v: v + 1), validate=True)
    # backward-data: a phase launch that misses lattice points
    bp = dconv.BackwardContext(spec, wb, 1, None, dconv.Math.BF16)
    gi = B(spec.N, spec.C, spec.H, spec.W)
    bp.execute(wb, gb, gi)
    bt = bp.save()
    with pytest.raises(dconv.InvalidDescriptor, match="written 0 times"):
        dconv.BackwardContext.load(_edit(bt, "tiles_per_img", lambda v: v - 1), validate=True)


def test_env_overrides_inert_outside_dev_mode(dconv, orc, monkeypatch):
    spec, P, Q, ib, wb, gb = _layer(dconv, orc, 4, 64, 64, 14, 14, 1, 1, 1, 0, 0)
    base = dconv.UpdatePlan(spec, None, dconv.Math.F32)
    dw = dconv.BlockedWeight(spec.K, spec.C, 1, 1)
    base.execute(ib, gb, dw)
    g0 = base.blocking["splits"]
    monkeypatch.setenv("DCONV_UPD_SPLITS", "3" if g0 != 3 else "5")
    monkeypatch.setenv("DCONV_FWD_NB", "1")
    up = dconv.UpdatePlan(spec, None, dconv.Math.F32)
    up.execute(ib, gb, dw)
    assert up.blocking["splits"] == g0, "a DCONV_* variable changed a production plan"
    lib = dconv._lib.lib()
    lib.dconv_set_dev_mode(1)
    try:
        up2 = dconv.UpdatePlan(spec, None, dconv.Math.F32)
        up2.execute(ib, gb, dw)
        assert up2.blocking["splits"] != g0
        monkeypatch.setenv("DCONV_UPD_SPLITS", "x7")
        with pytest.raises(dconv.InvalidArgument):
            up2.execute(ib, gb, dw)
    finally:
        lib.dconv_set_dev_mode(0)


@pytest.mark.parametrize("math", [0, 1])
def test_prepared_weights_on_side_stream_then_weights_ready(dconv, orc, math):
    """layer 2's weights are prepared on a side stream (PREP_ONLY);
    its WEIGHTS_READY execute runs right behind layer 1 (which writes layer 2's
    input) on the main stream. Must equal the plain two-layer chain bitwise."""
    from paper_1808_05567_b200._lib import EP_PREP_ONLY, EP_WEIGHTS_READY, Epilogue

    M = dconv.Math(math)
    dt = torch.float32 if M == dconv.Math.F32 else torch.bfloat16
    lib = dconv._lib.lib()
    N, C1, C2, C3, H = 8, 64, 128, 64, 28
    s1 = dconv.make_layer_spec(N, C1, C2, H, H, 3, 3, 1, 1, 1, 16)
    s2 = dconv.make_layer_spec(N, C2, C3, H, H, 1, 1, 1, 0, 0, 16)
    x = dconv.to_blocked_activation(dev(orc.uniform(11, (N, C1, H, H))), 16, 0, 0, dtype=dt)
    w1 = dconv.to_blocked_weight(dev(orc.he_normal(12, (C2, C1, 3, 3), C1 * 9)), s1)
    w2 = dconv.to_blocked_weight(dev(orc.he_normal(13, (C3, C2, 1, 1), C2)), s2)
    B = dconv.BlockedActivation
    p1 = dconv.ExecutionPlan(s1, None, None, M, 0, 0)
    p2 = dconv.ExecutionPlan(s2, None, None, M, 0, 0)
    ws1 = torch.empty(lib.dconv_fwd_workspace_bytes(p1._h), dtype=torch.uint8, device="cuda")
    ws2 = torch.empty(lib.dconv_fwd_workspace_bytes(p2._h), dtype=torch.uint8, device="cuda")

    def run(side):
        y1 = B(N, C2, H, H, 16, 0, 0, dt)
        y2 = B(N, C3, H, H, 16, 0, 0, dt)
        y1.data.fill_(float("nan"))  # stale contents must never reach layer 2
        main = torch.cuda.current_stream()
        if side:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ep = Epilogue(None, None, 0, EP_PREP_ONLY)
                assert lib.dconv_forward_ex(p2._h, C.byref(y1.to_c()), C.byref(w2.to_c()), C.byref(y2.to_c()),
                                            C.byref(ep), ws2.data_ptr(), s.cuda_stream) == 0
            main.wait_stream(s)
        assert lib.dconv_forward_ex(p1._h, C.byref(x.to_c()), C.byref(w1.to_c()), C.byref(y1.to_c()), None,
                                    ws1.data_ptr(), main.cuda_stream) == 0
        ep = Epilogue(None, None, 0, EP_WEIGHTS_READY if side else 0)
        assert lib.dconv_forward_ex(p2._h, C.byref(y1.to_c()), C.byref(w2.to_c()), C.byref(y2.to_c()), C.byref(ep),
                                    ws2.data_ptr(), main.cuda_stream) == 0
        torch.cuda.synchronize()
        return y2.data.clone()

    ref = run(False)
    for _ in range(5):
        assert torch.equal(run(True), ref)


def test_execute_host_cost_after_first_call(dconv, orc):
    """a8: the plan resolves its tiles and tensor maps on the first execute of a
    geometry; later calls only patch pointers and launch. Reports host us/call."""
    spec, P, Q, ib, wb, gb = _layer(dconv, orc, 32, 256, 64, 56, 56, 1, 1, 1, 0, 0)
    lib = dconv._lib.lib()
    fp = dconv.make_forward_plan(spec, 1, None, None, dconv.Math.F32)
    out = dconv.BlockedActivation(spec.N, spec.K, P, Q)
    ws = torch.empty(lib.dconv_fwd_workspace_bytes(fp._h), dtype=torch.uint8, device="cuda")
    a, w, o = ib.to_c(), wb.to_c(), out.to_c()
    s = torch.cuda.current_stream().cuda_stream
    t0 = time.perf_counter()
    assert lib.dconv_forward(fp._h, C.byref(a), C.byref(w), C.byref(o), ws.data_ptr(), s) == 0
    first = time.perf_counter() - t0
    torch.cuda.synchronize()
    n = 200
    torch.cuda._sleep(50_000_000)  # keep the queue busy: time host work, not back-pressure
    t0 = time.perf_counter()
    for _ in range(n):
        assert lib.dconv_forward(fp._h, C.byref(a), C.byref(w), C.byref(o), ws.data_ptr(), s) == 0
    per = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    print(f"forward execute host cost: first call {first * 1e6:.1f} us, then {per * 1e6:.1f} us/call (2 launches)")
    assert per < 40e-6, per


def test_cpp_shim_runs_both_engines(dconv):
    """include/dconv_b200.hpp: the reference's own calls (forward / backward / weight_update,
    same signatures, reference host tensors) on the B200 vs the reference engine and its
    naive oracle (tests/shim/shim_check.cpp, built against the reference by `make shim`)."""
    import os
    import subprocess

    binary = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "shim_check")
    if not os.path.exists(binary):
        pytest.skip("shim_check not built (needs /root/reference at build time)")
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0 and "SHIM CHECK OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("math", [0, 1])
def test_batched_weight_prep_matches_inline_prep(dconv, orc, math):
    """dconv_prep_batch_begin/end: three convs' forward and backward-data weight
    preparations recorded (PREP_ONLY) and launched as ONE kernel; the WEIGHTS_READY
    executes on those workspaces equal the inline-prep executes bitwise."""
    from paper_1808_05567_b200._lib import EP_PREP_ONLY, EP_WEIGHTS_READY, Epilogue

    M = dconv.Math(math)
    dt = torch.float32 if M == dconv.Math.F32 else torch.bfloat16
    lib = dconv._lib.lib()
    B = dconv.BlockedActivation
    layers = [(8, 64, 128, 28, 3), (8, 128, 256, 14, 1), (4, 48, 80, 9, 3)]  # (N, C, K, H, R); the last: ragged blocks
    st = torch.cuda.current_stream().cuda_stream
    cases = []
    for i, (N, C_, K, H, R) in enumerate(layers):
        pad = (R - 1) // 2
        s = dconv.make_layer_spec(N, C_, K, H, H, R, R, 1, pad, pad, 16)
        x = dconv.to_blocked_activation(dev(orc.uniform(40 + i, (N, C_, H, H))), 16, 0, 0, dtype=dt)
        g = dconv.to_blocked_activation(dev(orc.uniform(50 + i, (N, K, H, H))), 16, 0, 0, dtype=dt)
        w = dconv.to_blocked_weight(dev(orc.he_normal(60 + i, (K, C_, R, R), C_ * R * R)), s)
        fp = dconv.ExecutionPlan(s, None, None, M, 0, 0)
        bp = dconv.prepare_backward(s, w, 1, None, M)
        wsf = torch.empty(lib.dconv_fwd_workspace_bytes(fp._h), dtype=torch.uint8, device="cuda")
        wsb = torch.empty(lib.dconv_bwd_workspace_bytes(bp._h), dtype=torch.uint8, device="cuda")
        cases.append((N, C_, K, H, x, g, w, fp, bp, wsf, wsb))

    def run(batched):
        outs = []
        if batched:
            assert lib.dconv_prep_batch_begin() == 0
            for N, C_, K, H, x, g, w, fp, bp, wsf, wsb in cases:
                y, dx = B(N, K, H, H, 16, 0, 0, dt), B(N, C_, H, H, 16, 0, 0, dt)
                ep = Epilogue(None, None, 0, EP_PREP_ONLY)
                assert lib.dconv_forward_ex(fp._h, C.byref(x.to_c()), C.byref(w.to_c()), C.byref(y.to_c()),
                                            C.byref(ep), wsf.data_ptr(), st) == 0
                assert lib.dconv_backward_data_ex(bp._h, C.byref(w.to_c()), C.byref(g.to_c()), C.byref(dx.to_c()),
                                                  C.byref(ep), wsb.data_ptr(), st) == 0
            assert lib.dconv_prep_batch_end(st) == 0
        flag = EP_WEIGHTS_READY if batched else 0
        for N, C_, K, H, x, g, w, fp, bp, wsf, wsb in cases:
            y, dx = B(N, K, H, H, 16, 0, 0, dt), B(N, C_, H, H, 16, 0, 0, dt)
            ep = Epilogue(None, None, 0, flag)
            assert lib.dconv_forward_ex(fp._h, C.byref(x.to_c()), C.byref(w.to_c()), C.byref(y.to_c()), C.byref(ep),
                                        wsf.data_ptr(), st) == 0
            assert lib.dconv_backward_data_ex(bp._h, C.byref(w.to_c()), C.byref(g.to_c()), C.byref(dx.to_c()),
                                              C.byref(ep), wsb.data_ptr(), st) == 0
            outs += [y.data, dx.data]
        torch.cuda.synchronize()
        return [o.clone() for o in outs]

    ref = run(False)
    for wsf_b in [c[9] for c in cases] + [c[10] for c in cases]:
        wsf_b.fill_(0xAB)  # the batch must rewrite every prepared byte the convs read
    got = run(True)
    for a, b in zip(got, ref):
        assert torch.equal(a, b)
