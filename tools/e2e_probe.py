"""Dev tool: per-chunk device compute time vs the host-step pipeline (cfg2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402

math = d.Math.F32


def dev_step_ms(n):
    spec = d.make_layer_spec(n, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
    x = d.BlockedActivation(n, 256, 56, 56)
    x.data.uniform_(-1, 1)
    g = d.BlockedActivation(n, 64, 56, 56)
    g.data.uniform_(-1, 1)
    w = d.BlockedWeight(64, 256, 1, 1)
    w.data.normal_()
    y, dx, dw = d.BlockedActivation(n, 64, 56, 56), d.BlockedActivation(n, 256, 56, 56), d.BlockedWeight(64, 256, 1, 1)
    fp = d.make_forward_plan(spec, 1, None, None, math)
    bc = d.prepare_backward(spec, w, 1, None, math)
    up = d.UpdatePlan(spec, None, math)

    def step():
        fp.execute(x, w, y)
        bc.execute(w, g, dx)
        up.execute(x, g, dw)

    step()
    torch.cuda.synchronize()
    torch.cuda._sleep(5_000_000)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10


for n in (1, 2, 4, 8, 32):
    print("device F+B+U N =", n, round(dev_step_ms(n), 4), "ms")


def pipeline(nchunk, chunk, compute=True):
    """the host-step schedule re-done with torch streams + timing events"""
    spec = d.make_layer_spec(chunk, 256, 64, 56, 56, 1, 1, 1, 0, 0, 16)
    N = nchunk * chunk
    xs = 256 * 56 * 56
    gs = 64 * 56 * 56
    xh = torch.empty(N * xs).pin_memory()
    gh = torch.empty(N * gs).pin_memory()
    yh = torch.empty(N * gs).pin_memory()
    dxh = torch.empty(N * xs).pin_memory()
    X = [d.BlockedActivation(chunk, 256, 56, 56) for _ in range(2)]
    G = [d.BlockedActivation(chunk, 64, 56, 56) for _ in range(2)]
    Y = [d.BlockedActivation(chunk, 64, 56, 56) for _ in range(2)]
    DX = [d.BlockedActivation(chunk, 256, 56, 56) for _ in range(2)]
    w = d.BlockedWeight(64, 256, 1, 1)
    dw = d.BlockedWeight(64, 256, 1, 1)
    fp = d.make_forward_plan(spec, 1, None, None, math)
    bc = d.prepare_backward(spec, w, 1, None, math)
    up = d.UpdatePlan(spec, None, math)
    cs = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev_comp = [None, None]
    ev_out = [None, None]
    marks = []
    t0 = E()
    t0.record(cs)
    h2d.wait_stream(cs)
    d2h.wait_stream(cs)
    for i in range(nchunk):
        b = i & 1
        with torch.cuda.stream(h2d):
            if i >= 2:
                h2d.wait_event(ev_comp[b])
            a0 = E(); a0.record(h2d)
            X[b].data.copy_(xh[i * chunk * xs:(i + 1) * chunk * xs], non_blocking=True)
            G[b].data.copy_(gh[i * chunk * gs:(i + 1) * chunk * gs], non_blocking=True)
            a1 = E(); a1.record(h2d)
        cs.wait_event(a1)
        if i >= 2:
            cs.wait_event(ev_out[b])
        c0 = E(); c0.record(cs)
        if compute:
            fp.execute(X[b], w, Y[b])
            bc.execute(w, G[b], DX[b])
            up.execute(X[b], G[b], dw, accumulate=i > 0)
        c1 = E(); c1.record(cs)
        ev_comp[b] = c1
        with torch.cuda.stream(d2h):
            d2h.wait_event(c1)
            o0 = E(); o0.record(d2h)
            yh[i * chunk * gs:(i + 1) * chunk * gs].copy_(Y[b].data, non_blocking=True)
            dxh[i * chunk * xs:(i + 1) * chunk * xs].copy_(DX[b].data, non_blocking=True)
            o1 = E(); o1.record(d2h)
        ev_out[b] = o1
        marks.append((a0, a1, c0, c1, o0, o1))
    cs.wait_stream(d2h)
    t1 = E(); t1.record(cs)
    torch.cuda.synchronize()
    rel = lambda e: round(t0.elapsed_time(e), 3)  # noqa: E731
    for i, m in enumerate(marks):
        print(i, "h2d", rel(m[0]), rel(m[1]), "comp", rel(m[2]), rel(m[3]), "d2h", rel(m[4]), rel(m[5]))
    print("total", rel(t1))


for c in (4,):
    pipeline(8, c)
    pipeline(8, c)
    pipeline(8, c, compute=False)
