"""TEST INFRASTRUCTURE ONLY — composition oracle for the conv-stack executor.

The reference has no multi-layer backward (run_chain is forward-only,
harness.cpp:311-358), no residual add and no pooling, so the stack pieces
around the convs are "parity unpinned": this module composes the PINNED conv
oracles (oracle.c: conv_forward / conv_backward / conv_update, f64 accumulate)
with numpy ReLU, residual add and 3x3/s2/p1 max-pool, mirroring the
executor's graph semantics (paper_1808_05567_b200/executor.py)."""
import numpy as np

from . import oracle as orc


def maxpool_fwd(x):
    n, c, h, w = x.shape
    p, q = (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1
    out = np.full((n, c, p, q), -np.inf, np.float32)
    arg = np.zeros((n, c, p, q), np.int8)
    for dy in range(3):
        for dx in range(3):
            ys = 2 * np.arange(p) - 1 + dy
            xs = 2 * np.arange(q) - 1 + dx
            vy, vx = (ys >= 0) & (ys < h), (xs >= 0) & (xs < w)
            v = np.full((n, c, p, q), -np.inf, np.float32)
            v[:, :, vy[:, None] & vx[None, :]] = x[:, :, ys[vy]][:, :, :, xs[vx]].reshape(n, c, -1)
            better = v > out
            out = np.where(better, v, out)
            arg = np.where(better, dy * 3 + dx, arg)
    return out, arg


def maxpool_bwd(g, arg, h, w):
    n, c, p, q = g.shape
    gi = np.zeros((n, c, h, w), np.float32)
    for dy in range(3):
        for dx in range(3):
            sel = (arg == dy * 3 + dx)
            for y in range(p):
                iy = 2 * y - 1 + dy
                if iy < 0 or iy >= h:
                    continue
                for x in range(q):
                    ix = 2 * x - 1 + dx
                    if 0 <= ix < w:
                        gi[:, :, iy, ix] += np.where(sel[:, :, y, x], g[:, :, y, x], 0.0)
    return gi


def run(nodes, x, weights, dtop, conv_types, pool_type):
    """Forward + backward of the graph. Returns (acts, dws) with dws[name]."""
    acts = {"x": x}
    args = {}
    for nd in nodes:
        if isinstance(nd, pool_type):
            acts[nd.out], args[nd.name] = maxpool_fwd(acts[nd.src])
            continue
        n, c, h, w = acts[nd.src].shape
        s = orc.spec(n, nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, nd.pad, nd.pad, 16)
        z = orc.conv_forward(s, acts[nd.src], weights[nd.name])
        if nd.add:
            z = z + acts[nd.add]
        acts[nd.out] = np.maximum(z, 0) if nd.relu else z
    relu_out = {nd.out for nd in nodes if isinstance(nd, conv_types) and nd.relu}
    relu_out |= {nd.out for nd in nodes if isinstance(nd, pool_type) and nd.src in relu_out}
    grads = {}  # dL/dt (NOT through t's own relu)

    def acc(t, g):
        grads[t] = grads[t] + g if t in grads else g

    acc(nodes[-1].out, dtop)
    dws = {}
    for nd in reversed(nodes):
        g = grads[nd.out]
        if nd.out in relu_out and not isinstance(nd, pool_type):
            g = g * (acts[nd.out] > 0)
        if isinstance(nd, pool_type):
            _, _, h, w = acts[nd.src].shape
            acc(nd.src, maxpool_bwd(g, args[nd.name], h, w))
            continue
        n, c, h, w = acts[nd.src].shape
        s = orc.spec(n, nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, nd.pad, nd.pad, 16)
        dws[nd.name] = orc.conv_update(s, acts[nd.src], g)
        if nd.add:
            acc(nd.add, g)
        if nd.src != "x":
            acc(nd.src, orc.conv_backward(s, g, weights[nd.name]))
    return acts, dws
