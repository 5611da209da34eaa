"""Full-size parity of the BENCHMARKED plans (BASELINE configs 2 and 3), element
by element against the multithreaded CPU oracle (oracle/oracle.c: the
reference's naive f64-accumulating loops, reference.cpp:7-95, one thread per
output channel / image).

* weight update at the full minibatch (cfg2 N=32 with the bench's own plan,
  cfg3a / cfg3b N=64), both math modes, every dW element gated;
* the split-factor sweep of the weight update (acceptance.cpp:141-170 runs
  the COPY_REDUCE strategy at G in {1, 2, 4}; here the split-K factor G over
  {1, 8, 37, 74, auto}): every factor passes the gate and is bitwise
  reproducible run to run (acceptance.cpp:156-164);
* cfg3 forward / backward-data at full size in bf16 storage and math, checked
  on an image subset (outputs are independent per image).

Gates (BASELINE north_star): e = max|ref - got| / rms(ref) <= 1e-4
(fp32-accurate), <= 2e-2 (bf16). Set DCONV_PARITY_LOG=<path> to append one
JSON line per check (profiles/r02_parity_full_size.jsonl is such a log).
"""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOL = {0: 1e-4, 1: 2e-2}

SHAPES = {  # N, C, K, H, W, R, S, stride, pad_h, pad_w  (BASELINE.json configs[1], [2])
    "cfg2": (32, 256, 64, 56, 56, 1, 1, 1, 0, 0),
    "cfg3a": (64, 3, 64, 224, 224, 7, 7, 2, 3, 3),
    "cfg3b": (64, 512, 1024, 28, 28, 1, 1, 2, 0, 0),
}


def _log(rec):
    path = os.environ.get("DCONV_PARITY_LOG")
    print(json.dumps(rec))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def gate(orc, ref, got, math, what):
    n = orc.error_norms(ref, got)
    _log({"check": what, "math": "f32" if int(math) == 0 else "bf16", **{k: float(v) for k, v in n.items()}})
    assert n["max_over_rms"] <= TOL[int(math)], (what, n)
    return n


@pytest.fixture(scope="module")
def inputs(orc):
    cache = {}

    def get(cfg):
        if cfg not in cache:
            N, C_, K, H, W, R, S, st, ph, pw = SHAPES[cfg]
            s = orc.spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
            P, Q = orc.output_shape(s)
            # the bench's seeds: activations 0, weights 1, output gradients 2
            x = orc.uniform(0, (N, C_, H, W))
            w = orc.he_normal(1, (K, C_, R, S), C_ * R * S)
            g = orc.uniform(2, (N, K, P, Q))
            cache[cfg] = (s, x, w, g, orc.conv_update(s, x, g))
        return cache[cfg]

    return get


def _dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


def _blocked(d, cfg, x, g, storage):
    N, C_, K, H, W, R, S, st, ph, pw = SHAPES[cfg]
    spec = d.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    ib = d.to_blocked_activation(_dev(x), 16, ph, pw, dtype=storage)
    gb = d.to_blocked_activation(_dev(g), 16, 0, 0, dtype=storage)
    return spec, ib, gb


def _run_upd(d, spec, ib, gb, math, cfg=None):
    plan = d.UpdatePlan(spec, cfg, math)
    dw = d.BlockedWeight(spec.K, spec.C, spec.R, spec.S, 16, torch.float32, ib.data.device)
    plan.execute(ib, gb, dw)
    torch.cuda.synchronize()
    return plan, dw


@pytest.mark.parametrize("math", [0, 1], ids=["f32", "bf16"])
@pytest.mark.parametrize("cfg", ["cfg2", "cfg3a", "cfg3b"])
def test_full_batch_update_elementwise(dconv, orc, inputs, cfg, math):
    """The whole-minibatch dW of the plan the bench / executor runs, every
    element against the oracle. fp32-accurate runs on fp32 tensors; bf16 on
    bf16 tensors (the cfg4/cfg5 storage), compared with the oracle on the
    original fp32 inputs (quantisation error included)."""
    s, x, w, g, ref = inputs(cfg)
    M = dconv.Math(math)
    storage = torch.float32 if M == dconv.Math.F32 else torch.bfloat16
    spec, ib, gb = _blocked(dconv, cfg, x, g, storage)
    plan, dw = _run_upd(dconv, spec, ib, gb, M)
    blk = plan.blocking
    got = dconv.from_blocked_weight(dw).cpu().numpy()
    gate(orc, ref, got, M, f"{cfg} upd N={spec.N} splits={blk.get('splits')} mode={blk.get('mode')}")
    if cfg == "cfg2" and M == dconv.Math.F32:
        # the bench's cfg2 plan (bench.py: UpdatePlan(spec, None, F32)) is the 74-split TMEM-staged one
        assert blk.get("a_in_tmem") == 1, blk


@pytest.mark.parametrize("splits", [1, 8, 37, 74, 0], ids=["G1", "G8", "G37", "G74", "auto"])
def test_update_split_factor_sweep(dconv, orc, inputs, splits):
    """cfg2 at N=32, fp32-accurate: every split-K factor passes the gate and is
    bitwise reproducible; all factors agree with one another within the gate."""
    s, x, w, g, ref = inputs("cfg2")
    spec, ib, gb = _blocked(dconv, "cfg2", x, g, torch.float32)
    cfg = dconv.EngineConfig(upd_splits=splits)
    plan, a = _run_upd(dconv, spec, ib, gb, dconv.Math.F32, cfg)
    _, b = _run_upd(dconv, spec, ib, gb, dconv.Math.F32, cfg)
    if splits:
        assert plan.blocking["splits"] == splits, plan.blocking
    assert torch.equal(a.data, b.data), "weight update must be bitwise reproducible at a fixed split factor"
    gate(orc, ref, dconv.from_blocked_weight(a).cpu().numpy(), dconv.Math.F32,
         f"cfg2 upd split sweep G={plan.blocking['splits']}")


@pytest.mark.parametrize("cfg", ["cfg3a", "cfg3b"])
def test_cfg3_bf16_forward_backward_full_size(dconv, orc, inputs, cfg):
    """cfg3 in bf16 storage + bf16 math at the full N=64 (the oracle runs on a
    subset of images: FWD and BWD-data are independent per image)."""
    s, x, w, g, _ = inputs(cfg)
    N, C_, K, H, W, R, S, st, ph, pw = SHAPES[cfg]
    M = dconv.Math.BF16
    spec = dconv.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    ib = dconv.to_blocked_activation(_dev(x), 16, ph, pw, dtype=torch.bfloat16)
    wb = dconv.to_blocked_weight(_dev(w), spec)
    out = dconv.forward(spec, ib, wb, dconv.make_forward_plan(spec, 1, None, None, M))
    gb = dconv.to_blocked_activation(_dev(g), 16, 0, 0, dtype=torch.bfloat16)
    gi = dconv.backward_with(dconv.prepare_backward(spec, wb, 1, None, M), gb)
    got_f = dconv.from_blocked_activation(out, dtype=torch.float32).cpu().numpy()
    got_b = dconv.from_blocked_activation(gi, dtype=torch.float32).cpu().numpy()
    imgs = [0, N // 2, N - 1]
    sub = orc.spec(len(imgs), C_, K, H, W, R, S, st, ph, pw, 16)
    gate(orc, orc.conv_forward(sub, x[imgs], w), got_f[imgs], M, f"{cfg} fwd bf16 N={N} imgs={imgs}")
    rb = orc.conv_backward(sub, g[imgs], w)
    gb_sub = got_b[imgs]
    if R == 1 and S == 1 and st == 2:
        mask = np.ones_like(gb_sub, bool)
        mask[:, :, ::2, ::2] = False
        assert not gb_sub[mask].any(), "off-lattice dI must be exactly 0"
        rb, gb_sub = np.ascontiguousarray(rb[:, :, ::2, ::2]), np.ascontiguousarray(gb_sub[:, :, ::2, ::2])
    gate(orc, rb, gb_sub, M, f"{cfg} bwd bf16 N={N} imgs={imgs}")


@pytest.mark.parametrize("cfg", ["cfg2", "cfg3a", "cfg3b"])
def test_full_batch_forward_backward_all_images_f32(dconv, orc, inputs, cfg):
    """fp32-accurate FWD / BWD-data of the full minibatch, EVERY image against
    the multithreaded oracle (the bench's cfg2 plans included)."""
    s, x, w, g, _ = inputs(cfg)
    N, C_, K, H, W, R, S, st, ph, pw = SHAPES[cfg]
    M = dconv.Math.F32
    spec = dconv.make_layer_spec(N, C_, K, H, W, R, S, st, ph, pw, 16)
    ib = dconv.to_blocked_activation(_dev(x), spec)
    wb = dconv.to_blocked_weight(_dev(w), spec)
    out = dconv.forward(spec, ib, wb, dconv.make_forward_plan(spec, 1, None, None, M))
    gate(orc, orc.conv_forward(s, x, w), dconv.from_blocked_activation(out).cpu().numpy(), M, f"{cfg} fwd f32 N={N}")
    gb = dconv.to_blocked_activation(_dev(g), 16, 0, 0)
    gi = dconv.from_blocked_activation(dconv.backward_with(dconv.prepare_backward(spec, wb, 1, None, M), gb)).cpu().numpy()
    rb = orc.conv_backward(s, g, w)
    if R == 1 and S == 1 and st == 2:
        rb, gi = np.ascontiguousarray(rb[:, :, ::2, ::2]), np.ascontiguousarray(gi[:, :, ::2, ::2])
    gate(orc, rb, gi, M, f"{cfg} bwd f32 N={N}")
