"""The native layer-graph executor (dconv_graph_*) in data-parallel use.

* 2 ranks (gloo, both on the one GPU) each run their half of the minibatch;
  after the exchange the summed weight gradient equals the single-process
  full-batch executor's (fp32-accurate: l2_rel <= 1e-5) and the CPU oracle's
  per-layer update on the full batch;
* the NCCL path (native communicator, world 1 on one GPU): bucketed all-reduce
  inside the step, and the step captured into ONE CUDA graph with the
  collectives in it, replays to the same bits as the eager step;
* the SM budget for co-running collectives leaves results unchanged.
The reference's COPY_REDUCE over minibatch shards: propagation.cpp:357-375,
413-457; run_chain: harness.cpp:311-358.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
IMG, N_GLOBAL = 64, 4


def _inputs(orc, e, n0, n):
    """images n0 .. n0+n of the seeded global minibatch, and its top gradient"""
    from paper_1808_05567_b200 import api as d

    x = orc.uniform(0, (N_GLOBAL, 3, IMG, IMG))[n0:n0 + n]
    c, h, w = e.shapes[e.nodes[-1].out]
    dtop = orc.uniform(2, (N_GLOBAL, c, h, w))[n0:n0 + n]
    xt = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    dt = d.to_blocked_activation(torch.from_numpy(np.ascontiguousarray(dtop)).cuda(), 16, 0, 0, dtype=e.adt)
    return xt, dt


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1808_05567_b200 import api as d
    from paper_1808_05567_b200 import executor as ex

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nodes = ex.resnet50_conv_stack(IMG)
        n = N_GLOBAL // world
        e = ex.ConvStackExecutor(nodes, n, IMG, d.Math.F32, "cuda", group=dist.group.WORLD, lr=0.0,
                                 act_dtype=torch.float32, bucket_bytes=1 << 20)
        xt, dt = _inputs(orc, e, rank * n, n)
        e.load_input_nchw(xt)
        e.forward()
        e.backward(dt)  # native backward, then the gloo all-reduce of the flat gradient
        torch.cuda.synchronize()
        q.put((rank, e.flat.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_executor_equals_full_batch(dconv, orc):
    import multiprocessing as mp

    from paper_1808_05567_b200 import executor as ex

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert np.array_equal(res[0], res[1]), "all-reduced gradients differ between ranks"
    # single process, the whole minibatch
    nodes = ex.resnet50_conv_stack(IMG)
    e = ex.ConvStackExecutor(nodes, N_GLOBAL, IMG, dconv.Math.F32, "cuda", lr=0.0, act_dtype=torch.float32)
    xt, dt = _inputs(orc, e, 0, N_GLOBAL)
    e.load_input_nchw(xt)
    e.forward()
    e.backward(dt)
    torch.cuda.synchronize()
    full = e.flat.cpu().numpy()
    n = orc.error_norms(full, res[0])
    print("2-rank vs full batch flat dW:", n)
    assert n["l2_rel"] <= 1e-5, n
    # and every layer's summed gradient against the oracle update of the full batch
    # (in situ: the oracle on the executor's own activations and output gradients)
    worst = 0.0
    for nd in e.convs:
        c_, h_, w_ = e.shapes[nd.src]
        s = orc.spec(N_GLOBAL, nd.C, nd.K, h_, w_, nd.R, nd.S, nd.stride, nd.pad, nd.pad, 16)
        if nd.src == "x":  # load_input packs the images straight into the stem's s2d layout
            xs = orc.uniform(0, (N_GLOBAL, 3, IMG, IMG))
        else:
            xs = dconv.from_blocked_activation(e.act[nd.src]).cpu().numpy()
        gs = dconv.from_blocked_activation(e.grad[nd.out]).cpu().numpy()
        ref = orc.conv_update(s, xs, gs)
        sl = slice(*_slice_of(e, nd))
        got = dconv.from_blocked_weight(
            dconv.BlockedWeight(nd.K, nd.C, nd.R, nd.S, 16, torch.float32, "cuda",
                                data=torch.from_numpy(res[0][sl]).cuda())).cpu().numpy()
        m = orc.error_norms(ref, got)
        worst = max(worst, m["max_over_rms"])
        assert m["max_over_rms"] <= 1e-4, (nd.name, m)
    print("worst per-layer max/rms of the exchanged gradients:", worst)


def _slice_of(e, nd):
    base = e.flat.data_ptr()
    off = (e.dw[nd.name].data.data_ptr() - base) // 4
    return off, off + e.dw[nd.name].data.numel()


def test_nccl_step_in_one_cuda_graph_matches_eager(dconv, orc):
    """world 1 over a native NCCL communicator: the bucketed all-reduces run on the
    communication stream inside the step; the captured step replays bitwise."""
    import torch.distributed as dist

    from paper_1808_05567_b200 import executor as ex

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        nodes = ex.resnet50_conv_stack(IMG)
        B = 8
        kw = dict(lr=1e-6, act_dtype=torch.bfloat16, bucket_bytes=2 << 20)  # small: no divergence to inf
        e_ref = ex.ConvStackExecutor(nodes, B, IMG, dconv.Math.BF16, "cuda", **kw)
        e = ex.ConvStackExecutor(nodes, B, IMG, dconv.Math.BF16, "cuda", group=dist.group.WORLD, use_nccl=True, **kw)
        assert e.buckets() >= 3 and e.buckets() == len(e.bucketer.buckets)  # native rule == GradBucketer's
        x = torch.from_numpy(orc.uniform(0, (B, 3, IMG, IMG))).cuda()
        c, h, w = e.shapes[nodes[-1].out]
        dtop = dconv.to_blocked_activation(torch.from_numpy(orc.uniform(2, (B, c, h, w))).cuda(), 16, 0, 0,
                                           dtype=torch.bfloat16)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for ee in (e_ref, e):
                ee.load_input_nchw(x)
                ee.step(dtop)  # eager step (exchange + SGD)
        torch.cuda.synchronize()
        assert torch.equal(e_ref.flat, e.flat) and torch.equal(e_ref.wflat, e.wflat)
        # capture the NCCL executor's step into a CUDA graph; replay twice against two eager steps
        with torch.cuda.stream(s):
            e.capture(dtop)
        torch.cuda.synchronize()
        w0 = e.wflat.clone()
        e.wflat.copy_(e_ref.wflat)
        with torch.cuda.stream(s):
            for _ in range(2):
                e.replay()
                e_ref.step(dtop)
        torch.cuda.synchronize()
        assert e.launches_per_step() > 100
        assert torch.equal(e_ref.wflat, e.wflat), "graph replay differs from the eager step"
        assert not torch.equal(w0, e.wflat)
    finally:
        dist.destroy_process_group()


def test_sm_budget_keeps_results(dconv, orc):
    from paper_1808_05567_b200 import executor as ex

    lib = dconv._lib.lib()
    nodes = ex.resnet50_conv_stack(IMG)
    outs = []
    for budget in (0, 132):
        lib.dconv_set_sm_budget(budget)
        try:
            e = ex.ConvStackExecutor(nodes, 4, IMG, dconv.Math.BF16, "cuda", lr=0.0)
            x = torch.from_numpy(orc.uniform(0, (4, 3, IMG, IMG))).cuda()
            c, h, w = e.shapes[nodes[-1].out]
            dtop = dconv.to_blocked_activation(torch.from_numpy(orc.uniform(2, (4, c, h, w))).cuda(), 16, 0, 0,
                                               dtype=torch.bfloat16)
            e.load_input_nchw(x)
            e.step(dtop)
            torch.cuda.synchronize()
            outs.append(e.flat.clone())
            blk = e.act[nodes[-1].out].data.clone()
            outs.append(blk)
        finally:
            lib.dconv_set_sm_budget(0)
    # forward outputs are tiling-independent bitwise; the gradients only up to the
    # split-K order (the split factor follows the SM count)
    assert torch.equal(outs[1], outs[3])
    n = orc.error_norms(outs[0].cpu().numpy(), outs[2].cpu().numpy())
    assert n["l2_rel"] <= 1e-5, n
