"""Dev experiment: two half-batch executors on two streams (forward + backward each,
concurrently) vs one full-batch executor, device time per 256 images. Weights are
not shared here: this measures only whether the concurrency pays."""
import os, sys, torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1808_05567_b200 as d  # noqa: E402
from paper_1808_05567_b200 import executor as ex  # noqa: E402
nodes = ex.resnet50_conv_stack()


def mk(n):
    e = ex.ConvStackExecutor(nodes, n, 224, d.Math.BF16, "cuda", lr=0.0)
    e.act["x"].data.uniform_(-1, 1)
    c, h, w = e.shapes[nodes[-1].out]
    g = d.BlockedActivation(n, c, h, w, 16, 0, 0, torch.bfloat16)
    g.data.uniform_(-1, 1)
    return e, g


def bench(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


e, g = mk(256)
t_full = bench(lambda: e.step(g))
del e, g
torch.cuda.empty_cache()
(e1, g1), (e2, g2) = mk(128), mk(128)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def two():
    main = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(main)
    for s, e_, g_ in ((s1, e1, g1), (s2, e2, g2)):
        s.wait_event(ev)
        with torch.cuda.stream(s):
            e_.forward()
            e_.backward(g_)
    main.wait_stream(s1)
    main.wait_stream(s2)
    e1.sgd()


t_two = bench(two)
t_serial = bench(lambda: (e1.step(g1), e2.step(g2)))
print(f"full batch 256: {t_full:.2f} ms | two 128 concurrent: {t_two:.2f} ms | two 128 serial: {t_serial:.2f} ms")
