"""dev: eager step vs captured-graph replay of the native executor, per layer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1808_05567_b200 as d
from paper_1808_05567_b200 import executor as ex
from oracle import oracle as orc

IMG, B = 64, 8
nodes = ex.resnet50_conv_stack(IMG)
mk = lambda: ex.ConvStackExecutor(nodes, B, IMG, d.Math.BF16, "cuda", lr=float(os.environ.get("LR", "1e-3")),
                                  overlap_upd=os.environ.get("NOOV") is None)
a, b = mk(), mk()
x = torch.from_numpy(orc.uniform(0, (B, 3, IMG, IMG))).cuda()
c, h, w = a.shapes[nodes[-1].out]
dtop = d.to_blocked_activation(torch.from_numpy(orc.uniform(2, (B, c, h, w))).cuda(), 16, 0, 0, dtype=torch.bfloat16)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for e in (a, b):
        e.load_input_nchw(x)
    a.step(dtop); b.step(dtop)
torch.cuda.synchronize()
print("eager a==b", torch.equal(a.flat, b.flat), torch.equal(a.wflat, b.wflat))
with torch.cuda.stream(s):
    b.capture(dtop)
torch.cuda.synchronize()
for it in range(3):
    with torch.cuda.stream(s):
        a.step(dtop)
        b.replay()
    torch.cuda.synchronize()
    print("iter", it, "flat eq", torch.equal(a.flat, b.flat), "w eq", torch.equal(a.wflat, b.wflat),
          "top eq", torch.equal(a.act[nodes[-1].out].data, b.act[nodes[-1].out].data))
    for nd in nodes:
        if isinstance(nd, ex.ConvNode):
            if not torch.equal(a.dw[nd.name].data, b.dw[nd.name].data):
                dd = (a.dw[nd.name].data - b.dw[nd.name].data).abs().max().item()
                print("  dW differs", nd.name, dd)
        if not torch.equal(a.act[nd.out].data, b.act[nd.out].data):
            print("  act differs", nd.out)
            break
