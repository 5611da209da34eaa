"""Data-parallel layer-graph executor for conv stacks (ResNet-50 v1 conv stack).

The reference's `run_chain` (harness.cpp:311-358) runs a LINEAR chain of
forward convs, each layer writing its output straight into the next layer's
input surface. This executor is its training-time, multi-GPU generalisation:
a DAG of convs (bottleneck blocks with identity / projection shortcuts and the
stem max-pool) run forward, backward-data and weight-update on one B200 per
process, with the fp32 weight gradients summed across ranks by NCCL all-reduce
(the reference's COPY_REDUCE exchange promoted from threads to GPUs),
bucketed and overlapped with the backward of earlier layers.

Everything elementwise is fused into the conv epilogues of the C ABI
(`dconv_forward_ex` / `dconv_backward_data_ex`): ReLU and the residual add in
the forward, the ReLU mask and the two-branch gradient sum in the backward.
Activations are bf16 blocked tensors with halo 0 (padding is a TMA
out-of-bounds fill), weights fp32 masters in the blocked layout (prepared to
bf16 per pass), gradients fp32 for the weights.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib
from . import api as d
from ._lib import Act, Epilogue, Wt

# ------------------------------------------------------------------ graph


@dataclasses.dataclass
class ConvNode:
    name: str
    src: str              # input tensor
    out: str              # output tensor
    C: int
    K: int
    R: int
    S: int
    stride: int
    pad: int
    relu: bool = True
    add: Optional[str] = None  # residual added before the ReLU


@dataclasses.dataclass
class PoolNode:
    name: str
    src: str
    out: str


def resnet50_conv_stack(img: int = 224) -> List:
    """The 53 convs of ResNet-50 v1 (stride on the first 1x1 of a
    down-sampling block, SURVEY 8(d) cfg4 / Table I ids 6, 7, 11, 12, 16, 17)
    plus the stem max-pool. Tensor 'x' is the input image (3 channels)."""
    nodes: List = [ConvNode("stem", "x", "stem", 3, 64, 7, 7, 2, 3), PoolNode("pool", "stem", "s0")]
    cur, c_in = "s0", 64
    for si, (blocks, mid) in enumerate(((3, 64), (4, 128), (6, 256), (3, 512))):
        for bi in range(blocks):
            stride = 2 if (bi == 0 and si > 0) else 1
            out_c = 4 * mid
            pre = f"l{si + 1}b{bi}"
            sc = cur
            if bi == 0:  # projection shortcut (no ReLU; added before the block ReLU)
                nodes.append(ConvNode(pre + "p", cur, pre + "_p", c_in, out_c, 1, 1, stride, 0, relu=False))
                sc = pre + "_p"
            nodes.append(ConvNode(pre + "a", cur, pre + "_a", c_in, mid, 1, 1, stride, 0))
            nodes.append(ConvNode(pre + "b", pre + "_a", pre + "_b", mid, mid, 3, 3, 1, 1))
            nodes.append(ConvNode(pre + "c", pre + "_b", pre + "_o", mid, out_c, 1, 1, 1, 0, add=sc))
            cur, c_in = pre + "_o", out_c
    return nodes


def tensor_shapes(nodes: Sequence, img: int = 224, in_c: int = 3) -> Dict[str, tuple]:
    shapes = {"x": (in_c, img, img)}
    for nd in nodes:
        c, h, w = shapes[nd.src]
        if isinstance(nd, PoolNode):
            shapes[nd.out] = (c, (h + 2 - 3) // 2 + 1, (w + 2 - 3) // 2 + 1)
        else:
            shapes[nd.out] = (nd.K, (h + 2 * nd.pad - nd.R) // nd.stride + 1, (w + 2 * nd.pad - nd.S) // nd.stride + 1)
    return shapes


def step_flops_per_image(nodes: Sequence, img: int = 224, skip_stem_bwd: bool = True) -> int:
    """FWD + BWD-data + UPD pass_flops (harness.cpp:269-272, logical C) per image."""
    shapes = tensor_shapes(nodes, img)
    tot = 0
    for nd in nodes:
        if isinstance(nd, PoolNode):
            continue
        _, h, w = shapes[nd.src]
        _, p, q = shapes[nd.out]
        f = 2 * nd.K * nd.C * p * q * nd.R * nd.S
        tot += f * (2 if (skip_stem_bwd and nd.src == "x") else 3)
    return tot


# ------------------------------------------------------------------ gradient exchange


class GradBucketer:
    """Fixed-order bucketed all-reduce of a flat fp32 gradient buffer.

    Buckets are contiguous slices laid out in BACKWARD order (the first
    bucket is the last layers' gradients, ready first). `ready(i)` is called
    as each layer's gradient is final; a bucket is launched (async, on the
    communicator's stream) once all its layers are ready, so it overlaps the
    backward of earlier layers. Bucket boundaries and launch order are fixed,
    so the reduction is reproducible for a fixed world size and NCCL algorithm.
    """

    def __init__(self, flat: torch.Tensor, layer_slices: List[slice], bucket_bytes: int = 8 << 20, group=None):
        self.flat, self.group = flat, group
        self.buckets: List[List[int]] = []
        cur, cur_bytes = [], 0
        for i, sl in enumerate(layer_slices):
            cur.append(i)
            cur_bytes += (sl.stop - sl.start) * 4
            if cur_bytes >= bucket_bytes:
                self.buckets.append(cur)
                cur, cur_bytes = [], 0
        if cur:
            self.buckets.append(cur)
        self.slices = layer_slices
        self.of_layer = {i: b for b, ids in enumerate(self.buckets) for i in ids}
        self.pending: List = []
        self._left: List[int] = []

    def bucket_slice(self, b: int) -> slice:
        ids = self.buckets[b]
        return slice(self.slices[ids[0]].start, self.slices[ids[-1]].stop)

    def begin(self):
        self._left = [len(ids) for ids in self.buckets]
        self.pending = []

    def ready(self, layer: int, stream: Optional[torch.cuda.Stream] = None):
        b = self.of_layer[layer]
        self._left[b] -= 1
        if self._left[b] == 0:
            self._launch(b, stream)

    def _launch(self, b: int, stream):
        if self.group is None:
            return
        import torch.distributed as dist

        t = self.flat[self.bucket_slice(b)]
        if stream is not None:
            with torch.cuda.stream(stream):
                self.pending.append(dist.all_reduce(t, group=self.group, async_op=True))
        else:
            self.pending.append(dist.all_reduce(t, group=self.group, async_op=True))

    def finish(self):
        for w in self.pending:
            w.wait()
        self.pending = []


# ------------------------------------------------------------------ executor


class ConvStackExecutor:
    def __init__(self, nodes: Sequence, batch: int, img: int = 224, math: d.Math = d.Math.BF16,
                 device: str = "cuda", group=None, lr: float = 1e-4, seed: int = 1, bucket_bytes: int = 8 << 20,
                 act_dtype=torch.bfloat16, overlap_upd: bool = True):
        self.nodes, self.N, self.img, self.math, self.dev = list(nodes), batch, img, d.Math(math), torch.device(device)
        self.group, self.lr, self.adt = group, lr, act_dtype
        self.lib = _lib.lib()
        self.shapes = tensor_shapes(self.nodes, img)
        self.convs = [nd for nd in self.nodes if isinstance(nd, ConvNode)]
        relu_out = {nd.out for nd in self.nodes if isinstance(nd, ConvNode) and nd.relu}
        relu_out |= {nd.out for nd in self.nodes if isinstance(nd, PoolNode) and nd.src in relu_out}
        self.relu_out = relu_out
        # activations and their gradients (halo 0 blocked, bf16)
        self.act: Dict[str, d.BlockedActivation] = {}
        self.grad: Dict[str, d.BlockedActivation] = {}
        for name, (c, h, w) in self.shapes.items():
            self.act[name] = d.BlockedActivation(batch, c, h, w, 16, 0, 0, act_dtype, self.dev)
            if name != "x":
                self.grad[name] = d.BlockedActivation(batch, c, h, w, 16, 0, 0, act_dtype, self.dev)
        # a projection's output only feeds a residual add: its dL/dz is the block's dz
        for nd in self.convs:
            if nd.add is not None and nd.add in {c.out for c in self.convs if not c.relu}:
                self.grad[nd.add] = self.grad[nd.out]
        pools = [nd for nd in self.nodes if isinstance(nd, PoolNode)]
        self.argmax = {nd.name: torch.empty(self.act[nd.out].data.numel(), dtype=torch.uint8, device=self.dev)
                       for nd in pools}
        # weights: fp32 masters (He-normal, seeded host generator), flat fp32 gradient buffer in backward order
        self.w: Dict[str, d.BlockedWeight] = {}
        self.specs: Dict[str, d.ConvLayerSpec] = {}
        sizes = []
        for nd in self.convs:
            c, h, w = self.shapes[nd.src]
            spec = d.ConvLayerSpec(batch, nd.C, nd.K, h, w, nd.R, nd.S, nd.stride, nd.pad, nd.pad, 16)
            spec.validate()
            self.specs[nd.name] = spec
            host = torch.empty(nd.K, nd.C, nd.R, nd.S, dtype=torch.float32)
            std = float((2.0 / (nd.C * nd.R * nd.S)) ** 0.5)
            self.lib.dconv_fill_he_normal_host(seed * 1000 + len(sizes), std, host.data_ptr(), host.numel())
            self.w[nd.name] = d.to_blocked_weight(host.to(self.dev), spec)
            sizes.append(self.w[nd.name].data.numel())
        order = list(reversed(range(len(self.convs))))  # gradients become final in reverse order
        self.flat = torch.zeros(sum(sizes), dtype=torch.float32, device=self.dev)
        self.slices: List[slice] = [slice(0, 0)] * len(self.convs)
        off = 0
        for i in order:
            self.slices[i] = slice(off, off + sizes[i])
            off += sizes[i]
        self.dw = {nd.name: d.BlockedWeight(nd.K, nd.C, nd.R, nd.S, 16, torch.float32, self.dev,
                                            data=self.flat[self.slices[i]])
                   for i, nd in enumerate(self.convs)}
        # master weights in one flat buffer laid out like the gradients: SGD is ONE launch
        self.wflat = torch.empty_like(self.flat)
        for i, nd in enumerate(self.convs):
            self.wflat[self.slices[i]].copy_(self.w[nd.name].data.reshape(-1))
            self.w[nd.name] = d.BlockedWeight(nd.K, nd.C, nd.R, nd.S, 16, torch.float32, self.dev,
                                              data=self.wflat[self.slices[i]])
        n256 = self.flat.numel() // 256  # every blocked weight is a whole number of 16x16 lane blocks
        self._wflat_view = d.BlockedWeight(16, 16, 1, n256, 16, torch.float32, self.dev, data=self.wflat)
        self._gflat_view = d.BlockedWeight(16, 16, 1, n256, 16, torch.float32, self.dev, data=self.flat)
        self.bucketer = GradBucketer(self.flat, [self.slices[i] for i in order], bucket_bytes, group)
        self._bucket_index = {i: k for k, i in enumerate(order)}
        # narrow stride-2 input convs (the 7x7/s2 stem, C=3) run as a stride-1 conv over a
        # space-to-depth copy of their input: 4x4 taps over 12 of 16 lanes instead of
        # 49 taps over 3 of 16 (the MMA K dimension is a 16-lane channel block)
        self.s2d: Dict[str, dict] = {}
        for nd in self.convs:
            c, h, w = self.shapes[nd.src]
            if nd.stride == 2 and nd.C * 4 <= 16 and nd.R > 1 and nd.S > 1:
                _, P, Q = self.shapes[nd.out]
                r2, s2 = (nd.R + 1) // 2, (nd.S + 1) // 2
                hs, wsz = P + r2 - 1, Q + s2 - 1
                spec2 = d.ConvLayerSpec(batch, 4 * nd.C, nd.K, hs, wsz, r2, s2, 1, 0, 0, 16)
                spec2.validate()
                self.s2d[nd.name] = {
                    "spec": spec2,
                    "x": d.BlockedActivation(batch, 4 * nd.C, hs, wsz, 16, 0, 0, act_dtype, self.dev),
                    "w": d.BlockedWeight(nd.K, 4 * nd.C, r2, s2, 16, torch.float32, self.dev),
                    "dw": d.BlockedWeight(nd.K, 4 * nd.C, r2, s2, 16, torch.float32, self.dev),
                }
        # plans
        self.input_s2d = False  # set by load_input_nchw: the stem's s2d input is packed directly
        self.pspec = {n: (self.s2d[n]["spec"] if n in self.s2d else s) for n, s in self.specs.items()}
        self.fplan = {n: d.ExecutionPlan(s, None, None, self.math, 0, 0) for n, s in self.pspec.items()}
        self.bplan = {n: d.BackwardContext(s, None, 1, None, self.math) for n, s in self.specs.items()
                      if self._needs_bwd(n)}
        self.uplan = {n: d.UpdatePlan(s, None, self.math) for n, s in self.pspec.items()}
        self.comm_stream = torch.cuda.Stream(self.dev) if group is not None else None
        self._ev = {i: torch.cuda.Event() for i in range(len(self.convs))}
        # weight updates (+ their split reductions) run on a side stream, concurrent with the
        # backward-data chain: each kernel's last-wave tail is filled by the other's CTAs and
        # the small reduction kernels leave the critical path. A layer's update is forked
        # once its output gradient is final; SGD joins.
        self.upd_stream = torch.cuda.Stream(self.dev) if (self.dev.type == "cuda" and overlap_upd) else None
        self._ev_gready = {i: torch.cuda.Event() for i in range(len(self.convs))}

    def _needs_bwd(self, name):
        nd = next(n for n in self.convs if n.name == name)
        return nd.src != "x"  # the stem's backward-data (image gradient) is skipped

    # -------------------------------------------------------------- passes
    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def _ep(self, add=None, mask=None, relu=False):
        return Epilogue(add.data.data_ptr() if add is not None else None,
                        mask.data.data_ptr() if mask is not None else None, 1 if relu else 0)

    def forward(self):
        for nd in self.nodes:
            if isinstance(nd, PoolNode):
                _check(self.lib.dconv_maxpool_fwd(C.byref(self.act[nd.src].to_c()), C.byref(self.act[nd.out].to_c()),
                                                  self.argmax[nd.name].data_ptr(), self._stream()))
                continue
            self.conv_forward(nd)

    def conv_forward(self, nd: ConvNode):
        plan = self.fplan[nd.name]
        ep = self._ep(add=self.act[nd.add] if nd.add else None, relu=nd.relu)
        ws = plan._ws.get(self.lib.dconv_fwd_workspace_bytes(plan._h), self.dev)
        src, wt = self.act[nd.src], self.w[nd.name]
        if nd.name in self.s2d:
            sd = self.s2d[nd.name]
            if not (nd.src == "x" and self.input_s2d):  # load_input_nchw packed it already
                _check(self.lib.dconv_s2d_act(C.byref(src.to_c()), C.byref(sd["x"].to_c()), nd.pad, self._stream()))
            _check(self.lib.dconv_s2d_wt(C.byref(wt.to_c()), C.byref(sd["w"].to_c()), 0, self._stream()))
            src, wt = sd["x"], sd["w"]
        _check(self.lib.dconv_forward_ex(plan._h, C.byref(src.to_c()), C.byref(wt.to_c()),
                                         C.byref(self.act[nd.out].to_c()), C.byref(ep), ws, self._stream()))

    def load_input_nchw(self, nchw: torch.Tensor):
        """Pack this step's images (N, 3, H, W fp32 on the device) into the executor's
        input: straight into the stem's space-to-depth layout when the stem runs that
        way (one pass, no full-resolution 16-lane copy), else the blocked tensor 'x'.
        Steps after this skip the stem's own space-to-depth."""
        stem = next((nd for nd in self.convs if nd.src == "x"), None)
        if stem is not None and stem.name in self.s2d:
            n, c, h, w = nchw.shape
            _check(self.lib.dconv_pack_s2d(nchw.data_ptr(), n, c, h, w, C.byref(self.s2d[stem.name]["x"].to_c()),
                                           stem.pad, self._stream()))
            self.input_s2d = True
        else:
            _check(self.lib.dconv_pack_act(nchw.data_ptr(), 0, C.byref(self.act["x"].to_c()), self._stream()))

    def conv_update(self, nd: ConvNode):
        up = self.uplan[nd.name]
        src, dw = self.act[nd.src], self.dw[nd.name]
        if nd.name in self.s2d:  # s2d copy of the input was made by the forward of this step
            src, dw = self.s2d[nd.name]["x"], self.s2d[nd.name]["dw"]
        a, g = src.to_c(), self.grad[nd.out].to_c()
        ws = up._ws.get(self.lib.dconv_upd_workspace_bytes(up._h, C.byref(a), C.byref(g)), self.dev)
        _check(self.lib.dconv_weight_update(up._h, C.byref(a), C.byref(g), C.byref(dw.to_c()), 0, ws,
                                            self._stream()))
        if nd.name in self.s2d:
            _check(self.lib.dconv_s2d_wt(C.byref(self.dw[nd.name].to_c()), C.byref(dw.to_c()), 1, self._stream()))

    def backward(self, dtop: d.BlockedActivation):
        """Gradient buffers hold dL/dz (already through the ReLU of their tensor)."""
        top = self.nodes[-1].out
        mask = self.act[top] if top in self.relu_out else None
        self.grad[top].data.copy_(dtop.data)
        if mask is not None:
            self.grad[top].data.mul_((mask.data > 0).to(self.grad[top].data.dtype))
        self.bucketer.begin()
        written = set()
        for idx in reversed(range(len(self.nodes))):
            nd = self.nodes[idx]
            if isinstance(nd, PoolNode):
                if nd.src in self.relu_out:  # ReLU mask of the pooled input, read off the pooled output
                    _check(self.lib.dconv_maxpool_bwd_pooled_mask(
                        C.byref(self.grad[nd.out].to_c()), self.argmax[nd.name].data_ptr(),
                        C.byref(self.grad[nd.src].to_c()), C.byref(self.act[nd.out].to_c()), self._stream()))
                else:
                    _check(self.lib.dconv_maxpool_bwd(C.byref(self.grad[nd.out].to_c()),
                                                      self.argmax[nd.name].data_ptr(),
                                                      C.byref(self.grad[nd.src].to_c()), None, self._stream()))
                written.add(nd.src)
                continue
            ci = self.convs.index(nd)
            g_out = self.grad[nd.out]  # = dL/dz of this conv (its epilogue's pre-activation), final here
            if self.upd_stream is not None:
                self._ev_gready[ci].record()
                self.upd_stream.wait_event(self._ev_gready[ci])
                with torch.cuda.stream(self.upd_stream):
                    self.conv_update(nd)  # weight gradient
                    if self.group is not None:
                        self._ev[ci].record()
                        self.comm_stream.wait_event(self._ev[ci])
            else:
                self.conv_update(nd)
                if self.group is not None:
                    self._ev[ci].record()
                    self.comm_stream.wait_event(self._ev[ci])
            self.bucketer.ready(self._bucket_index[ci], self.comm_stream)
            # residual branch: a projection shares this dz (aliased buffer); an identity
            # shortcut's contribution is folded into the input-gradient epilogue below
            if nd.src == "x":
                continue
            # data gradient of the conv input, through the ReLU of that tensor, summing branches
            gi = self.grad[nd.src]
            mask = self.act[nd.src] if nd.src in self.relu_out else None
            add = None
            if nd.src in written:
                add = gi  # second contribution: accumulate in place
            else:
                ident = [c for c in self.convs if c.add == nd.src]  # identity shortcut consumer of src
                if ident:
                    add = self.grad[ident[0].out]
            bp = self.bplan[nd.name]
            ws = bp._ws.get(self.lib.dconv_bwd_workspace_bytes(bp._h), self.dev)
            ep = self._ep(add=add, mask=mask)
            _check(self.lib.dconv_backward_data_ex(bp._h, C.byref(self.w[nd.name].to_c()), C.byref(g_out.to_c()),
                                                   C.byref(gi.to_c()), C.byref(ep), ws, self._stream()))
            written.add(nd.src)
        if self.upd_stream is not None:
            torch.cuda.current_stream().wait_stream(self.upd_stream)  # join: every dW final

    def sgd(self):
        self.bucketer.finish()
        if self.group is not None:
            import torch.distributed as dist

            self.flat.div_(dist.get_world_size(self.group))
        _check(self.lib.dconv_sgd(C.byref(self._wflat_view.to_c()), C.byref(self._gflat_view.to_c()), self.lr,
                                  self._stream()))

    def step(self, dtop: d.BlockedActivation):
        self.forward()
        self.backward(dtop)
        self.sgd()

    def launches_per_step(self) -> int:
        n = 0
        for nd in self.nodes:
            if isinstance(nd, PoolNode):
                n += 2
                continue
            n += self.fplan[nd.name].launches()
            src = self.s2d[nd.name]["x"] if nd.name in self.s2d else self.act[nd.src]
            n += self.uplan[nd.name].launches(src, self.grad[nd.out])
            if nd.name in self.s2d:
                n += 3  # input / filter space-to-depth, gradient back
            if nd.name in self.bplan:
                n += self.bplan[nd.name].launches()
        return n + 1  # one SGD launch over the flat weights


def _check(st):
    d._check(st)
