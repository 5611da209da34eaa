"""Data-parallel layer-graph executor for conv stacks (ResNet-50 v1 conv stack).

The reference's `run_chain` (harness.cpp:311-358) runs a LINEAR chain of
forward convs, each layer writing its output straight into the next layer's
input surface. Its training-time, multi-GPU generalisation is native code:
`dconv_graph_*` in the C ABI (csrc/graph.cu) runs a DAG of convs (bottleneck
blocks with identity / projection shortcuts and the stem max-pool) forward,
backward-data and weight-update, with ReLU / residual add / ReLU mask /
branch sums fused into the conv epilogues, weight updates on a side stream,
the fp32 weight gradients all-reduced by NCCL in buckets (the reference's
COPY_REDUCE exchange promoted from threads to GPUs) overlapped with the
backward of earlier layers, SGD, and one CUDA graph per step at any world size.

This module describes the graph (ResNet-50's 53 convs), and ConvStackExecutor
is a thin handle over the native executor exposing its tensors as torch views.
With a gloo process group (CPU tests, several ranks sharing one GPU) the
gradient exchange runs in Python (torch.distributed) between the native
backward and apply calls; with an NCCL group the native executor owns its
own communicator (same ranks) and the exchange is inside the step / graph.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Dict, List, Optional, Sequence

import torch

from . import _lib
from . import api as d
from ._lib import Act, GraphCfg, GraphNode, Wt

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
    """Fixed-order bucketed all-reduce of a flat fp32 gradient buffer (the
    exchange of ConvStackExecutor over a gloo group; the native executor,
    csrc/graph.cu, cuts its NCCL buckets by the same rule on its own stream).

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

_DT = {torch.float32: 0, torch.bfloat16: 1}


def _nccl_comm(group, lib):
    """A native NCCL communicator over the ranks of `group` (id made on rank 0)."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    idbuf = C.create_string_buffer(128)
    if rank == 0:
        d._check(lib.dconv_nccl_unique_id(idbuf, 128))
    obj = [bytes(idbuf.raw)]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    comm = C.c_void_p()
    d._check(lib.dconv_nccl_comm_create(obj[0], 128, world, rank, C.byref(comm)))
    return comm


class ConvStackExecutor:
    """Handle over the native executor (dconv_graph_*). `nodes` use tensor names;
    tensor 'x' is the input image."""

    def __init__(self, nodes: Sequence, batch: int, img: int = 224, math: d.Math = d.Math.BF16,
                 device: str = "cuda", group=None, lr: float = 1e-4, seed: int = 1, bucket_bytes: int = 8 << 20,
                 act_dtype=torch.bfloat16, overlap_upd: bool = True, use_nccl: Optional[bool] = None):
        self.nodes, self.N, self.img, self.math = list(nodes), batch, img, d.Math(math)
        self.dev = torch.device(device)
        if self.dev.type == "cuda" and self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        self.group, self.lr, self.adt = group, lr, act_dtype
        self.lib = _lib.lib()
        self.shapes = tensor_shapes(self.nodes, img)
        self.convs = [nd for nd in self.nodes if isinstance(nd, ConvNode)]
        relu_out = {nd.out for nd in self.convs if nd.relu}
        relu_out |= {nd.out for nd in self.nodes if isinstance(nd, PoolNode) and nd.src in relu_out}
        self.relu_out = relu_out  # tensors produced by a ReLU (their gradients carry its mask)
        ids = {"x": 0}
        for i, nd in enumerate(self.nodes):
            ids[nd.out] = i + 1
        self.ids = ids
        arr = (GraphNode * len(self.nodes))()
        for i, nd in enumerate(self.nodes):
            if isinstance(nd, PoolNode):
                arr[i] = GraphNode(_lib.NODE_MAXPOOL, ids[nd.src], -1, 0, 0, 0, 0, 0, 0, 0, 0)
            else:
                arr[i] = GraphNode(_lib.NODE_CONV, ids[nd.src], ids[nd.add] if nd.add else -1, nd.C, nd.K, nd.R,
                                   nd.S, nd.stride, nd.pad, nd.pad, int(nd.relu))
        cfg = GraphCfg()
        self.lib.dconv_graph_config_default(C.byref(cfg))
        cfg.lr, cfg.seed, cfg.bucket_bytes = lr, seed, bucket_bytes
        cfg.overlap_update, cfg.act_dtype = int(overlap_upd), _DT[act_dtype]
        self._comm = None
        self._py_exchange = False
        if group is not None:
            import torch.distributed as dist

            cfg.world, cfg.rank = dist.get_world_size(group), dist.get_rank(group)
            if use_nccl is None:
                use_nccl = dist.get_backend(group) == "nccl"
            if use_nccl:
                self._comm = _nccl_comm(group, self.lib)
                cfg.nccl_comm = self._comm
            else:
                self._py_exchange = cfg.world > 1
        self._bucket_bytes = bucket_bytes
        self._h = C.c_void_p()
        with torch.cuda.device(self.dev):
            d._check(self.lib.dconv_graph_create(arr, len(self.nodes), batch, 3, img, img, int(self.math),
                                                 C.byref(cfg), C.byref(self._h)))
        self._views()

    def _views(self):
        lib, di = self.lib, self.dev.index
        self.act: Dict[str, d.BlockedActivation] = {}
        self.grad: Dict[str, d.BlockedActivation] = {}
        for name, i in self.ids.items():
            for grad, dst in ((0, self.act), (1, self.grad)):
                if grad and i == 0:
                    continue
                a = Act()
                d._check(lib.dconv_graph_tensor(self._h, i, grad, C.byref(a)))
                numel = a.n * -(-a.c // 16) * a.h * a.w * 16
                dst[name] = d.BlockedActivation(a.n, a.c, a.h, a.w, 16, 0, 0, self.adt, self.dev,
                                                data=_lib.device_view(a.data, numel, self.adt, di))
        self.w: Dict[str, d.BlockedWeight] = {}
        self.dw: Dict[str, d.BlockedWeight] = {}
        for ci, nd in enumerate(self.convs):
            w, g, node = Wt(), Wt(), C.c_int()
            d._check(lib.dconv_graph_conv(self._h, ci, C.byref(node), C.byref(w), C.byref(g)))
            for src, dst in ((w, self.w), (g, self.dw)):
                numel = -(-src.k // 16) * -(-src.c // 16) * src.r * src.s * 256
                dst[nd.name] = d.BlockedWeight(src.k, src.c, src.r, src.s, 16, torch.float32, self.dev,
                                               data=_lib.device_view(src.data, numel, torch.float32, di))
        for attr, fn in (("flat", lib.dconv_graph_grads), ("wflat", lib.dconv_graph_weights)):
            p, n = C.c_void_p(), C.c_size_t()
            d._check(fn(self._h, C.byref(p), C.byref(n)))
            setattr(self, attr, _lib.device_view(p.value, n.value, torch.float32, di))
        # the gloo path exchanges the same flat buffer in fixed backward-order buckets
        order = sorted(self.convs, key=lambda nd: self.dw[nd.name].data.data_ptr())
        base = self.flat.data_ptr()
        slices = []
        for nd in order:
            off = (self.dw[nd.name].data.data_ptr() - base) // 4
            slices.append(slice(off, off + self.dw[nd.name].data.numel()))
        self.bucketer = GradBucketer(self.flat, slices, self._bucket_bytes, self.group if self._py_exchange else None)
        self.specs = {nd.name: d.ConvLayerSpec(self.N, nd.C, nd.K, *self.shapes[nd.src][1:], nd.R, nd.S, nd.stride,
                                               nd.pad, nd.pad, 16) for nd in self.convs}

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h is not None and h.value:
                self.lib.dconv_graph_destroy(h)
                self._h = None
            if getattr(self, "_comm", None) is not None:
                self.lib.dconv_nccl_comm_destroy(self._comm)
                self._comm = None
        except Exception:  # interpreter shutdown
            pass

    # -------------------------------------------------------------- passes
    def _stream(self):
        return torch.cuda.current_stream(self.dev).cuda_stream

    def load_input_nchw(self, nchw: torch.Tensor):
        """This step's images (N, 3, H, W fp32 on the device), packed straight into
        the stem's space-to-depth layout (one pass)."""
        d._check(self.lib.dconv_graph_load_input(self._h, nchw.data_ptr(), self._stream()))

    def forward(self):
        d._check(self.lib.dconv_graph_forward(self._h, self._stream()))

    def backward(self, dtop: d.BlockedActivation):
        """Leaves the (all-reduced) weight gradients in `flat` / `dw`."""
        d._check(self.lib.dconv_graph_backward(self._h, C.byref(dtop.to_c()), self._stream()))
        if self._py_exchange:  # host-side (gloo) exchange, bucket by bucket in backward order
            self.bucketer.begin()
            for k in range(len(self.bucketer.slices)):
                self.bucketer.ready(k)
            self.bucketer.finish()

    def sgd(self):
        d._check(self.lib.dconv_graph_apply(self._h, self._stream()))

    def step(self, dtop: d.BlockedActivation):
        if self._py_exchange:
            self.forward()
            self.backward(dtop)
            self.sgd()
        else:
            d._check(self.lib.dconv_graph_step(self._h, C.byref(dtop.to_c()), self._stream()))

    def capture(self, dtop: d.BlockedActivation):
        """Capture one step (exchange included) into a CUDA graph on the current stream."""
        if self._py_exchange:
            raise d.Unsupported("capture: the gloo exchange runs on the host")
        d._check(self.lib.dconv_graph_capture(self._h, C.byref(dtop.to_c()), self._stream()))

    def replay(self):
        d._check(self.lib.dconv_graph_replay(self._h, self._stream()))

    def profile(self, dtop: d.BlockedActivation, reps: int = 3) -> Dict[str, Dict[str, float]]:
        """per-conv device ms of each pass timed alone (dconv_graph_profile); clobbers tensors"""
        ms = (C.c_float * (3 * len(self.convs)))()
        d._check(self.lib.dconv_graph_profile(self._h, C.byref(dtop.to_c()), reps, ms, self._stream()))
        return {nd.name: {"F": ms[3 * i], "B": ms[3 * i + 1], "U": ms[3 * i + 2]} for i, nd in enumerate(self.convs)}

    def launches_per_step(self) -> int:
        """kernels launched by the last step (ours; NCCL's excluded)."""
        return self.lib.dconv_graph_launches(self._h)

    def buckets(self) -> int:
        return self.lib.dconv_graph_buckets(self._h)
