"""Python mirror of the reference's dconv execute API over B200 device memory.

Names, argument meaning and error behaviour follow the reference artifact
(/root/reference/proj/core/include/dconv/*.hpp); every call goes through the
C ABI of libdconv_b200.so (include/dconv_b200.h). Tensors are device-resident
torch tensors holding exactly the reference's blocked layouts
([n][c_b][h+2hh][w+2hw][vlen] activations, [k_b][c_b][r][s][c][k] weights),
in fp32 (the reference type) or bf16.

Execute calls are stream-ordered on torch's current CUDA stream; the
synchronous contract of the reference (results are final on return) holds
when ``sync=True`` (the default), which synchronises that stream.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import json
from typing import Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import Act, EngineCfg, Fusion, Spec, Wt

# ------------------------------------------------------------------ errors (errors.hpp:8-57)


class Error(RuntimeError):
    pass


class NonIntegralShape(Error):
    pass


class InvalidLayerSpec(Error):
    pass


class ShapeMismatch(Error):
    pass


class InvalidDescriptor(Error):
    pass


class OverflowRisk(Error):
    pass


class PlanInfeasible(Error):
    pass


class EmptyTrace(Error):
    pass


class PlanTensorMismatch(Error):
    pass


class InfeasibleStrategy(Error):
    pass


class ChainShapeMismatch(Error):
    pass


class ParseError(Error):
    pass


class CudaError(Error):
    pass


class Unsupported(Error):
    pass


class InvalidArgument(Error):
    pass


_EXC = {1: NonIntegralShape, 2: InvalidLayerSpec, 3: ShapeMismatch, 4: InvalidDescriptor, 5: OverflowRisk,
        6: PlanInfeasible, 7: EmptyTrace, 8: PlanTensorMismatch, 9: InfeasibleStrategy, 10: ChainShapeMismatch,
        11: ParseError, 100: CudaError, 101: Unsupported, 102: InvalidArgument}


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.lib().dconv_last_error().decode(errors="replace")
        raise _EXC.get(status, Error)(msg)


def _stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


# ------------------------------------------------------------------ descriptor (layer_spec.hpp:12-49)


@dataclasses.dataclass
class ConvLayerSpec:
    N: int = 1
    C: int = 1
    K: int = 1
    H: int = 1
    W: int = 1
    R: int = 1
    S: int = 1
    stride: int = 1
    pad_h: int = 0
    pad_w: int = 0
    vlen: int = 16

    def cb(self) -> int:
        return -(-self.C // self.vlen)

    def kb(self) -> int:
        return -(-self.K // self.vlen)

    def P(self) -> int:
        return (self.H + 2 * self.pad_h - self.R) // self.stride + 1

    def Q(self) -> int:
        return (self.W + 2 * self.pad_w - self.S) // self.stride + 1

    def validate(self) -> None:
        _check(_lib.lib().dconv_spec_validate(C.byref(self.to_c())))

    def to_c(self) -> Spec:
        return Spec(self.N, self.C, self.K, self.H, self.W, self.R, self.S, self.stride, self.pad_h, self.pad_w,
                    self.vlen)


def make_layer_spec(N, C_, K, H, W, R, S, stride, *args) -> ConvLayerSpec:
    """make_layer_spec (layer_spec.cpp:20-43): (…, stride[, vlen]) with the "same"
    default pad (R-1)/2 for odd filters, or (…, stride, pad_h, pad_w, vlen)."""
    if len(args) in (0, 1):
        vlen = args[0] if args else 16
        pad_h = (R - 1) // 2 if R % 2 == 1 else 0
        pad_w = (S - 1) // 2 if S % 2 == 1 else 0
    elif len(args) == 3:
        pad_h, pad_w, vlen = args
    else:
        raise TypeError("make_layer_spec(N, C, K, H, W, R, S, stride[, vlen]) or (..., stride, pad_h, pad_w, vlen)")
    s = ConvLayerSpec(N, C_, K, H, W, R, S, stride, pad_h, pad_w, vlen)
    s.validate()
    return s


def derive_output_shape(spec: ConvLayerSpec) -> Tuple[int, int]:
    """layer_spec.cpp:45-51 (floor division of the padded span)."""
    P, Q = C.c_int(), C.c_int()
    _check(_lib.lib().dconv_output_shape(C.byref(spec.to_c()), C.byref(P), C.byref(Q)))
    return P.value, Q.value


def pass_flops(spec: ConvLayerSpec) -> int:
    """harness.cpp:269-272."""
    return int(_lib.lib().dconv_pass_flops(C.byref(spec.to_c())))


# ------------------------------------------------------------------ tensors (blocked.hpp)

_DT = {torch.float32: 0, torch.bfloat16: 1}


def _ceil(a, b):
    return -(-a // b)


class BlockedActivation:
    """BlockedActivationT (blocked.hpp:16-80) over a flat device tensor."""

    def __init__(self, n, c, h, w, vlen=16, halo_h=0, halo_w=0, dtype=torch.float32, device="cuda", data=None):
        self.n, self.c, self.h, self.w, self.vlen, self.halo_h, self.halo_w = n, c, h, w, vlen, halo_h, halo_w
        numel = n * _ceil(c, vlen) * (h + 2 * halo_h) * (w + 2 * halo_w) * vlen
        if data is None:
            data = torch.zeros(numel, dtype=dtype, device=device)
        if data.numel() != numel or not data.is_contiguous():
            raise ShapeMismatch("BlockedActivation: storage size / contiguity mismatch")
        self.data = data

    def cb(self):
        return _ceil(self.c, self.vlen)

    def hp(self):
        return self.h + 2 * self.halo_h

    def wp(self):
        return self.w + 2 * self.halo_w

    def offset(self, img, block, ph, pw):
        """blocked.hpp:47-51."""
        return (((img * self.cb() + block) * self.hp() + ph) * self.wp() + pw) * self.vlen

    def view5(self):
        return self.data.view(self.n, self.cb(), self.hp(), self.wp(), self.vlen)

    def fill_zero(self):
        self.data.zero_()

    def zero_halo(self, sync=True):
        _check(_lib.lib().dconv_zero_halo(C.byref(self.to_c()), _stream_ptr()))
        if sync:
            torch.cuda.current_stream().synchronize()

    def to_c(self) -> Act:
        return Act(self.data.data_ptr(), self.n, self.c, self.h, self.w, self.vlen, self.halo_h, self.halo_w,
                   _DT[self.data.dtype])


class BlockedWeight:
    """BlockedWeightT (blocked.hpp:84-125) over a flat device tensor."""

    def __init__(self, k, c, r, s, vlen=16, dtype=torch.float32, device="cuda", data=None):
        self.k, self.c, self.r, self.s, self.vlen = k, c, r, s, vlen
        numel = _ceil(k, vlen) * _ceil(c, vlen) * r * s * vlen * vlen
        if data is None:
            data = torch.zeros(numel, dtype=dtype, device=device)
        if data.numel() != numel or not data.is_contiguous():
            raise ShapeMismatch("BlockedWeight: storage size / contiguity mismatch")
        self.data = data

    def kb(self):
        return _ceil(self.k, self.vlen)

    def cb(self):
        return _ceil(self.c, self.vlen)

    def offset(self, kblk, cblk, fr, fs):
        """blocked.hpp:112-115."""
        return (((kblk * self.cb() + cblk) * self.r + fr) * self.s + fs) * self.vlen * self.vlen

    def to_c(self) -> Wt:
        return Wt(self.data.data_ptr(), self.k, self.c, self.r, self.s, self.vlen, _DT[self.data.dtype])


def _sync(sync):
    if sync:
        torch.cuda.current_stream().synchronize()


def to_blocked_activation(nchw: torch.Tensor, spec_or_vlen=16, halo_h=0, halo_w=0, dtype=None, sync=True):
    """to_blocked_activation (blocked.hpp:133-155): device pack kernel.
    Accepts (tensor, spec) -> halo = spec padding, or (tensor, vlen, halo_h, halo_w)."""
    if isinstance(spec_or_vlen, ConvLayerSpec):
        s = spec_or_vlen
        if tuple(nchw.shape) != (s.N, s.C, s.H, s.W):
            raise ShapeMismatch(f"to_blocked_activation: expected [{s.N},{s.C},{s.H},{s.W}], got {list(nchw.shape)}")
        vlen, halo_h, halo_w = s.vlen, s.pad_h, s.pad_w
    else:
        vlen = spec_or_vlen
    src = nchw.contiguous()
    n, c, h, w = src.shape
    out = BlockedActivation(n, c, h, w, vlen, halo_h, halo_w, dtype or src.dtype, src.device,
                            data=torch.empty(n * _ceil(c, vlen) * (h + 2 * halo_h) * (w + 2 * halo_w) * vlen,
                                             dtype=dtype or src.dtype, device=src.device))
    _check(_lib.lib().dconv_pack_act(src.data_ptr(), _DT[src.dtype], C.byref(out.to_c()), _stream_ptr()))
    _sync(sync)
    return out


def from_blocked_activation(blk: BlockedActivation, spec: Optional[ConvLayerSpec] = None, dtype=None, sync=True):
    """from_blocked_activation (blocked.hpp:157-178)."""
    if spec is not None and (blk.n, blk.c, blk.h, blk.w) != (spec.N, spec.C, spec.H, spec.W):
        raise ShapeMismatch("from_blocked_activation: blocked dims disagree with spec")
    out = torch.empty(blk.n, blk.c, blk.h, blk.w, dtype=dtype or blk.data.dtype, device=blk.data.device)
    _check(_lib.lib().dconv_unpack_act(C.byref(blk.to_c()), out.data_ptr(), _DT[out.dtype], _stream_ptr()))
    _sync(sync)
    return out


def to_blocked_weight(kcrs: torch.Tensor, spec_or_vlen=16, dtype=None, sync=True) -> BlockedWeight:
    """to_blocked_weight (blocked.hpp:180-200)."""
    if isinstance(spec_or_vlen, ConvLayerSpec):
        s = spec_or_vlen
        if tuple(kcrs.shape) != (s.K, s.C, s.R, s.S):
            raise ShapeMismatch(f"to_blocked_weight: expected [{s.K},{s.C},{s.R},{s.S}], got {list(kcrs.shape)}")
        vlen = s.vlen
    else:
        vlen = spec_or_vlen
    src = kcrs.contiguous()
    k, c, r, s_ = src.shape
    out = BlockedWeight(k, c, r, s_, vlen, dtype or src.dtype, src.device,
                        data=torch.empty(_ceil(k, vlen) * _ceil(c, vlen) * r * s_ * vlen * vlen,
                                         dtype=dtype or src.dtype, device=src.device))
    _check(_lib.lib().dconv_pack_wt(src.data_ptr(), _DT[src.dtype], C.byref(out.to_c()), _stream_ptr()))
    _sync(sync)
    return out


def from_blocked_weight(blk: BlockedWeight, dtype=None, sync=True) -> torch.Tensor:
    """from_blocked_weight (blocked.hpp:202-213)."""
    out = torch.empty(blk.k, blk.c, blk.r, blk.s, dtype=dtype or blk.data.dtype, device=blk.data.device)
    _check(_lib.lib().dconv_unpack_wt(C.byref(blk.to_c()), out.data_ptr(), _DT[out.dtype], _stream_ptr()))
    _sync(sync)
    return out


def transform_weight_stride1(w: BlockedWeight, sync=True) -> BlockedWeight:
    """transform_weight_stride1 (propagation.hpp:20-33)."""
    out = BlockedWeight(w.c, w.k, w.r, w.s, w.vlen, w.data.dtype, w.data.device)
    _check(_lib.lib().dconv_transform_weight_dual(C.byref(w.to_c()), C.byref(out.to_c()), _stream_ptr()))
    _sync(sync)
    return out


def copy_with_halo(src: BlockedActivation, halo_h: int, halo_w: int, sync=True) -> BlockedActivation:
    """copy_with_halo (propagation.hpp:35-49)."""
    out = BlockedActivation(src.n, src.c, src.h, src.w, src.vlen, halo_h, halo_w, src.data.dtype, src.data.device,
                            data=torch.empty(src.n * src.cb() * (src.h + 2 * halo_h) * (src.w + 2 * halo_w) *
                                             src.vlen, dtype=src.data.dtype, device=src.data.device))
    _check(_lib.lib().dconv_copy_with_halo(C.byref(src.to_c()), C.byref(out.to_c()), _stream_ptr()))
    _sync(sync)
    return out


# ------------------------------------------------------------------ config / fusion


class FusedOpKind(enum.IntEnum):
    """kernel_streams.hpp:29."""
    RELU = 0
    BIAS_ADD = 1
    BIAS_RELU = 2


@dataclasses.dataclass
class FusedOp:
    kind: FusedOpKind = FusedOpKind.RELU
    bias: Sequence[float] = ()


@dataclasses.dataclass
class EngineConfig:
    """config.hpp:10-20 plus the sm_100a tile-selector overrides (0 = auto)."""
    min_accumulators: int = 8
    max_accumulators: int = 28
    cache_budget_bytes: int = 512 * 1024
    prefetch_lookahead: int = 1
    prefetch_enabled: bool = True
    streaming_stores: bool = False
    acc_chain_limit: int = 512
    i16_bound_in: int = 256
    i16_bound_wt: int = 256
    tile_mb: int = 0
    tile_nb: int = 0
    stages: int = 0
    upd_splits: int = 0

    def to_c(self) -> EngineCfg:
        return EngineCfg(self.min_accumulators, self.max_accumulators, self.cache_budget_bytes,
                         self.prefetch_lookahead, int(self.prefetch_enabled), int(self.streaming_stores),
                         self.acc_chain_limit, self.i16_bound_in, self.i16_bound_wt, self.tile_mb, self.tile_nb,
                         self.stages, self.upd_splits)


class Math(enum.IntEnum):
    """Arithmetic of the tensor-core passes (KernelDType analog, microkernel.hpp:16)."""
    F32 = 0   # fp32-accurate: exact bf16x3 split, 6 products, fp32 accumulate
    BF16 = 1  # bf16 operands, fp32 accumulate


def _fusion_c(op: Optional[FusedOp]):
    if op is None:
        return None, None
    bias = (C.c_float * len(op.bias))(*op.bias) if len(op.bias) else None
    f = Fusion(int(op.kind), C.cast(bias, C.POINTER(C.c_float)) if bias is not None else None, len(op.bias))
    return f, bias


class _Workspace:
    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device) -> int:
        nbytes = max(int(nbytes), 256)
        dev = torch.device(device)
        if dev.type == "cuda" and dev.index is None:  # "cuda" == the current device: compare like with like
            dev = torch.device("cuda", torch.cuda.current_device())
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != dev:
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        return self.buf.data_ptr()


def _validate(fn, handle, a, b) -> dict:
    """validate_plan analog (kernel_streams.cpp:461-617): raises InvalidDescriptor
    on a violated property, else returns the validator's JSON summary."""
    buf = C.create_string_buffer(1 << 16)
    st = fn(handle, C.byref(a.to_c()), C.byref(b.to_c()), buf, len(buf))
    _check(st)
    return json.loads(buf.value.decode() or "{}")


def _save(fn, handle) -> str:
    """save_plan (kernel_streams.cpp:619-688) analog: the plan and its resolved launches as DCPL text."""
    need = C.c_size_t()
    _check(fn(handle, None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    _check(fn(handle, buf, len(buf), C.byref(need)))
    return buf.value.decode()


def _plan_header(text: str) -> dict:
    rec = {}
    for line in text.splitlines():
        parts = line.split()
        if parts and parts[0] in ("kind", "spec", "math", "out_halo") and parts[0] not in rec:
            rec[parts[0]] = parts[1:]
        if parts and parts[0] == "entries":
            break
    if "spec" not in rec:
        raise ParseError("load_plan: no spec record")
    return rec


def _load(fn, text: str, validate: bool):
    """load_plan (kernel_streams.cpp:690-788) analog; validate=True also runs the plan validator."""
    h = C.c_void_p()
    raw = text.encode()
    _check(fn(raw, len(raw), int(validate), C.byref(h)))
    rec = _plan_header(text)
    spec = ConvLayerSpec(*[int(v) for v in rec["spec"]])
    return h, spec, Math(int(rec["math"][0])), rec


def _describe(fn, handle) -> dict:
    buf = C.create_string_buffer(4096)
    fn(handle, buf, len(buf))
    try:
        return json.loads(buf.value.decode())
    except ValueError:
        return {"raw": buf.value.decode()}


# ------------------------------------------------------------------ forward (propagation.hpp:53-64)


class ExecutionPlan:
    """ExecutionPlan analog (kernel_streams.hpp:90-101): the per-layer launch plan."""

    def __init__(self, spec: ConvLayerSpec, fusion: Optional[FusedOp], cfg: Optional[EngineConfig], math: Math,
                 out_halo_h: int, out_halo_w: int, threads: int = 1):
        self.spec, self.fusion, self.math = spec, fusion, Math(math)
        self.out_halo_h, self.out_halo_w, self.threads = out_halo_h, out_halo_w, threads
        self._h = C.c_void_p()
        f, self._bias_keep = _fusion_c(fusion)
        cfg_c = cfg.to_c() if cfg is not None else None
        _check(_lib.lib().dconv_fwd_plan_create(C.byref(spec.to_c()), C.byref(f) if f else None,
                                                C.byref(cfg_c) if cfg_c else None, int(math), out_halo_h,
                                                out_halo_w, C.byref(self._h)))
        self._ws = _Workspace()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dconv_fwd_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def blocking(self) -> dict:
        """chosen tile (LayerReport.blocking analog, harness.hpp:48)."""
        return _describe(_lib.lib().dconv_fwd_plan_describe, self._h)

    def launches(self) -> int:
        return _lib.lib().dconv_fwd_launches(self._h)

    def validate(self, inp: BlockedActivation, out: BlockedActivation) -> dict:
        return _validate(_lib.lib().dconv_fwd_plan_validate, self._h, inp, out)

    def save(self) -> str:
        return _save(_lib.lib().dconv_fwd_plan_save, self._h)

    @classmethod
    def load(cls, text: str, validate: bool = True) -> "ExecutionPlan":
        h, spec, math, rec = _load(_lib.lib().dconv_fwd_plan_load, text, validate)
        self = cls.__new__(cls)
        self.spec, self.fusion, self.math, self.threads = spec, None, math, 1
        self.out_halo_h, self.out_halo_w = (int(v) for v in rec["out_halo"])
        self._h, self._bias_keep, self._ws = h, None, _Workspace()
        return self

    def execute(self, inp: BlockedActivation, wt: BlockedWeight, out: BlockedActivation) -> None:
        ws = self._ws.get(_lib.lib().dconv_fwd_workspace_bytes(self._h), inp.data.device)
        _check(_lib.lib().dconv_forward(self._h, C.byref(inp.to_c()), C.byref(wt.to_c()), C.byref(out.to_c()), ws,
                                        _stream_ptr()))


def make_forward_plan(spec: ConvLayerSpec, threads: int = 1, fusion: Optional[FusedOp] = None,
                      cfg: Optional[EngineConfig] = None, dtype: Math = Math.F32, out_halo_h: int = 0,
                      out_halo_w: int = 0) -> ExecutionPlan:
    """make_forward_plan (propagation.cpp:42-54). `threads` is accepted for API
    compatibility; the GPU tile scheduler replaces the thread partition."""
    spec.validate()
    return ExecutionPlan(spec, fusion, cfg, dtype, out_halo_h, out_halo_w, threads)


def _check_forward_tensors(spec, inp, wt):
    """propagation.cpp:12-19."""
    if (inp.n, inp.c, inp.h, inp.w, inp.vlen) != (spec.N, spec.C, spec.H, spec.W, spec.vlen):
        raise ShapeMismatch("forward: input does not match the layer spec")
    if (wt.k, wt.c, wt.r, wt.s, wt.vlen) != (spec.K, spec.C, spec.R, spec.S, spec.vlen):
        raise ShapeMismatch("forward: weight does not match the layer spec")


def forward_into(plan: ExecutionPlan, inp: BlockedActivation, wt: BlockedWeight, out: BlockedActivation,
                 sync: bool = True, strict_surface: bool = True) -> None:
    """forward_into (propagation.cpp:56-61): out is fully rewritten (interior +
    zero halo). With strict_surface the input halo must equal the padding, as
    the reference's check_plan_tensors requires (kernel_streams.cpp:122-141)."""
    s = plan.spec
    _check_forward_tensors(s, inp, wt)
    if strict_surface and (inp.halo_h, inp.halo_w) != (s.pad_h, s.pad_w):
        raise PlanTensorMismatch("forward: input halo does not match the plan's input surface")
    plan.execute(inp, wt, out)
    _sync(sync)


def forward(spec: ConvLayerSpec, inp: BlockedActivation, wt: BlockedWeight, plan: ExecutionPlan,
            out_dtype=torch.float32, sync: bool = True) -> BlockedActivation:
    """forward (propagation.cpp:63-74)."""
    _check_forward_tensors(spec, inp, wt)
    P, Q = derive_output_shape(spec)
    out = BlockedActivation(spec.N, spec.K, P, Q, spec.vlen, plan.out_halo_h, plan.out_halo_w, out_dtype,
                            inp.data.device,
                            data=torch.empty(spec.N * spec.kb() * (P + 2 * plan.out_halo_h) *
                                             (Q + 2 * plan.out_halo_w) * spec.vlen, dtype=out_dtype,
                                             device=inp.data.device))
    forward_into(plan, inp, wt, out, sync=sync)
    return out


def apply_fused_op(act: BlockedActivation, op: FusedOp, sync=True) -> None:
    """apply_fused_op (propagation.cpp:193-215), post-hoc on the interior."""
    f, keep = _fusion_c(op)
    _check(_lib.lib().dconv_apply_fused_op(C.byref(act.to_c()), C.byref(f), _stream_ptr()))
    _sync(sync)
    del keep


# ------------------------------------------------------------------ backward-data (propagation.hpp:83-101)


class BackwardRoute(enum.IntEnum):
    DUALITY_STRIDE1 = 0
    DUALITY_1x1 = 1
    GENERIC_GEMM = 2  # stride-phase decomposition on sm_100a


def choose_backward_route(spec: ConvLayerSpec) -> BackwardRoute:
    """propagation.cpp:35-40."""
    if spec.stride == 1 and spec.pad_h <= spec.R - 1 and spec.pad_w <= spec.S - 1:
        return BackwardRoute.DUALITY_STRIDE1
    if spec.R == 1 and spec.S == 1:
        return BackwardRoute.DUALITY_1x1
    return BackwardRoute.GENERIC_GEMM


class BackwardContext:
    """BackwardContext (propagation.hpp:83-91). The reference bakes the
    transformed weights in; on the GPU the weights are an execute-time input
    (they change every step), so the context keeps a reference to them."""

    def __init__(self, spec: ConvLayerSpec, wt: Optional[BlockedWeight], threads: int, cfg: Optional[EngineConfig],
                 math: Math):
        self.spec, self.wt, self.threads, self.math = spec, wt, threads, Math(math)
        self._h = C.c_void_p()
        cfg_c = cfg.to_c() if cfg is not None else None
        _check(_lib.lib().dconv_bwd_plan_create(C.byref(spec.to_c()), C.byref(cfg_c) if cfg_c else None, int(math),
                                                C.byref(self._h)))
        self.route = BackwardRoute(_lib.lib().dconv_bwd_route(self._h))
        self._ws = _Workspace()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dconv_bwd_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def blocking(self) -> dict:
        return _describe(_lib.lib().dconv_bwd_plan_describe, self._h)

    def launches(self) -> int:
        return _lib.lib().dconv_bwd_launches(self._h)

    def validate(self, grad_out: BlockedActivation, grad_in: BlockedActivation) -> dict:
        return _validate(_lib.lib().dconv_bwd_plan_validate, self._h, grad_out, grad_in)

    def save(self) -> str:
        return _save(_lib.lib().dconv_bwd_plan_save, self._h)

    @classmethod
    def load(cls, text: str, validate: bool = True, wt: Optional[BlockedWeight] = None) -> "BackwardContext":
        h, spec, math, _ = _load(_lib.lib().dconv_bwd_plan_load, text, validate)
        self = cls.__new__(cls)
        self.spec, self.wt, self.threads, self.math = spec, wt, 1, math
        self._h, self._ws = h, _Workspace()
        self.route = BackwardRoute(_lib.lib().dconv_bwd_route(self._h))
        return self

    def execute(self, wt: BlockedWeight, grad_out: BlockedActivation, grad_in: BlockedActivation) -> None:
        ws = self._ws.get(_lib.lib().dconv_bwd_workspace_bytes(self._h), grad_out.data.device)
        _check(_lib.lib().dconv_backward_data(self._h, C.byref(wt.to_c()), C.byref(grad_out.to_c()),
                                              C.byref(grad_in.to_c()), ws, _stream_ptr()))


def prepare_backward(spec: ConvLayerSpec, wt: BlockedWeight, threads: int = 1, cfg: Optional[EngineConfig] = None,
                     dtype: Math = Math.F32) -> BackwardContext:
    """prepare_backward (propagation.cpp:217-276)."""
    spec.validate()
    if (wt.k, wt.c, wt.r, wt.s, wt.vlen) != (spec.K, spec.C, spec.R, spec.S, spec.vlen):
        raise ShapeMismatch("backward: weight does not match the layer spec")
    return BackwardContext(spec, wt, threads, cfg, dtype)


def backward_with(ctx: BackwardContext, grad_out: BlockedActivation, wt: Optional[BlockedWeight] = None,
                  out_halo: Optional[Tuple[int, int]] = None, out_dtype=None, sync=True) -> BlockedActivation:
    """backward_with (propagation.cpp:278-348). The result carries halo 0 for
    the stride-1 route and halo = pad for the strided routes, like the reference."""
    s = ctx.spec
    P, Q = derive_output_shape(s)
    if (grad_out.n, grad_out.c, grad_out.h, grad_out.w, grad_out.vlen) != (s.N, s.K, P, Q, s.vlen):
        raise ShapeMismatch("backward: grad_out does not match the layer spec")
    if out_halo is None:
        out_halo = (0, 0) if ctx.route == BackwardRoute.DUALITY_STRIDE1 else (s.pad_h, s.pad_w)
    dt = out_dtype or grad_out.data.dtype
    gi = BlockedActivation(s.N, s.C, s.H, s.W, s.vlen, out_halo[0], out_halo[1], dt, grad_out.data.device,
                           data=torch.empty(s.N * s.cb() * (s.H + 2 * out_halo[0]) * (s.W + 2 * out_halo[1]) * s.vlen,
                                            dtype=dt, device=grad_out.data.device))
    ctx.execute(wt if wt is not None else ctx.wt, grad_out, gi)
    _sync(sync)
    return gi


def backward(spec: ConvLayerSpec, grad_out: BlockedActivation, wt: BlockedWeight, threads: int = 1,
             cfg: Optional[EngineConfig] = None, dtype: Math = Math.F32) -> BlockedActivation:
    """backward (propagation.cpp:350-355)."""
    return backward_with(prepare_backward(spec, wt, threads, cfg, dtype), grad_out)


# ------------------------------------------------------------------ weight update (propagation.hpp:103-117)


class UpdateMode(enum.IntEnum):
    TASK_PARALLEL = 0
    COPY_REDUCE = 1
    HYBRID = 2


@dataclasses.dataclass
class WeightUpdateStrategy:
    """WeightUpdateStrategy (planner.hpp:66-73). On the GPU `copies` is the
    split-K factor G: G partial dW copies over disjoint pixel ranges reduced in
    fixed index order (COPY_REDUCE)."""
    mode: UpdateMode = UpdateMode.COPY_REDUCE
    copies: int = 1
    threads: int = 1


class UpdatePlan:
    def __init__(self, spec: ConvLayerSpec, cfg: Optional[EngineConfig], math: Math):
        self.spec, self.math = spec, Math(math)
        self._h = C.c_void_p()
        cfg_c = cfg.to_c() if cfg is not None else None
        _check(_lib.lib().dconv_upd_plan_create(C.byref(spec.to_c()), C.byref(cfg_c) if cfg_c else None, int(math),
                                                C.byref(self._h)))
        self._ws = _Workspace()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dconv_upd_plan_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def splits(self) -> int:
        return _lib.lib().dconv_upd_splits(self._h)

    @property
    def blocking(self) -> dict:
        return _describe(_lib.lib().dconv_upd_plan_describe, self._h)

    def launches(self, inp, grad_out) -> int:
        return _lib.lib().dconv_upd_launches(self._h, C.byref(inp.to_c()), C.byref(grad_out.to_c()))

    def validate(self, inp: BlockedActivation, grad_out: BlockedActivation) -> dict:
        return _validate(_lib.lib().dconv_upd_plan_validate, self._h, inp, grad_out)

    def save(self) -> str:
        return _save(_lib.lib().dconv_upd_plan_save, self._h)

    @classmethod
    def load(cls, text: str, validate: bool = True) -> "UpdatePlan":
        h, spec, math, _ = _load(_lib.lib().dconv_upd_plan_load, text, validate)
        self = cls.__new__(cls)
        self.spec, self.math = spec, math
        self._h, self._ws = h, _Workspace()
        return self

    def execute(self, inp: BlockedActivation, grad_out: BlockedActivation, dw: BlockedWeight, accumulate=False):
        a, g = inp.to_c(), grad_out.to_c()
        ws = self._ws.get(_lib.lib().dconv_upd_workspace_bytes(self._h, C.byref(a), C.byref(g)), inp.data.device)
        _check(_lib.lib().dconv_weight_update(self._h, C.byref(a), C.byref(g), C.byref(dw.to_c()), int(accumulate),
                                              ws, _stream_ptr()))


def choose_update_strategy(spec: ConvLayerSpec, threads: int = 1, cfg: Optional[EngineConfig] = None,
                           dtype: Math = Math.F32) -> WeightUpdateStrategy:
    """choose_update_strategy (planner.cpp:107-143) -> the split-K factor."""
    plan = UpdatePlan(spec, cfg, dtype)
    g = plan.splits
    return WeightUpdateStrategy(UpdateMode.COPY_REDUCE if g > 1 else UpdateMode.TASK_PARALLEL, g, threads)


def choose_spatial_blocking(spec: ConvLayerSpec, cfg: Optional[EngineConfig] = None) -> Tuple[int, int]:
    """choose_spatial_blocking (planner.cpp:153-173); the GPU plan streams whole
    output rows per stage, so the blocking is (1 row band, Q)."""
    P, Q = derive_output_shape(spec)
    return 1, Q


def weight_update(spec: ConvLayerSpec, inp: BlockedActivation, grad_out: BlockedActivation,
                  strategy: Optional[WeightUpdateStrategy] = None, b_p: int = 1, b_q: int = 0,
                  cfg: Optional[EngineConfig] = None, dtype: Math = Math.F32, out_dtype=torch.float32,
                  sync=True) -> BlockedWeight:
    """weight_update (propagation.cpp:377-458) with the reference's validation."""
    spec.validate()
    P, Q = derive_output_shape(spec)
    if (inp.n, inp.c, inp.h, inp.w, inp.vlen) != (spec.N, spec.C, spec.H, spec.W, spec.vlen):
        raise ShapeMismatch("weight_update: input does not match the layer spec")
    if inp.halo_h < spec.pad_h or inp.halo_w < spec.pad_w:
        raise ShapeMismatch("weight_update: input halo smaller than the padding")
    if (grad_out.n, grad_out.c, grad_out.h, grad_out.w, grad_out.vlen) != (spec.N, spec.K, P, Q, spec.vlen):
        raise ShapeMismatch("weight_update: grad_out does not match the layer spec")
    if b_q == 0:
        b_q = Q
    if b_p < 1 or b_q < 1 or P % b_p != 0 or Q % b_q != 0:
        raise InfeasibleStrategy("weight_update: blocking must divide (P, Q)")
    if strategy is not None:
        if strategy.threads < 1 or strategy.copies < 1 or strategy.threads % strategy.copies != 0:
            raise InfeasibleStrategy("weight_update: copies must divide threads")
    c = cfg or EngineConfig()
    if strategy is not None and strategy.copies > 1 and c.upd_splits == 0:
        c = dataclasses.replace(c, upd_splits=strategy.copies)
    plan = UpdatePlan(spec, c, dtype)
    dw = BlockedWeight(spec.K, spec.C, spec.R, spec.S, spec.vlen, out_dtype, inp.data.device,
                       data=torch.empty(spec.kb() * spec.cb() * spec.R * spec.S * spec.vlen * spec.vlen,
                                        dtype=out_dtype, device=inp.data.device))
    plan.execute(inp, grad_out, dw)
    _sync(sync)
    return dw


class HostStep:
    """One layer step (forward, backward-data, weight update) on HOST tensors:
    the reference's execute contract (forward_into propagation.cpp:56-61,
    backward_with :237-261, weight_update :377-458 all take host memory and
    return finished results). The batch streams through the GPU in image
    chunks with copies and kernels overlapped (dconv_host_step_run). Host
    tensors are CPU BlockedActivation / BlockedWeight storages; pin them
    (``pin_memory()``) for full-duplex overlap."""

    def __init__(self, spec: ConvLayerSpec, math: Math = Math.F32, chunk_images: int = 0):
        self.spec, self.math = spec, Math(math)
        self._h = C.c_void_p()
        _check(_lib.lib().dconv_host_step_create(C.byref(spec.to_c()), int(math), int(chunk_images),
                                                 C.byref(self._h)))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                _lib.lib().dconv_host_step_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    @property
    def chunk(self) -> int:
        return _lib.lib().dconv_host_step_chunk(self._h)

    def launches(self) -> int:
        return _lib.lib().dconv_host_step_launches(self._h)

    def run(self, x: Optional[BlockedActivation], w: Optional[BlockedWeight], dy: Optional[BlockedActivation],
            y: Optional[BlockedActivation] = None, dx: Optional[BlockedActivation] = None,
            dw: Optional[BlockedWeight] = None, sync: bool = True) -> None:
        for t in (x, w, dy, y, dx, dw):
            if t is not None and t.data.device.type != "cpu":
                raise InvalidArgument("HostStep.run: tensors must live in host memory")
        ref = lambda t: C.byref(t.to_c()) if t is not None else None  # noqa: E731
        _check(_lib.lib().dconv_host_step_run(self._h, ref(x), ref(w), ref(dy), ref(y), ref(dx), ref(dw),
                                              _stream_ptr()))
        _sync(sync)
