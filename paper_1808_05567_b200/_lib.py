"""ctypes binding of the C ABI in include/dconv_b200.h (libdconv_b200.so).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
``-gencode arch=compute_100a,code=sm_100a``). There is no fallback: if the
library is missing or fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libdconv_b200.so")


class Spec(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "C", "K", "H", "W", "R", "S", "stride", "pad_h", "pad_w", "vlen")]


class Act(C.Structure):
    _fields_ = [("data", C.c_void_p)] + [(n, C.c_int) for n in ("n", "c", "h", "w", "vlen", "halo_h", "halo_w",
                                                                  "dtype")]


class Wt(C.Structure):
    _fields_ = [("data", C.c_void_p)] + [(n, C.c_int) for n in ("k", "c", "r", "s", "vlen", "dtype")]


class Fusion(C.Structure):
    _fields_ = [("kind", C.c_int), ("bias", C.POINTER(C.c_float)), ("bias_len", C.c_int)]


EP_WEIGHTS_READY = 1  # dconv_epilogue_t.flags (include/dconv_b200.h)
EP_PREP_ONLY = 2


class Epilogue(C.Structure):
    _fields_ = [("add", C.c_void_p), ("mask", C.c_void_p), ("relu", C.c_int), ("flags", C.c_int)]


class GraphNode(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("kind", "src", "add", "C", "K", "R", "S", "stride", "pad_h", "pad_w", "relu")]


class GraphCfg(C.Structure):
    _fields_ = [("lr", C.c_float), ("seed", C.c_int), ("bucket_bytes", C.c_int64), ("world", C.c_int),
                ("rank", C.c_int), ("nccl_comm", C.c_void_p), ("overlap_update", C.c_int), ("act_dtype", C.c_int)]


NODE_CONV, NODE_MAXPOOL = 0, 1


class EngineCfg(C.Structure):
    _fields_ = [("min_accumulators", C.c_int), ("max_accumulators", C.c_int), ("cache_budget_bytes", C.c_int64),
                ("prefetch_lookahead", C.c_int), ("prefetch_enabled", C.c_int), ("streaming_stores", C.c_int),
                ("acc_chain_limit", C.c_int), ("i16_bound_in", C.c_int), ("i16_bound_wt", C.c_int),
                ("tile_mb", C.c_int), ("tile_nb", C.c_int), ("stages", C.c_int), ("upd_splits", C.c_int)]


# status codes (include/dconv_b200.h) -> reference exception class names (errors.hpp:8-57)
STATUS_NAMES = {
    1: "NonIntegralShape", 2: "InvalidLayerSpec", 3: "ShapeMismatch", 4: "InvalidDescriptor", 5: "OverflowRisk",
    6: "PlanInfeasible", 7: "EmptyTrace", 8: "PlanTensorMismatch", 9: "InfeasibleStrategy",
    10: "ChainShapeMismatch", 11: "ParseError", 100: "CudaError", 101: "Unsupported", 102: "InvalidArgument",
}

# every symbol the header declares (tests check the export table against this list)
EXPORTS = [
    "dconv_last_error", "dconv_status_string", "dconv_version", "dconv_engine_config_default", "dconv_make_spec",
    "dconv_spec_validate", "dconv_output_shape", "dconv_pass_flops", "dconv_act_elems", "dconv_wt_elems",
    "dconv_pack_act", "dconv_unpack_act", "dconv_pack_wt", "dconv_unpack_wt", "dconv_transform_weight_dual",
    "dconv_copy_with_halo", "dconv_zero_halo", "dconv_apply_fused_op", "dconv_fill_uniform_host",
    "dconv_fill_he_normal_host", "dconv_fwd_plan_create", "dconv_fwd_plan_destroy", "dconv_fwd_plan_describe",
    "dconv_fwd_workspace_bytes", "dconv_forward", "dconv_fwd_launches", "dconv_bwd_plan_create",
    "dconv_bwd_plan_destroy", "dconv_bwd_route", "dconv_bwd_plan_describe", "dconv_bwd_workspace_bytes",
    "dconv_backward_data", "dconv_bwd_launches", "dconv_upd_plan_create", "dconv_upd_plan_destroy",
    "dconv_upd_splits", "dconv_upd_plan_describe", "dconv_upd_workspace_bytes", "dconv_weight_update",
    "dconv_upd_launches", "dconv_profile", "dconv_profile_last_ms", "dconv_forward_ex", "dconv_backward_data_ex",
    "dconv_maxpool_fwd", "dconv_maxpool_bwd", "dconv_maxpool_bwd_pooled_mask", "dconv_sgd", "dconv_s2d_act", "dconv_s2d_wt", "dconv_pack_s2d", "dconv_host_step_create", "dconv_host_step_destroy",
    "dconv_host_step_chunk", "dconv_host_step_run", "dconv_host_step_launches", "dconv_fwd_plan_validate",
    "dconv_bwd_plan_validate", "dconv_upd_plan_validate", "dconv_set_dev_mode", "dconv_fwd_plan_save",
    "dconv_fwd_plan_load", "dconv_bwd_plan_save", "dconv_bwd_plan_load", "dconv_upd_plan_save", "dconv_upd_plan_load",
    "dconv_graph_config_default", "dconv_graph_create", "dconv_graph_destroy", "dconv_graph_load_input",
    "dconv_graph_forward", "dconv_graph_backward", "dconv_graph_apply", "dconv_graph_step", "dconv_graph_capture",
    "dconv_graph_replay", "dconv_graph_launches", "dconv_graph_num_tensors", "dconv_graph_num_convs",
    "dconv_graph_buckets", "dconv_graph_tensor", "dconv_graph_conv", "dconv_graph_grads", "dconv_graph_weights",
    "dconv_nccl_unique_id", "dconv_nccl_comm_create", "dconv_nccl_comm_destroy", "dconv_relu_mask", "dconv_scale_wt",
    "dconv_set_sm_budget", "dconv_graph_profile", "dconv_subsample2", "dconv_prep_batch_begin", "dconv_prep_batch_end",
]


def _bind(lib):
    P = C.POINTER
    vp, i, sz, i64 = C.c_void_p, C.c_int, C.c_size_t, C.c_int64
    sig = {
        "dconv_last_error": (C.c_char_p, []),
        "dconv_status_string": (C.c_char_p, [i]),
        "dconv_version": (i, []),
        "dconv_engine_config_default": (None, [P(EngineCfg)]),
        "dconv_make_spec": (i, [i] * 11 + [P(Spec)]),
        "dconv_spec_validate": (i, [P(Spec)]),
        "dconv_output_shape": (i, [P(Spec), P(i), P(i)]),
        "dconv_pass_flops": (i64, [P(Spec)]),
        "dconv_act_elems": (i64, [P(Act)]),
        "dconv_wt_elems": (i64, [P(Wt)]),
        "dconv_pack_act": (i, [vp, i, P(Act), vp]),
        "dconv_unpack_act": (i, [P(Act), vp, i, vp]),
        "dconv_pack_wt": (i, [vp, i, P(Wt), vp]),
        "dconv_unpack_wt": (i, [P(Wt), vp, i, vp]),
        "dconv_transform_weight_dual": (i, [P(Wt), P(Wt), vp]),
        "dconv_copy_with_halo": (i, [P(Act), P(Act), vp]),
        "dconv_zero_halo": (i, [P(Act), vp]),
        "dconv_apply_fused_op": (i, [P(Act), P(Fusion), vp]),
        "dconv_fill_uniform_host": (None, [C.c_uint64, C.c_float, C.c_float, vp, i64]),
        "dconv_fill_he_normal_host": (None, [C.c_uint64, C.c_float, vp, i64]),
        "dconv_fwd_plan_create": (i, [P(Spec), P(Fusion), P(EngineCfg), i, i, i, P(vp)]),
        "dconv_fwd_plan_destroy": (None, [vp]),
        "dconv_fwd_plan_describe": (i, [vp, C.c_char_p, sz]),
        "dconv_fwd_workspace_bytes": (sz, [vp]),
        "dconv_forward": (i, [vp, P(Act), P(Wt), P(Act), vp, vp]),
        "dconv_fwd_launches": (i, [vp]),
        "dconv_bwd_plan_create": (i, [P(Spec), P(EngineCfg), i, P(vp)]),
        "dconv_bwd_plan_destroy": (None, [vp]),
        "dconv_bwd_route": (i, [vp]),
        "dconv_bwd_plan_describe": (i, [vp, C.c_char_p, sz]),
        "dconv_bwd_workspace_bytes": (sz, [vp]),
        "dconv_backward_data": (i, [vp, P(Wt), P(Act), P(Act), vp, vp]),
        "dconv_bwd_launches": (i, [vp]),
        "dconv_upd_plan_create": (i, [P(Spec), P(EngineCfg), i, P(vp)]),
        "dconv_upd_plan_destroy": (None, [vp]),
        "dconv_upd_splits": (i, [vp]),
        "dconv_upd_plan_describe": (i, [vp, C.c_char_p, sz]),
        "dconv_upd_workspace_bytes": (sz, [vp, P(Act), P(Act)]),
        "dconv_weight_update": (i, [vp, P(Act), P(Act), P(Wt), i, vp, vp]),
        "dconv_upd_launches": (i, [vp, P(Act), P(Act)]),
        "dconv_profile": (i, [i]),
        "dconv_forward_ex": (i, [vp, P(Act), P(Wt), P(Act), P(Epilogue), vp, vp]),
        "dconv_backward_data_ex": (i, [vp, P(Wt), P(Act), P(Act), P(Epilogue), vp, vp]),
        "dconv_maxpool_fwd": (i, [P(Act), P(Act), vp, vp]),
        "dconv_maxpool_bwd": (i, [P(Act), vp, P(Act), vp, vp]),
        "dconv_sgd": (i, [P(Wt), P(Wt), C.c_float, vp]),
        "dconv_maxpool_bwd_pooled_mask": (i, [P(Act), vp, P(Act), P(Act), vp]),
        "dconv_s2d_act": (i, [P(Act), P(Act), i, vp]),
        "dconv_subsample2": (i, [P(Act), P(Act), i, vp]),
        "dconv_prep_batch_begin": (i, []),
        "dconv_prep_batch_end": (i, [vp]),
        "dconv_s2d_wt": (i, [P(Wt), P(Wt), i, vp]),
        "dconv_pack_s2d": (i, [vp, i, i, i, i, P(Act), i, vp]),
        "dconv_host_step_create": (i, [P(Spec), i, i, P(vp)]),
        "dconv_host_step_destroy": (None, [vp]),
        "dconv_host_step_chunk": (i, [vp]),
        "dconv_host_step_run": (i, [vp, P(Act), P(Wt), P(Act), P(Act), P(Act), P(Wt), vp]),
        "dconv_host_step_launches": (i, [vp]),
        "dconv_fwd_plan_validate": (i, [vp, P(Act), P(Act), C.c_char_p, sz]),
        "dconv_bwd_plan_validate": (i, [vp, P(Act), P(Act), C.c_char_p, sz]),
        "dconv_upd_plan_validate": (i, [vp, P(Act), P(Act), C.c_char_p, sz]),
        "dconv_profile_last_ms": (C.c_float, [i]),
        "dconv_set_dev_mode": (i, [i]),
        "dconv_fwd_plan_save": (i, [vp, C.c_char_p, sz, P(sz)]),
        "dconv_fwd_plan_load": (i, [C.c_char_p, sz, i, P(vp)]),
        "dconv_bwd_plan_save": (i, [vp, C.c_char_p, sz, P(sz)]),
        "dconv_bwd_plan_load": (i, [C.c_char_p, sz, i, P(vp)]),
        "dconv_upd_plan_save": (i, [vp, C.c_char_p, sz, P(sz)]),
        "dconv_upd_plan_load": (i, [C.c_char_p, sz, i, P(vp)]),
        "dconv_graph_config_default": (None, [P(GraphCfg)]),
        "dconv_graph_create": (i, [P(GraphNode), i, i, i, i, i, i, P(GraphCfg), P(vp)]),
        "dconv_graph_destroy": (None, [vp]),
        "dconv_graph_load_input": (i, [vp, vp, vp]),
        "dconv_graph_forward": (i, [vp, vp]),
        "dconv_graph_backward": (i, [vp, P(Act), vp]),
        "dconv_graph_apply": (i, [vp, vp]),
        "dconv_graph_step": (i, [vp, P(Act), vp]),
        "dconv_graph_capture": (i, [vp, P(Act), vp]),
        "dconv_graph_replay": (i, [vp, vp]),
        "dconv_graph_launches": (i, [vp]),
        "dconv_graph_profile": (i, [vp, P(Act), i, P(C.c_float), vp]),
        "dconv_graph_num_tensors": (i, [vp]),
        "dconv_graph_num_convs": (i, [vp]),
        "dconv_graph_buckets": (i, [vp]),
        "dconv_graph_tensor": (i, [vp, i, i, P(Act)]),
        "dconv_graph_conv": (i, [vp, i, P(i), P(Wt), P(Wt)]),
        "dconv_graph_grads": (i, [vp, P(vp), P(sz)]),
        "dconv_graph_weights": (i, [vp, P(vp), P(sz)]),
        "dconv_nccl_unique_id": (i, [C.c_char_p, sz]),
        "dconv_nccl_comm_create": (i, [C.c_char_p, sz, i, i, P(vp)]),
        "dconv_nccl_comm_destroy": (i, [vp]),
        "dconv_relu_mask": (i, [P(Act), P(Act), vp]),
        "dconv_scale_wt": (i, [P(Wt), C.c_float, vp]),
        "dconv_set_sm_budget": (i, [i]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = None


def lib():
    """Load libdconv_b200.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc sm_100a) first")
        _lib = _bind(C.CDLL(LIB_PATH))
    return _lib


# ------------------------------------------------------------------ device views (DLPack)
# Tensors owned by the library (the graph executor's activations, gradients and
# flat weight buffers) are exposed to torch as aliasing views through a DLPack
# capsule: no copy; the owner must outlive the view.


class _DLDevice(C.Structure):
    _fields_ = [("device_type", C.c_int32), ("device_id", C.c_int32)]


class _DLDataType(C.Structure):
    _fields_ = [("code", C.c_uint8), ("bits", C.c_uint8), ("lanes", C.c_uint16)]


class _DLTensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("device", _DLDevice), ("ndim", C.c_int32), ("dtype", _DLDataType),
                ("shape", C.POINTER(C.c_int64)), ("strides", C.POINTER(C.c_int64)), ("byte_offset", C.c_uint64)]


class _DLManagedTensor(C.Structure):
    pass


_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", C.c_void_p),
                             ("deleter", C.CFUNCTYPE(None, C.POINTER(_DLManagedTensor)))]

_KEEP = []  # ctypes storage referenced by live capsules


def device_view(ptr: int, numel: int, dtype, device_index: int):
    """A 1-D torch tensor aliasing `numel` elements of device memory at `ptr`."""
    import torch

    code, bits = {torch.float32: (2, 32), torch.bfloat16: (4, 16), torch.uint8: (1, 8)}[dtype]
    shape = (C.c_int64 * 1)(numel)
    mt = _DLManagedTensor()
    mt.dl_tensor = _DLTensor(C.c_void_p(ptr), _DLDevice(2, device_index), 1, _DLDataType(code, bits, 1),
                             C.cast(shape, C.POINTER(C.c_int64)), None, 0)
    mt.manager_ctx = None
    mt.deleter = C.CFUNCTYPE(None, C.POINTER(_DLManagedTensor))()
    _KEEP.append((shape, mt))
    new = C.pythonapi.PyCapsule_New
    new.restype = C.py_object
    new.argtypes = [C.c_void_p, C.c_char_p, C.c_void_p]
    cap = new(C.addressof(mt), b"dltensor", None)
    return torch.utils.dlpack.from_dlpack(cap)
