"""dconv-b200: the reference's blocked direct-convolution execute path
(arxiv 1808.05567 artifact) on B200 / sm_100a.

The C ABI (include/dconv_b200.h, libdconv_b200.so) is the product; this
package is its Python mirror of the reference API (see api.py). Importing it
requires the built library — there is no CPU fallback.
"""
from ._lib import lib as _load_lib
from .api import (  # noqa: F401
    BackwardContext, BackwardRoute, BlockedActivation, BlockedWeight, ChainShapeMismatch, ConvLayerSpec, CudaError,
    EmptyTrace, EngineConfig, Error, ExecutionPlan, FusedOp, FusedOpKind, InfeasibleStrategy, InvalidArgument,
    HostStep, InvalidDescriptor, InvalidLayerSpec, Math, NonIntegralShape, OverflowRisk, ParseError, PlanInfeasible,
    PlanTensorMismatch, ShapeMismatch, Unsupported, UpdateMode, UpdatePlan, WeightUpdateStrategy, apply_fused_op,
    backward, backward_with, choose_backward_route, choose_spatial_blocking, choose_update_strategy, copy_with_halo,
    derive_output_shape, forward, forward_into, from_blocked_activation, from_blocked_weight, make_forward_plan,
    make_layer_spec, pass_flops, prepare_backward, to_blocked_activation, to_blocked_weight,
    transform_weight_stride1, weight_update,
)

_load_lib()  # fail loudly at import if the sm_100a library is missing
