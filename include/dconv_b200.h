/*
 * dconv_b200 — C ABI of the B200 (sm_100a) direct-convolution engine.
 *
 * Drop-in boundary for the reference artifact's conv execute calls
 * (arxiv 1808.05567 artifact, /root/reference/proj). Every entry point
 * below replaces one reference interface, cited as file:line (paths relative
 * to proj/core). Plain C types only: device pointers, sizes, an opaque plan
 * handle and a CUDA stream. All execute calls are ASYNCHRONOUS on `stream`;
 * the synchronous reference contract (execute returns finished results) is
 * restored by the C++ shim / Python mirror, which synchronise the stream.
 *
 * Layouts are the reference's, element for element:
 *   activations  [n][c_b][h + 2*halo_h][w + 2*halo_w][vlen]  (blocked.hpp:47-51)
 *   weights      [k_b][c_b][r][s][c][k]                      (blocked.hpp:112-115)
 * stored as fp32 (the reference type) or bf16.
 *
 * Errors: every function returns a dconv_status_t whose non-zero values map
 * 1:1 onto the reference exception classes (errors.hpp:8-57); the message is
 * available from dconv_last_error() (thread-local).
 */
#ifndef DCONV_B200_H
#define DCONV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dconv_stream_t; /* == cudaStream_t */

typedef enum dconv_status {
  DCONV_OK = 0,
  DCONV_ERR_NON_INTEGRAL_SHAPE = 1,   /* errors.hpp:14 NonIntegralShape */
  DCONV_ERR_INVALID_LAYER_SPEC = 2,   /* errors.hpp:18 InvalidLayerSpec */
  DCONV_ERR_SHAPE_MISMATCH = 3,       /* errors.hpp:22 ShapeMismatch */
  DCONV_ERR_INVALID_DESCRIPTOR = 4,   /* errors.hpp:26 InvalidDescriptor */
  DCONV_ERR_OVERFLOW_RISK = 5,        /* errors.hpp:30 OverflowRisk */
  DCONV_ERR_PLAN_INFEASIBLE = 6,      /* errors.hpp:34 PlanInfeasible */
  DCONV_ERR_EMPTY_TRACE = 7,          /* errors.hpp:38 EmptyTrace */
  DCONV_ERR_PLAN_TENSOR_MISMATCH = 8, /* errors.hpp:42 PlanTensorMismatch */
  DCONV_ERR_INFEASIBLE_STRATEGY = 9,  /* errors.hpp:46 InfeasibleStrategy */
  DCONV_ERR_CHAIN_SHAPE_MISMATCH = 10,/* errors.hpp:50 ChainShapeMismatch */
  DCONV_ERR_PARSE = 11,               /* errors.hpp:54 ParseError */
  DCONV_ERR_CUDA = 100,               /* CUDA runtime / driver failure */
  DCONV_ERR_UNSUPPORTED = 101,        /* valid for the reference, not implemented on sm_100a */
  DCONV_ERR_INVALID_ARGUMENT = 102    /* null pointer, bad enum */
} dconv_status_t;

/* ConvLayerSpec (layer_spec.hpp:12-38), field for field */
typedef struct dconv_spec {
  int N, C, K, H, W, R, S, stride, pad_h, pad_w, vlen;
} dconv_spec_t;

typedef enum dconv_dtype { DCONV_F32 = 0, DCONV_BF16 = 1 } dconv_dtype_t;

/* arithmetic of the tensor-core passes */
typedef enum dconv_math {
  DCONV_MATH_F32 = 0, /* fp32-accurate: exact 3-way bf16 split, 6 products, fp32 accumulate */
  DCONV_MATH_BF16 = 1 /* bf16 operands, fp32 accumulate */
} dconv_math_t;

/* BlockedActivationT (blocked.hpp:16-80) over device memory */
typedef struct dconv_act {
  void* data;
  int n, c, h, w, vlen, halo_h, halo_w;
  int dtype; /* dconv_dtype_t */
} dconv_act_t;

/* BlockedWeightT (blocked.hpp:84-125) over device memory */
typedef struct dconv_wt {
  void* data;
  int k, c, r, s, vlen;
  int dtype;
} dconv_wt_t;

/* FusedOp (kernel_streams.hpp:29-34); bias is a HOST array of K floats */
typedef enum dconv_fused_kind {
  DCONV_FUSE_NONE = -1,
  DCONV_FUSE_RELU = 0,
  DCONV_FUSE_BIAS_ADD = 1,
  DCONV_FUSE_BIAS_RELU = 2
} dconv_fused_kind_t;
typedef struct dconv_fusion {
  int kind;
  const float* bias; /* host, K entries (BIAS_*), copied at plan creation */
  int bias_len;
} dconv_fusion_t;

/* EngineConfig (config.hpp:10-20) plus sm_100a tile-selector overrides
 * (0 = automatic). The CPU tunables are accepted for API compatibility. */
typedef struct dconv_engine_config {
  int min_accumulators, max_accumulators;
  int64_t cache_budget_bytes;
  int prefetch_lookahead, prefetch_enabled, streaming_stores;
  int acc_chain_limit, i16_bound_in, i16_bound_wt;
  int tile_mb;    /* FWD/BWD: 128-row m-blocks per CTA */
  int tile_nb;    /* 16-channel output blocks per CTA */
  int stages;     /* smem pipeline depth */
  int upd_splits; /* UPD split-K factor */
} dconv_engine_config_t;

/* ---------------------------------------------------------------- basics */
const char* dconv_last_error(void);
const char* dconv_status_string(int status);
int dconv_version(void);
void dconv_engine_config_default(dconv_engine_config_t* cfg); /* config.hpp:10-20 */

/* make_layer_spec (layer_spec.cpp:20-43); pad_h/pad_w < 0 = "same" default (R-1)/2 */
int dconv_make_spec(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w, int vlen,
                    dconv_spec_t* out);
int dconv_spec_validate(const dconv_spec_t* spec);                 /* layer_spec.cpp:7-18 */
int dconv_output_shape(const dconv_spec_t* spec, int* P, int* Q);  /* layer_spec.cpp:45-51 */
int64_t dconv_pass_flops(const dconv_spec_t* spec);                /* harness.cpp:269-272 */
int64_t dconv_act_elems(const dconv_act_t* a);                     /* blocked.hpp:29-34 */
int64_t dconv_wt_elems(const dconv_wt_t* w);                       /* blocked.hpp:92-97 */

/* ---------------------------------------------------------------- layouts (device, async) */
/* to_blocked_activation (blocked.hpp:133-155): NCHW -> blocked, halo and tail lanes zero */
int dconv_pack_act(const void* nchw, int src_dtype, const dconv_act_t* dst, dconv_stream_t stream);
/* from_blocked_activation (blocked.hpp:157-178) */
int dconv_unpack_act(const dconv_act_t* src, void* nchw, int dst_dtype, dconv_stream_t stream);
/* to_blocked_weight / from_blocked_weight (blocked.hpp:180-213) */
int dconv_pack_wt(const void* kcrs, int src_dtype, const dconv_wt_t* dst, dconv_stream_t stream);
int dconv_unpack_wt(const dconv_wt_t* src, void* kcrs, int dst_dtype, dconv_stream_t stream);
/* transform_weight_stride1 (propagation.hpp:20-33): dst has k = src.c, c = src.k */
int dconv_transform_weight_dual(const dconv_wt_t* src, const dconv_wt_t* dst, dconv_stream_t stream);
/* copy_with_halo (propagation.hpp:35-49) */
int dconv_copy_with_halo(const dconv_act_t* src, const dconv_act_t* dst, dconv_stream_t stream);
/* BlockedActivationT::zero_halo (blocked.hpp:67-79) */
int dconv_zero_halo(const dconv_act_t* act, dconv_stream_t stream);
/* apply_fused_op (propagation.cpp:193-215): post-hoc op on the interior */
int dconv_apply_fused_op(const dconv_act_t* act, const dconv_fusion_t* op, dconv_stream_t stream);
/* host-side seeded generators shared by bench and tests (util.hpp:40-71 splitmix64) */
void dconv_fill_uniform_host(uint64_t seed, float lo, float hi, float* out, int64_t n);
void dconv_fill_he_normal_host(uint64_t seed, float stddev, float* out, int64_t n);

/* ---------------------------------------------------------------- forward */
typedef struct dconv_fwd_plan* dconv_fwd_plan_t;
/* make_forward_plan (propagation.cpp:42-54): tile selection replaces
 * choose_loop_order / select_register_blocking / partition_threads / dryrun */
int dconv_fwd_plan_create(const dconv_spec_t* spec, const dconv_fusion_t* fusion, const dconv_engine_config_t* cfg,
                          int math, int out_halo_h, int out_halo_w, dconv_fwd_plan_t* plan);
void dconv_fwd_plan_destroy(dconv_fwd_plan_t plan);
/* JSON description of the chosen tiles (LayerReport.blocking analog, harness.hpp:48) */
int dconv_fwd_plan_describe(dconv_fwd_plan_t plan, char* buf, size_t len);
size_t dconv_fwd_workspace_bytes(dconv_fwd_plan_t plan);
/* forward_into (propagation.cpp:56-61): writes the interior and zeroes the
 * output halo; any input halo is accepted (padding is an OOB zero fill). */
int dconv_forward(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_wt_t* wt, const dconv_act_t* out,
                  void* workspace, dconv_stream_t stream);
/* number of this library's kernels one dconv_forward launches */
int dconv_fwd_launches(dconv_fwd_plan_t plan);

/* Graph-executor epilogue (run_chain analog, harness.cpp:311-358, extended to
 * training): v = acc (+bias) (+add[px]); relu; v *= (mask[px] > 0).
 * add / mask are device tensors with the OUTPUT's geometry and dtype (null = off):
 * add carries a residual (forward) or the other branch's gradient (backward),
 * mask the forward activation whose ReLU the gradient passes back through. */
typedef struct dconv_epilogue {
  const void* add;
  const void* mask;
  int relu;
  /* DCONV_EP_PREP_ONLY: only prepare the weights into `workspace` (they depend on
   * the weights alone: a caller may run this on another stream, ahead of time);
   * DCONV_EP_WEIGHTS_READY: the workspace already holds them, skip the preparation */
  int flags;
} dconv_epilogue_t;
#define DCONV_EP_WEIGHTS_READY 1
#define DCONV_EP_PREP_ONLY 2
int dconv_forward_ex(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_wt_t* wt, const dconv_act_t* out,
                     const dconv_epilogue_t* ep, void* workspace, dconv_stream_t stream);

/* ---------------------------------------------------------------- backward-data */
typedef struct dconv_bwd_plan* dconv_bwd_plan_t;
typedef enum dconv_bwd_route {
  DCONV_BWD_DUALITY_STRIDE1 = 0, /* propagation.hpp:11 */
  DCONV_BWD_DUALITY_1x1 = 1,
  DCONV_BWD_GENERIC = 2          /* stride-phase decomposition (GENERIC_GEMM analog) */
} dconv_bwd_route_t;
/* prepare_backward (propagation.cpp:217-276); weights are passed per execute call */
int dconv_bwd_plan_create(const dconv_spec_t* spec, const dconv_engine_config_t* cfg, int math,
                          dconv_bwd_plan_t* plan);
void dconv_bwd_plan_destroy(dconv_bwd_plan_t plan);
int dconv_bwd_route(dconv_bwd_plan_t plan); /* choose_backward_route (propagation.cpp:35-40) */
int dconv_bwd_plan_describe(dconv_bwd_plan_t plan, char* buf, size_t len);
size_t dconv_bwd_workspace_bytes(dconv_bwd_plan_t plan);
/* backward_with (propagation.cpp:278-348): dI interior written, dI halo zeroed,
 * off-lattice entries of strided routes exactly 0 */
int dconv_backward_data(dconv_bwd_plan_t plan, const dconv_wt_t* wt, const dconv_act_t* grad_out,
                        const dconv_act_t* grad_in, void* workspace, dconv_stream_t stream);
int dconv_bwd_launches(dconv_bwd_plan_t plan);
/* backward_data with the graph epilogue; for strided layers `add` must be null
 * or grad_in->data itself (in-place gradient accumulation) */
int dconv_backward_data_ex(dconv_bwd_plan_t plan, const dconv_wt_t* wt, const dconv_act_t* grad_out,
                           const dconv_act_t* grad_in, const dconv_epilogue_t* ep, void* workspace,
                           dconv_stream_t stream);

/* Batched weight preparation (executor extension; no reference counterpart): between
 * dconv_prep_batch_begin() and dconv_prep_batch_end(stream), dconv_forward_ex /
 * dconv_backward_data_ex calls with DCONV_EP_PREP_ONLY made by the calling thread
 * record their weight preparation instead of launching it; _end launches every recorded
 * preparation as ONE kernel on `stream` (its job table is a kernel parameter, so the
 * launch is graph-capturable). The convs then run with DCONV_EP_WEIGHTS_READY on the
 * same workspaces -- one launch per step instead of one per conv. */
int dconv_prep_batch_begin(void);
int dconv_prep_batch_end(dconv_stream_t stream);

/* ---------------------------------------------------------------- graph-executor ops */
/* 3x3 / stride 2 / pad 1 max pool (ResNet stem) on halo-0 blocked tensors;
 * argmax: n*c_b*P*Q*16 bytes, consumed by the backward (gather, no atomics) */
int dconv_maxpool_fwd(const dconv_act_t* in, const dconv_act_t* out, void* argmax, dconv_stream_t stream);
/* mask (nullable, grad_in's geometry): ReLU backward of the pooled activation */
int dconv_maxpool_bwd(const dconv_act_t* grad_out, const void* argmax, const dconv_act_t* grad_in, const void* mask,
                      dconv_stream_t stream);
/* stride-2 lattice of a halo-0 blocked tensor (inverse = 0: sub[n][c][y][x] =
 * in[n][c][2y][2x]) and back (inverse = 1: in = the lattice values of sub, exact
 * zeros elsewhere): a stride-2 1x1 conv is a stride-1 1x1 conv over the lattice,
 * and its backward-data the lattice scatter of that conv's (the reference runs it
 * as DUALITY_1x1, propagation.cpp:35-40, 277-355); sub = ((h+1)/2, (w+1)/2) */
int dconv_subsample2(const dconv_act_t* in, const dconv_act_t* sub, int inverse, dconv_stream_t stream);
/* space-to-depth for a stride-2 conv on a narrow input (the 7x7/s2/p3 stem):
 * xs[n][i][j][(dy*2+dx)*C+c] = x[n][c][2i+dy-pad][2j+dx-pad], C <= 4 -> 4C
 * channels; the conv becomes stride 1 with a ceil(R/2) x ceil(S/2) filter */
int dconv_s2d_act(const dconv_act_t* x, const dconv_act_t* xs, int pad, dconv_stream_t stream);
/* the NCHW fp32 image (C <= 4) packed straight into that space-to-depth layout
 * (input packing and dconv_s2d_act in one pass) */
int dconv_pack_s2d(const float* nchw, int n, int c, int h, int w, const dconv_act_t* xs, int pad,
                   dconv_stream_t stream);
/* filter for that conv (inverse = 0: w -> w2) and its gradient back (inverse = 1:
 * w2 -> w, i.e. dW from the stride-1 conv's dW2); fp32 blocked weights */
int dconv_s2d_wt(const dconv_wt_t* w, const dconv_wt_t* w2, int inverse, dconv_stream_t stream);
/* same backward with the ReLU mask of the pooled INPUT taken from the pooled
 * OUTPUT (grad_out's geometry): at the argmax the input equals the window max,
 * so "input > 0" == "output > 0" -- a quarter of the mask bytes */
int dconv_maxpool_bwd_pooled_mask(const dconv_act_t* grad_out, const void* argmax, const dconv_act_t* grad_in,
                                   const dconv_act_t* pooled, dconv_stream_t stream);
/* w -= lr * g on fp32 blocked weights */
int dconv_sgd(const dconv_wt_t* w, const dconv_wt_t* g, float lr, dconv_stream_t stream);

/* ---------------------------------------------------------------- weight update */
typedef struct dconv_upd_plan* dconv_upd_plan_t;
/* choose_update_strategy + choose_spatial_blocking (planner.cpp:107-173):
 * split-K factor and pixel band per stage */
int dconv_upd_plan_create(const dconv_spec_t* spec, const dconv_engine_config_t* cfg, int math,
                          dconv_upd_plan_t* plan);
void dconv_upd_plan_destroy(dconv_upd_plan_t plan);
int dconv_upd_splits(dconv_upd_plan_t plan); /* WeightUpdateStrategy.copies analog */
int dconv_upd_plan_describe(dconv_upd_plan_t plan, char* buf, size_t len);
/* workspace depends on the operand dtypes / halos (fp32 operands are split once into bf16 pieces) */
size_t dconv_upd_workspace_bytes(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out);
/* weight_update (propagation.cpp:377-458) + reduce_weight_copies (:357-375):
 * fixed-order split reduction -> bitwise reproducible. accumulate != 0 adds into dw. */
int dconv_weight_update(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out,
                        const dconv_wt_t* grad_w, int accumulate, void* workspace, dconv_stream_t stream);
int dconv_upd_launches(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out);

/* ---------------------------------------------------------------- plan validation */
/* validate_plan (kernel_streams.cpp:461-617) analog: re-derives the plan's tile
 * schedule for these tensors on the host and checks that every output element
 * is written exactly once (tiles, CTA striding, lattices, zero fills), that the
 * staged boxes cover every row the MMAs read, and the smem / TMEM / ring / box
 * limits; UPD: split ranges and tap groups partition their index spaces.
 * DCONV_ERR_INVALID_DESCRIPTOR on the first violation; `report` (may be null)
 * receives a JSON summary. No device work. */
int dconv_fwd_plan_validate(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_act_t* out, char* report,
                            size_t len);
int dconv_bwd_plan_validate(dconv_bwd_plan_t plan, const dconv_act_t* grad_out, const dconv_act_t* grad_in,
                            char* report, size_t len);
int dconv_upd_plan_validate(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out,
                            char* report, size_t len);

/* ---------------------------------------------------------------- plan serialization */
/* save_plan / load_plan (kernel_streams.cpp:619-788; KSPL v1) analog, text
 * format "DCPL 1": the plan descriptor plus every launch the plan has resolved
 * (tile shapes, ring depths, grid, split-K factor, tap tables, epilogue) per
 * tensor geometry. save: writes a NUL-terminated text into buf (len bytes;
 * buf = NULL only reports the size in *needed). load: rebuilds the plan and
 * seeds its launch cache, so the reloaded plan executes exactly the saved
 * tiles (bitwise-identical results); validate != 0 runs the plan validator on
 * every loaded launch (DCONV_ERR_INVALID_DESCRIPTOR if one fails). Malformed
 * text: DCONV_ERR_PARSE (errors.hpp:54). */
int dconv_fwd_plan_save(dconv_fwd_plan_t plan, char* buf, size_t len, size_t* needed);
int dconv_fwd_plan_load(const char* text, size_t len, int validate, dconv_fwd_plan_t* plan);
int dconv_bwd_plan_save(dconv_bwd_plan_t plan, char* buf, size_t len, size_t* needed);
int dconv_bwd_plan_load(const char* text, size_t len, int validate, dconv_bwd_plan_t* plan);
int dconv_upd_plan_save(dconv_upd_plan_t plan, char* buf, size_t len, size_t* needed);
int dconv_upd_plan_load(const char* text, size_t len, int validate, dconv_upd_plan_t* plan);

/* ---------------------------------------------------------------- host-buffer step */
/* One layer step on HOST tensors (pinned for overlap), the reference's
 * execute contract (propagation.cpp:56-61 forward_into, :237-261 backward_with,
 * :377-458 weight_update take host memory): the batch streams through the GPU
 * in chunks of `chunk_images` (0 = N/4) with H2D of chunk i+1, the kernels of
 * chunk i and D2H of chunk i-1 overlapped on internal streams. Descriptor
 * `data` fields are HOST pointers. A null y / dx / dw skips that pass. The
 * call is asynchronous on `stream`, which completes after every copy. */
typedef struct dconv_host_step* dconv_host_step_t;
int dconv_host_step_create(const dconv_spec_t* spec, int math, int chunk_images, dconv_host_step_t* step);
void dconv_host_step_destroy(dconv_host_step_t step);
int dconv_host_step_chunk(dconv_host_step_t step);
int dconv_host_step_run(dconv_host_step_t step, const dconv_act_t* x, const dconv_wt_t* w, const dconv_act_t* dy,
                        const dconv_act_t* y, const dconv_act_t* dx, const dconv_wt_t* dw, dconv_stream_t stream);
/* kernels launched by the last run */
int dconv_host_step_launches(dconv_host_step_t step);

/* ---------------------------------------------------------------- layer-graph executor */
/* run_chain (harness.cpp:311-358; ChainLayer harness.hpp:84-95) grown into the
 * data-parallel training step of a conv DAG: forward (ReLU / residual add fused),
 * backward-data (ReLU mask / branch sum fused), weight updates on a side stream,
 * NCCL all-reduce of the fp32 weight gradients in buckets (backward order,
 * overlapped with the backward of earlier layers; COPY_REDUCE over minibatch
 * shards, propagation.cpp:357-375, promoted to GPUs), SGD; capturable into one
 * CUDA graph per step at any world size. Tensors are blocked, halo 0, vlen 16. */
typedef enum dconv_node_kind { DCONV_NODE_CONV = 0, DCONV_NODE_MAXPOOL = 1 /* 3x3, stride 2, pad 1 */ } dconv_node_kind_t;
typedef struct dconv_graph_node {
  int kind;
  int src; /* input tensor id: 0 = the graph input, node i writes tensor i + 1 */
  int add; /* conv: tensor id added before the ReLU (residual), -1 = none */
  int C, K, R, S, stride, pad_h, pad_w;
  int relu; /* conv: ReLU on the output */
} dconv_graph_node_t;
typedef struct dconv_graph_config {
  float lr;             /* SGD learning rate */
  int seed;             /* He-normal weights: splitmix64 seed * 1000 + conv index */
  int64_t bucket_bytes; /* gradient all-reduce bucket size */
  int world, rank;      /* data-parallel shard of the global minibatch */
  void* nccl_comm;      /* ncclComm_t (dconv_nccl_comm_create) or NULL: no exchange (world 1, or the
                           caller all-reduces dconv_graph_grads itself between backward and apply) */
  int overlap_update;   /* 1: weight updates on a side stream, concurrent with backward-data */
  int act_dtype;        /* activation storage (DCONV_BF16; DCONV_F32 for fp32-accurate math) */
} dconv_graph_config_t;
typedef struct dconv_graph* dconv_graph_t;
void dconv_graph_config_default(dconv_graph_config_t* cfg);
/* the chain checks of run_chain (harness.cpp:331-341): DCONV_ERR_CHAIN_SHAPE_MISMATCH */
int dconv_graph_create(const dconv_graph_node_t* nodes, int n_nodes, int batch, int in_c, int in_h, int in_w,
                       int math, const dconv_graph_config_t* cfg, dconv_graph_t* graph);
void dconv_graph_destroy(dconv_graph_t graph);
/* this step's images: NCHW fp32 on the device (packed into the input / the stem's layout) */
int dconv_graph_load_input(dconv_graph_t graph, const float* nchw, dconv_stream_t stream);
int dconv_graph_forward(dconv_graph_t graph, dconv_stream_t stream);
/* dtop: gradient of the last tensor (its ReLU applied here); leaves dW in dconv_graph_grads,
 * all-reduced when a communicator is set */
int dconv_graph_backward(dconv_graph_t graph, const dconv_act_t* dtop, dconv_stream_t stream);
/* waits for the exchange, averages over `world`, SGD on the flat master weights */
int dconv_graph_apply(dconv_graph_t graph, dconv_stream_t stream);
int dconv_graph_step(dconv_graph_t graph, const dconv_act_t* dtop, dconv_stream_t stream); /* all three */
/* capture one step into a CUDA graph on `stream` (non-default), then replay it */
int dconv_graph_capture(dconv_graph_t graph, const dconv_act_t* dtop, dconv_stream_t stream);
int dconv_graph_replay(dconv_graph_t graph, dconv_stream_t stream);
int dconv_graph_launches(dconv_graph_t graph); /* kernels of the last step (NCCL's excluded) */
/* per-layer device time (LayerReport analog, harness.hpp:36-60): runs one step, then
 * times each conv's forward, backward-data and weight update alone on `stream`
 * (best of 2 x `reps` back-to-back calls); ms[3*conv + {0,1,2}]. Overwrites the
 * step's tensors. */
int dconv_graph_profile(dconv_graph_t graph, const dconv_act_t* dtop, int reps, float* ms, dconv_stream_t stream);
int dconv_graph_num_tensors(dconv_graph_t graph);
int dconv_graph_num_convs(dconv_graph_t graph);
int dconv_graph_buckets(dconv_graph_t graph);
int dconv_graph_tensor(dconv_graph_t graph, int id, int grad, dconv_act_t* out);
int dconv_graph_conv(dconv_graph_t graph, int conv, int* node, dconv_wt_t* w, dconv_wt_t* dw);
/* flat fp32 buffers laid out in backward order: weight gradients / master weights */
int dconv_graph_grads(dconv_graph_t graph, float** flat, size_t* n);
int dconv_graph_weights(dconv_graph_t graph, float** flat, size_t* n);
/* NCCL communicator helpers (libnccl.so.2 loaded at run time): the id (128 bytes) is
 * made on one rank and broadcast by the caller */
int dconv_nccl_unique_id(char* id, size_t len);
int dconv_nccl_comm_create(const char* id, size_t len, int world, int rank, void** comm);
int dconv_nccl_comm_destroy(void* comm);

/* graph-executor element ops: g *= (act > 0); w *= scale (fp32) */
int dconv_relu_mask(const dconv_act_t* grad, const dconv_act_t* act, dconv_stream_t stream);
int dconv_scale_wt(const dconv_wt_t* w, float scale, dconv_stream_t stream);
/* cap the SMs a persistent conv kernel occupies (0 = all): leaves room for
 * collectives running concurrently; applies to launches resolved afterwards */
int dconv_set_sm_budget(int sms);

/* ---------------------------------------------------------------- developer mode */
/* on != 0: the DCONV_* experiment variables of tools/ (tile / ring / split
 * overrides) take effect and plan caches are bypassed. Off by default: the
 * environment cannot change a production plan. */
int dconv_set_dev_mode(int on);

/* ---------------------------------------------------------------- profiling */
/* enable != 0: bracket each pass's main conv kernel(s) with CUDA events on the
 * launch stream (0 forward, 1 backward-data, 2 weight-update) */
int dconv_profile(int enable);
/* device time of the last bracketed launch of pass `which` in ms (synchronises
 * on its stop event); -1 if none */
float dconv_profile_last_ms(int which);

#ifdef __cplusplus
}
#endif
#endif /* DCONV_B200_H */
