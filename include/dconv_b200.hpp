/*
 * dconv_b200.hpp — header-compatible C++ shim: the reference's execute API on a B200.
 *
 * The reference artifact's calls (namespace dconv, /root/reference/proj/core):
 *   make_forward_plan / forward_into / forward       propagation.hpp:53-64
 *   prepare_backward / backward_with / backward      propagation.hpp:93-101
 *   choose_update_strategy / choose_spatial_blocking planner.hpp:87-94
 *   weight_update                                    propagation.hpp:113-117
 * re-declared in namespace dconv_b200 with the SAME signatures over the reference's
 * own types (dconv::ConvLayerSpec, dconv::BlockedActivation / BlockedWeight host
 * tensors, dconv::FusedOp, dconv::EngineConfig, dconv::WeightUpdateStrategy) and
 * its exception classes (errors.hpp:8-57), implemented over the C ABI
 * (dconv_b200.h). A caller switches engines by namespace:
 *
 *   #include <dconv/propagation.hpp>      // the reference's headers first
 *   #include "dconv_b200.hpp"
 *   namespace eng = dconv_b200;            // was: namespace eng = dconv;
 *   auto plan = eng::make_forward_plan(spec, threads);
 *   eng::forward_into(plan, in, wt, out);
 *
 * Contract kept: tensors are host memory, every call returns finished results
 * (synchronous), the output of forward_into is fully overwritten (halo zeroed),
 * backward_with returns dI with halo 0 on the stride-1 dual route and halo = pad
 * otherwise (propagation.cpp:279-355), validation throws the reference's
 * exceptions. Differences: `threads` is accepted and ignored; the tensors are
 * staged through device buffers per call (device-resident callers use the C ABI
 * directly: no copies, asynchronous on a stream); plans are move-only handles.
 * Math: fp32-accurate (DCONV_MATH_F32) unless a plan is made with DCONV_MATH_BF16.
 */
#ifndef DCONV_B200_HPP
#define DCONV_B200_HPP

#include <cuda_runtime.h>

#include <memory>
#include <optional>
#include <string>
#include <utility>

#include "dconv_b200.h"

namespace dconv_b200 {

// ------------------------------------------------------------------ errors
[[noreturn]] inline void raise_status(int st, const std::string& where) {
  const std::string msg = where + ": " + dconv_last_error();
  switch (st) {
    case DCONV_ERR_NON_INTEGRAL_SHAPE: throw dconv::NonIntegralShape(msg);
    case DCONV_ERR_INVALID_LAYER_SPEC: throw dconv::InvalidLayerSpec(msg);
    case DCONV_ERR_SHAPE_MISMATCH: throw dconv::ShapeMismatch(msg);
    case DCONV_ERR_INVALID_DESCRIPTOR: throw dconv::InvalidDescriptor(msg);
    case DCONV_ERR_OVERFLOW_RISK: throw dconv::OverflowRisk(msg);
    case DCONV_ERR_PLAN_INFEASIBLE: throw dconv::PlanInfeasible(msg);
    case DCONV_ERR_EMPTY_TRACE: throw dconv::EmptyTrace(msg);
    case DCONV_ERR_PLAN_TENSOR_MISMATCH: throw dconv::PlanTensorMismatch(msg);
    case DCONV_ERR_INFEASIBLE_STRATEGY: throw dconv::InfeasibleStrategy(msg);
    case DCONV_ERR_CHAIN_SHAPE_MISMATCH: throw dconv::ChainShapeMismatch(msg);
    case DCONV_ERR_PARSE: throw dconv::ParseError(msg, 0);
    default: throw dconv::Error(msg);
  }
}
inline void check(int st, const char* where) {
  if (st != DCONV_OK) raise_status(st, where);
}
inline void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw dconv::Error(std::string(where) + ": " + cudaGetErrorString(e));
}

namespace detail {
inline dconv_spec_t spec_c(const dconv::ConvLayerSpec& s) {
  return dconv_spec_t{s.N, s.C, s.K, s.H, s.W, s.R, s.S, s.stride, s.pad_h, s.pad_w, s.vlen};
}
inline dconv_engine_config_t cfg_c(const dconv::EngineConfig& c, int upd_splits = 0) {
  dconv_engine_config_t e;
  dconv_engine_config_default(&e);
  e.min_accumulators = c.min_accumulators;
  e.max_accumulators = c.max_accumulators;
  e.cache_budget_bytes = c.cache_budget_bytes;
  e.prefetch_lookahead = c.prefetch_lookahead;
  e.prefetch_enabled = c.prefetch_enabled ? 1 : 0;
  e.streaming_stores = c.streaming_stores ? 1 : 0;
  e.acc_chain_limit = c.acc_chain_limit;
  e.i16_bound_in = c.i16_bound_in;
  e.i16_bound_wt = c.i16_bound_wt;
  e.upd_splits = upd_splits;
  return e;
}
// a device buffer (freed on scope exit)
struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { cuda_check(cudaMalloc(&p, bytes ? bytes : 256), "cudaMalloc"); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
};
template <class A>
size_t bytes_of(const A& a) {
  return a.data.size() * sizeof(float);
}
inline dconv_act_t act_c(void* dev, const dconv::BlockedActivation& a) {
  return dconv_act_t{dev, a.n, a.c, a.h, a.w, a.vlen, a.halo_h, a.halo_w, DCONV_F32};
}
inline dconv_wt_t wt_c(void* dev, const dconv::BlockedWeight& w) {
  return dconv_wt_t{dev, w.k, w.c, w.r, w.s, w.vlen, DCONV_F32};
}
// the shim's own stream: every call synchronises it before returning
inline cudaStream_t stream() {
  static cudaStream_t s = [] {
    cudaStream_t t;
    cuda_check(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking), "cudaStreamCreate");
    return t;
  }();
  return s;
}
inline void upload(Dev& d, const void* h, size_t n) {
  cuda_check(cudaMemcpyAsync(d.p, h, n, cudaMemcpyHostToDevice, stream()), "H2D");
}
inline void download(void* h, const Dev& d, size_t n) {
  cuda_check(cudaMemcpyAsync(h, d.p, n, cudaMemcpyDeviceToHost, stream()), "D2H");
  cuda_check(cudaStreamSynchronize(stream()), "sync");
}
}  // namespace detail

// ------------------------------------------------------------------ forward (propagation.hpp:53-64)
struct ExecutionPlan {
  dconv::ConvLayerSpec spec;
  int out_halo_h = 0, out_halo_w = 0;
  int math = DCONV_MATH_F32;
  std::shared_ptr<dconv_fwd_plan> handle;  // dconv_fwd_plan_destroy on release
};

inline ExecutionPlan make_forward_plan(const dconv::ConvLayerSpec& spec, int threads,
                                       const std::optional<dconv::FusedOp>& fusion = {},
                                       const dconv::EngineConfig& cfg = {}, int math = DCONV_MATH_F32,
                                       int out_halo_h = 0, int out_halo_w = 0) {
  (void)threads;
  spec.validate();
  const dconv_spec_t s = detail::spec_c(spec);
  const dconv_engine_config_t c = detail::cfg_c(cfg);
  dconv_fusion_t f{DCONV_FUSE_NONE, nullptr, 0};
  if (fusion) {
    f.kind = static_cast<int>(fusion->kind);  // RELU, BIAS_ADD, BIAS_RELU (kernel_streams.hpp:27)
    f.bias = fusion->bias.empty() ? nullptr : fusion->bias.data();
    f.bias_len = static_cast<int>(fusion->bias.size());
  }
  dconv_fwd_plan_t h = nullptr;
  check(dconv_fwd_plan_create(&s, fusion ? &f : nullptr, &c, math, out_halo_h, out_halo_w, &h), "make_forward_plan");
  ExecutionPlan p;
  p.spec = spec;
  p.out_halo_h = out_halo_h;
  p.out_halo_w = out_halo_w;
  p.math = math;
  p.handle.reset(h, dconv_fwd_plan_destroy);
  return p;
}

// writes the interior and zeroes the halo of `out` (propagation.cpp:56-61)
inline void forward_into(const ExecutionPlan& plan, const dconv::BlockedActivation& in,
                         const dconv::BlockedWeight& wt, dconv::BlockedActivation& out) {
  const dconv::ConvLayerSpec& s = plan.spec;
  // check_plan_tensors (kernel_streams.cpp:122-141): the input surface is the plan's
  if (in.halo_h != s.pad_h || in.halo_w != s.pad_w)
    throw dconv::PlanTensorMismatch("forward_into: input halo differs from the plan's input surface");
  detail::Dev di(detail::bytes_of(in)), dw(detail::bytes_of(wt)), dout(detail::bytes_of(out)),
      ws(dconv_fwd_workspace_bytes(plan.handle.get()));
  detail::upload(di, in.data.data(), detail::bytes_of(in));
  detail::upload(dw, wt.data.data(), detail::bytes_of(wt));
  const dconv_act_t a = detail::act_c(di.p, in), o = detail::act_c(dout.p, out);
  const dconv_wt_t w = detail::wt_c(dw.p, wt);
  check(dconv_forward(plan.handle.get(), &a, &w, &o, ws.p, reinterpret_cast<dconv_stream_t>(detail::stream())),
        "forward_into");
  detail::download(out.data.data(), dout, detail::bytes_of(out));
}

inline dconv::BlockedActivation forward(const dconv::ConvLayerSpec& spec, const dconv::BlockedActivation& in,
                                        const dconv::BlockedWeight& wt, const ExecutionPlan& plan) {
  const auto [P, Q] = dconv::derive_output_shape(spec);
  dconv::BlockedActivation out(spec.N, spec.K, P, Q, spec.vlen, plan.out_halo_h, plan.out_halo_w);
  dconv_b200::forward_into(plan, in, wt, out);
  return out;
}

// ------------------------------------------------------------------ backward-data (propagation.hpp:83-101)
enum class BackwardRoute { DUALITY_STRIDE1 = 0, DUALITY_1x1 = 1, GENERIC_GEMM = 2 };

struct BackwardContext {
  BackwardRoute route = BackwardRoute::GENERIC_GEMM;
  dconv::ConvLayerSpec spec;
  dconv::BlockedWeight wt;  // the weights (untransformed: the GPU prepares them per call)
  int math = DCONV_MATH_F32;
  std::shared_ptr<dconv_bwd_plan> handle;
};

inline BackwardContext prepare_backward(const dconv::ConvLayerSpec& spec, const dconv::BlockedWeight& wt,
                                        int threads, const dconv::EngineConfig& cfg = {},
                                        int math = DCONV_MATH_F32) {
  (void)threads;
  spec.validate();
  const dconv_spec_t s = detail::spec_c(spec);
  const dconv_engine_config_t c = detail::cfg_c(cfg);
  dconv_bwd_plan_t h = nullptr;
  check(dconv_bwd_plan_create(&s, &c, math, &h), "prepare_backward");
  BackwardContext ctx;
  ctx.spec = spec;
  ctx.wt = wt;
  ctx.math = math;
  ctx.handle.reset(h, dconv_bwd_plan_destroy);
  ctx.route = static_cast<BackwardRoute>(dconv_bwd_route(h));
  return ctx;
}

inline dconv::BlockedActivation backward_with(const BackwardContext& ctx, const dconv::BlockedActivation& grad_out) {
  const dconv::ConvLayerSpec& s = ctx.spec;
  const auto [P, Q] = dconv::derive_output_shape(s);
  if (grad_out.n != s.N || grad_out.c != s.K || grad_out.h != P || grad_out.w != Q || grad_out.vlen != s.vlen)
    throw dconv::ShapeMismatch("backward: grad_out does not match the layer spec");
  const bool dual1 = ctx.route == BackwardRoute::DUALITY_STRIDE1;
  dconv::BlockedActivation gi(s.N, s.C, s.H, s.W, s.vlen, dual1 ? 0 : s.pad_h, dual1 ? 0 : s.pad_w);
  detail::Dev dgo(detail::bytes_of(grad_out)), dw(detail::bytes_of(ctx.wt)), dgi(detail::bytes_of(gi)),
      ws(dconv_bwd_workspace_bytes(ctx.handle.get()));
  detail::upload(dgo, grad_out.data.data(), detail::bytes_of(grad_out));
  detail::upload(dw, ctx.wt.data.data(), detail::bytes_of(ctx.wt));
  const dconv_act_t go = detail::act_c(dgo.p, grad_out), g = detail::act_c(dgi.p, gi);
  const dconv_wt_t w = detail::wt_c(dw.p, ctx.wt);
  check(dconv_backward_data(ctx.handle.get(), &w, &go, &g, ws.p, reinterpret_cast<dconv_stream_t>(detail::stream())),
        "backward_with");
  if (!dual1) check(dconv_zero_halo(&g, reinterpret_cast<dconv_stream_t>(detail::stream())), "backward_with");
  detail::download(gi.data.data(), dgi, detail::bytes_of(gi));
  return gi;
}

inline dconv::BlockedActivation backward(const dconv::ConvLayerSpec& spec, const dconv::BlockedActivation& grad_out,
                                         const dconv::BlockedWeight& wt, int threads,
                                         const dconv::EngineConfig& cfg = {}) {
  return dconv_b200::backward_with(dconv_b200::prepare_backward(spec, wt, threads, cfg), grad_out);
}

// ------------------------------------------------------------------ weight update (planner.hpp:87-94, propagation.hpp:113-117)
// On the GPU the strategy's `copies` is the split-K factor G: G partial dW copies
// over disjoint pixel ranges summed in fixed index order (COPY_REDUCE).
inline dconv::WeightUpdateStrategy choose_update_strategy(const dconv::ConvLayerSpec& spec, int threads,
                                                          const dconv::EngineConfig& cfg = {}) {
  spec.validate();
  const dconv_spec_t s = detail::spec_c(spec);
  const dconv_engine_config_t c = detail::cfg_c(cfg);
  dconv_upd_plan_t h = nullptr;
  check(dconv_upd_plan_create(&s, &c, DCONV_MATH_F32, &h), "choose_update_strategy");
  const int g = dconv_upd_splits(h);
  dconv_upd_plan_destroy(h);
  dconv::WeightUpdateStrategy st;
  st.mode = g > 1 ? dconv::UpdateMode::COPY_REDUCE : dconv::UpdateMode::TASK_PARALLEL;
  st.copies = g;
  st.threads = threads < g ? g : threads;
  return st;
}

// the GPU streams whole output rows per stage: the blocking is (1, Q)
inline std::pair<int, int> choose_spatial_blocking(const dconv::ConvLayerSpec& spec, const dconv::EngineConfig& = {}) {
  return {1, dconv::derive_output_shape(spec).second};
}

inline dconv::BlockedWeight weight_update(const dconv::ConvLayerSpec& spec, const dconv::BlockedActivation& in,
                                          const dconv::BlockedActivation& grad_out,
                                          const dconv::WeightUpdateStrategy& strategy, int b_p, int b_q,
                                          const dconv::EngineConfig& cfg = {}, int math = DCONV_MATH_F32) {
  spec.validate();
  const auto [P, Q] = dconv::derive_output_shape(spec);
  // propagation.cpp:383-393
  if (in.n != spec.N || in.c != spec.C || in.h != spec.H || in.w != spec.W || in.vlen != spec.vlen)
    throw dconv::ShapeMismatch("weight_update: input does not match the layer spec");
  if (in.halo_h < spec.pad_h || in.halo_w < spec.pad_w)
    throw dconv::ShapeMismatch("weight_update: input halo smaller than the padding");
  if (grad_out.n != spec.N || grad_out.c != spec.K || grad_out.h != P || grad_out.w != Q ||
      grad_out.vlen != spec.vlen)
    throw dconv::ShapeMismatch("weight_update: grad_out does not match the layer spec");
  if (b_p < 1 || b_q < 1 || P % b_p != 0 || Q % b_q != 0)
    throw dconv::InfeasibleStrategy("weight_update: blocking must divide (P, Q)");
  if (strategy.threads < 1 || strategy.copies < 1 || strategy.threads % strategy.copies != 0)
    throw dconv::InfeasibleStrategy("weight_update: copies must divide threads");
  const dconv_spec_t s = detail::spec_c(spec);
  const dconv_engine_config_t c = detail::cfg_c(cfg, strategy.copies > 1 ? strategy.copies : 0);
  dconv_upd_plan_t h = nullptr;
  check(dconv_upd_plan_create(&s, &c, math, &h), "weight_update");
  std::unique_ptr<dconv_upd_plan, void (*)(dconv_upd_plan_t)> plan(h, dconv_upd_plan_destroy);
  dconv::BlockedWeight dw(spec.K, spec.C, spec.R, spec.S, spec.vlen);
  detail::Dev din(detail::bytes_of(in)), dgo(detail::bytes_of(grad_out)), ddw(detail::bytes_of(dw));
  detail::upload(din, in.data.data(), detail::bytes_of(in));
  detail::upload(dgo, grad_out.data.data(), detail::bytes_of(grad_out));
  const dconv_act_t a = detail::act_c(din.p, in), g = detail::act_c(dgo.p, grad_out);
  const dconv_wt_t w = detail::wt_c(ddw.p, dw);
  detail::Dev ws(dconv_upd_workspace_bytes(h, &a, &g));
  check(dconv_weight_update(h, &a, &g, &w, 0, ws.p, reinterpret_cast<dconv_stream_t>(detail::stream())),
        "weight_update");
  detail::download(dw.data.data(), ddw, detail::bytes_of(dw));
  return dw;
}

}  // namespace dconv_b200

#endif  // DCONV_B200_HPP
