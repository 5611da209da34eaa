// TEST / BASELINE INFRASTRUCTURE ONLY.
// A thin extern "C" driver over the UNMODIFIED reference artifact
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libdconv_ref.so). It exposes
//  * the reference naive oracles and blocked conversions, used by
//    tests/test_oracle.py to pin oracle/oracle.c bitwise, and
//  * the reference direct engine's FWD / BWD / UPD execute calls, timed the
//    way the reference harness times them (harness.cpp:55-72, 180-185,
//    208-222, 247-257), used as bench.py's CPU baseline / reference arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>

#include "dconv/blocked.hpp"
#include "dconv/harness.hpp"
#include "dconv/planner.hpp"
#include "dconv/propagation.hpp"
#include "dconv/reference.hpp"

using namespace dconv;

namespace {
thread_local std::string g_err;

ConvLayerSpec spec_of(const int* s) {
  return make_layer_spec(s[0], s[1], s[2], s[3], s[4], s[5], s[6], s[7], s[8], s[9], s[10]);
}
TensorF wrap(const float* p, int64_t a, int64_t b, int64_t c, int64_t d) {
  TensorF t(a, b, c, d);
  std::memcpy(t.data(), p, sizeof(float) * t.size());
  return t;
}
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int64_t ref_pass_flops(const int* s) {
  int64_t v = -1;
  guarded([&] { v = pass_flops(spec_of(s)); });
  return v;
}

// reference.cpp:99-128 naive oracles on canonical tensors
int ref_conv_forward_naive(const int* s, const float* in, const float* wt, float* out) {
  return guarded([&] {
    const ConvLayerSpec sp = spec_of(s);
    const auto [P, Q] = derive_output_shape(sp);
    const TensorF o = conv_forward_naive(sp, wrap(in, sp.N, sp.C, sp.H, sp.W), wrap(wt, sp.K, sp.C, sp.R, sp.S));
    std::memcpy(out, o.data(), sizeof(float) * o.size());
    (void)P;
    (void)Q;
  });
}
int ref_conv_backward_naive(const int* s, const float* go, const float* wt, float* gi) {
  return guarded([&] {
    const ConvLayerSpec sp = spec_of(s);
    const auto [P, Q] = derive_output_shape(sp);
    const TensorF o = conv_backward_naive(sp, wrap(go, sp.N, sp.K, P, Q), wrap(wt, sp.K, sp.C, sp.R, sp.S));
    std::memcpy(gi, o.data(), sizeof(float) * o.size());
  });
}
int ref_conv_update_naive(const int* s, const float* in, const float* go, float* gw) {
  return guarded([&] {
    const ConvLayerSpec sp = spec_of(s);
    const auto [P, Q] = derive_output_shape(sp);
    const TensorF o = conv_update_naive(sp, wrap(in, sp.N, sp.C, sp.H, sp.W), wrap(go, sp.N, sp.K, P, Q));
    std::memcpy(gw, o.data(), sizeof(float) * o.size());
  });
}

// harness.cpp:274-278 random_f32 with Rng(seed)
void ref_random_f32(uint64_t seed, float* out, int64_t n) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.next_f32();
}

// blocked.hpp conversions and propagation.hpp:20-33 dual transform
int ref_to_blocked_act(const float* nchw, int n, int c, int h, int w, int vlen, int hh, int hw, float* out) {
  return guarded([&] {
    const auto b = to_blocked_activation(wrap(nchw, n, c, h, w), vlen, hh, hw);
    std::memcpy(out, b.data.data(), sizeof(float) * b.data.size());
  });
}
int ref_to_blocked_wt(const float* kcrs, int k, int c, int r, int s, int vlen, float* out) {
  return guarded([&] {
    const auto b = to_blocked_weight(wrap(kcrs, k, c, r, s), vlen);
    std::memcpy(out, b.data.data(), sizeof(float) * b.data.size());
  });
}
int ref_transform_weight_stride1(const float* kcrs, int k, int c, int r, int s, int vlen, float* out) {
  return guarded([&] {
    const auto b = transform_weight_stride1(to_blocked_weight(wrap(kcrs, k, c, r, s), vlen));
    std::memcpy(out, b.data.data(), sizeof(float) * b.data.size());
  });
}

// Reference direct engine, one pass, canonical tensors in/out. pass: 0 F, 1 B, 2 U.
// Setup (plan / context / strategy) is untimed as in bench_layer; the execute
// call is timed `iters` times after one warm-up. Returns best and mean ms and
// leaves the last result in `out` (NKPQ / NCHW / KCRS).
int ref_direct_pass(const int* s, int pass, int threads, int iters, const float* a, const float* b, float* out,
                    double* best_ms, double* avg_ms) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const ConvLayerSpec sp = spec_of(s);
    const auto [P, Q] = derive_output_shape(sp);
    double best = std::numeric_limits<double>::infinity(), sum = 0.0;
    auto timed = [&](auto&& fn) {
      fn();
      for (int i = 0; i < iters; ++i) {
        const auto t0 = Clock::now();
        fn();
        const double ms = std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
        best = ms < best ? ms : best;
        sum += ms;
      }
    };
    if (pass == 0) {
      const BlockedActivation ib = to_blocked_activation(wrap(a, sp.N, sp.C, sp.H, sp.W), sp);
      const BlockedWeight wb = to_blocked_weight(wrap(b, sp.K, sp.C, sp.R, sp.S), sp);
      const ExecutionPlan plan = make_forward_plan(sp, threads);
      BlockedActivation o(sp.N, sp.K, P, Q, sp.vlen);
      timed([&] { forward_into(plan, ib, wb, o); });
      const TensorF t = from_blocked_activation(o);
      std::memcpy(out, t.data(), sizeof(float) * t.size());
    } else if (pass == 1) {
      const BlockedActivation gb = to_blocked_activation(wrap(a, sp.N, sp.K, P, Q), sp.vlen, 0, 0);
      const BlockedWeight wb = to_blocked_weight(wrap(b, sp.K, sp.C, sp.R, sp.S), sp);
      const BackwardContext ctx = prepare_backward(sp, wb, threads);
      BlockedActivation gi;
      timed([&] { gi = backward_with(ctx, gb); });
      const TensorF t = from_blocked_activation(gi);
      std::memcpy(out, t.data(), sizeof(float) * t.size());
    } else {
      const BlockedActivation ib = to_blocked_activation(wrap(a, sp.N, sp.C, sp.H, sp.W), sp);
      const BlockedActivation gb = to_blocked_activation(wrap(b, sp.N, sp.K, P, Q), sp.vlen, 0, 0);
      const WeightUpdateStrategy st = choose_update_strategy(sp, threads);
      const auto [bp, bq] = choose_spatial_blocking(sp);
      BlockedWeight dw;
      timed([&] { dw = weight_update(sp, ib, gb, st, bp, bq); });
      const TensorF t = from_blocked_weight(dw);
      std::memcpy(out, t.data(), sizeof(float) * t.size());
    }
    *best_ms = best;
    *avg_ms = iters > 0 ? sum / iters : 0.0;
  });
}

}  // extern "C"
