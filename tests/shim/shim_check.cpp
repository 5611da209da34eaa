// TEST INFRASTRUCTURE: compiles include/dconv_b200.hpp (the header-compatible C++
// shim) against the reference's own headers and runs the SAME calls through both
// engines -- namespace dconv (the reference CPU direct engine, linked from
// oracle/_ref/libdconv_ref.so) and namespace dconv_b200 (the B200 through the C ABI)
// -- on reference-generated inputs (Rng / random_f32, harness.cpp:274-278), checking
// the B200 results against the reference's naive oracle (reference.cpp:99-128).
// Built by oracle/Makefile (`make shim`, needs /root/reference) into oracle/_ref/;
// tests/test_capi.py builds it, tests/test_gpu_plans.py runs it on the GPU.
#include <dconv/blocked.hpp>
#include <dconv/harness.hpp>
#include <dconv/norms.hpp>
#include <dconv/planner.hpp>
#include <dconv/propagation.hpp>
#include <dconv/reference.hpp>

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "dconv_b200.hpp"

namespace {

double max_over_rms(const dconv::TensorF& ref, const dconv::TensorF& got) {
  double mx = 0, ss = 0;
  for (int64_t i = 0; i < ref.size(); ++i) {
    mx = std::fmax(mx, std::fabs(static_cast<double>(ref.data()[i]) - got.data()[i]));
    ss += static_cast<double>(ref.data()[i]) * ref.data()[i];
  }
  const double rms = std::sqrt(ss / std::max<int64_t>(1, ref.size()));
  return rms > 0 ? mx / rms : mx;
}

int failures = 0;

void gate(const char* what, const dconv::TensorF& ref, const dconv::TensorF& got, const dconv::TensorF& cpu) {
  const double e = max_over_rms(ref, got), ec = max_over_rms(ref, cpu);
  const bool ok = e <= 1e-4;
  std::printf("%-34s b200 max/rms %.3e   reference engine %.3e   %s\n", what, e, ec, ok ? "ok" : "FAIL");
  failures += ok ? 0 : 1;
}

}  // namespace

int main() {
  // (N, C, K, H, W, R, S, stride): 3x3/s1 (dual route), 1x1/s2 (lattice route), 7x7/s2 stem (generic)
  const int shapes[][8] = {{2, 32, 48, 14, 14, 3, 3, 1}, {2, 64, 32, 14, 14, 1, 1, 2}, {2, 3, 32, 30, 30, 7, 7, 2}};
  try {
    for (const auto& sh : shapes) {
      const dconv::ConvLayerSpec spec = dconv::make_layer_spec(sh[0], sh[1], sh[2], sh[3], sh[4], sh[5], sh[6], sh[7]);
      const auto [P, Q] = dconv::derive_output_shape(spec);
      dconv::Rng rng(17);
      const dconv::TensorF x = dconv::random_f32(rng, spec.N, spec.C, spec.H, spec.W);
      const dconv::TensorF w = dconv::random_f32(rng, spec.K, spec.C, spec.R, spec.S);
      const dconv::TensorF g = dconv::random_f32(rng, spec.N, spec.K, P, Q);
      const auto ib = dconv::to_blocked_activation(x, spec);
      const auto wb = dconv::to_blocked_weight(w, spec);
      const auto gb = dconv::to_blocked_activation(g, spec.vlen, 0, 0);
      char tag[96];
      // forward: identical calls, two engines
      const auto out_b = dconv_b200::forward(spec, ib, wb, dconv_b200::make_forward_plan(spec, 4));
      const auto out_c = dconv::forward(spec, ib, wb, dconv::make_forward_plan(spec, 4));
      std::snprintf(tag, sizeof(tag), "forward  %dx%d/s%d C%d K%d", spec.R, spec.S, spec.stride, spec.C, spec.K);
      gate(tag, dconv::conv_forward_naive(spec, x, w), dconv::from_blocked_activation(out_b),
           dconv::from_blocked_activation(out_c));
      // backward-data
      const auto gi_b = dconv_b200::backward(spec, gb, wb, 4);
      const auto gi_c = dconv::backward(spec, gb, wb, 4);
      if (gi_b.halo_h != gi_c.halo_h || gi_b.halo_w != gi_c.halo_w) {
        std::printf("backward halo differs from the reference route's (%d,%d vs %d,%d)\n", gi_b.halo_h, gi_b.halo_w,
                    gi_c.halo_h, gi_c.halo_w);
        ++failures;
      }
      std::snprintf(tag, sizeof(tag), "backward %dx%d/s%d C%d K%d", spec.R, spec.S, spec.stride, spec.C, spec.K);
      gate(tag, dconv::conv_backward_naive(spec, g, w), dconv::from_blocked_activation(gi_b),
           dconv::from_blocked_activation(gi_c));
      // weight update
      const auto st_b = dconv_b200::choose_update_strategy(spec, 4);
      const auto [bp, bq] = dconv_b200::choose_spatial_blocking(spec);
      const auto dw_b = dconv_b200::weight_update(spec, ib, gb, st_b, bp, bq);
      const auto st_c = dconv::choose_update_strategy(spec, 4);
      const auto [cp, cq] = dconv::choose_spatial_blocking(spec);
      const auto dw_c = dconv::weight_update(spec, ib, gb, st_c, cp, cq);
      std::snprintf(tag, sizeof(tag), "update   %dx%d/s%d C%d K%d G=%d", spec.R, spec.S, spec.stride, spec.C, spec.K,
                    st_b.copies);
      gate(tag, dconv::conv_update_naive(spec, x, g), dconv::from_blocked_weight(dw_b), dconv::from_blocked_weight(dw_c));
    }
    // the reference's exceptions come through the shim
    bool thrown = false;
    try {
      const dconv::ConvLayerSpec spec = dconv::make_layer_spec(1, 16, 16, 6, 6, 3, 3, 1);
      dconv::BlockedActivation bad(1, 16, 6, 6, 16, 0, 0);  // halo 0 != pad 1
      dconv::BlockedWeight wb(16, 16, 3, 3, 16);
      dconv::BlockedActivation out(1, 16, 6, 6, 16);
      dconv_b200::forward_into(dconv_b200::make_forward_plan(spec, 1), bad, wb, out);
    } catch (const dconv::PlanTensorMismatch&) {
      thrown = true;
    }
    std::printf("PlanTensorMismatch on a foreign input surface: %s\n", thrown ? "ok" : "FAIL");
    failures += thrown ? 0 : 1;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s\n", failures ? "SHIM CHECK FAILED" : "SHIM CHECK OK");
  return failures ? 1 : 0;
}
