// Plan validation — the GPU analog of the reference's `validate_plan`
// (kernel_streams.cpp:461-617), which replays a plan's recorded streams and
// checks that every output tile is written exactly once, that every offset
// stays inside its tensor, and that the APPLY records follow each tile's last
// reduction step. Here the plan is a tile schedule, so the validator re-derives
// on the host exactly what the kernels will do for the given tensors:
//  * FWD / BWD phases: every (image, output pixel, output block) the epilogue
//    writes is written by exactly one (tile, row, block) — including the
//    persistent CTA striding, multi-image tiles, virtual-row padding columns,
//    the stride lattice and the 1x1/s2 zero fill;
//  * staging geometry: the staged activation box covers every row the MMA
//    reads (taps shifted), TMA box extents <= 256, smem within the per-CTA
//    limit, TMEM columns <= 512, ring depths within the barrier arrays;
//  * UPD: split ranges partition the stage list exactly once per tile, tap
//    groups partition the taps, the stages cover every output pixel, and the
//    partial buffer holds every (split, tap, c, k).
// A failure returns DCONV_ERR_INVALID_DESCRIPTOR (errors.hpp:26) with the
// first violated property; success fills a JSON summary.
//
// Included at the end of dconv_capi.cu.
#pragma once
#include <vector>

namespace {

inline int P_chk(const dconv_spec_t& s) { return out_P(s); }

struct VReport {
  std::string err;
  long long outputs = 0, writes = 0, tiles = 0;
  void fail_if(bool bad, const std::string& what) {
    if (bad && err.empty()) err = what;
  }
};

// tile schedule coverage of one FWD-kernel launch over an output lattice of
// n_img x P x Q pixels x kb_out blocks (counts in `cnt`)
void cover_launch(const FwdLaunch& L, std::vector<uint8_t>& cnt, VReport& r) {
  const FwdParams& p = L.p;
  const int n_mtiles = p.mimg > 0 ? cdiv(p.n_img, p.mimg) : p.n_img * p.tiles_per_img;
  const int n_tiles = n_mtiles * p.n_ntiles;
  const int v_end = p.P * p.wsub;
  r.tiles += n_tiles;
  // persistent striding: CTA c takes tiles c, c + grid, ... -> each tile once
  std::vector<uint8_t> seen(static_cast<size_t>(n_tiles), 0);
  for (unsigned c = 0; c < L.grid.x; ++c)
    for (int t = static_cast<int>(c); t < n_tiles; t += static_cast<int>(L.grid.x)) ++seen[t];
  for (int t = 0; t < n_tiles; ++t) r.fail_if(seen[t] != 1, "tile " + std::to_string(t) + " scheduled " +
                                                                   std::to_string(seen[t]) + " times");
  const int M = 128 * p.mb;
  for (int t = 0; t < n_tiles && r.err.empty(); ++t) {
    const int ntile = t % p.n_ntiles, mt = t / p.n_ntiles;
    int n, v0;
    if (p.mimg > 0) {
      n = mt * p.mimg;
      v0 = 0;
    } else {
      n = mt / p.tiles_per_img;
      v0 = (mt % p.tiles_per_img) * M;
    }
    for (int row = 0; row < M; ++row) {
      int v = v0 + row, nn = n;
      bool valid;
      if (p.mimg > 0) {
        const int pitch = p.img_pitch > 0 ? p.img_pitch : v_end;
        const int img = v / pitch;
        nn = n + img;
        v -= img * pitch;
        valid = img < p.mimg && nn < p.n_img;
      } else {
        valid = v < v_end;
      }
      const int pp = v / p.wsub, qq = v - (v / p.wsub) * p.wsub;
      valid = valid && qq < p.Q && pp < p.P;
      if (!valid) continue;
      for (int g = 0; g < p.nb; ++g) {
        const int kb = ntile * p.nb + g;
        if (kb >= p.kb_out) continue;
        uint8_t& c = cnt[((static_cast<size_t>(nn) * p.P + pp) * p.Q + qq) * p.kb_out + kb];
        if (c < 255) ++c;
        ++r.writes;
      }
    }
  }
}

// the launch computes the problem it is attached to (a loaded or corrupted plan
// is rejected before the coverage replay indexes anything)
void check_problem(const FwdLaunch& L, int n_img, int P, int Q, int kb_out, int cb_red, VReport& r) {
  const FwdParams& p = L.p;
  r.fail_if(p.n_img != n_img || p.P != P || p.Q != Q || p.kb_out != kb_out || p.cb_in != cb_red,
            "launch problem (images, output extents, channel blocks) differs from the tensors");
  r.fail_if(p.mb < 1 || p.mb > 4 || p.nb < 1 || p.nb > 16 || p.wsub < p.Q || p.tiles_per_img < 0 || p.mimg < 0 ||
                p.n_ntiles < 1 || p.n_ntiles * p.nb < kb_out || p.kc < 1 || p.kc > 4,
            "tile shape outside the kernel's limits");
  r.fail_if(p.n_phases < 1 || p.n_phases > kMaxPhases || p.n_taps < 1 || p.n_taps > kMaxTaps || p.w_taps < 1,
            "tap tables outside the kernel's limits");
  r.fail_if(L.grid.x < 1 || L.grid.y != 1 || L.grid.z != 1, "grid must be (ctas, 1, 1)");
}

// staging geometry of one launch
void check_geometry(const FwdLaunch& L, int maxshift, VReport& r) {
  const FwdParams& p = L.p;
  const int M = 128 * p.mb;
  if (p.img_pitch > 0) {
    r.fail_if(p.mimg < 1 || p.mimg * p.img_pitch > M || p.img_pitch % p.wsub != 0 ||
                  (p.mimg + 1) * p.img_pitch < M + maxshift || p.a_load_px > p.a_px,
              "packed tile: images / staged rows do not cover the rows the MMA reads");
  } else if (p.mimg > 0) {
    r.fail_if(p.a_load_px > p.a_px, "multi-image tile loads more pixels than its slot holds");
  } else if (p.linear) {
    // rows v_off .. v_off + M - 1 shifted by up to maxshift must be staged
    r.fail_if(M + maxshift > p.a_px, "linear tile: staged pixels " + std::to_string(p.a_px) + " < rows read " +
                                         std::to_string(M + maxshift));
  } else {
    r.fail_if((p.wsub - 1) + M + maxshift > p.a_px, "rows tile: staged rows do not cover the shifted taps");
    r.fail_if(p.wsub * p.stride > 256 || (p.a_px / p.wsub) * p.stride > 256, "TMA box extent > 256");
  }
  r.fail_if(L.stages < 1 || L.stages > kMaxStages || L.raw_stages > kMaxStages || L.w_stages > kMaxStages,
            "ring depth outside 1..kMaxStages");
  r.fail_if(L.smem > static_cast<size_t>(kSmemBudget), "shared memory " + std::to_string(L.smem) + " > budget");
  const int acc_cols = ((L.pieces == 3 && p.split_acc) ? 2 : 1) * p.mb * 16 * p.nb;
  const int ring = L.ts ? L.stages * L.pieces * 8 * p.kc : 0;
  r.fail_if(p.acc_bufs * acc_cols + ring > 512, "TMEM columns > 512");
  // multi-block stages: any single-tap plan; multi-tap plans only with bf16 activations
  // (one box of kc planes lands straight in the MMA layout)
  r.fail_if(p.kc < 1 || (p.kc > 1 && p.n_taps != 1 && (L.raw_f32 || L.ts)),
            "multi-block multi-tap stages need bf16 activations");
}

std::string vjson(const VReport& r, const std::string& extra) {
  return "{\"ok\":" + std::string(r.err.empty() ? "true" : "false") + ",\"tiles\":" + std::to_string(r.tiles) +
         ",\"outputs\":" + std::to_string(r.outputs) + ",\"writes\":" + std::to_string(r.writes) + extra + "}";
}

}  // namespace

extern "C" {

int dconv_fwd_plan_validate(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_act_t* out, char* report,
                            size_t len) {
  if (plan && plan->inner && in && out) {  // vlen != 16: the twin's launch on the re-blocked tensors
    const dconv_act_t a = act_as16(*in, in->data, plan->spec.pad_h, plan->spec.pad_w);
    const dconv_act_t b = act_as16(*out, out->data, out->halo_h, out->halo_w);
    return dconv_fwd_plan_validate(plan->inner, &a, &b, report, len);
  }
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_act(in, "validate input");
    check_act(out, "validate output");
    const dconv_spec_t& s = plan->spec;
    const int P = out_P(s), Q = out_Q(s);
    if (in->n != s.N || in->c != s.C || in->h != s.H || in->w != s.W || out->n != s.N || out->c != s.K ||
        out->h != P || out->w != Q)
      fail(DCONV_ERR_SHAPE_MISMATCH, "validate: tensors do not match the layer spec");
    // the launch the plan will execute for these tensors (cached, or loaded by
    // dconv_plan_load: a reloaded plan is validated exactly as it will run)
    FwdLaunch L;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      L = fwd_entry(plan, *in, *out).L.at(0);
    }
    struct {
      int kb_out;
    } pb{cdiv(s.K, 16)};
    VReport r;
    std::vector<uint8_t> cnt(static_cast<size_t>(s.N) * P * Q * pb.kb_out, 0);
    r.outputs = static_cast<long long>(cnt.size());
    check_problem(L, s.N, P, Q, pb.kb_out, cdiv(s.C, 16), r);
    if (r.err.empty()) cover_launch(L, cnt, r);
    check_geometry(L, plan->taps.r2max * L.p.wsub + plan->taps.s2max, r);
    for (size_t i = 0; i < cnt.size() && r.err.empty(); ++i)
      r.fail_if(cnt[i] != 1, "output element " + std::to_string(i) + " written " + std::to_string(cnt[i]) + " times");
    r.fail_if(dconv_fwd_workspace_bytes(plan) < prep_bytes(plan->pieces, cdiv(s.C, 16), L.p.n_taps, pb.kb_out),
              "workspace smaller than the prepared weights");
    copy_out(vjson(r, ",\"plan\":" + json_tile(L)), report, len);
    if (!r.err.empty()) fail(DCONV_ERR_INVALID_DESCRIPTOR, "plan validation: " + r.err);
  });
}

int dconv_bwd_plan_validate(dconv_bwd_plan_t plan, const dconv_act_t* grad_out, const dconv_act_t* grad_in,
                            char* report, size_t len) {
  if (plan && plan->inner && grad_out && grad_in) {
    const dconv_act_t a = act_as16(*grad_out, grad_out->data, 0, 0);
    const dconv_act_t b = act_as16(*grad_in, grad_in->data, 0, 0);
    return dconv_bwd_plan_validate(plan->inner, &a, &b, report, len);
  }
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_act(grad_out, "validate grad_out");
    check_act(grad_in, "validate grad_in");
    const dconv_spec_t& s = plan->spec;
    if (grad_in->n != s.N || grad_in->c != s.C || grad_in->h != s.H || grad_in->w != s.W)
      fail(DCONV_ERR_SHAPE_MISMATCH, "validate: grad_in does not match the layer spec");
    const int kb = cdiv(s.C, 16);
    // dI pixel (y, x) belongs to phase (y % st, x % st) at lattice point (y / st, x / st)
    std::vector<uint8_t> cnt(static_cast<size_t>(s.N) * s.H * s.W * kb, 0);
    VReport r;
    r.outputs = static_cast<long long>(cnt.size());
    const bool fill = bwd_fill(plan, false);
    std::vector<FwdLaunch> Ls;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      Ls = bwd_entry(plan, *grad_out, *grad_in, false).L;
    }
    size_t conv_i = 0;
    std::string phases = "[";
    for (auto& ph : plan->phases) {
      const int ly = cdiv(s.H - ph.a, s.stride), lx = cdiv(s.W - ph.b, s.stride);
      if (ph.zero) {
        if (!fill)  // zero-lattice pass writes every lattice point once
          for (int n = 0; n < s.N; ++n)
            for (int y = 0; y < ly; ++y)
              for (int x = 0; x < lx; ++x)
                for (int b = 0; b < kb; ++b) {
                  ++cnt[((static_cast<size_t>(n) * s.H + ph.a + s.stride * y) * s.W + ph.b + s.stride * x) * kb + b];
                  ++r.writes;
                }
        phases += std::string(phases.size() > 1 ? "," : "") + (fill ? "\"filled\"" : "\"zero\"");
        continue;
      }
      if (conv_i >= Ls.size()) {
        r.fail_if(true, "plan has fewer phase launches than tap phases");
        break;
      }
      const FwdLaunch& L = Ls[conv_i++];
      VReport pr;
      check_problem(L, s.N, ly, lx, kb, cdiv(s.K, 16), pr);
      r.fail_if(!pr.err.empty(), pr.err);
      if (!r.err.empty()) break;
      std::vector<uint8_t> lat(static_cast<size_t>(s.N) * L.p.P * L.p.Q * L.p.kb_out, 0);
      cover_launch(L, lat, pr);
      check_geometry(L, ph.taps.r2max * L.p.wsub + ph.taps.s2max, pr);
      r.fail_if(!pr.err.empty(), pr.err);
      r.tiles += pr.tiles;
      for (int n = 0; n < s.N; ++n)
        for (int y = 0; y < ly; ++y)
          for (int x = 0; x < lx; ++x)
            for (int b = 0; b < kb; ++b) {
              const uint8_t c = lat[((static_cast<size_t>(n) * ly + y) * lx + x) * L.p.kb_out + b];
              const int yy = ph.a + s.stride * y, xx = ph.b + s.stride * x;
              cnt[((static_cast<size_t>(n) * s.H + yy) * s.W + xx) * kb + b] += c;
              r.writes += c;
              if (fill && c)  // the tap phase also writes the three zero neighbours it owns
                for (int dy = 0; dy < 2; ++dy)
                  for (int dx = 0; dx < 2; ++dx)
                    if ((dy | dx) && yy + dy < s.H && xx + dx < s.W) {
                      ++cnt[((static_cast<size_t>(n) * s.H + yy + dy) * s.W + xx + dx) * kb + b];
                      ++r.writes;
                    }
            }
      phases += std::string(phases.size() > 1 ? "," : "") + json_tile(L);
    }
    phases += "]";
    for (size_t i = 0; i < cnt.size() && r.err.empty(); ++i)
      r.fail_if(cnt[i] != 1, "grad_in element " + std::to_string(i) + " written " + std::to_string(cnt[i]) + " times");
    copy_out(vjson(r, ",\"route\":" + std::to_string(plan->route) + ",\"phases\":" + phases), report, len);
    if (!r.err.empty()) fail(DCONV_ERR_INVALID_DESCRIPTOR, "plan validation: " + r.err);
  });
}

int dconv_upd_plan_validate(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out,
                            char* report, size_t len) {
  if (plan && plan->inner && in && grad_out) {
    const dconv_act_t a = act_as16(*in, in->data, plan->spec.pad_h, plan->spec.pad_w);
    const dconv_act_t b = act_as16(*grad_out, grad_out->data, 0, 0);
    return dconv_upd_plan_validate(plan->inner, &a, &b, report, len);
  }
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_act(in, "validate input");
    check_act(grad_out, "validate grad_out");
    const dconv_spec_t& s = plan->spec;
    UpdLaunch L;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      L = upd_entry(plan, *in, *grad_out).L;
    }
    const UpdParams& p = L.p;
    VReport r;
    r.fail_if(L.stages < 1 || L.stages > kMaxStages || L.raw_stages > kMaxStages || L.pc_stages > kMaxStages,
              "ring depth outside 1..kMaxStages");
    r.fail_if(p.n_tgroups < 1 || p.n_tgroups > kMaxTapGroups || p.n_taps != s.R * s.S || p.splits < 1 ||
                  p.vs < 16 || p.vs % 16 != 0 || p.nb < 1 || p.nb > 16 || p.n_img != s.N ||
                  p.stages_per_img < 1 ||
                  p.stages_total != (p.pimg > 0 ? (p.n_img + p.pimg - 1) / p.pimg : p.n_img * p.stages_per_img) ||
                  (p.pimg > 0 && (p.stages_per_img != 1 || p.vs < p.pimg * p.img_pitch || p.img_pitch < P_chk(s) * p.wsub)),
              "launch tables outside the kernel's limits");
    r.fail_if(static_cast<int>(L.grid.z) != p.splits || static_cast<int>(L.grid.x) % p.n_tgroups != 0,
              "grid does not match (c-tiles x tap groups, k-tiles, splits)");
    if (!r.err.empty()) fail(DCONV_ERR_INVALID_DESCRIPTOR, "plan validation: " + r.err);
    // a CTA covers p.mc consecutive 128-channel c-tiles
    const int n_ctiles = static_cast<int>(L.grid.x) / p.n_tgroups * (p.mc > 1 ? p.mc : 1),
              n_ktiles = static_cast<int>(L.grid.y);
    r.tiles = static_cast<long long>(L.grid.x) * L.grid.y * L.grid.z;
    // split ranges partition [0, stages_total) exactly once
    std::vector<uint8_t> st(static_cast<size_t>(p.stages_total), 0);
    const int per = (p.stages_total + p.splits - 1) / p.splits;
    for (int sp = 0; sp < p.splits; ++sp)
      for (int g = sp * per; g < std::min(p.stages_total, (sp + 1) * per); ++g) ++st[g];
    for (int g = 0; g < p.stages_total; ++g)
      r.fail_if(st[g] != 1, "stage " + std::to_string(g) + " reduced " + std::to_string(st[g]) + " times");
    // tap groups partition the taps (cross-stacked: every (A slot, dO copy) pair is one tap)
    std::vector<uint8_t> tp(static_cast<size_t>(p.n_taps), 0);
    r.fail_if(p.xs > 1 && (p.xs > 4 || p.xs_S != s.S || s.stride != 1 || p.stack < 2 || p.tg != p.xs),
              "cross-stacked plan outside the kernel's limits");
    for (int g = 0; g < p.n_tgroups && r.err.empty(); ++g)
      for (int t = p.tg_tap0[g]; t < p.tg_tap0[g] + p.tg_ntaps[g]; ++t) {
        if (p.xs > 1) {
          if (t < 0 || t >= kMaxXsSlots) continue;
          for (int j = 0; j < p.xs; ++j) {
            const int tr = p.xs_slot_r[t], tc = p.xs_slot_s[t] + j;
            if (tr >= 0 && tr < s.R && tc >= 0 && tc < s.S) ++tp[tr * s.S + tc];
          }
        } else if (t >= 0 && t < p.n_taps) {
          ++tp[t];
        }
      }
    for (int t = 0; t < p.n_taps; ++t) r.fail_if(tp[t] != 1, "tap " + std::to_string(t) + " not covered once");
    // stages cover every output pixel of every image; channel tiles cover C and K
    const int P = out_P(s), Q = out_Q(s);
    r.fail_if(p.stages_per_img * p.vs < (p.linear ? P * Q : P * p.wsub) ||
                  (!p.linear && p.stages_per_img * p.rows_ps < P),
              "stages do not cover the output plane");
    r.fail_if(!p.linear && p.wsub < Q, "virtual row pitch narrower than the output row");
    r.fail_if(n_ctiles * 128 < (p.stack > 1 ? 16 * p.cb_eff : s.C) || n_ktiles * 16 * p.nb < s.K,
              "channel tiles do not cover C / K");
    r.fail_if(p.c_pad < n_ctiles * 128 || p.k_pad < n_ktiles * 16 * p.nb, "partial buffer too small");
    r.fail_if(L.smem > static_cast<size_t>(kSmemBudget), "shared memory over budget");
    r.outputs = static_cast<long long>(s.R) * s.S * s.C * s.K;
    r.writes = static_cast<long long>(p.splits) * p.n_taps * p.c_pad * p.k_pad;
    copy_out(vjson(r, ",\"splits\":" + std::to_string(p.splits) + ",\"stages_total\":" +
                          std::to_string(p.stages_total) + ",\"tap_groups\":" + std::to_string(p.n_tgroups)),
             report, len);
    if (!r.err.empty()) fail(DCONV_ERR_INVALID_DESCRIPTOR, "plan validation: " + r.err);
  });
}

}  // extern "C"
