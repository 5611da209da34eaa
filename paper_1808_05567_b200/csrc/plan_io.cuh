// Plan serialization — the GPU analog of the reference's KSPL save_plan /
// load_plan (kernel_streams.cpp:619-788). A plan here is its descriptor (spec,
// math, fusion, output surface, engine config) plus the RESOLVED launches it
// has cached per tensor geometry: tile shapes, ring depths, grid, split-K
// factor, tap tables and epilogue decisions. Loading a plan seeds its launch
// cache, so a reloaded plan executes exactly the saved tiles (bitwise-identical
// results, test_kernel_streams.cpp:234-257) without re-running the tile search.
//
// Format "DCPL 1": UTF-8 text, one record per line, `name v0 v1 ...` — kept
// editable on purpose, so tests can inject faults into a saved plan and check
// that validation catches them (test_kernel_streams.cpp:152-175). With
// validate = 1, dconv_*_plan_load runs the plan validator (validate.cuh) on
// every loaded launch against tensors of its recorded geometry and rejects the
// plan (DCONV_ERR_INVALID_DESCRIPTOR) on the first violated property.
//
// Included at the end of dconv_capi.cu, after validate.cuh.
#pragma once
#include <sstream>

namespace {

#define DCONV_FWD_INT_FIELDS(X)                                                                                     \
  X(n_img) X(in_cb) X(cb_in) X(kb_out) X(P) X(Q) X(wsub) X(tiles_per_img) X(mb) X(nb) X(acc_bufs) X(linear)       \
  X(mimg) X(a_px) X(a_load_px) X(lin_boxes) X(in_row0) X(in_col0) X(stride) X(n_phases) X(taps_box) X(w_taps)    \
  X(kc) X(w_resident) X(w_all) X(tma_store) X(out_fill) X(split_acc) X(ts_epi2) X(epi_groups) X(fill_h_end)       \
  X(fill_w_end) X(n_taps) X(n_ntiles) X(out_bf16) X(out_cb) X(out_hp) X(out_wp) X(out_y0) X(out_x0) X(out_scale)  \
  X(out_halo_h) X(out_halo_w) X(img_pitch) X(a_sw128)
#define DCONV_FWD_ARRAYS(X) \
  X(phase_row, kMaxPhases) X(phase_col, kMaxPhases) X(phase_ntaps, kMaxPhases) X(phase_tap0, kMaxPhases) X(tap_shift, kMaxTaps)

#define DCONV_UPD_INT_FIELDS(X)                                                                                    \
  X(n_img) X(in_cb) X(do_cb) X(cb_in) X(kb_out) X(P) X(Q) X(wsub) X(linear) X(rows_ps) X(vs) X(a_px) X(in_rows)  \
  X(in_row0) X(in_col0) X(stride) X(stages_per_img) X(stages_total) X(splits) X(nb) X(tg) X(n_tgroups) X(stack)  \
  X(cb_eff) X(half) X(sw32) X(mc) X(lsu) X(n_taps) X(c_pad) X(k_pad) X(drain) X(drain_bufs) X(xs) X(xs_S) X(pimg) X(img_pitch) X(epi_tma)
#define DCONV_UPD_ARRAYS(X)                                                                                     \
  X(tg_phase, kMaxTapGroups) X(tg_tap0, kMaxTapGroups) X(tg_ntaps, kMaxTapGroups) X(phase_row, kMaxPhases)      \
  X(phase_col, kMaxPhases) X(tap_shift, kMaxTaps) X(tap_src, kMaxTaps) X(tap_ph, kMaxTaps) X(tap_r2, kMaxTaps) \
  X(tap_s2, kMaxTaps) X(xs_slot_r, kMaxXsSlots) X(xs_slot_s, kMaxXsSlots)

using Rec = std::map<std::string, std::vector<long long>>;

void put(std::ostringstream& os, const char* name, std::initializer_list<long long> v) {
  os << name;
  for (long long x : v) os << ' ' << x;
  os << '\n';
}
template <class T>
void put_arr(std::ostringstream& os, const char* name, const T* a, int n) {
  os << name;
  for (int i = 0; i < n; ++i) os << ' ' << static_cast<long long>(a[i]);
  os << '\n';
}

void save_fwd_launch(std::ostringstream& os, const FwdLaunch& L) {
  os << "launch fwd\n";
  put(os, "grid", {L.grid.x, L.grid.y, L.grid.z});
  put(os, "rings", {L.stages, L.raw_stages, L.w_stages});
  put(os, "smem", {static_cast<long long>(L.smem), static_cast<long long>(L.smem_launch),
                   static_cast<long long>(L.raw_slot)});
  put(os, "mode", {L.raw_f32 ? 1 : 0, L.pieces, L.ts ? 1 : 0});
#define X(f) put(os, #f, {L.p.f});
  DCONV_FWD_INT_FIELDS(X)
#undef X
#define X(f, n) put_arr(os, #f, L.p.f, n);
  DCONV_FWD_ARRAYS(X)
#undef X
  os << "end\n";
}

void save_upd_launch(std::ostringstream& os, const UpdLaunch& L) {
  os << "launch upd\n";
  put(os, "grid", {L.grid.x, L.grid.y, L.grid.z});
  put(os, "rings", {L.stages, L.raw_stages, L.pc_stages, L.passes});
  put(os, "smem", {static_cast<long long>(L.smem)});
  put(os, "ws", {static_cast<long long>(L.ws_in), static_cast<long long>(L.ws_do),
                 static_cast<long long>(L.ws_partial)});
  put(os, "mode", {L.split_in ? 1 : 0, L.split_do ? 1 : 0, L.raw ? 1 : 0, L.cat ? 1 : 0, L.tsa ? 1 : 0});
#define X(f) put(os, #f, {L.p.f});
  DCONV_UPD_INT_FIELDS(X)
#undef X
#define X(f, n) put_arr(os, #f, L.p.f, n);
  DCONV_UPD_ARRAYS(X)
#undef X
  os << "end\n";
}

// ---------------------------------------------------------------- parsing
struct Reader {
  std::istringstream is;
  explicit Reader(const std::string& s) : is(s) {}
  // next non-empty line split into (name, values)
  bool next(std::string& name, std::vector<long long>& v, std::string* rest = nullptr) {
    std::string line;
    while (std::getline(is, line)) {
      if (line.empty()) continue;
      std::istringstream ls(line);
      ls >> name;
      v.clear();
      std::string tok;
      if (rest) rest->clear();
      while (ls >> tok) {
        char* end = nullptr;
        const long long x = std::strtoll(tok.c_str(), &end, 10);
        if (end == tok.c_str() || *end) {
          if (rest) {
            *rest = tok;
            continue;
          }
          fail(DCONV_ERR_PARSE, "plan: bad number '" + tok + "' in record '" + name + "'");
        }
        v.push_back(x);
      }
      return true;
    }
    return false;
  }
  std::vector<long long> expect(const char* name, size_t n) {
    std::string nm;
    std::vector<long long> v;
    if (!next(nm, v) || nm != name) fail(DCONV_ERR_PARSE, std::string("plan: expected record '") + name + "'");
    if (n && v.size() != n) fail(DCONV_ERR_PARSE, std::string("plan: record '") + name + "' has the wrong length");
    return v;
  }
  // a launch body: records up to "end"
  Rec body() {
    Rec r;
    std::string nm;
    std::vector<long long> v;
    while (next(nm, v)) {
      if (nm == "end") return r;
      r[nm] = v;
    }
    fail(DCONV_ERR_PARSE, "plan: truncated launch record");
  }
};

const std::vector<long long>& field(const Rec& r, const char* name, size_t n) {
  auto it = r.find(name);
  if (it == r.end()) fail(DCONV_ERR_PARSE, std::string("plan: launch misses '") + name + "'");
  if (it->second.size() != n) fail(DCONV_ERR_PARSE, std::string("plan: '") + name + "' has the wrong length");
  return it->second;
}

FwdLaunch load_fwd_launch(const Rec& r) {
  FwdLaunch L;
  std::memset(&L.p, 0, sizeof(L.p));
  const auto& g = field(r, "grid", 3);
  L.grid = dim3(static_cast<unsigned>(g[0]), static_cast<unsigned>(g[1]), static_cast<unsigned>(g[2]));
  const auto& rg = field(r, "rings", 3);
  L.stages = static_cast<int>(rg[0]);
  L.raw_stages = static_cast<int>(rg[1]);
  L.w_stages = static_cast<int>(rg[2]);
  const auto& sm = field(r, "smem", 3);
  L.smem = static_cast<size_t>(sm[0]);
  L.smem_launch = static_cast<size_t>(sm[1]);
  L.raw_slot = static_cast<size_t>(sm[2]);
  const auto& md = field(r, "mode", 3);
  L.raw_f32 = md[0] != 0;
  L.pieces = static_cast<int>(md[1]);
  L.ts = md[2] != 0;
#define X(f) L.p.f = static_cast<int>(field(r, #f, 1)[0]);
  DCONV_FWD_INT_FIELDS(X)
#undef X
#define X(f, n)                                               \
  {                                                           \
    const auto& a = field(r, #f, n);                          \
    for (int i = 0; i < n; ++i) L.p.f[i] = static_cast<int>(a[i]); \
  }
  DCONV_FWD_ARRAYS(X)
#undef X
  return L;
}

UpdLaunch load_upd_launch(const Rec& r) {
  UpdLaunch L;
  std::memset(&L.p, 0, sizeof(L.p));
  const auto& g = field(r, "grid", 3);
  L.grid = dim3(static_cast<unsigned>(g[0]), static_cast<unsigned>(g[1]), static_cast<unsigned>(g[2]));
  const auto& rg = field(r, "rings", 4);
  L.stages = static_cast<int>(rg[0]);
  L.raw_stages = static_cast<int>(rg[1]);
  L.pc_stages = static_cast<int>(rg[2]);
  L.passes = static_cast<int>(rg[3]);
  L.smem = static_cast<size_t>(field(r, "smem", 1)[0]);
  const auto& ws = field(r, "ws", 3);
  L.ws_in = static_cast<size_t>(ws[0]);
  L.ws_do = static_cast<size_t>(ws[1]);
  L.ws_partial = static_cast<size_t>(ws[2]);
  const auto& md = field(r, "mode", 5);
  L.split_in = md[0] != 0;
  L.split_do = md[1] != 0;
  L.raw = md[2] != 0;
  L.cat = md[3] != 0;
  L.tsa = md[4] != 0;
#define X(f) L.p.f = static_cast<int>(field(r, #f, 1)[0]);
  DCONV_UPD_INT_FIELDS(X)
#undef X
#define X(f, n)                                               \
  {                                                           \
    const auto& a = field(r, #f, n);                          \
    for (int i = 0; i < n; ++i) L.p.f[i] = static_cast<int>(a[i]); \
  }
  DCONV_UPD_ARRAYS(X)
#undef X
  return L;
}

// ---------------------------------------------------------------- header
void save_header(std::ostringstream& os, const char* kind, const dconv_spec_t& s, int math, bool has_cfg,
                 const dconv_engine_config_t& cfg) {
  os << "DCPL 1\n" << "kind " << kind << '\n';
  put(os, "spec", {s.N, s.C, s.K, s.H, s.W, s.R, s.S, s.stride, s.pad_h, s.pad_w, s.vlen});
  put(os, "math", {math});
  if (has_cfg)
    put(os, "cfg", {cfg.min_accumulators, cfg.max_accumulators, cfg.cache_budget_bytes, cfg.prefetch_lookahead,
                    cfg.prefetch_enabled, cfg.streaming_stores, cfg.acc_chain_limit, cfg.i16_bound_in,
                    cfg.i16_bound_wt, cfg.tile_mb, cfg.tile_nb, cfg.stages, cfg.upd_splits});
  else
    put(os, "cfg", {});
}

struct Header {
  dconv_spec_t spec;
  int math;
  bool has_cfg;
  dconv_engine_config_t cfg;
};

Header read_header(Reader& rd, const char* kind) {
  std::string nm, word;
  std::vector<long long> v;
  if (!rd.next(nm, v) || nm != "DCPL") fail(DCONV_ERR_PARSE, "load_plan: bad magic");
  if (v.size() != 1 || v[0] != 1) fail(DCONV_ERR_PARSE, "load_plan: unsupported version");
  if (!rd.next(nm, v, &word) || nm != "kind" || word != kind)
    fail(DCONV_ERR_PARSE, std::string("load_plan: not a ") + kind + " plan");
  Header h;
  const auto sp = rd.expect("spec", 11);
  h.spec = {static_cast<int>(sp[0]), static_cast<int>(sp[1]), static_cast<int>(sp[2]), static_cast<int>(sp[3]),
            static_cast<int>(sp[4]), static_cast<int>(sp[5]), static_cast<int>(sp[6]), static_cast<int>(sp[7]),
            static_cast<int>(sp[8]), static_cast<int>(sp[9]), static_cast<int>(sp[10])};
  h.math = static_cast<int>(rd.expect("math", 1)[0]);
  const auto c = rd.expect("cfg", 0);
  h.has_cfg = !c.empty();
  std::memset(&h.cfg, 0, sizeof(h.cfg));
  if (h.has_cfg) {
    if (c.size() != 13) fail(DCONV_ERR_PARSE, "load_plan: cfg record has the wrong length");
    h.cfg.cache_budget_bytes = c[2];
    int* f[12] = {&h.cfg.min_accumulators, &h.cfg.max_accumulators, &h.cfg.prefetch_lookahead,
                  &h.cfg.prefetch_enabled, &h.cfg.streaming_stores, &h.cfg.acc_chain_limit, &h.cfg.i16_bound_in,
                  &h.cfg.i16_bound_wt, &h.cfg.tile_mb, &h.cfg.tile_nb, &h.cfg.stages, &h.cfg.upd_splits};
    const int src[12] = {0, 1, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12};
    for (int i = 0; i < 12; ++i) *f[i] = static_cast<int>(c[src[i]]);
  }
  return h;
}

GeoKey read_key(const std::vector<long long>& v) {
  if (v.size() != 16) fail(DCONV_ERR_PARSE, "load_plan: entry key has the wrong length");
  GeoKey k;
  for (int i = 0; i < 16; ++i) k[i] = static_cast<int>(v[i]);
  return k;
}

// tensors of a cache key's geometry (for validating a loaded launch; never dereferenced)
void key_tensors(const GeoKey& k, dconv_act_t& a, dconv_act_t& b) {
  std::memset(&a, 0, sizeof(a));
  std::memset(&b, 0, sizeof(b));
  a.data = b.data = reinterpret_cast<void*>(256);
  a.n = k[0], a.c = k[1], a.h = k[2], a.w = k[3], a.halo_h = k[4], a.halo_w = k[5], a.dtype = k[6], a.vlen = 16;
  b.n = k[7], b.c = k[8], b.h = k[9], b.w = k[10], b.halo_h = k[11], b.halo_w = k[12], b.dtype = k[13], b.vlen = 16;
}

size_t emit(const std::string& text, char* buf, size_t len, size_t* needed) {
  if (needed) *needed = text.size() + 1;
  if (buf && len > text.size()) {
    std::memcpy(buf, text.data(), text.size() + 1);
    return text.size();
  }
  if (buf) fail(DCONV_ERR_INVALID_ARGUMENT, "plan save: buffer too small (" + std::to_string(text.size() + 1) + " bytes needed)");
  return 0;
}

}  // namespace

extern "C" {

int dconv_set_dev_mode(int on) {
  g_dev_mode = on != 0;
  return DCONV_OK;
}

// ---------------------------------------------------------------- forward
int dconv_fwd_plan_save(dconv_fwd_plan_t plan, char* buf, size_t len, size_t* needed) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    if (plan->inner) fail(DCONV_ERR_UNSUPPORTED, "plan save: vlen != 16 plans re-block around a vlen-16 twin");
    std::ostringstream os;
    save_header(os, "fwd", plan->spec, plan->math, plan->has_cfg, plan->cfg);
    put(os, "out_halo", {plan->out_halo_h, plan->out_halo_w});
    std::vector<float> bias;
    if (plan->bias_dev && (plan->fuse_kind == DCONV_FUSE_BIAS_ADD || plan->fuse_kind == DCONV_FUSE_BIAS_RELU)) {
      bias.resize(plan->spec.K);
      cuda_check(cudaMemcpy(bias.data(), plan->bias_dev, bias.size() * sizeof(float), cudaMemcpyDeviceToHost),
                 "bias read");
    }
    os << "fusion " << plan->fuse_kind << ' ' << bias.size();
    for (float f : bias) {
      uint32_t u;
      std::memcpy(&u, &f, 4);
      os << ' ' << u;  // exact bit patterns
    }
    os << '\n';
    std::lock_guard<std::mutex> lk(plan->mu);
    put(os, "entries", {static_cast<long long>(plan->cache.size())});
    for (auto& kv : plan->cache) {
      put_arr(os, "entry", kv.first.data(), 16);
      for (auto& L : kv.second.L) save_fwd_launch(os, L);
    }
    emit(os.str(), buf, len, needed);
  });
}

int dconv_fwd_plan_load(const char* text, size_t len, int validate, dconv_fwd_plan_t* out) {
  dconv_fwd_plan_t plan = nullptr;
  const int st = guarded([&] {
    if (!text || !out) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    Reader rd(std::string(text, strnlen(text, len)));
    const Header h = read_header(rd, "fwd");
    const auto oh = rd.expect("out_halo", 2);
    std::string nm;
    std::vector<long long> v;
    if (!rd.next(nm, v) || nm != "fusion" || v.size() < 2 || v.size() != 2 + static_cast<size_t>(v[1]))
      fail(DCONV_ERR_PARSE, "load_plan: bad fusion record");
    std::vector<float> bias(static_cast<size_t>(v[1]));
    for (size_t i = 0; i < bias.size(); ++i) {
      const uint32_t u = static_cast<uint32_t>(v[2 + i]);
      std::memcpy(&bias[i], &u, 4);
    }
    dconv_fusion_t fu = {static_cast<int>(v[0]), bias.empty() ? nullptr : bias.data(), static_cast<int>(bias.size())};
    const int rc = dconv_fwd_plan_create(&h.spec, fu.kind ? &fu : nullptr, h.has_cfg ? &h.cfg : nullptr, h.math,
                                         static_cast<int>(oh[0]), static_cast<int>(oh[1]), &plan);
    if (rc != DCONV_OK) fail(rc, g_err);
    const long long n = rd.expect("entries", 1)[0];
    for (long long i = 0; i < n; ++i) {
      const GeoKey key = read_key(rd.expect("entry", 16));
      std::string w;
      if (!rd.next(nm, v, &w) || nm != "launch" || w != "fwd") fail(DCONV_ERR_PARSE, "load_plan: expected a launch");
      FwdEntry e;
      e.L.push_back(load_fwd_launch(rd.body()));
      e.desc = json_tile(e.L[0]);
      plan->cache[key] = std::move(e);
      if (validate) {
        dconv_act_t a, b;
        key_tensors(key, a, b);
        const int vr = dconv_fwd_plan_validate(plan, &a, &b, nullptr, 0);
        if (vr != DCONV_OK) fail(vr, g_err);
      }
    }
    *out = plan;
  });
  if (st != DCONV_OK && plan) dconv_fwd_plan_destroy(plan);
  return st;
}

// ---------------------------------------------------------------- backward-data
int dconv_bwd_plan_save(dconv_bwd_plan_t plan, char* buf, size_t len, size_t* needed) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    if (plan->inner) fail(DCONV_ERR_UNSUPPORTED, "plan save: vlen != 16 plans re-block around a vlen-16 twin");
    std::ostringstream os;
    save_header(os, "bwd", plan->spec, plan->math, plan->has_cfg, plan->cfg);
    std::lock_guard<std::mutex> lk(plan->mu);
    put(os, "entries", {static_cast<long long>(plan->cache.size())});
    for (auto& kv : plan->cache) {
      put_arr(os, "entry", kv.first.data(), 16);
      put(os, "launches", {static_cast<long long>(kv.second.L.size())});
      for (auto& L : kv.second.L) save_fwd_launch(os, L);
    }
    emit(os.str(), buf, len, needed);
  });
}

int dconv_bwd_plan_load(const char* text, size_t len, int validate, dconv_bwd_plan_t* out) {
  dconv_bwd_plan_t plan = nullptr;
  const int st = guarded([&] {
    if (!text || !out) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    Reader rd(std::string(text, strnlen(text, len)));
    const Header h = read_header(rd, "bwd");
    const int rc = dconv_bwd_plan_create(&h.spec, h.has_cfg ? &h.cfg : nullptr, h.math, &plan);
    if (rc != DCONV_OK) fail(rc, g_err);
    const long long n = rd.expect("entries", 1)[0];
    std::string nm, w;
    std::vector<long long> v;
    for (long long i = 0; i < n; ++i) {
      const GeoKey key = read_key(rd.expect("entry", 16));
      const long long nl = rd.expect("launches", 1)[0];
      FwdEntry e;
      for (long long j = 0; j < nl; ++j) {
        if (!rd.next(nm, v, &w) || nm != "launch" || w != "fwd") fail(DCONV_ERR_PARSE, "load_plan: expected a launch");
        e.L.push_back(load_fwd_launch(rd.body()));
      }
      // descriptor JSON in the execute order of the phases
      const bool accumulate = key[14] != 0, fill = bwd_fill(plan, accumulate);
      e.desc = "{\"route\":" + std::to_string(plan->route) + ",\"phases\":[";
      size_t li = 0;
      for (size_t k = 0; k < plan->phases.size(); ++k) {
        if (k) e.desc += ",";
        if (plan->phases[k].zero)
          e.desc += accumulate ? "\"skip\"" : fill ? "\"filled\"" : "\"zero\"";
        else if (li < e.L.size())
          e.desc += json_tile(e.L[li++]);
      }
      e.desc += "]}";
      plan->cache[key] = std::move(e);
      if (validate) {
        if (accumulate) continue;  // validated as the plain (non-accumulating) surface below
        dconv_act_t a, b;
        key_tensors(key, a, b);
        const int vr = dconv_bwd_plan_validate(plan, &a, &b, nullptr, 0);
        if (vr != DCONV_OK) fail(vr, g_err);
      }
    }
    *out = plan;
  });
  if (st != DCONV_OK && plan) dconv_bwd_plan_destroy(plan);
  return st;
}

// ---------------------------------------------------------------- weight update
int dconv_upd_plan_save(dconv_upd_plan_t plan, char* buf, size_t len, size_t* needed) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    if (plan->inner) fail(DCONV_ERR_UNSUPPORTED, "plan save: vlen != 16 plans re-block around a vlen-16 twin");
    std::ostringstream os;
    save_header(os, "upd", plan->spec, plan->math, plan->has_cfg, plan->cfg);
    std::lock_guard<std::mutex> lk(plan->mu);
    put(os, "entries", {static_cast<long long>(plan->cache.size())});
    for (auto& kv : plan->cache) {
      put_arr(os, "entry", kv.first.data(), 16);
      save_upd_launch(os, kv.second->L);
    }
    emit(os.str(), buf, len, needed);
  });
}

int dconv_upd_plan_load(const char* text, size_t len, int validate, dconv_upd_plan_t* out) {
  dconv_upd_plan_t plan = nullptr;
  const int st = guarded([&] {
    if (!text || !out) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    Reader rd(std::string(text, strnlen(text, len)));
    const Header h = read_header(rd, "upd");
    const int rc = dconv_upd_plan_create(&h.spec, h.has_cfg ? &h.cfg : nullptr, h.math, &plan);
    if (rc != DCONV_OK) fail(rc, g_err);
    const long long n = rd.expect("entries", 1)[0];
    std::string nm, w;
    std::vector<long long> v;
    for (long long i = 0; i < n; ++i) {
      const GeoKey key = read_key(rd.expect("entry", 16));
      if (!rd.next(nm, v, &w) || nm != "launch" || w != "upd") fail(DCONV_ERR_PARSE, "load_plan: expected a launch");
      auto* e = new UpdEntry();
      e->L = load_upd_launch(rd.body());
      e->desc = json_upd(e->L, plan->pieces);
      auto it = plan->cache.find(key);
      if (it != plan->cache.end()) delete it->second;
      plan->cache[key] = e;
      if (validate) {
        dconv_act_t a, b;
        key_tensors(key, a, b);
        const int vr = dconv_upd_plan_validate(plan, &a, &b, nullptr, 0);
        if (vr != DCONV_OK) fail(vr, g_err);
      }
    }
    *out = plan;
  });
  if (st != DCONV_OK && plan) dconv_upd_plan_destroy(plan);
  return st;
}

}  // extern "C"
