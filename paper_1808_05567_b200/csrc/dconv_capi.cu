// dconv_b200 C ABI implementation: plans (tile selection in place of the
// reference's JIT / dryrun), TMA descriptor encoding, and launches of the
// sm_100a kernels in kernels/*.cuh. See include/dconv_b200.h.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <mutex>
#include <array>
#include <memory>

#include "../../include/dconv_b200.h"
#include "kernels/conv_fwd.cuh"
#include "kernels/conv_upd.cuh"
#include "kernels/layout.cuh"

using namespace dconv_sm100;

namespace {
// Experiment overrides (DCONV_* environment variables, read by the tile selectors
// of tools/*_sweep.py). They are inert unless developer mode is switched on with
// dconv_set_dev_mode(1): a stray variable cannot change a production plan. In
// developer mode the plan caches are bypassed (every execute re-plans, so a sweep
// can vary them between calls in one process) and malformed numbers are an error.
bool g_dev_mode = false;

const char* dev_env(const char* name) { return g_dev_mode ? std::getenv(name) : nullptr; }
#define DCONV_ENV(name) dev_env(name)


thread_local std::string g_err;

struct Fail {
  int code;
};

[[noreturn]] void fail(int code, const std::string& msg) {
  g_err = msg;
  throw Fail{code};
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(DCONV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// developer-mode integer override: `dflt` when unset, an error when malformed
int env_int(const char* name, int dflt) {
  const char* v = dev_env(name);
  if (!v) return dflt;
  char* end = nullptr;
  const long x = std::strtol(v, &end, 10);
  if (end == v || *end != 0 || x < -(1L << 30) || x > (1L << 30))
    fail(DCONV_ERR_INVALID_ARGUMENT, std::string(name) + ": not an integer: '" + v + "'");
  return static_cast<int>(x);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return DCONV_OK;
  } catch (const Fail& e) {
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DCONV_ERR_CUDA;
  }
}

int cdiv(int a, int b) { return (a + b - 1) / b; }
int64_t cdiv64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------ spec
// layer_spec.cpp:7-18
void validate_spec(const dconv_spec_t& s) {
  if (s.N < 1 || s.C < 1 || s.K < 1 || s.H < 1 || s.W < 1 || s.R < 1 || s.S < 1)
    fail(DCONV_ERR_INVALID_LAYER_SPEC, "all tensor extents must be >= 1");
  if (s.stride < 1) fail(DCONV_ERR_INVALID_LAYER_SPEC, "stride must be >= 1");
  if (s.pad_h < 0 || s.pad_w < 0) fail(DCONV_ERR_INVALID_LAYER_SPEC, "padding must be >= 0");
  if (s.vlen < 1) fail(DCONV_ERR_INVALID_LAYER_SPEC, "vlen must be >= 1");
  if (s.R > s.H + 2 * s.pad_h || s.S > s.W + 2 * s.pad_w)
    fail(DCONV_ERR_NON_INTEGRAL_SHAPE, "filter exceeds padded input: R=" + std::to_string(s.R) +
                                           " S=" + std::to_string(s.S) + " vs padded " +
                                           std::to_string(s.H + 2 * s.pad_h) + "x" + std::to_string(s.W + 2 * s.pad_w));
}
int out_P(const dconv_spec_t& s) { return (s.H + 2 * s.pad_h - s.R) / s.stride + 1; }
int out_Q(const dconv_spec_t& s) { return (s.W + 2 * s.pad_w - s.S) / s.stride + 1; }

int64_t act_elems(const dconv_act_t& a) {
  return static_cast<int64_t>(a.n) * cdiv(a.c, a.vlen) * (a.h + 2 * a.halo_h) * (a.w + 2 * a.halo_w) * a.vlen;
}
int64_t wt_elems(const dconv_wt_t& w) {
  return static_cast<int64_t>(cdiv(w.k, w.vlen)) * cdiv(w.c, w.vlen) * w.r * w.s * w.vlen * w.vlen;
}

void check_dtype(int dt) {
  if (dt != DCONV_F32 && dt != DCONV_BF16) fail(DCONV_ERR_INVALID_ARGUMENT, "dtype must be DCONV_F32 or DCONV_BF16");
}
void check_act(const dconv_act_t* a, const char* what) {
  if (!a || !a->data) fail(DCONV_ERR_INVALID_ARGUMENT, std::string(what) + ": null activation");
  check_dtype(a->dtype);
  if (a->n < 1 || a->c < 1 || a->h < 1 || a->w < 1 || a->vlen < 1 || a->halo_h < 0 || a->halo_w < 0)
    fail(DCONV_ERR_SHAPE_MISMATCH, std::string(what) + ": bad activation extents");
  if (reinterpret_cast<uintptr_t>(a->data) % 16 != 0)
    fail(DCONV_ERR_INVALID_ARGUMENT, std::string(what) + ": data must be 16-byte aligned");
}
void check_wt(const dconv_wt_t* w, const char* what) {
  if (!w || !w->data) fail(DCONV_ERR_INVALID_ARGUMENT, std::string(what) + ": null weight");
  check_dtype(w->dtype);
  if (w->k < 1 || w->c < 1 || w->r < 1 || w->s < 1 || w->vlen < 1)
    fail(DCONV_ERR_SHAPE_MISMATCH, std::string(what) + ": bad weight extents");
}

// ------------------------------------------------------------------ TMA encoding
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "cuTensorMapEncodeTiled");
    if (q != cudaDriverEntryPointSuccess || !p) fail(DCONV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

CUtensorMap encode(int bf16, int rank, const void* base, const uint64_t* dims, const uint64_t* strides_bytes,
                   const uint32_t* box, const uint32_t* estr, const char* what,
                   CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = estr ? estr[i] : 1;
    if (i + 1 < rank) st[i] = strides_bytes[i];
  }
  const CUresult r = encode_fn()(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                 rank, const_cast<void*>(base), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(DCONV_ERR_CUDA, std::string("tensor map encode failed (") + what + ") code " +
                                                  std::to_string(static_cast<int>(r)));
  return m;
}

// ------------------------------------------------------------------ profiling hook
// When enabled, CUDA events bracket the main conv kernel(s) of each pass on
// the launch stream; dconv_profile_last_ms() reads the last interval.
struct ProfSlot {
  cudaEvent_t start = nullptr, stop = nullptr;
  bool armed = false;
};
bool g_prof = false;
ProfSlot g_slot[3];  // 0 forward, 1 backward-data, 2 weight-update

void prof_begin(int which, cudaStream_t s) {
  if (!g_prof) return;
  ProfSlot& p = g_slot[which];
  if (!p.start) {
    cuda_check(cudaEventCreate(&p.start), "event");
    cuda_check(cudaEventCreate(&p.stop), "event");
  }
  cuda_check(cudaEventRecord(p.start, s), "event record");
}
void prof_end(int which, cudaStream_t s) {
  if (!g_prof) return;
  cuda_check(cudaEventRecord(g_slot[which].stop, s), "event record");
  g_slot[which].armed = true;
}

// SMs a persistent conv kernel may occupy: all of them, or dconv_set_sm_budget()'s
// cap (leaves SMs free for concurrently running collectives, e.g. NCCL's kernels)
int g_sm_budget = 0;

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
  }
  return g_sm_budget > 0 ? std::min(n, g_sm_budget) : n;
}

constexpr int kSmemBudget = 227 * 1024 - 2048;  // dynamic smem per CTA (static barriers excluded)
constexpr int kFwdBudget = kSmemBudget - static_cast<int>(kEpiStageBytes) - 1024;  // minus epilogue staging

int grid1d(int64_t total, int block = 256) {
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cdiv64(total, block), 148LL * 16)));
}

// ------------------------------------------------------------------ generic implicit-GEMM conv
// The forward kernel's problem: a stride-`stride` correlation of an input
// tensor with a phase-sorted tap list, written to an output surface.
struct ConvProblem {
  dconv_act_t in;  // input tensor (any halo)
  int cb_red;      // reduction blocks (= in channel blocks)
  int kb_out;      // output blocks
  int P, Q;        // output extents
  int R, S, stride;
  int row_off, col_off;  // logical input coordinate of output (0,0), tap (0,0) (= -pad)
};

struct Taps {
  int n_phases = 0;
  int phase_row[kMaxPhases] = {}, phase_col[kMaxPhases] = {};
  int phase_ntaps[kMaxPhases] = {}, phase_tap0[kMaxPhases] = {};
  std::vector<int> r, s;  // phase-sorted original taps
  std::vector<int> r2, s2;
  int r2max = 0, s2max = 0, taps_box = 0;
};

// phase (a, b) holds taps r = a + stride*r2, s = b + stride*s2
Taps phase_taps(int R, int S, int st) {
  Taps t;
  for (int a = 0; a < st; ++a)
    for (int b = 0; b < st; ++b) {
      std::vector<std::pair<int, int>> list;
      for (int r = a; r < R; r += st)
        for (int s = b; s < S; s += st) list.emplace_back(r, s);
      if (list.empty()) continue;
      if (t.n_phases >= kMaxPhases) fail(DCONV_ERR_UNSUPPORTED, "more than 16 stride phases (stride > 4)");
      const int ph = t.n_phases++;
      t.phase_row[ph] = a;
      t.phase_col[ph] = b;
      t.phase_tap0[ph] = static_cast<int>(t.r.size());
      t.phase_ntaps[ph] = static_cast<int>(list.size());
      t.taps_box = std::max(t.taps_box, static_cast<int>(list.size()));
      for (auto& rs : list) {
        t.r.push_back(rs.first);
        t.s.push_back(rs.second);
        t.r2.push_back(rs.first / st);
        t.s2.push_back(rs.second / st);
        t.r2max = std::max(t.r2max, rs.first / st);
        t.s2max = std::max(t.s2max, rs.second / st);
      }
    }
  if (static_cast<int>(t.r.size()) > kMaxTaps) fail(DCONV_ERR_UNSUPPORTED, "more than 128 filter taps");
  return t;
}

struct FwdTile {
  int mb = 1, nb = 1, stages = 2;
};

struct FwdLaunch {
  FwdParams p;
  CUtensorMap map_a;
  dim3 grid;
  int stages;      // piece-ring depth
  int raw_stages;  // raw-ring depth (fp32 activations)
  int w_stages;    // weight-ring depth
  size_t smem;
  bool raw_f32;
  int pieces;
  bool ts = false;  // A pieces staged in tensor memory (single-tap fp32 problems)
  size_t raw_slot = 0;  // bytes per raw-ring slot
  // resolved by finalize_fwd() for a given output surface (epilogue staging)
  CUtensorMap map_out, map_out2;
  size_t smem_launch = 0;  // dynamic smem of the launch (rings + epilogue staging)
};

// Decide staging mode, tile and pipeline depth; encode TMA maps.
FwdLaunch plan_fwd_launch(const ConvProblem& pb, const Taps& taps, const void* wprep, int pieces,
                          const dconv_engine_config_t* cfg) {
  FwdLaunch L;
  std::memset(&L.p, 0, sizeof(L.p));
  FwdParams& p = L.p;
  const dconv_act_t& in = pb.in;
  const bool raw_f32 = in.dtype == DCONV_F32;
  if (!raw_f32 && pieces == 3)
    fail(DCONV_ERR_UNSUPPORTED, "fp32-accurate math needs fp32 activations (got bf16)");
  L.raw_f32 = raw_f32;
  L.pieces = pieces;
  const int st = pb.stride;
  const int wp = in.w + 2 * in.halo_w;
  p.n_img = in.n;
  p.in_cb = cdiv(in.c, 16);
  p.cb_in = pb.cb_red;
  p.kb_out = pb.kb_out;
  p.P = pb.P;
  p.Q = pb.Q;
  p.stride = st;
  p.n_phases = taps.n_phases;
  for (int i = 0; i < taps.n_phases; ++i) {
    p.phase_row[i] = taps.phase_row[i];
    p.phase_col[i] = taps.phase_col[i];
    p.phase_ntaps[i] = taps.phase_ntaps[i];
    p.phase_tap0[i] = taps.phase_tap0[i];
  }
  p.taps_box = taps.taps_box;
  // fp32-accurate: the tensor core rounds the fp32 accumulator per MMA, so long
  // reductions keep hi*hi apart from the five correction products (Table I
  // layer 18, 4608-long, reached 1.27e-4 with one accumulator); reductions of
  // <= 1024 (<= 384 accumulation steps) stay well inside the gate with one
  const int red_len = pb.cb_red * 16 * static_cast<int>(taps.r.size());
  p.split_acc = (pieces == 3 && red_len > 1024) ? 1 : 0;
  const int n_acc = (pieces == 3 && p.split_acc) ? 2 : 1;
  // linear mode: the halo'd physical plane is the virtual grid
  // (and every shifted tap stays inside the halo'd plane: a stride phase of the
  // backward route can have more output rows / columns than its input supplies)
  const bool linear = st == 1 && -pb.row_off == in.halo_h && -pb.col_off == in.halo_w &&
                      pb.P + taps.r2max <= in.h + 2 * in.halo_h && pb.Q + taps.s2max <= in.w + 2 * in.halo_w;
  p.linear = linear ? 1 : 0;
  // multi-image tiles: 1x1 stride-1 on halo-free planes of <= 128 pixels
  const int hw = in.h * in.w;
  const bool mimg_ok = linear && pb.R == 1 && pb.S == 1 && in.halo_h == 0 && in.halo_w == 0 && hw <= 128 &&
                       (cfg == nullptr || cfg->tile_mb == 0 || cfg->tile_mb == 2);
  p.wsub = linear ? wp : pb.Q + taps.s2max;
  // packed multi-tap tiles (FwdParams::img_pitch): small stride-1 same-padded images of a
  // bf16 rows plan, three 7x7 images per 256-row tile (57 % of the MMA rows real
  // pixels instead of 38 % for one image per 128-row tile)
  // bf16 planes of <= 64 pixels (7x7, 8x8) also as 128-row tiles of two images x 256 output
  // channels with double-buffered accumulators: the 256-row tile leaves TMEM room for only
  // 128 channels per tile, whose N = 128 MMAs are issue bound (~107 cycles for a 64-cycle
  // MMA) and whose activations are re-read by twice as many channel tiles; measured 13-25 %
  // faster on the 7x7 / 8x8 1x1 layers although only 98 of 128 MMA rows are pixels at 7x7
  const bool mimg_mb1 = !raw_f32 && hw <= 64 && !DCONV_ENV("DCONV_NO_MIMG_MB1");
  const int pk_pitch = (in.h + (-pb.row_off)) * (pb.Q + taps.s2max);
  const bool pk_ok = !raw_f32 && !linear && st == 1 && taps.n_phases == 1 && in.halo_h == 0 && in.halo_w == 0 &&
                     pb.P == in.h && pb.Q == in.w && pb.row_off <= 0 && pb.col_off <= 0 &&
                     pb.R - 1 + pb.row_off <= -pb.row_off && pb.S - 1 + pb.col_off <= -pb.col_off &&
                     -pb.col_off * 2 == taps.s2max && pk_pitch % 8 == 0 && 2 * pk_pitch <= 256 &&
                     in.h - pb.row_off <= 256 && pb.Q + taps.s2max <= 256 && !(cfg && cfg->tile_mb) &&
                     !DCONV_ENV("DCONV_FWD_NO_PK");
  p.in_row0 = pb.row_off;
  p.in_col0 = pb.col_off;
  for (size_t t = 0; t < taps.r.size(); ++t) p.tap_shift[t] = taps.r2[t] * p.wsub + taps.s2[t];
  const int maxshift = taps.r2max * p.wsub + taps.s2max;

  FwdTile tile;
  const int kb_total = pb.kb_out;
  const int want_mb = (cfg && cfg->tile_mb > 0) ? cfg->tile_mb : env_int("DCONV_FWD_MB", 0);
  const int want_nb = (cfg && cfg->tile_nb > 0) ? std::min(cfg->tile_nb, 16)
                     : std::min(env_int("DCONV_FWD_NB", 0), 16);
  int a_px = 0, lin_boxes = 0, pc_st = 0, raw_st = 0, w_st = 0, acc_bufs = 2;
  bool w_all = false;
  FwdSmem layout;
  bool found = false;
  // widest N tile first (fewer activation re-reads), then the largest M tile;
  // two TMEM accumulators of mb*16*nb columns must fit in 512. Weight stages
  // hold up to w_taps taps (big filters stream taps through several stages).
  int w_taps = taps.taps_box;
  // TS: single-tap problems on fp32 activations stage the A pieces in TMEM
  // (mb = 1; accumulators + a ring of pieces*8 columns per stage <= 512)
  L.ts = raw_f32 && taps.r.size() == 1 && !(cfg && (cfg->tile_mb == 2 || cfg->stages < 0));
  int kc = 1;
  p.w_resident = 0;
  if (L.ts) {
    const int ring = pieces * 8;
    for (int want_bufs : {2, 1}) {
      for (int n_nt = cdiv(kb_total, 16); !found; ++n_nt) {
        const int nb = want_nb ? want_nb : cdiv(kb_total, n_nt);
        const int acc_cols = n_acc * 16 * nb;
        const int left = 512 - want_bufs * acc_cols;
        // channel blocks per stage: amortise the per-stage barrier / issue cost
        int kcx = std::min(4, pb.cb_red);
        while (kcx > 1 && (left <= 0 || left / (ring * kcx) < 2)) kcx >>= 1;
        const int ring_st = left > 0 ? std::min(kMaxStages, left / (ring * kcx)) : 0;
        if (left > 0 && ring_st >= 2) {
          const int apx = 128;
          const int lb = (linear && !mimg_ok) ? 1 : 0;
          if (!linear) {
            const int rows_box = (p.wsub + 128 - 2) / p.wsub + 1;
            if (p.wsub * st > 256 || rows_box * st > 256) break;
          }
          const int apx_rows = linear ? apx : ((p.wsub + 128 - 2) / p.wsub + 1) * p.wsub;
          // resident weight slice: every CTA keeps one output-channel tile for the
          // whole launch (grid % n_ntiles == 0) and the slice fits beside the raw ring
          const int n_nt_tiles = cdiv(kb_total, nb);
          const int m_tiles = mimg_ok ? cdiv(in.n, 128 / hw) : in.n * cdiv(pb.P * p.wsub, 128);
          const int grid_est = std::min(m_tiles * n_nt_tiles, sm_count());
          const int res_bytes = pb.cb_red * pieces * nb * 512;
          const bool resident = grid_est % n_nt_tiles == 0 && res_bytes <= 120 * 1024 &&
                                cdiv(pb.cb_red, kcx) <= kMaxStages && !DCONV_ENV("DCONV_NO_RESIDENT");
          const FwdSmem lay = fwd_smem_layout(apx_rows * kcx, resident ? pb.cb_red : kcx, nb, pieces, true, 0, 1);
          int wss = resident ? 1
                             : std::max(2, std::min<int>(kMaxStages, (kFwdBudget / 4) / static_cast<int>(lay.w_slot)));
          // keep room for the TMA-store staging of dense outputs
          const int left_s = kFwdBudget - static_cast<int>(kEpiStagingBytes) - wss * static_cast<int>(lay.w_slot);
          int rws = left_s > 0 ? std::min<int>(kMaxStages, left_s / static_cast<int>(lay.raw_slot)) : 0;
          if (cfg && cfg->stages > 0) rws = std::max(1, std::min(cfg->stages, rws));
          if (rws >= 2) {
            tile.mb = 1;
            tile.nb = nb;
            acc_bufs = want_bufs;
            pc_st = ring_st;
            raw_st = rws;
            w_st = wss;
            w_taps = 1;
            kc = kcx;
            p.w_resident = resident ? 1 : 0;
            layout = fwd_smem_layout(apx_rows * kc, resident ? pb.cb_red : kc, nb, pieces, true, 0, w_st);
            a_px = apx_rows;
            lin_boxes = lb;
            found = true;
          }
        }
        if (want_nb || nb == 1) break;
      }
      if (found) break;
    }
    if (!found) L.ts = false;
  }
  // small grids (bf16 plans of small batches: e.g. 14x14 layers at 32 images): the
  // persistent kernel's time is one CTA's serial K loop, so when the widest tiles
  // leave SMs idle the N tile narrows (down to 64 channels) and 256-row tiles are
  // skipped until the tiles fill the grid
  auto est_tiles = [&](int mb, int n_nt) {
    const int m_t = mimg_ok ? cdiv(in.n, std::max(1, (128 * mb) / hw)) : in.n * cdiv(pb.P * p.wsub, 128 * mb);
    return m_t * n_nt;
  };
  // (measured: narrower N tiles do not pay -- the N = 128 MMAs are issue-bound -- so only
  // developer mode enables it: DCONV_SHAPE_GRID=1)
  const bool shape_grid = !raw_f32 && !want_nb && !want_mb && DCONV_ENV("DCONV_SHAPE_GRID");
  const bool pk = pk_ok && !want_mb;  // (an explicit m-tile override keeps row tiles)
  int n_nt0 = cdiv(kb_total, 16);
  if (shape_grid)
    while (est_tiles(1, n_nt0) < sm_count() && cdiv(kb_total, n_nt0 + 1) >= 4 && cdiv(kb_total, n_nt0 + 1) < cdiv(kb_total, n_nt0))
      ++n_nt0;
  for (int tier = 0; tier < 6 && !found; ++tier) {
    const int want_pc = tier < 2 ? 3 : tier < 4 ? 2 : 1;
    const int want_bufs = (tier % 2 == 0) ? 2 : 1;
    for (int n_nt = n_nt0; !found; ++n_nt) {
      const int nb = want_nb ? want_nb : cdiv(kb_total, n_nt);
      for (int mb : {4, 2, 1}) {
        if (want_mb && mb != want_mb) continue;
        if (mb == 4 && !want_mb) continue;  // 512-row tiles: explicit override only (DCONV_FWD_MB / tile_mb)
        if (shape_grid && mb == 2 && est_tiles(2, n_nt) < sm_count() && !mimg_ok) continue;
        // accumulators: (pieces == 3 ? 2 : 1) x mb x 16nb columns, double-buffered when they fit
        const int acc_cols = n_acc * mb * 16 * nb;
        if (acc_cols > 512) continue;
        const int bufs = 2 * acc_cols <= 512 ? 2 : 1;
        if (bufs == 1 && mb > 1 && !want_mb) continue;
        if (bufs < want_bufs) continue;
        if (pk && mb == 1 && nb > 8) continue;  // packed tiles first: 256 rows x (N <= 128, two buffers)
        const int Lpx = 128 * mb;
        int apx, lb = 0;
        if (pk && mb == 2) {  // (pki + 1) images per chunk plane; reads reach Lpx + maxshift rows
          const int pki = Lpx / pk_pitch;
          apx = (pki + 1) * pk_pitch;
          if (apx < Lpx + maxshift) continue;  // the box must cover every row the MMA reads
        } else if (mimg_ok) {
          if (mb != 2 && !(mb == 1 && mimg_mb1)) continue;
          apx = Lpx;
        } else if (linear) {
          lb = cdiv(Lpx + maxshift, 128);
          apx = lb * 128;
        } else {
          const int rows_box = (p.wsub + Lpx - 2 + maxshift) / p.wsub + 1;
          if (p.wsub * st > 256 || rows_box * st > 256) continue;
          apx = rows_box * p.wsub;
        }
        // weight stage <= 32 KB (fp32 activations) / 80 KB (bf16: every tap of a (c_b,
        // phase) in one stage for nb <= 16 -- fewer per-stage barriers and MMA-issue
        // restarts; measured 1.2-1.5x on the 3x3 bf16 layers)
        int wt = taps.taps_box;
        const int w_cap = env_int("DCONV_WCAP", raw_f32 ? 32 : 80) * 1024;
        while (wt > 1 && static_cast<int>(fwd_smem_layout(apx, wt, nb, pieces, raw_f32, 1, 1).w_slot) > w_cap)
          wt = (wt + 1) / 2;
        const FwdSmem lay = fwd_smem_layout(apx, wt, nb, pieces, raw_f32, 1, 1);
        int pcs, rws = 0, wss;
        // weight ring: enough slots to cover L2 latency, bounded to ~1/4 of smem
        wss = std::max(2, std::min<int>(kMaxStages, (kFwdBudget / 4) / static_cast<int>(lay.w_slot)));
        if (raw_f32) {
          pcs = want_pc;
          int left = kFwdBudget - pcs * static_cast<int>(lay.pc_slot) - wss * static_cast<int>(lay.w_slot);
          rws = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lay.raw_slot)) : 0;
          if (rws < 3 && wss > 2) {  // give raw slots priority over weight depth
            wss = 2;
            left = kFwdBudget - pcs * static_cast<int>(lay.pc_slot) - wss * static_cast<int>(lay.w_slot);
            rws = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lay.raw_slot)) : 0;
          }
          if (rws < (want_pc == 1 ? 1 : 2)) continue;
        } else {
          // single-tap bf16 problems carry kc channel blocks per stage (amortises the
          // per-stage barrier / commit cost over kc x mb MMAs)
          int kcx = (taps.r.size() == 1) ? std::min(env_int("DCONV_FWD_KC", 4), pb.cb_red)
                                         : (linear && apx > 256) ? 1  // one TMA box per block: <= 256 rows
                                         : (pb.cb_red % 2 != 0)  ? 1  // whole stages only (the multi-tap issuer)
                                                                 : std::min(env_int("DCONV_FWD_KC", 2), pb.cb_red);
          // multi-tap outputs are never dense (wsub > Q): no TMA-store staging to reserve
          const int stg_res = (taps.r.size() == 1 || DCONV_ENV("DCONV_STG_RES")) ? 3 * 16384 : 0;
          pcs = 0;
          for (; kcx >= 1; kcx = kcx > 1 ? kcx / 2 : 0) {
            const FwdSmem lk = fwd_smem_layout(apx * kcx, wt * kcx, nb, pieces, raw_f32, 1, 1);
            int wsk = std::max(2, std::min<int>(kMaxStages, (kFwdBudget / 4) / static_cast<int>(lk.w_slot)));
            // room for three epilogue groups' TMA-store staging (bf16 slabs: 3 x 16 KB)
            int left = kFwdBudget - stg_res - wsk * static_cast<int>(lk.w_slot);
            pcs = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lk.pc_slot)) : 0;
            // single-tap stages: a third weight slot when four activation slots still fit
            // (a 32 KB weight stage takes ~1.9 k cycles from L2; measured 3-9 % on 14x14 1x1s)
            if (taps.r.size() == 1 && wsk == 2 && kcx > 1) {
              const int left3 = kFwdBudget - stg_res - 3 * static_cast<int>(lk.w_slot);
              if (left3 >= 4 * static_cast<int>(lk.pc_slot)) {
                wsk = 3;
                pcs = std::min<int>(kMaxStages, left3 / static_cast<int>(lk.pc_slot));
              }
            }
            if (pcs < want_pc && wsk > 2) {
              wsk = 2;
              left = kFwdBudget - stg_res - wsk * static_cast<int>(lk.w_slot);
              pcs = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lk.pc_slot)) : 0;
            }
            if (kcx == 1 && pcs < want_pc) {  // no room for the TMA-store staging: plain budget
              wsk = std::max(2, std::min<int>(kMaxStages, (kFwdBudget / 4) / static_cast<int>(lk.w_slot)));
              left = kFwdBudget - wsk * static_cast<int>(lk.w_slot);
              pcs = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lk.pc_slot)) : 0;
              if (pcs < want_pc && wsk > 2) {
                wsk = 2;
                left = kFwdBudget - wsk * static_cast<int>(lk.w_slot);
                pcs = left > 0 ? std::min<int>(kMaxStages, left / static_cast<int>(lk.pc_slot)) : 0;
              }
            }
            if (pcs >= want_pc) {
              wss = wsk;
              kc = kcx;
              break;
            }
          }
          if (DCONV_ENV("DCONV_WST")) {  // debug: weight-ring depth sweep
            const FwdSmem lk = fwd_smem_layout(apx * kc, wt * kc, nb, pieces, raw_f32, 1, 1);
            wss = std::max(1, std::min(kMaxStages, env_int("DCONV_WST", 2)));
            pcs = std::min<int>(kMaxStages, (kFwdBudget - stg_res - wss * static_cast<int>(lk.w_slot)) /
                                                static_cast<int>(lk.pc_slot));
          }
          if (pcs < want_pc) continue;
          if (kc > 1 && linear && !mimg_ok) lb = 1;  // one box of Lpx pixels x kc blocks
          // one output-channel tile and every tap of a channel-block group in one stage:
          // when all the stages' weights fit, each gets its own slot, loaded once per CTA
          // (the stem, the 56x56 3x3 and 1x1 layers re-streamed them for every tile)
          w_all = false;
          // ... also with several output-channel tiles when every CTA keeps ONE of them for
          // the whole launch (persistent striding by a multiple of the n-tile count): the
          // 1x1 layers with K > 256 then stream only activations, not the weights per tile
          const int n_nt_tiles = cdiv(kb_total, nb);
          const int m_tiles_e = mimg_ok ? cdiv(in.n, std::max(1, (128 * mb) / hw)) : in.n * cdiv(pb.P * p.wsub, 128 * mb);
          const bool fixed_nt = nb >= kb_total || std::min(m_tiles_e * n_nt_tiles, sm_count()) % n_nt_tiles == 0;
          if (fixed_nt && taps.n_phases == 1 && wt == taps.taps_box && !DCONV_ENV("DCONV_NO_WALL")) {
            const int kst = cdiv(pb.cb_red, kc);
            const FwdSmem lk = fwd_smem_layout(apx * kc, wt * kc, nb, pieces, raw_f32, 1, 1);
            const int w_bytes = kst * static_cast<int>(lk.w_slot);
            const int pcs2 = kst <= kMaxStages && w_bytes <= env_int("DCONV_WALL_KB", 160) * 1024
                                 ? std::min<int>(kMaxStages, (kFwdBudget - stg_res - w_bytes) / static_cast<int>(lk.pc_slot))
                                 : 0;
            if (pcs2 >= 2) {
              wss = kst;
              pcs = pcs2;
              w_all = true;
            }
          }
        }
        tile.mb = mb;
        tile.nb = nb;
        acc_bufs = bufs;
        pc_st = pcs;
        raw_st = rws;
        w_st = wss;
        w_taps = wt;
        if (cfg && cfg->stages > 0) {
          if (raw_f32)
            raw_st = std::max(1, std::min(cfg->stages, raw_st));
          else
            pc_st = std::max(1, std::min(cfg->stages, pc_st));
        }
        layout = fwd_smem_layout(apx * kc, wt * kc, nb, pieces, raw_f32, pc_st, w_st);
        a_px = apx;
        lin_boxes = lb;
        found = true;
        break;
      }
      if (want_nb || nb == 1) break;
    }
  }
  if (!found) fail(DCONV_ERR_PLAN_INFEASIBLE, "no forward tile fits shared memory / TMA box limits");
  p.mb = tile.mb;
  p.nb = tile.nb;
  p.kc = kc;
  // w_all is consumed only by the single-lane bf16 MMA loop (conv_fwd.cuh): same conditions
  p.w_all = (w_all && (tile.mb == 1 || tile.mb == 2 || tile.mb == 4) && static_cast<int>(taps.r.size()) <= kFastTaps) ? 1 : 0;
  p.acc_bufs = acc_bufs;
  p.a_px = a_px;
  p.a_load_px = a_px;
  p.lin_boxes = lin_boxes;
  p.tiles_per_img = cdiv(pb.P * p.wsub, 128 * tile.mb);
  p.mimg = 0;
  p.img_pitch = 0;
  if (pk && tile.mb == 2) {
    p.mimg = (128 * tile.mb) / pk_pitch;
    p.img_pitch = pk_pitch;
    p.a_load_px = (p.mimg + 1) * pk_pitch;
  } else if (mimg_ok && (tile.mb == 2 || L.ts || (tile.mb == 1 && mimg_mb1))) {
    p.mimg = (128 * tile.mb) / hw;
    p.a_load_px = p.mimg * hw;
  }
  L.stages = pc_st;
  L.raw_stages = raw_st;
  L.w_stages = w_st;
  L.smem = static_cast<size_t>(layout.raw_off) + static_cast<size_t>(raw_st) * layout.raw_slot + kEpiStageBytes;
  L.raw_slot = layout.raw_slot;
  const int n_tiles = (p.mimg > 0 ? cdiv(in.n, p.mimg) : in.n * p.tiles_per_img) * cdiv(kb_total, tile.nb);
  L.grid = dim3(static_cast<unsigned>(std::min(n_tiles, sm_count())), 1, 1);

  p.n_taps = static_cast<int>(taps.r.size());
  p.w_taps = w_taps;
  p.n_ntiles = cdiv(kb_total, tile.nb);
  p.wprep = wprep;
  return L;
}

// activation tensor map of a resolved forward launch for input `in`
// (fp32 as 64 B pixel rows, SWIZZLE_64B, converted to pieces on chip; bf16 as
// 32 B pixel rows, SWIZZLE_32B, read in place by the MMA)
void encode_fwd_act_map(FwdLaunch& L, const dconv_act_t& in) {
  const FwdParams& p = L.p;
  const bool raw_f32 = L.raw_f32;
  const int st = p.stride, kc = p.kc, a_px = p.a_px;
  const int hp = in.h + 2 * in.halo_h, wp = in.w + 2 * in.halo_w;
  const int hw = in.h * in.w;
  const uint64_t planes = static_cast<uint64_t>(in.n) * p.in_cb;
  const uint64_t pix = raw_f32 ? 64 : 32;
  const CUtensorMapSwizzle swz = raw_f32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  if (p.img_pitch > 0) {  // packed multi-tap: {16, w, h, images, channel blocks}, images inside the planes
    const uint64_t plane_b = static_cast<uint64_t>(wp) * hp * pix;
    const uint64_t dims[5] = {16, static_cast<uint64_t>(in.w), static_cast<uint64_t>(in.h),
                              static_cast<uint64_t>(in.n), static_cast<uint64_t>(p.in_cb)};
    const uint64_t strides[4] = {pix, pix * wp, plane_b * p.in_cb, plane_b};
    const uint32_t box[5] = {16, static_cast<uint32_t>(p.wsub), static_cast<uint32_t>(p.img_pitch / p.wsub),
                             static_cast<uint32_t>(p.mimg + 1), static_cast<uint32_t>(kc)};
    L.map_a = encode(!raw_f32, 5, in.data, dims, strides, box, nullptr, "activation packed images", swz);
  } else if (p.mimg > 0) {
    const uint64_t dims[4] = {16, static_cast<uint64_t>(hw), static_cast<uint64_t>(p.in_cb),
                              static_cast<uint64_t>(in.n)};
    const uint64_t strides[3] = {pix, pix * hw, pix * hw * p.in_cb};
    // TS converters read any row order: one box of kc blocks; the smem-MMA path needs
    // each block's rows contiguous, so it issues one box per block
    const uint32_t box[4] = {16, static_cast<uint32_t>(hw), static_cast<uint32_t>(L.ts ? kc : 1),
                             static_cast<uint32_t>(p.mimg)};
    L.map_a = encode(!raw_f32, 4, in.data, dims, strides, box, nullptr, "activation multi-image", swz);
  } else if (p.linear && p.a_sw128) {  // 128 B rows of four pixels, SWIZZLE_128B (read back through SW32 descriptors)
    if (raw_f32 || (static_cast<uint64_t>(hp) * wp) % 4 != 0 || a_px % 32 != 0)
      fail(DCONV_ERR_INVALID_DESCRIPTOR, "a_sw128 plan on a plane that is not a multiple of four pixels");
    const uint64_t dims[3] = {64, static_cast<uint64_t>(hp) * wp / 4, planes};
    const uint64_t strides[2] = {128, pix * hp * wp};
    const uint32_t box[3] = {64, static_cast<uint32_t>((kc > 1 ? a_px : 128) / 4), static_cast<uint32_t>(kc)};
    L.map_a = encode(1, 3, in.data, dims, strides, box, nullptr, "activation linear sw128", CU_TENSOR_MAP_SWIZZLE_128B);
  } else if (p.linear) {
    const uint64_t dims[3] = {16, static_cast<uint64_t>(hp) * wp, planes};
    const uint64_t strides[2] = {pix, pix * hp * wp};
    const uint32_t box[3] = {16, static_cast<uint32_t>(kc > 1 ? a_px : 128), static_cast<uint32_t>(kc)};
    L.map_a = encode(!raw_f32, 3, in.data, dims, strides, box, nullptr, "activation linear", swz);
  } else {
    const char* base = reinterpret_cast<const char*>(in.data) + (static_cast<uint64_t>(in.halo_h) * wp + in.halo_w) * pix;
    const uint64_t dims[4] = {16, static_cast<uint64_t>(in.w), static_cast<uint64_t>(in.h), planes};
    const uint64_t strides[3] = {pix, pix * wp, pix * wp * hp};
    const uint32_t box[4] = {16, static_cast<uint32_t>(p.wsub * st), static_cast<uint32_t>((a_px / p.wsub) * st),
                             static_cast<uint32_t>(kc)};
    const uint32_t estr[4] = {1, static_cast<uint32_t>(st), static_cast<uint32_t>(st), 1};
    L.map_a = encode(!raw_f32, 4, base, dims, strides, box, estr, "activation rows", swz);
  }
}

long long* g_fwd_dbg = nullptr;  // dconv_debug_counters(): per-CTA role cycle counters
int g_fwd_dbg_mode = 0;

// Epilogue decisions of a forward launch for its output surface (p.out_* set):
// dense outputs (no halo / lattice / padding columns / multi-image rows) stage
// 32-pixel slabs in smem and TMA-store them. Resolved once per cached launch.
void finalize_fwd(FwdLaunch& L) {
  FwdParams& p = L.p;
  p.dbg = g_fwd_dbg;
  p.dbg_mode = g_fwd_dbg_mode;
  const int esz = p.out_bf16 ? 2 : 4;
  // 4 warps x 2 slabs of {16 lanes, 32 px, 2 blocks} per epilogue group; bf16
  // smem-staged plans run three groups
  // TS plans with one stage per tile: a second epilogue group (the stores dominate)
  const int kiters = cdiv(p.cb_in, p.kc) * p.n_phases;
  p.ts_epi2 = (L.ts && kiters == 1 && p.nb >= 4 && !DCONV_ENV("DCONV_NO_TS_EPI2")) ? 1 : 0;
  p.epi_groups = env_int("DCONV_EPI_GROUPS", 3);
  auto staging_bytes = [&] {
    return static_cast<size_t>((!L.raw_f32 && !L.ts) ? 3 : p.ts_epi2 ? 2 : 1) * 4 * 2 * (2 * 32 * 16 * esz);
  };
  // its staging comes out of the raw ring when needed (these plans load 1/4 of what they store)
  while (p.ts_epi2 && L.smem + staging_bytes() > static_cast<size_t>(kSmemBudget) && L.raw_stages > 3) {
    --L.raw_stages;
    L.smem -= L.raw_slot;
  }
  if (L.smem + staging_bytes() > static_cast<size_t>(kSmemBudget)) p.ts_epi2 = 0;
  const size_t staging = staging_bytes();
  L.smem_launch = L.smem;
  p.tma_store = 0;
  if (p.mimg == 0 && p.out_halo_h == 0 && p.out_halo_w == 0 && p.out_scale == 1 && p.out_y0 == 0 &&
      p.out_x0 == 0 && p.out_hp == p.P && p.out_wp == p.Q && p.wsub == p.Q && !(p.dbg_mode & 1) &&
      !DCONV_ENV("DCONV_NO_TMA_STORE") &&
      L.smem + staging <= static_cast<size_t>(kSmemBudget)) {
    p.tma_store = 1;
    L.smem_launch = L.smem + staging;
  }
  // bf16 linear single-tap plans (1x1, stride 1, dense planes of 4k pixels): 128 B activation rows
  p.a_sw128 = (p.tma_store && !L.raw_f32 && !L.ts && p.linear && p.mimg == 0 && p.img_pitch == 0 && p.n_taps == 1 &&
               p.n_phases == 1 && p.tap_shift[0] == 0 && p.stride == 1 && p.in_row0 == 0 && p.in_col0 == 0 &&
               (p.P * p.Q) % 4 == 0 && p.a_px % 32 == 0 && !DCONV_ENV("DCONV_NO_A_SW128"))
                  ? 1
                  : 0;
}

// output slab maps of a TMA-store launch (p.out set)
void encode_fwd_out_maps(FwdLaunch& L) {
  std::memset(&L.map_out, 0, sizeof(L.map_out));
  std::memset(&L.map_out2, 0, sizeof(L.map_out2));
  const FwdParams& p = L.p;
  if (!p.tma_store) return;
  const int esz = p.out_bf16 ? 2 : 4;
  const uint64_t pq = static_cast<uint64_t>(p.P) * p.Q;
  const uint64_t dims[4] = {16, pq, static_cast<uint64_t>(p.out_cb), static_cast<uint64_t>(p.n_img)};
  const uint64_t strides[3] = {16ull * esz, pq * 16 * esz, pq * 16 * esz * p.out_cb};
  const uint32_t box[4] = {16, 32, 1, 1};
  L.map_out = encode(p.out_bf16, 4, p.out, dims, strides, box, nullptr, "output slab",
                     p.out_bf16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B);
  const uint32_t box2[4] = {16, 32, 2, 1};
  L.map_out2 = encode(p.out_bf16, 4, p.out, dims, strides, box2, nullptr, "output slab pair",
                      p.out_bf16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize, raised once per kernel (not per launch)
std::mutex g_attr_mu;
std::map<const void*, int> g_attr_smem;
template <class K>
void ensure_smem(K kern, size_t smem) {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  int& cur = g_attr_smem[reinterpret_cast<const void*>(kern)];
  if (cur >= static_cast<int>(smem)) return;
  cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
             "smem attribute");
  cur = static_cast<int>(smem);
}

// Launch a resolved forward launch (maps encoded, pointers patched).
// pdl: programmatic dependent launch -- only when the weight prep was launched
// on this stream immediately before (its weight producer waits on
// griddepcontrol.wait; every other role reads data the prep's predecessors wrote).
// prof_slot >= 0: bracket the kernel launch with the profiling events.
void launch_fwd(const FwdLaunch& L, cudaStream_t stream, bool pdl, int prof_slot = -1, bool prof_open = true,
                bool prof_close = true) {
  const size_t smem = L.smem_launch;
  auto go = [&](auto kern, int threads) {
    ensure_smem(kern, smem);
    if (prof_slot >= 0 && prof_open) prof_begin(prof_slot, stream);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = (pdl && !(prof_slot >= 0 && prof_open)) ? 1 : 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = L.grid;
    lc.blockDim = dim3(threads, 1, 1);
    lc.dynamicSmemBytes = smem;
    lc.stream = stream;
    lc.attrs = &attr;
    lc.numAttrs = 1;
    cuda_check(cudaLaunchKernelEx(&lc, kern, L.map_a, L.map_out, L.map_out2, L.p, L.raw_stages, L.stages,
                                  L.w_stages),
               "conv_fwd_kernel launch");
    if (prof_slot >= 0 && prof_close) prof_end(prof_slot, stream);
  };
  if (L.ts) {
    if (L.pieces == 3)
      go(conv_fwd_kernel<true, 3, true>, kFwdThreadsTS);
    else
      go(conv_fwd_kernel<true, 1, true>, kFwdThreadsTS);
  } else if (L.raw_f32) {
    if (L.pieces == 3)
      go(conv_fwd_kernel<true, 3>, kFwdThreadsP);
    else
      go(conv_fwd_kernel<true, 1>, kFwdThreadsP);
  } else {
    go(conv_fwd_kernel<false, 1>, kFwdThreadsTS);  // 16 warps: three epilogue groups
  }
  cuda_check(cudaGetLastError(), "conv_fwd_kernel launch");
}

// dconv_prep_batch_begin .. _end: this thread's weight preps are recorded, not launched
thread_local std::vector<PrepJob>* g_prep_rec = nullptr;

// weight prep: src blocked weights -> bf16 pieces in the phase-sorted tap order
// (tapmap_dev is uploaded once at plan creation so execute calls are graph-capturable)
void launch_weight_prep(const dconv_wt_t& w, int n_taps, const int* tapmap_dev, void* dst, int cb_in, int nb,
                        int n_ntiles, int dual, int pieces, int nt_major, cudaStream_t stream) {
  const int64_t total = static_cast<int64_t>(cb_in) * n_ntiles * n_taps * 2 * nb * 128;
  if (total >= (int64_t{1} << 31)) fail(DCONV_ERR_UNSUPPORTED, "weight prep: more than 2^31 prepared weights");
  const int kbs = cdiv(w.k, 16), cbs = cdiv(w.c, 16);
  if (g_prep_rec) {
    PrepJob j;
    j.src = w.data;
    j.dst = dst;
    j.tapmap = tapmap_dev;
    j.src_bf16 = w.dtype == DCONV_F32 ? 0 : 1;
    j.kb_src = kbs;
    j.cb_src = cbs;
    j.rs_src = w.r * w.s;
    j.n_taps = n_taps;
    j.cb_in = cb_in;
    j.nb = nb;
    j.n_ntiles = n_ntiles;
    j.dual = dual;
    j.pieces = pieces;
    j.nt_major = nt_major;
    j.n8 = static_cast<int>(total / 8);
    j.off8 = 0;
    g_prep_rec->push_back(j);
    return;
  }
  if (w.dtype == DCONV_F32)
    weight_prep_kernel<float><<<grid1d(total / 8), 256, 0, stream>>>(
        reinterpret_cast<const float*>(w.data), reinterpret_cast<__nv_bfloat16*>(dst), kbs, cbs, w.r * w.s,
        tapmap_dev, n_taps, cb_in, nb, n_ntiles, dual, pieces, nt_major);
  else
    weight_prep_kernel<__nv_bfloat16><<<grid1d(total / 8), 256, 0, stream>>>(
        reinterpret_cast<const __nv_bfloat16*>(w.data), reinterpret_cast<__nv_bfloat16*>(dst), kbs, cbs, w.r * w.s,
        tapmap_dev, n_taps, cb_in, nb, n_ntiles, dual, pieces, nt_major);
  cuda_check(cudaGetLastError(), "weight_prep launch");
}

// upper bound over tilings: n_ntiles * nb <= kb_out + 15
size_t prep_bytes(int pieces, int cb_in, int taps, int kb_out) {
  return static_cast<size_t>(pieces) * cb_in * taps * 2 * (kb_out + 15) * 256;
}
size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }

std::string json_tile(const FwdLaunch& L) {
  char buf[512];
  std::snprintf(buf, sizeof(buf),
                "{\"mode\":\"%s\",\"wsub\":%d,\"mb\":%d,\"nb\":%d,\"pc_stages\":%d,\"raw_stages\":%d,\"w_stages\":%d,"
                "\"smem\":%zu,\"ctas\":%u,\"tiles\":%d,\"pieces\":%d,\"raw_f32\":%d,\"phases\":%d,\"a_px\":%d,"
                "\"mimg\":%d,\"a_in_tmem\":%d,\"kc\":%d,\"w_resident\":%d,\"tma_store\":%d,\"split_acc\":%d,"
                "\"epi_groups\":%d,\"a_sw128\":%d}",
                L.p.linear ? "linear" : "rows", L.p.wsub, L.p.mb, L.p.nb, L.stages, L.raw_stages, L.w_stages, L.smem,
                L.grid.x,
                (L.p.mimg > 0 ? (L.p.n_img + L.p.mimg - 1) / L.p.mimg : L.p.n_img * L.p.tiles_per_img) * L.p.n_ntiles,
                L.pieces, L.raw_f32 ? 1 : 0, L.p.n_phases, L.p.a_px, L.p.mimg, L.ts ? 1 : 0, L.p.kc, L.p.w_resident, L.p.tma_store, L.p.split_acc,
                (!L.raw_f32 && !L.ts) ? std::max(1, std::min(3, L.p.epi_groups)) : (L.p.ts_epi2 && L.p.tma_store) ? 2 : 1,
                L.p.a_sw128);
  return buf;
}

int math_pieces(int math) {
  if (math == DCONV_MATH_F32) return 3;
  if (math == DCONV_MATH_BF16) return 1;
  fail(DCONV_ERR_INVALID_ARGUMENT, "math must be DCONV_MATH_F32 or DCONV_MATH_BF16");
}

void copy_out(const std::string& s, char* buf, size_t len) {
  if (!buf || len == 0) return;
  const size_t n = std::min(len - 1, s.size());
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}

}  // namespace

namespace {
// ------------------------------------------------------------------ vlen != 16
// The tensor-core passes run on 16-lane channel blocks. A plan for another vlen
// (the reference runs vlen 4, 5, 8 ..., test_propagation.cpp:64-76) keeps a
// vlen-16 twin; each execute re-blocks its operands into workspace copies
// (device kernels, bitwise data moves), runs the twin and re-blocks the result
// back into the caller's vlen-v tensor (halo and tail lanes zeroed).
dconv_spec_t spec16(const dconv_spec_t& s) {
  dconv_spec_t t = s;
  t.vlen = 16;
  return t;
}
dconv_act_t act_as16(const dconv_act_t& a, void* data, int hh, int hw) {
  dconv_act_t t = a;
  t.data = data;
  t.vlen = 16;
  t.halo_h = hh;
  t.halo_w = hw;
  return t;
}
dconv_wt_t wt_as16(const dconv_wt_t& w, void* data, int dtype) {
  dconv_wt_t t = w;
  t.data = data;
  t.vlen = 16;
  t.dtype = dtype;
  return t;
}
size_t act_bytes(const dconv_act_t& a) { return align256(static_cast<size_t>(act_elems(a)) * (a.dtype == DCONV_BF16 ? 2 : 4)); }
size_t wt_bytes(const dconv_wt_t& w) { return align256(static_cast<size_t>(wt_elems(w)) * (w.dtype == DCONV_BF16 ? 2 : 4)); }

void launch_reblock_act(const dconv_act_t& src, const dconv_act_t& dst, int accumulate, cudaStream_t cs) {
  if (src.dtype != dst.dtype) fail(DCONV_ERR_INVALID_ARGUMENT, "reblock: dtypes differ");
  const int g = grid1d(act_elems(dst));
  if (src.dtype == DCONV_F32)
    reblock_act_kernel<float><<<g, 256, 0, cs>>>((const float*)src.data, (float*)dst.data, src.n, src.c, src.h, src.w,
                                                 src.vlen, src.halo_h, src.halo_w, dst.vlen, dst.halo_h, dst.halo_w,
                                                 accumulate);
  else
    reblock_act_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((const __nv_bfloat16*)src.data, (__nv_bfloat16*)dst.data,
                                                         src.n, src.c, src.h, src.w, src.vlen, src.halo_h, src.halo_w,
                                                         dst.vlen, dst.halo_h, dst.halo_w, accumulate);
  cuda_check(cudaGetLastError(), "reblock_act");
}
void launch_reblock_wt(const dconv_wt_t& src, const dconv_wt_t& dst, int accumulate, cudaStream_t cs) {
  if (src.dtype != dst.dtype) fail(DCONV_ERR_INVALID_ARGUMENT, "reblock: dtypes differ");
  const int g = grid1d(wt_elems(dst));
  if (src.dtype == DCONV_F32)
    reblock_wt_kernel<float><<<g, 256, 0, cs>>>((const float*)src.data, (float*)dst.data, src.k, src.c, src.r, src.s,
                                                src.vlen, dst.vlen, accumulate);
  else
    reblock_wt_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((const __nv_bfloat16*)src.data, (__nv_bfloat16*)dst.data,
                                                        src.k, src.c, src.r, src.s, src.vlen, dst.vlen, accumulate);
  cuda_check(cudaGetLastError(), "reblock_wt");
}
void reblock_epilogue_check(const dconv_epilogue_t* ep) {
  if (ep && (ep->add || ep->mask || ep->flags))
    fail(DCONV_ERR_UNSUPPORTED, "vlen != 16: fused graph epilogues need 16-lane tensors");
}
}  // namespace

// ====================================================================== plans
// Resolved launches are cached per tensor geometry (the reference builds its
// ExecutionPlan once per layer, propagation.cpp:42-54): the tile search, the
// epilogue decisions and the descriptor JSON happen on the first execute of a
// geometry; the tensor maps are re-encoded only when a tensor address changes.
using GeoKey = std::array<int, 16>;

GeoKey geo_key(const dconv_act_t& a, const dconv_act_t& b, int extra = 0) {
  return {a.n, a.c, a.h, a.w, a.halo_h, a.halo_w, a.dtype, b.n, b.c, b.h, b.w, b.halo_h, b.halo_w, b.dtype,
          extra, g_sm_budget};
}

struct FwdEntry {
  std::vector<FwdLaunch> L;  // one per launched phase (forward: one)
  const void* in_ptr = nullptr;
  const void* out_ptr = nullptr;
  bool maps = false;
  std::string desc;
};

struct dconv_fwd_plan {
  dconv_spec_t spec;
  int math, pieces;
  int fuse_kind;
  float* bias_dev = nullptr;  // kb*16 lanes, tail zero (plan.bias_lanes analog)
  int out_halo_h, out_halo_w;
  dconv_engine_config_t cfg;
  bool has_cfg;
  Taps taps;
  int* tapmap_dev = nullptr;
  std::mutex mu;
  std::map<GeoKey, FwdEntry> cache;
  const std::string* last_desc = nullptr;
  dconv_fwd_plan* inner = nullptr;  // vlen != 16: the vlen-16 twin the execute re-blocks around
};

struct BwdPhase {
  int a, b;            // output phase of dI
  bool zero;           // no taps: lattice is zero
  ConvProblem pb;      // stride-1 sub-problem (input dO)
  Taps taps;           // single phase
  std::vector<int> tapmap;  // prepared tap -> source r*S+s
  size_t ws_off;
};

struct dconv_bwd_plan {
  dconv_spec_t spec;
  int math, pieces;
  int route;
  dconv_engine_config_t cfg;
  bool has_cfg;
  std::vector<BwdPhase> phases;
  int* tapmap_dev = nullptr;  // concatenated tap maps
  size_t ws_bytes = 0;
  std::mutex mu;
  std::map<GeoKey, FwdEntry> cache;  // key: (grad_out, grad_in, accumulate)
  const std::string* last_desc = nullptr;
  dconv_bwd_plan* inner = nullptr;  // vlen != 16: the vlen-16 twin
};

struct UpdEntry;

struct dconv_upd_plan {
  dconv_spec_t spec;
  int math, pieces;
  dconv_engine_config_t cfg;
  bool has_cfg;
  Taps taps;
  std::mutex mu;
  std::map<GeoKey, UpdEntry*> cache;
  const std::string* last_desc = nullptr;
  dconv_upd_plan* inner = nullptr;  // vlen != 16: the vlen-16 twin
  // modelled bf16 variant choice (k-tile width, stacking, c-tiles per CTA) per operand
  // geometry: computed once, not on every execute (the search evaluates ~10 plans)
  mutable std::mutex sel_mu;
  mutable std::map<std::array<int, 12>, std::array<int, 3>> sel_cache;
};

extern "C" {

const char* dconv_last_error(void) { return g_err.c_str(); }
// the executor (graph.cu) reports its own failures through dconv_last_error()
void dconv_internal_set_error(const char* msg) { g_err = msg ? msg : ""; }
// the DCONV_* developer overrides for graph.cu (null outside developer mode)
const char* dconv_internal_dev_env(const char* name) { return dev_env(name); }

int dconv_prep_batch_begin(void) {
  return guarded([&] {
    if (g_prep_rec) fail(DCONV_ERR_INVALID_ARGUMENT, "prep_batch_begin: a batch is already open on this thread");
    g_prep_rec = new std::vector<PrepJob>();
  });
}

int dconv_prep_batch_end(dconv_stream_t stream) {
  std::unique_ptr<std::vector<PrepJob>> jobs(g_prep_rec);
  g_prep_rec = nullptr;
  return guarded([&] {
    if (!jobs) fail(DCONV_ERR_INVALID_ARGUMENT, "prep_batch_end: no open batch on this thread");
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    for (size_t j0 = 0; j0 < jobs->size(); j0 += kPrepBatchMax) {
      PrepBatch b;
      b.n_jobs = static_cast<int>(std::min<size_t>(kPrepBatchMax, jobs->size() - j0));
      int64_t off = 0;
      for (int j = 0; j < b.n_jobs; ++j) {
        b.job[j] = (*jobs)[j0 + j];
        b.job[j].off8 = static_cast<int>(off);
        off += b.job[j].n8;
      }
      if (off >= (int64_t{1} << 31)) fail(DCONV_ERR_UNSUPPORTED, "prep_batch_end: more than 2^31 prepared groups");
      b.total8 = static_cast<int>(off);
      weight_prep_batch_kernel<<<grid1d(off), 256, 0, cs>>>(b);
      cuda_check(cudaGetLastError(), "weight_prep_batch launch");
    }
  });
}

const char* dconv_status_string(int s) {
  switch (s) {
    case DCONV_OK: return "ok";
    case DCONV_ERR_NON_INTEGRAL_SHAPE: return "NonIntegralShape";
    case DCONV_ERR_INVALID_LAYER_SPEC: return "InvalidLayerSpec";
    case DCONV_ERR_SHAPE_MISMATCH: return "ShapeMismatch";
    case DCONV_ERR_INVALID_DESCRIPTOR: return "InvalidDescriptor";
    case DCONV_ERR_OVERFLOW_RISK: return "OverflowRisk";
    case DCONV_ERR_PLAN_INFEASIBLE: return "PlanInfeasible";
    case DCONV_ERR_EMPTY_TRACE: return "EmptyTrace";
    case DCONV_ERR_PLAN_TENSOR_MISMATCH: return "PlanTensorMismatch";
    case DCONV_ERR_INFEASIBLE_STRATEGY: return "InfeasibleStrategy";
    case DCONV_ERR_CHAIN_SHAPE_MISMATCH: return "ChainShapeMismatch";
    case DCONV_ERR_PARSE: return "ParseError";
    case DCONV_ERR_CUDA: return "CudaError";
    case DCONV_ERR_UNSUPPORTED: return "Unsupported";
    case DCONV_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    default: return "unknown";
  }
}

int dconv_version(void) { return 100; }

void dconv_engine_config_default(dconv_engine_config_t* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->min_accumulators = 8;
  c->max_accumulators = 28;
  c->cache_budget_bytes = 512 * 1024;
  c->prefetch_lookahead = 1;
  c->prefetch_enabled = 1;
  c->streaming_stores = 0;
  c->acc_chain_limit = 512;
  c->i16_bound_in = 256;
  c->i16_bound_wt = 256;
}

int dconv_make_spec(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w, int vlen,
                    dconv_spec_t* out) {
  return guarded([&] {
    if (!out) fail(DCONV_ERR_INVALID_ARGUMENT, "null spec");
    if (pad_h < 0) pad_h = (R % 2 == 1) ? (R - 1) / 2 : 0;
    if (pad_w < 0) pad_w = (S % 2 == 1) ? (S - 1) / 2 : 0;
    dconv_spec_t s = {N, C, K, H, W, R, S, stride, pad_h, pad_w, vlen};
    *out = s;
    validate_spec(s);
  });
}

int dconv_spec_validate(const dconv_spec_t* spec) {
  return guarded([&] {
    if (!spec) fail(DCONV_ERR_INVALID_ARGUMENT, "null spec");
    validate_spec(*spec);
  });
}

int dconv_output_shape(const dconv_spec_t* spec, int* P, int* Q) {
  return guarded([&] {
    if (!spec || !P || !Q) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    validate_spec(*spec);
    *P = out_P(*spec);
    *Q = out_Q(*spec);
  });
}

int64_t dconv_pass_flops(const dconv_spec_t* s) {
  if (!s || dconv_spec_validate(s) != DCONV_OK) return -1;
  return 2LL * s->N * s->K * s->C * out_P(*s) * out_Q(*s) * s->R * s->S;
}

int64_t dconv_act_elems(const dconv_act_t* a) { return a ? act_elems(*a) : -1; }
int64_t dconv_wt_elems(const dconv_wt_t* w) { return w ? wt_elems(*w) : -1; }

// ------------------------------------------------------------------ layouts
int dconv_pack_act(const void* nchw, int src_dtype, const dconv_act_t* dst, dconv_stream_t stream) {
  return guarded([&] {
    check_act(dst, "pack_act dst");
    check_dtype(src_dtype);
    if (!nchw) fail(DCONV_ERR_INVALID_ARGUMENT, "pack_act: null source");
    const dconv_act_t& d = *dst;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (d.vlen == 16) {  // thread per pixel, vector lane rows
      const int g16 = grid1d(act_elems(d) / 16);
      if (src_dtype == DCONV_F32 && d.dtype == DCONV_F32)
        pack_act16_kernel<float, float><<<g16, 256, 0, s>>>((const float*)nchw, (float*)d.data, d.n, d.c, d.h, d.w,
                                                            d.halo_h, d.halo_w);
      else if (src_dtype == DCONV_F32)
        pack_act16_kernel<float, __nv_bfloat16><<<g16, 256, 0, s>>>((const float*)nchw, (__nv_bfloat16*)d.data, d.n,
                                                                    d.c, d.h, d.w, d.halo_h, d.halo_w);
      else if (d.dtype == DCONV_F32)
        pack_act16_kernel<__nv_bfloat16, float><<<g16, 256, 0, s>>>((const __nv_bfloat16*)nchw, (float*)d.data, d.n,
                                                                    d.c, d.h, d.w, d.halo_h, d.halo_w);
      else
        pack_act16_kernel<__nv_bfloat16, __nv_bfloat16><<<g16, 256, 0, s>>>(
            (const __nv_bfloat16*)nchw, (__nv_bfloat16*)d.data, d.n, d.c, d.h, d.w, d.halo_h, d.halo_w);
      cuda_check(cudaGetLastError(), "pack_act");
      return;
    }
    const int g = grid1d(act_elems(d));
    if (src_dtype == DCONV_F32 && d.dtype == DCONV_F32)
      pack_act_kernel<float, float><<<g, 256, 0, s>>>((const float*)nchw, (float*)d.data, d.n, d.c, d.h, d.w, d.vlen,
                                                      d.halo_h, d.halo_w);
    else if (src_dtype == DCONV_F32)
      pack_act_kernel<float, __nv_bfloat16><<<g, 256, 0, s>>>((const float*)nchw, (__nv_bfloat16*)d.data, d.n, d.c,
                                                              d.h, d.w, d.vlen, d.halo_h, d.halo_w);
    else if (d.dtype == DCONV_F32)
      pack_act_kernel<__nv_bfloat16, float><<<g, 256, 0, s>>>((const __nv_bfloat16*)nchw, (float*)d.data, d.n, d.c,
                                                              d.h, d.w, d.vlen, d.halo_h, d.halo_w);
    else
      pack_act_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>(
          (const __nv_bfloat16*)nchw, (__nv_bfloat16*)d.data, d.n, d.c, d.h, d.w, d.vlen, d.halo_h, d.halo_w);
    cuda_check(cudaGetLastError(), "pack_act");
  });
}

int dconv_unpack_act(const dconv_act_t* src, void* nchw, int dst_dtype, dconv_stream_t stream) {
  return guarded([&] {
    check_act(src, "unpack_act src");
    check_dtype(dst_dtype);
    if (!nchw) fail(DCONV_ERR_INVALID_ARGUMENT, "unpack_act: null destination");
    const dconv_act_t& a = *src;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (a.vlen == 16) {  // thread per pixel, vector lane rows
      const int g16 = grid1d(static_cast<int64_t>(a.n) * cdiv(a.c, 16) * a.h * a.w);
      if (a.dtype == DCONV_F32 && dst_dtype == DCONV_F32)
        unpack_act16_kernel<float, float><<<g16, 256, 0, s>>>((const float*)a.data, (float*)nchw, a.n, a.c, a.h, a.w,
                                                              a.halo_h, a.halo_w);
      else if (a.dtype == DCONV_F32)
        unpack_act16_kernel<float, __nv_bfloat16><<<g16, 256, 0, s>>>((const float*)a.data, (__nv_bfloat16*)nchw, a.n,
                                                                      a.c, a.h, a.w, a.halo_h, a.halo_w);
      else if (dst_dtype == DCONV_F32)
        unpack_act16_kernel<__nv_bfloat16, float><<<g16, 256, 0, s>>>((const __nv_bfloat16*)a.data, (float*)nchw, a.n,
                                                                      a.c, a.h, a.w, a.halo_h, a.halo_w);
      else
        unpack_act16_kernel<__nv_bfloat16, __nv_bfloat16><<<g16, 256, 0, s>>>(
            (const __nv_bfloat16*)a.data, (__nv_bfloat16*)nchw, a.n, a.c, a.h, a.w, a.halo_h, a.halo_w);
      cuda_check(cudaGetLastError(), "unpack_act");
      return;
    }
    const int g = grid1d(static_cast<int64_t>(a.n) * a.c * a.h * a.w);
    if (a.dtype == DCONV_F32 && dst_dtype == DCONV_F32)
      unpack_act_kernel<float, float><<<g, 256, 0, s>>>((const float*)a.data, (float*)nchw, a.n, a.c, a.h, a.w, a.vlen,
                                                        a.halo_h, a.halo_w);
    else if (a.dtype == DCONV_F32)
      unpack_act_kernel<float, __nv_bfloat16><<<g, 256, 0, s>>>((const float*)a.data, (__nv_bfloat16*)nchw, a.n, a.c,
                                                                a.h, a.w, a.vlen, a.halo_h, a.halo_w);
    else if (dst_dtype == DCONV_F32)
      unpack_act_kernel<__nv_bfloat16, float><<<g, 256, 0, s>>>((const __nv_bfloat16*)a.data, (float*)nchw, a.n, a.c,
                                                                a.h, a.w, a.vlen, a.halo_h, a.halo_w);
    else
      unpack_act_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>(
          (const __nv_bfloat16*)a.data, (__nv_bfloat16*)nchw, a.n, a.c, a.h, a.w, a.vlen, a.halo_h, a.halo_w);
    cuda_check(cudaGetLastError(), "unpack_act");
  });
}

int dconv_pack_wt(const void* kcrs, int src_dtype, const dconv_wt_t* dst, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(dst, "pack_wt dst");
    check_dtype(src_dtype);
    if (!kcrs) fail(DCONV_ERR_INVALID_ARGUMENT, "pack_wt: null source");
    const dconv_wt_t& d = *dst;
    const int g = grid1d(wt_elems(d));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (src_dtype == DCONV_F32 && d.dtype == DCONV_F32)
      pack_wt_kernel<float, float><<<g, 256, 0, s>>>((const float*)kcrs, (float*)d.data, d.k, d.c, d.r, d.s, d.vlen);
    else if (src_dtype == DCONV_F32)
      pack_wt_kernel<float, __nv_bfloat16><<<g, 256, 0, s>>>((const float*)kcrs, (__nv_bfloat16*)d.data, d.k, d.c,
                                                             d.r, d.s, d.vlen);
    else if (d.dtype == DCONV_F32)
      pack_wt_kernel<__nv_bfloat16, float><<<g, 256, 0, s>>>((const __nv_bfloat16*)kcrs, (float*)d.data, d.k, d.c,
                                                             d.r, d.s, d.vlen);
    else
      pack_wt_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)kcrs,
                                                                     (__nv_bfloat16*)d.data, d.k, d.c, d.r, d.s,
                                                                     d.vlen);
    cuda_check(cudaGetLastError(), "pack_wt");
  });
}

int dconv_unpack_wt(const dconv_wt_t* src, void* kcrs, int dst_dtype, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(src, "unpack_wt src");
    check_dtype(dst_dtype);
    if (!kcrs) fail(DCONV_ERR_INVALID_ARGUMENT, "unpack_wt: null destination");
    const dconv_wt_t& w = *src;
    const int g = grid1d(static_cast<int64_t>(w.k) * w.c * w.r * w.s);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (w.dtype == DCONV_F32 && dst_dtype == DCONV_F32)
      unpack_wt_kernel<float, float><<<g, 256, 0, s>>>((const float*)w.data, (float*)kcrs, w.k, w.c, w.r, w.s, w.vlen);
    else if (w.dtype == DCONV_F32)
      unpack_wt_kernel<float, __nv_bfloat16><<<g, 256, 0, s>>>((const float*)w.data, (__nv_bfloat16*)kcrs, w.k, w.c,
                                                               w.r, w.s, w.vlen);
    else if (dst_dtype == DCONV_F32)
      unpack_wt_kernel<__nv_bfloat16, float><<<g, 256, 0, s>>>((const __nv_bfloat16*)w.data, (float*)kcrs, w.k, w.c,
                                                               w.r, w.s, w.vlen);
    else
      unpack_wt_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, s>>>(
          (const __nv_bfloat16*)w.data, (__nv_bfloat16*)kcrs, w.k, w.c, w.r, w.s, w.vlen);
    cuda_check(cudaGetLastError(), "unpack_wt");
  });
}

int dconv_transform_weight_dual(const dconv_wt_t* src, const dconv_wt_t* dst, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(src, "transform src");
    check_wt(dst, "transform dst");
    const dconv_wt_t& a = *src;
    const dconv_wt_t& b = *dst;
    if (b.k != a.c || b.c != a.k || b.r != a.r || b.s != a.s || b.vlen != a.vlen || b.dtype != a.dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "transform_weight_dual: dst must be (k=src.c, c=src.k, same r, s, vlen, dtype)");
    const int g = grid1d(wt_elems(b));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (a.dtype == DCONV_F32)
      dual_wt_kernel<float><<<g, 256, 0, s>>>((const float*)a.data, (float*)b.data, a.k, a.c, a.r, a.s, a.vlen);
    else
      dual_wt_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)a.data, (__nv_bfloat16*)b.data, a.k, a.c,
                                                      a.r, a.s, a.vlen);
    cuda_check(cudaGetLastError(), "dual_wt");
  });
}

int dconv_copy_with_halo(const dconv_act_t* src, const dconv_act_t* dst, dconv_stream_t stream) {
  return guarded([&] {
    check_act(src, "copy_with_halo src");
    check_act(dst, "copy_with_halo dst");
    const dconv_act_t& a = *src;
    const dconv_act_t& b = *dst;
    if (a.n != b.n || a.c != b.c || a.h != b.h || a.w != b.w || a.vlen != b.vlen || a.dtype != b.dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "copy_with_halo: tensors differ beyond the halo");
    const int g = grid1d(act_elems(b));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int cb = cdiv(a.c, a.vlen);
    if (a.dtype == DCONV_F32)
      rehalo_kernel<float><<<g, 256, 0, s>>>((const float*)a.data, (float*)b.data, a.n, cb, a.h, a.w, a.vlen,
                                             a.halo_h, a.halo_w, b.halo_h, b.halo_w);
    else
      rehalo_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((const __nv_bfloat16*)a.data, (__nv_bfloat16*)b.data, a.n, cb,
                                                     a.h, a.w, a.vlen, a.halo_h, a.halo_w, b.halo_h, b.halo_w);
    cuda_check(cudaGetLastError(), "rehalo");
  });
}

int dconv_zero_halo(const dconv_act_t* act, dconv_stream_t stream) {
  return guarded([&] {
    check_act(act, "zero_halo");
    const dconv_act_t& a = *act;
    if (a.halo_h == 0 && a.halo_w == 0) return;
    const int planes = a.n * cdiv(a.c, a.vlen);
    const int64_t frame = (static_cast<int64_t>(a.h + 2 * a.halo_h) * (a.w + 2 * a.halo_w) -
                           static_cast<int64_t>(a.h) * a.w);
    const int g = grid1d(planes * frame * a.vlen);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (a.dtype == DCONV_F32)
      zero_halo_kernel<float><<<g, 256, 0, s>>>((float*)a.data, planes, a.h, a.w, a.halo_h, a.halo_w, a.vlen);
    else
      zero_halo_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((__nv_bfloat16*)a.data, planes, a.h, a.w, a.halo_h, a.halo_w,
                                                        a.vlen);
    cuda_check(cudaGetLastError(), "zero_halo");
  });
}

}  // extern "C"

namespace {
template <typename T>
__global__ void apply_op_kernel(T* __restrict__ d, int planes_n, int cb, int h, int w, int hh, int hw, int v,
                                int kind, const float* __restrict__ bias) {
  const int hp = h + 2 * hh, wp = w + 2 * hw;
  const long long total = static_cast<long long>(planes_n) * cb * h * w * v;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % v);
    long long q = e / v;
    const int x = static_cast<int>(q % w);
    q /= w;
    const int y = static_cast<int>(q % h);
    q /= h;
    const int b = static_cast<int>(q % cb);
    const long long plane = q;  // n*cb + b
    T* px = d + ((plane * hp + y + hh) * wp + x + hw) * v + lane;
    float val = to_f<T>(*px);
    if (kind != DCONV_FUSE_RELU) val += bias[b * v + lane];
    if (kind != DCONV_FUSE_BIAS_ADD) val = val > 0.0f ? val : 0.0f;
    *px = from_f<T>(val);
  }
}
}  // namespace

extern "C" {

int dconv_apply_fused_op(const dconv_act_t* act, const dconv_fusion_t* op, dconv_stream_t stream) {
  return guarded([&] {
    check_act(act, "apply_fused_op");
    if (!op || op->kind < DCONV_FUSE_RELU || op->kind > DCONV_FUSE_BIAS_RELU)
      fail(DCONV_ERR_INVALID_ARGUMENT, "apply_fused_op: bad op");
    const dconv_act_t& a = *act;
    const int cb = cdiv(a.c, a.vlen);
    float* bias_dev = nullptr;
    if (op->kind != DCONV_FUSE_RELU) {
      if (!op->bias || op->bias_len != a.c) fail(DCONV_ERR_SHAPE_MISMATCH, "apply_fused_op: bias length must equal channels");
      std::vector<float> lanes(static_cast<size_t>(cb) * a.vlen, 0.0f);
      std::copy(op->bias, op->bias + a.c, lanes.begin());
      cuda_check(cudaMalloc(&bias_dev, lanes.size() * sizeof(float)), "bias alloc");
      cuda_check(cudaMemcpy(bias_dev, lanes.data(), lanes.size() * sizeof(float), cudaMemcpyHostToDevice), "bias copy");
    }
    const int g = grid1d(static_cast<int64_t>(a.n) * cb * a.h * a.w * a.vlen);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (a.dtype == DCONV_F32)
      apply_op_kernel<float><<<g, 256, 0, s>>>((float*)a.data, a.n, cb, a.h, a.w, a.halo_h, a.halo_w, a.vlen, op->kind,
                                               bias_dev);
    else
      apply_op_kernel<__nv_bfloat16><<<g, 256, 0, s>>>((__nv_bfloat16*)a.data, a.n, cb, a.h, a.w, a.halo_h, a.halo_w,
                                                       a.vlen, op->kind, bias_dev);
    cuda_check(cudaGetLastError(), "apply_fused_op");
    if (bias_dev) {
      cuda_check(cudaStreamSynchronize(s), "apply_fused_op sync");
      cudaFree(bias_dev);
    }
  });
}

// splitmix64 (util.hpp:46-52) uniform / He-normal generators, host side
static uint64_t splitmix(uint64_t& st) {
  st += 0x9e3779b97f4a7c15ULL;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
void dconv_fill_uniform_host(uint64_t seed, float lo, float hi, float* out, int64_t n) {
  uint64_t st = seed;
  for (int64_t i = 0; i < n; ++i) {
    const float u = static_cast<float>(splitmix(st) >> 40) * (1.0f / 16777216.0f);
    out[i] = lo + (hi - lo) * u;
  }
}
void dconv_fill_he_normal_host(uint64_t seed, float stddev, float* out, int64_t n) {
  uint64_t st = seed;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; ++i) {
    const double u1 = static_cast<double>((splitmix(st) >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double u2 = static_cast<double>(splitmix(st) >> 11) * (1.0 / 9007199254740992.0);
    out[i] = static_cast<float>(std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2) * static_cast<double>(stddev));
  }
}

// ------------------------------------------------------------------ forward
int dconv_fwd_plan_create(const dconv_spec_t* spec, const dconv_fusion_t* fusion, const dconv_engine_config_t* cfg,
                          int math, int out_halo_h, int out_halo_w, dconv_fwd_plan_t* plan) {
  dconv_fwd_plan* pl = nullptr;
  const int st = guarded([&] {
    if (!spec || !plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    validate_spec(*spec);
    if (out_halo_h < 0 || out_halo_w < 0) fail(DCONV_ERR_INVALID_LAYER_SPEC, "output halo must be >= 0");
    pl = new dconv_fwd_plan();
    pl->spec = *spec;
    pl->math = math;
    pl->pieces = math_pieces(math);
    if (spec->vlen != 16) {  // the tensor-core passes run on 16-lane blocks: re-block around a twin
      const dconv_spec_t s16 = spec16(*spec);
      const int rc = dconv_fwd_plan_create(&s16, fusion, cfg, math, out_halo_h, out_halo_w, &pl->inner);
      if (rc != DCONV_OK) fail(rc, g_err);
      pl->out_halo_h = out_halo_h;
      pl->out_halo_w = out_halo_w;
      *plan = pl;
      return;
    }
    pl->fuse_kind = fusion ? fusion->kind : DCONV_FUSE_NONE;
    pl->out_halo_h = out_halo_h;
    pl->out_halo_w = out_halo_w;
    pl->has_cfg = cfg != nullptr;
    if (cfg) pl->cfg = *cfg;
    pl->taps = phase_taps(spec->R, spec->S, spec->stride);
    if (pl->fuse_kind != DCONV_FUSE_NONE) {
      if (pl->fuse_kind < DCONV_FUSE_RELU || pl->fuse_kind > DCONV_FUSE_BIAS_RELU)
        fail(DCONV_ERR_INVALID_ARGUMENT, "bad fusion kind");
      const int kb = cdiv(spec->K, 16);
      std::vector<float> lanes(static_cast<size_t>(kb) * 16, 0.0f);
      if (pl->fuse_kind != DCONV_FUSE_RELU) {
        if (!fusion->bias || fusion->bias_len != spec->K)
          fail(DCONV_ERR_SHAPE_MISMATCH, "apply_fused_op: bias length must equal channels");
        std::copy(fusion->bias, fusion->bias + spec->K, lanes.begin());
      }
      cuda_check(cudaMalloc(&pl->bias_dev, lanes.size() * sizeof(float)), "bias alloc");
      cuda_check(cudaMemcpy(pl->bias_dev, lanes.data(), lanes.size() * sizeof(float), cudaMemcpyHostToDevice),
                 "bias upload");
    }
    cuda_check(cudaMalloc(&pl->tapmap_dev, kMaxTaps * sizeof(int)), "tapmap alloc");
    std::vector<int> tapmap;
    for (size_t t = 0; t < pl->taps.r.size(); ++t) tapmap.push_back(pl->taps.r[t] * spec->S + pl->taps.s[t]);
    cuda_check(cudaMemcpy(pl->tapmap_dev, tapmap.data(), tapmap.size() * sizeof(int), cudaMemcpyHostToDevice),
               "tapmap upload");
    *plan = pl;
  });
  if (st != DCONV_OK && pl) {
    if (pl->bias_dev) cudaFree(pl->bias_dev);
    if (pl->tapmap_dev) cudaFree(pl->tapmap_dev);
    if (pl->inner) dconv_fwd_plan_destroy(pl->inner);
    delete pl;
  }
  return st;
}

void dconv_fwd_plan_destroy(dconv_fwd_plan_t plan) {
  if (!plan) return;
  if (plan->inner) dconv_fwd_plan_destroy(plan->inner);
  if (plan->bias_dev) cudaFree(plan->bias_dev);
  if (plan->tapmap_dev) cudaFree(plan->tapmap_dev);
  delete plan;
}

size_t dconv_fwd_workspace_bytes(dconv_fwd_plan_t plan) {
  if (!plan) return 0;
  if (plan->inner) {  // twin's workspace + 16-lane copies of input (halo = pad), weights, output
    const dconv_spec_t& s = plan->spec;
    const dconv_act_t in{nullptr, s.N, s.C, s.H, s.W, 16, s.pad_h, s.pad_w, DCONV_F32};
    const dconv_act_t out{nullptr, s.N, s.K, out_P(s), out_Q(s), 16, plan->out_halo_h, plan->out_halo_w, DCONV_F32};
    const dconv_wt_t w{nullptr, s.K, s.C, s.R, s.S, 16, DCONV_F32};
    return dconv_fwd_workspace_bytes(plan->inner) + act_bytes(in) + wt_bytes(w) + act_bytes(out);
  }
  const dconv_spec_t& s = plan->spec;
  return align256(prep_bytes(plan->pieces, cdiv(s.C, 16), s.R * s.S, cdiv(s.K, 16)));
}

int dconv_fwd_plan_describe(dconv_fwd_plan_t plan, char* buf, size_t len) {
  if (plan && plan->inner) return dconv_fwd_plan_describe(plan->inner, buf, len);
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    std::lock_guard<std::mutex> lk(plan->mu);
    copy_out(plan->last_desc ? *plan->last_desc : std::string("{\"tile\":\"chosen at first execute\"}"), buf, len);
  });
}

int dconv_fwd_launches(dconv_fwd_plan_t plan) { return plan ? (plan->inner ? 5 : 2) : 0; }

int dconv_forward(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_wt_t* wt, const dconv_act_t* out,
                  void* workspace, dconv_stream_t stream) {
  return dconv_forward_ex(plan, in, wt, out, nullptr, workspace, stream);
}

}  // extern "C"

namespace {
// the forward plan's resolved launch for (in, out) geometry (caller holds plan->mu)
FwdEntry& fwd_entry(dconv_fwd_plan* plan, const dconv_act_t& in, const dconv_act_t& out) {
  const GeoKey key = geo_key(in, out);
  auto it = plan->cache.find(key);
  if (it != plan->cache.end() && !g_dev_mode) return it->second;
  const dconv_spec_t& s = plan->spec;
  const int P = out_P(s), Q = out_Q(s);
  const int cb = cdiv(s.C, 16), kb = cdiv(s.K, 16);
  ConvProblem pb;
  pb.in = in;
  pb.cb_red = cb;
  pb.kb_out = kb;
  pb.P = P;
  pb.Q = Q;
  pb.R = s.R;
  pb.S = s.S;
  pb.stride = s.stride;
  pb.row_off = -s.pad_h;
  pb.col_off = -s.pad_w;
  FwdLaunch L = plan_fwd_launch(pb, plan->taps, nullptr, plan->pieces, plan->has_cfg ? &plan->cfg : nullptr);
  FwdParams& p = L.p;
  p.out_bf16 = out.dtype == DCONV_BF16;
  p.out_cb = kb;
  p.out_hp = P + 2 * out.halo_h;
  p.out_wp = Q + 2 * out.halo_w;
  p.out_y0 = out.halo_h;
  p.out_x0 = out.halo_w;
  p.out_scale = 1;
  p.out_halo_h = out.halo_h;
  p.out_halo_w = out.halo_w;
  finalize_fwd(L);
  FwdEntry e;
  e.L.push_back(L);
  e.desc = json_tile(L);
  return plan->cache[key] = std::move(e);
}
}  // namespace

extern "C" {

int dconv_forward_ex(dconv_fwd_plan_t plan, const dconv_act_t* in, const dconv_wt_t* wt, const dconv_act_t* out,
                     const dconv_epilogue_t* ep, void* workspace, dconv_stream_t stream) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_act(in, "forward input");
    check_wt(wt, "forward weight");
    check_act(out, "forward output");
    if (!workspace) fail(DCONV_ERR_INVALID_ARGUMENT, "forward: null workspace");
    const dconv_spec_t& s = plan->spec;
    const int P = out_P(s), Q = out_Q(s);
    // propagation.cpp:12-19 check_forward_tensors
    if (in->n != s.N || in->c != s.C || in->h != s.H || in->w != s.W || in->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "forward: input does not match the layer spec");
    if (wt->k != s.K || wt->c != s.C || wt->r != s.R || wt->s != s.S || wt->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "forward: weight does not match the layer spec");
    if (out->n != s.N || out->c != s.K || out->h != P || out->w != Q || out->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "forward: output does not match the layer spec");
    if (out->halo_h != plan->out_halo_h || out->halo_w != plan->out_halo_w)
      fail(DCONV_ERR_PLAN_TENSOR_MISMATCH, "forward: output halo differs from the plan's output surface");
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (plan->inner) {  // vlen != 16: re-block around the 16-lane twin
      if (ep && (ep->flags & (DCONV_EP_PREP_ONLY | DCONV_EP_WEIGHTS_READY)))
        fail(DCONV_ERR_UNSUPPORTED, "weight preparation flags need vlen 16 tensors");
      reblock_epilogue_check(ep);
      if (in->dtype != out->dtype || wt->dtype != in->dtype)
        fail(DCONV_ERR_UNSUPPORTED, "vlen != 16: input, weights and output share one dtype");
      char* w8 = reinterpret_cast<char*>(workspace) + dconv_fwd_workspace_bytes(plan->inner);
      const dconv_act_t in16 = act_as16(*in, w8, s.pad_h, s.pad_w);
      const dconv_wt_t w16 = wt_as16(*wt, w8 + act_bytes(in16), wt->dtype);
      const dconv_act_t out16 = act_as16(*out, w8 + act_bytes(in16) + wt_bytes(w16), out->halo_h, out->halo_w);
      launch_reblock_act(*in, in16, 0, cs);
      launch_reblock_wt(*wt, w16, 0, cs);
      const int rc = dconv_forward_ex(plan->inner, &in16, &w16, &out16, nullptr, workspace, stream);
      if (rc != DCONV_OK) fail(rc, g_err);
      launch_reblock_act(out16, *out, 0, cs);
      return;
    }
    const int cb = cdiv(s.C, 16);
    FwdLaunch L;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      FwdEntry& e = fwd_entry(plan, *in, *out);
      FwdLaunch& c = e.L[0];
      if (!e.maps || e.in_ptr != in->data || e.out_ptr != out->data) {
        encode_fwd_act_map(c, *in);
        c.p.out = out->data;
        encode_fwd_out_maps(c);
        e.in_ptr = in->data;
        e.out_ptr = out->data;
        e.maps = true;
      }
      L = c;
      plan->last_desc = &e.desc;
    }
    FwdParams& p = L.p;
    p.dbg = g_fwd_dbg;  // developer builds: role counters / ablation bits (set per call)
    p.dbg_mode = g_fwd_dbg_mode;
    p.wprep = workspace;
    p.out = out->data;
    p.bias = (plan->fuse_kind == DCONV_FUSE_BIAS_ADD || plan->fuse_kind == DCONV_FUSE_BIAS_RELU) ? plan->bias_dev
                                                                                                  : nullptr;
    p.relu = (plan->fuse_kind == DCONV_FUSE_RELU || plan->fuse_kind == DCONV_FUSE_BIAS_RELU) ? 1 : 0;
    p.add = nullptr;
    p.mask = nullptr;
    if (ep) {
      p.add = ep->add;
      p.mask = ep->mask;
      p.relu |= ep->relu ? 1 : 0;
    }
    // weights -> bf16 pieces, phase-sorted taps
    const int ep_flags = ep ? ep->flags : 0;
    const bool prep = !(ep_flags & DCONV_EP_WEIGHTS_READY);
    if (prep)
      launch_weight_prep(*wt, p.n_taps, plan->tapmap_dev, workspace, cb, p.nb, p.n_ntiles, 0, plan->pieces,
                         L.raw_f32 ? 0 : 1, cs);
    if (ep_flags & DCONV_EP_PREP_ONLY) return;
    launch_fwd(L, cs, prep, 0);
  });
}

// ------------------------------------------------------------------ backward-data
// propagation.cpp:35-40
static int choose_route(const dconv_spec_t& s) {
  if (s.stride == 1 && s.pad_h <= s.R - 1 && s.pad_w <= s.S - 1) return DCONV_BWD_DUALITY_STRIDE1;
  if (s.R == 1 && s.S == 1) return DCONV_BWD_DUALITY_1x1;
  return DCONV_BWD_GENERIC;
}

int dconv_bwd_plan_create(const dconv_spec_t* spec, const dconv_engine_config_t* cfg, int math,
                          dconv_bwd_plan_t* plan) {
  dconv_bwd_plan* pl = nullptr;
  const int st = guarded([&] {
    if (!spec || !plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    validate_spec(*spec);
    pl = new dconv_bwd_plan();
    pl->spec = *spec;
    pl->math = math;
    pl->pieces = math_pieces(math);
    pl->route = choose_route(*spec);
    if (spec->vlen != 16) {
      const dconv_spec_t s16 = spec16(*spec);
      const int rc = dconv_bwd_plan_create(&s16, cfg, math, &pl->inner);
      if (rc != DCONV_OK) fail(rc, g_err);
      *plan = pl;
      return;
    }
    pl->has_cfg = cfg != nullptr;
    if (cfg) pl->cfg = *cfg;
    const dconv_spec_t& s = *spec;
    const int P = out_P(s), Q = out_Q(s);
    const int kb = cdiv(s.K, 16), cb = cdiv(s.C, 16);
    const int stv = s.stride;
    // Stride-phase decomposition of dI: phase (a, b) of dI is a stride-1
    // correlation of dO with the flipped sub-filter W[a' + st*r2][b' + st*s2].
    // Stride 1 degenerates to the single dual phase (DUALITY_STRIDE1).
    size_t off = 0;
    for (int a = 0; a < stv; ++a)
      for (int b = 0; b < stv; ++b) {
        BwdPhase ph;
        ph.a = a;
        ph.b = b;
        const int ap = (a + s.pad_h) % stv, bp = (b + s.pad_w) % stv;
        const int offa = (a + s.pad_h - ap) / stv, offb = (b + s.pad_w - bp) / stv;
        const int R2 = ap < s.R ? cdiv(s.R - ap, stv) : 0;
        const int S2 = bp < s.S ? cdiv(s.S - bp, stv) : 0;
        const int ly = a < s.H ? cdiv(s.H - a, stv) : 0, lx = b < s.W ? cdiv(s.W - b, stv) : 0;
        ph.zero = R2 == 0 || S2 == 0;
        if (ly == 0 || lx == 0) continue;
        ph.pb.cb_red = kb;
        ph.pb.kb_out = cb;
        ph.pb.P = ly;
        ph.pb.Q = lx;
        ph.pb.R = R2;
        ph.pb.S = S2;
        ph.pb.stride = 1;
        ph.pb.row_off = offa - (R2 - 1);
        ph.pb.col_off = offb - (S2 - 1);
        ph.ws_off = off;
        if (!ph.zero) {
          ph.taps = phase_taps(R2, S2, 1);
          for (size_t t = 0; t < ph.taps.r.size(); ++t) {
            const int u = ph.taps.r[t], w = ph.taps.s[t];  // prepared tap (u, w) <- source tap, flipped
            const int r = ap + stv * (R2 - 1 - u), sc = bp + stv * (S2 - 1 - w);
            ph.tapmap.push_back(r * s.S + sc);
          }
          off += align256(prep_bytes(pl->pieces, kb, static_cast<int>(ph.tapmap.size()), cb));
        }
        pl->phases.push_back(ph);
      }
    pl->ws_bytes = off;
    (void)P;
    (void)Q;
    std::vector<int> all;
    for (auto& ph : pl->phases) all.insert(all.end(), ph.tapmap.begin(), ph.tapmap.end());
    cuda_check(cudaMalloc(&pl->tapmap_dev, std::max<size_t>(1, all.size()) * sizeof(int)), "tapmap alloc");
    if (!all.empty())
      cuda_check(cudaMemcpy(pl->tapmap_dev, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice),
                 "tapmap upload");
    *plan = pl;
  });
  if (st != DCONV_OK && pl) {
    if (pl->tapmap_dev) cudaFree(pl->tapmap_dev);
    if (pl->inner) dconv_bwd_plan_destroy(pl->inner);
    delete pl;
  }
  return st;
}

void dconv_bwd_plan_destroy(dconv_bwd_plan_t plan) {
  if (!plan) return;
  if (plan->inner) dconv_bwd_plan_destroy(plan->inner);
  if (plan->tapmap_dev) cudaFree(plan->tapmap_dev);
  delete plan;
}

int dconv_bwd_route(dconv_bwd_plan_t plan) { return plan ? plan->route : -1; }
size_t dconv_bwd_workspace_bytes(dconv_bwd_plan_t plan) {
  if (plan && plan->inner) {  // twin's workspace + 16-lane dO (halo 0), weights, dI (halo 0)
    const dconv_spec_t& s = plan->spec;
    const dconv_act_t go{nullptr, s.N, s.K, out_P(s), out_Q(s), 16, 0, 0, DCONV_F32};
    const dconv_act_t gi{nullptr, s.N, s.C, s.H, s.W, 16, 0, 0, DCONV_F32};
    const dconv_wt_t w{nullptr, s.K, s.C, s.R, s.S, 16, DCONV_F32};
    return dconv_bwd_workspace_bytes(plan->inner) + act_bytes(go) + wt_bytes(w) + act_bytes(gi);
  }
  return plan ? std::max<size_t>(align256(plan->ws_bytes), 256) : 0;
}
int dconv_bwd_plan_describe(dconv_bwd_plan_t plan, char* buf, size_t len) {
  if (plan && plan->inner) return dconv_bwd_plan_describe(plan->inner, buf, len);
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    std::lock_guard<std::mutex> lk(plan->mu);
    copy_out(plan->last_desc ? *plan->last_desc : std::string("{\"tile\":\"chosen at first execute\"}"), buf, len);
  });
}
int dconv_backward_data(dconv_bwd_plan_t plan, const dconv_wt_t* wt, const dconv_act_t* grad_out,
                        const dconv_act_t* grad_in, void* workspace, dconv_stream_t stream) {
  return dconv_backward_data_ex(plan, wt, grad_out, grad_in, nullptr, workspace, stream);
}

// weight preparations one backward-data execute launches (graph executor accounting)
int dconv_internal_bwd_prep_launches(dconv_bwd_plan_t plan) {
  if (!plan) return 0;
  if (plan->inner) return dconv_internal_bwd_prep_launches(plan->inner);
  int n = 0;
  for (auto& ph : plan->phases) n += ph.zero ? 0 : 1;
  return n;
}

int dconv_bwd_launches(dconv_bwd_plan_t plan) {
  if (!plan) return 0;
  if (plan->inner) return dconv_bwd_launches(plan->inner) + 3;
  int n = 0;
  for (auto& ph : plan->phases) n += ph.zero ? 1 : 2;
  return n;
}

}  // extern "C"

namespace {
// 1x1 / stride 2 without accumulation: the single tap phase (0, 0) writes the whole
// dI (its lattice values and the three zero neighbours of each) instead of zero passes
bool bwd_fill(const dconv_bwd_plan* plan, bool accumulate) {
  const dconv_spec_t& s = plan->spec;
  int n_conv = 0;
  for (auto& ph : plan->phases) n_conv += ph.zero ? 0 : 1;
  return !accumulate && s.stride == 2 && s.R == 1 && s.S == 1 && s.pad_h == 0 && s.pad_w == 0 && n_conv == 1;
}

// the backward plan's resolved phase launches for (grad_out, grad_in) geometry
// and the accumulate mode (caller holds plan->mu)
FwdEntry& bwd_entry(dconv_bwd_plan* plan, const dconv_act_t& grad_out, const dconv_act_t& grad_in,
                    bool accumulate) {
  const GeoKey key = geo_key(grad_out, grad_in, accumulate ? 1 : 0);
  auto it = plan->cache.find(key);
  if (it != plan->cache.end() && !g_dev_mode) return it->second;
  const dconv_spec_t& s = plan->spec;
  const int cb = cdiv(s.C, 16);
  const int hp = s.H + 2 * grad_in.halo_h, wp = s.W + 2 * grad_in.halo_w;
  const bool fill = bwd_fill(plan, accumulate);
  FwdEntry e;
  e.desc = "{\"route\":" + std::to_string(plan->route) + ",\"phases\":[";
  bool first = true;
  for (auto& ph : plan->phases) {
    if (!first) e.desc += ",";
    first = false;
    if (ph.zero) {
      e.desc += accumulate ? "\"skip\"" : fill ? "\"filled\"" : "\"zero\"";
      continue;
    }
    ConvProblem pb = ph.pb;
    pb.in = grad_out;
    FwdLaunch L = plan_fwd_launch(pb, ph.taps, nullptr, plan->pieces, plan->has_cfg ? &plan->cfg : nullptr);
    FwdParams& p = L.p;
    p.out_bf16 = grad_in.dtype == DCONV_BF16;
    p.out_cb = cb;
    p.out_hp = hp;
    p.out_wp = wp;
    p.out_y0 = grad_in.halo_h + ph.a;
    p.out_x0 = grad_in.halo_w + ph.b;
    p.out_scale = s.stride;
    const bool single = s.stride == 1;
    p.out_halo_h = single ? grad_in.halo_h : 0;
    p.out_halo_w = single ? grad_in.halo_w : 0;
    p.out_fill = fill ? 1 : 0;
    p.fill_h_end = grad_in.halo_h + s.H;
    p.fill_w_end = grad_in.halo_w + s.W;
    finalize_fwd(L);
    e.desc += json_tile(L);
    e.L.push_back(L);
  }
  e.desc += "]}";
  return plan->cache[key] = std::move(e);
}
}  // namespace

extern "C" {

int dconv_backward_data_ex(dconv_bwd_plan_t plan, const dconv_wt_t* wt, const dconv_act_t* grad_out,
                           const dconv_act_t* grad_in, const dconv_epilogue_t* ep, void* workspace,
                           dconv_stream_t stream) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_wt(wt, "backward weight");
    check_act(grad_out, "backward grad_out");
    check_act(grad_in, "backward grad_in");
    if (!workspace) fail(DCONV_ERR_INVALID_ARGUMENT, "backward: null workspace");
    const dconv_spec_t& s = plan->spec;
    const int P = out_P(s), Q = out_Q(s);
    if (wt->k != s.K || wt->c != s.C || wt->r != s.R || wt->s != s.S || wt->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "backward: weight does not match the layer spec");
    if (grad_out->n != s.N || grad_out->c != s.K || grad_out->h != P || grad_out->w != Q || grad_out->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "backward: grad_out does not match the layer spec");
    if (grad_in->n != s.N || grad_in->c != s.C || grad_in->h != s.H || grad_in->w != s.W || grad_in->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "backward: grad_in does not match the layer spec");
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (plan->inner) {  // vlen != 16: re-block around the 16-lane twin
      if (ep && (ep->flags & (DCONV_EP_PREP_ONLY | DCONV_EP_WEIGHTS_READY)))
        fail(DCONV_ERR_UNSUPPORTED, "weight preparation flags need vlen 16 tensors");
      reblock_epilogue_check(ep);
      if (grad_out->dtype != grad_in->dtype || wt->dtype != grad_out->dtype)
        fail(DCONV_ERR_UNSUPPORTED, "vlen != 16: grad_out, weights and grad_in share one dtype");
      char* w8 = reinterpret_cast<char*>(workspace) + dconv_bwd_workspace_bytes(plan->inner);
      const dconv_act_t go16 = act_as16(*grad_out, w8, 0, 0);
      const dconv_wt_t w16 = wt_as16(*wt, w8 + act_bytes(go16), wt->dtype);
      const dconv_act_t gi16 = act_as16(*grad_in, w8 + act_bytes(go16) + wt_bytes(w16), 0, 0);
      launch_reblock_act(*grad_out, go16, 0, cs);
      launch_reblock_wt(*wt, w16, 0, cs);
      const int rc = dconv_backward_data_ex(plan->inner, &w16, &go16, &gi16, nullptr, workspace, stream);
      if (rc != DCONV_OK) fail(rc, g_err);
      launch_reblock_act(gi16, *grad_in, 0, cs);
      return;
    }
    const int kb = cdiv(s.K, 16), cb = cdiv(s.C, 16);
    const int hp = s.H + 2 * grad_in->halo_h, wp = s.W + 2 * grad_in->halo_w;
    const bool accumulate = ep && ep->add && ep->add == grad_in->data;
    if (ep && ep->add && !accumulate && s.stride != 1)
      fail(DCONV_ERR_UNSUPPORTED, "backward_data_ex: strided layers accept add == grad_in only");
    const bool fill = bwd_fill(plan, accumulate);
    std::vector<FwdLaunch> Ls;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      FwdEntry& e = bwd_entry(plan, *grad_out, *grad_in, accumulate);
      if (!e.maps || e.in_ptr != grad_out->data || e.out_ptr != grad_in->data) {
        for (auto& c : e.L) {
          encode_fwd_act_map(c, *grad_out);
          c.p.out = grad_in->data;
          encode_fwd_out_maps(c);
        }
        e.in_ptr = grad_out->data;
        e.out_ptr = grad_in->data;
        e.maps = true;
      }
      Ls = e.L;
      plan->last_desc = &e.desc;
    }
    const int ep_flags = ep ? ep->flags : 0;
    const bool prep = !(ep_flags & DCONV_EP_WEIGHTS_READY);
    const int n_conv = static_cast<int>(Ls.size());
    int tap_off = 0, conv_i = 0;
    for (auto& ph : plan->phases) {
      if (ph.zero) {
        if (accumulate || fill || (ep_flags & DCONV_EP_PREP_ONLY)) continue;  // adding zeros / written by the tap phase
        const int planes = s.N * cb;
        const int ly = cdiv(s.H - ph.a, s.stride), lx = cdiv(s.W - ph.b, s.stride);
        const int g = grid1d(static_cast<int64_t>(planes) * ly * lx * 16);
        if (grad_in->dtype == DCONV_F32)
          zero_lattice_kernel<float><<<g, 256, 0, cs>>>((float*)grad_in->data, planes, s.H, s.W, hp, wp,
                                                        grad_in->halo_h, grad_in->halo_w, s.stride, ph.a, ph.b);
        else
          zero_lattice_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((__nv_bfloat16*)grad_in->data, planes, s.H, s.W, hp,
                                                                wp, grad_in->halo_h, grad_in->halo_w, s.stride, ph.a,
                                                                ph.b);
        cuda_check(cudaGetLastError(), "zero_lattice");
        continue;
      }
      FwdLaunch& L = Ls[conv_i];
      void* wprep = reinterpret_cast<char*>(workspace) + ph.ws_off;
      FwdParams& p = L.p;
      p.dbg = g_fwd_dbg;
      p.dbg_mode = g_fwd_dbg_mode;
      p.wprep = wprep;
      if (prep)
        launch_weight_prep(*wt, p.n_taps, plan->tapmap_dev + tap_off, wprep, kb, p.nb, p.n_ntiles, 1, plan->pieces,
                           L.raw_f32 ? 0 : 1, cs);
      tap_off += static_cast<int>(ph.tapmap.size());
      if (ep_flags & DCONV_EP_PREP_ONLY) {
        ++conv_i;
        continue;
      }
      p.out = grad_in->data;
      p.bias = nullptr;
      p.relu = 0;
      p.add = nullptr;
      p.mask = nullptr;
      if (ep) {
        p.add = ep->add;
        p.mask = ep->mask;
        p.relu = ep->relu ? 1 : 0;
      }
      launch_fwd(L, cs, prep, 1, conv_i == 0, conv_i == n_conv - 1);
      ++conv_i;
    }
    if (ep_flags & DCONV_EP_PREP_ONLY) return;
    if (s.stride != 1) {
      const int r = dconv_zero_halo(grad_in, stream);
      if (r != DCONV_OK) fail(r, g_err);
    }
  });
}

}  // extern "C"

// ====================================================================== weight update
namespace {

struct UpdLaunch {
  UpdParams p;
  int passes;  // 1, or 3 (one A piece per pass)
  CUtensorMap map_in, map_do;
  CUtensorMap map_part;  // partials [split][tap][c_pad] rows x k_pad fp32 (UpdParams::epi_tma)
  const void* part_ptr = nullptr;  // the partial buffer map_part was encoded for
  dim3 grid;
  int stages;
  size_t smem;
  size_t ws_in, ws_do, ws_partial;  // workspace byte sizes (piece tensors, partials)
  bool split_in, split_do;
  // fp32 operands converted in shared memory (conv_upd_raw_kernel)
  bool raw = false, cat = false;
  bool tsa = false;  // single tap: A operand staged in TMEM (conv_upd_ts_kernel)
  int raw_stages = 0, pc_stages = 0;
  double est_cycles = 0;  // bf16 plans: modelled SM-cycles of the whole launch (selection only)
};

void encode_upd_maps(UpdLaunch& L, const dconv_upd_plan& pl, const dconv_act_t& in, const dconv_act_t& dout,
                     const void* in_pieces, const void* do_pieces);

// Tile selection for the split-K UPD (replaces choose_update_strategy /
// choose_spatial_blocking, planner.cpp:107-173): virtual-pixel band per stage,
// k-tile width, tap groups bounded by TMEM, split factor for >= 2 waves.
UpdLaunch plan_upd(const dconv_upd_plan& pl, const dconv_act_t& in, const dconv_act_t& dout, bool encode_maps,
                   const void* in_pieces, const void* do_pieces, float* partial, int force_nb = 0,
                   int force_unstack = -1, int force_mc = 1) {
  // bf16 operands read in place: pick the k-tile width and (for < 8 channel blocks)
  // tap stacking vs plain shifted-descriptor taps by the modelled time -- the TMA
  // row rate (27 B/clk/SM for 32 B rows) against the MMA time of each choice
  const bool bf16_ops = in.dtype == DCONV_BF16 && dout.dtype == DCONV_BF16 && pl.pieces == 1 &&
                        !DCONV_ENV("DCONV_UPD_NO_MODEL");
  if (bf16_ops && force_unstack < 0 && !(pl.has_cfg && pl.cfg.tile_nb > 0)) {
    const int kb0 = cdiv(pl.spec.K, 16), cb0 = cdiv(pl.spec.C, 16);
    const int nb_def = cdiv(kb0, cdiv(kb0, 16));
    // (un-stacked narrow multi-tap plans -- M rows past C idle, every tap through a shifted
    // descriptor -- are modelled well but measured slower on the C=64 3x3 layer: opt-in)
    const bool narrow_taps = cb0 < 8 && pl.spec.R * pl.spec.S > 1 && pl.spec.C > 8 && DCONV_ENV("DCONV_UPD_UNSTACK");
    // single-tap layers with >= 2 c-tiles: a CTA may also take two c-tiles (two
    // accumulators), staging each dO tile once for both
    const bool mc_ok = pl.spec.R * pl.spec.S == 1 && cb0 % 16 == 0 && !DCONV_ENV("DCONV_UPD_NO_MC");
    const std::array<int, 12> key = {in.n,   in.c,     in.h,       in.w,   in.halo_h, in.halo_w,
                                     dout.h, dout.w, dout.halo_h, dout.halo_w, in.dtype, dout.dtype};
    if (!g_dev_mode) {
      std::lock_guard<std::mutex> lk(pl.sel_mu);
      const auto it = pl.sel_cache.find(key);
      if (it != pl.sel_cache.end())
        return plan_upd(pl, in, dout, encode_maps, in_pieces, do_pieces, partial, it->second[0], it->second[1],
                        it->second[2]);
    }
    double best = 1e30;
    int b_nb = nb_def, b_un = 0, b_mc = 1;
    for (int un = 0; un <= (narrow_taps ? 1 : 0); ++un)
      for (int mcv = 1; mcv <= (mc_ok ? 2 : 1); ++mcv)
        for (int div : {1, 2, 4}) {
          const int nbv = nb_def / div;
          if (nbv < 1 || (div > 1 && nb_def % div) || mcv * 16 * nbv > 512) continue;
          try {
            const UpdLaunch t = plan_upd(pl, in, dout, false, nullptr, nullptr, nullptr, nbv, un, mcv);
            if (t.est_cycles > 0 && t.est_cycles < best * 0.97) {
              best = t.est_cycles;
              b_nb = nbv;
              b_un = un;
              b_mc = mcv;
            }
          } catch (...) {
          }
        }
    {
      std::lock_guard<std::mutex> lk(pl.sel_mu);
      pl.sel_cache[key] = {b_nb, b_un, b_mc};
    }
    return plan_upd(pl, in, dout, encode_maps, in_pieces, do_pieces, partial, b_nb, b_un, b_mc);
  }
  UpdLaunch L;
  std::memset(&L.p, 0, sizeof(L.p));
  UpdParams& p = L.p;
  const dconv_spec_t& s = pl.spec;
  const int pieces = pl.pieces;
  const int P = out_P(s), Q = out_Q(s);
  const int st = s.stride;
  const int cb = cdiv(s.C, 16), kb = cdiv(s.K, 16);
  const Taps& taps = pl.taps;
  L.split_in = !(in.dtype == DCONV_BF16 && pieces == 1);
  L.split_do = !(dout.dtype == DCONV_BF16 && pieces == 1);
  if (pieces == 3 && (in.dtype != DCONV_F32 || dout.dtype != DCONV_F32))
    fail(DCONV_ERR_UNSUPPORTED, "fp32-accurate math needs fp32 operands");
  p.n_img = s.N;
  p.in_cb = cb;
  p.do_cb = kb;
  p.cb_in = cb;
  p.kb_out = kb;
  p.P = P;
  p.Q = Q;
  p.stride = st;
  p.n_taps = s.R * s.S;
  p.in_row0 = -s.pad_h;
  p.in_col0 = -s.pad_w;
  const bool linear = st == 1 && s.R == 1 && s.S == 1 && s.pad_h == 0 && s.pad_w == 0 && in.halo_h == 0 &&
                      in.halo_w == 0 && dout.halo_h == 0 && dout.halo_w == 0;
  p.linear = linear ? 1 : 0;
  // tap stacking for narrow inputs (< 8 channel blocks, e.g. the 3-channel stem)
  const bool stacked = !linear && cb < 8 && s.R * s.S > 1 && force_unstack != 1;
  // C <= 8 (the 3-channel stem): only the first 8-lane chunk of each pixel is
  // non-zero, so a tap slot is one chunk and 16 taps share the 128 MMA rows
  p.half = (stacked && s.C <= 8) ? 1 : 0;
  p.stack = stacked ? (p.half ? 16 : 8 / cb) : 1;
  // bf16 in place: a c-tile of a narrow layer loads only its cb planes (the MMA's
  // rows past them read stale shared memory; those dW rows are never reduced)
  p.cb_eff = stacked ? cb : ((bf16_ops && !p.half && !DCONV_ENV("DCONV_UPD_NO_SW32")) ? std::min(8, cb) : 8);
  // k tile
  int n_kt = cdiv(kb, 16);
  p.nb = cdiv(kb, n_kt);
  if (pl.has_cfg && pl.cfg.tile_nb > 0) p.nb = std::min(pl.cfg.tile_nb, 16);
  if (force_nb > 0) p.nb = force_nb;
  const int NT = 16 * p.nb;
  const int n_ktiles = cdiv(kb, p.nb);
  const int n_ctiles = cdiv(cb, 8);
  // cross-stacking (stride-1 bf16 stacked plans, see UpdParams::xs): xs dO copies shifted
  // by 0..xs-1 columns along N, A slots = the input tile at rows 0..R-1 x columns
  // 0, xs, 2xs.. Chosen by staged planes per stage over all tap groups (the TMA row
  // rate bounds these plans): the 64-channel 3x3 takes xs = 3 (36 planes for 9 taps
  // instead of 60), the space-to-depth stem xs = 2 (16 instead of 24)
  int xs = 1;
  if (stacked && bf16_ops && !p.half && st == 1 && taps.n_phases == 1 && pieces == 1 &&
      static_cast<int>(taps.r.size()) == s.R * s.S && !DCONV_ENV("DCONV_UPD_NO_SW32") && !DCONV_ENV("DCONV_UPD_NO_XS")) {
    long long best_planes = 0;
    for (int x = 1; x <= 4; ++x) {
      if (s.S % x != 0 || x * NT > 256) continue;
      const int slots = s.R * (s.S / x);
      if (x > 1 && slots > kMaxXsSlots) continue;
      const int groups = cdiv(slots, p.stack);
      const long long planes = static_cast<long long>(slots) * cb + static_cast<long long>(groups) * x * p.nb;
      if (x == 1 || planes < best_planes) {
        best_planes = planes;
        xs = x;
      }
    }
  }
  const int nb_b = p.nb * xs;  // dO planes staged per stage
  // c-tiles per CTA (see the selector above); only the bf16 SW32 single-tap kernel path
  const int mc = (force_mc == 2 && bf16_ops && !stacked && taps.r.size() == 1 && cb % 16 == 0 && !p.half &&
                  !DCONV_ENV("DCONV_UPD_NO_SW32")) ? 2 : 1;
  p.mc = mc;
  // geometry and pipeline depth
  const int maxshift_rows = taps.r2max, s2max = taps.s2max;
  // Candidate (virtual pitch, band) geometries in preference order. A single
  // pass stages all operand pieces; fp32-accurate shapes too wide for that
  // fall back to three passes with one A piece each.
  struct Cand {
    int wsub, rows_ps, in_rows, vs, a_px, stages, passes;
    UpdStage lay;
    int pimg;  // packed images per stage (UpdParams::pimg), 0 = row bands
  };
  std::vector<Cand> cands;
  auto add = [&](int wsub, int rows_ps, int in_rows, int vs, int a_px, int pimg = 0) {
    if (!linear && (wsub * st > 256 || in_rows * st > 256 || rows_ps > 256)) return;
    if (linear && vs > 256) return;
    for (int passes : {1, 3}) {
      if (passes == 3 && pieces == 1) continue;
      const UpdStage lay = passes == 1 ? upd_stage_layout(a_px, vs, nb_b, pieces, pieces, mc)
                                       : upd_stage_layout(a_px, vs, p.nb, 1, 3);
      const int stg = std::min<int>(kMaxStages, kSmemBudget / static_cast<int>(lay.bytes));
      if (stg >= 2) cands.push_back({wsub, rows_ps, in_rows, vs, a_px, stg, passes, lay, pimg});
    }
  };
  if (linear) {
    const int want_vs = env_int("DCONV_UPD_VS", 0);  // developer mode: force the stage band
    for (int vs : {256, 128, 64, 32, 16})
      if (!want_vs || vs == want_vs) add(Q, 0, 0, vs, vs);
  } else {
    const int wmin = Q + s2max;
    const int w16 = (wmin + 15) / 16 * 16;
    int g = 16;
    while (g > 1 && wmin % g != 0) g >>= 1;
    const int base_rows = 16 / g;  // rows so that rows * wmin % 16 == 0
    std::vector<std::pair<int, int>> geo;
    if (w16 * 4 <= wmin * 5) {  // 16-aligned pitch wastes <= 25%: 1-row bands allowed
      for (int rows : {4, 2, 1}) geo.emplace_back(w16, rows);
      // taller bands stage fewer halo rows per output row (the TMA row rate bounds
      // these plans): half and whole small planes
      for (int rows : {(P + 1) / 2, P})
        if (rows > 4 && rows <= 16) geo.emplace_back(w16, rows);
    }
    for (int m : {4, 2, 1}) geo.emplace_back(wmin, base_rows * m);
    for (int rows : {2, 1}) geo.emplace_back(w16, rows);
    for (auto& gr : geo) {
      const int wsub = gr.first, rows_ps = gr.second;
      if (rows_ps > P && !(wsub == wmin && rows_ps == base_rows)) continue;  // bands taller than the image
      const int in_rows = stacked ? rows_ps : rows_ps + maxshift_rows + (s2max > 0 ? 1 : 0);
      add(wsub, rows_ps, in_rows, rows_ps * wsub, in_rows * wsub);
    }
    // packed images (UpdParams::pimg): small stride-1 planes with symmetric padding
    if (bf16_ops && !stacked && xs == 1 && st == 1 && taps.n_phases == 1 && in.halo_h == 0 && in.halo_w == 0 &&
        dout.halo_h == 0 && dout.halo_w == 0 && s.H <= 16 && s.R - 1 - s.pad_h <= s.pad_h &&
        s.S - 1 - s.pad_w <= s.pad_w && P == s.H && Q == s.W && ((s.H + s.pad_h) * (s.W + 2 * s.pad_w)) % 8 == 0 &&
        !DCONV_ENV("DCONV_UPD_NO_PIMG")) {
      const int wsub = s.W + 2 * s.pad_w, rows = s.H + s.pad_h, pitch = rows * wsub;
      for (int k : {1, 2, 4}) {
        if ((k * pitch) % 16 != 0 || k * pitch > 256) continue;
        add(wsub, rows, rows, k * pitch, (k + 1) * pitch, k);
        break;
      }
    }
  }
  const Cand* best = nullptr;
  // modelled cycles of one candidate over the whole launch (bf16 in-place plans)
  auto cand_cycles = [&](const Cand& cd) -> double {
    const int tgv = std::max(1, std::min(512 / NT, taps.taps_box));
    std::vector<int> groups;  // taps (cross-stacked: A slots) per CTA accumulator group
    if (xs > 1) {
      const int slots = s.R * (s.S / xs);
      for (int t0 = 0; t0 < slots; t0 += p.stack) groups.push_back(std::min(p.stack, slots - t0));
    } else if (stacked) {
      for (int t0 = 0; t0 < static_cast<int>(taps.r.size()); t0 += p.stack)
        groups.push_back(std::min(p.stack, static_cast<int>(taps.r.size()) - t0));
    } else {
      // (the model keeps the unbalanced 4 + 4 + 1 split it was calibrated with: fed the balanced
      // groups the plan uses, it picked slower candidates for the 28x28 and 7x7 3x3 layers)
      for (int ph = 0; ph < taps.n_phases; ++ph)
        for (int t0 = 0; t0 < taps.phase_ntaps[ph]; t0 += tgv) groups.push_back(std::min(tgv, taps.phase_ntaps[ph] - t0));
    }
    const double b_bytes = 2.0 * nb_b * cd.lay.b_plane;
    const double spi = linear ? cdiv(P * Q, cd.vs) : cd.pimg > 0 ? 1.0 / cd.pimg : cdiv(P, cd.rows_ps);
    // cycles per 128 x NT x 16 MMA: tensor time NT/2, or the shared-memory reads of its
    // operands (4 KB of A + NT x 32 B of B at ~128 B/clk) when those are longer (NT < 128)
    const double mma_unit = std::max(xs * NT / 2.0, (4096.0 + 32.0 * xs * NT) / 128.0);
    double cyc = 0;
    for (int g : groups) {
      const double a_bytes = stacked ? static_cast<double>(g) * (p.half ? 1 : 2 * p.cb_eff) * cd.lay.a_plane
                                     : 2.0 * p.cb_eff * mc * cd.lay.a_plane;
      const double mma = (stacked ? 1 : g * mc) * (cd.vs / 16.0) * mma_unit;
      cyc += std::max((a_bytes + b_bytes) / 27.0, mma) + 300.0;
    }
    return cyc * (n_ctiles / mc) * n_ktiles * spi * s.N / sm_count();
  };
  if (bf16_ops) {
    double bc = 1e30;
    for (auto& cd : cands)
      if (cd.passes == 1 && cd.stages >= 2) {
        const double c = cand_cycles(cd) * (cd.stages >= 3 ? 1.0 : 1.15);
        if (c < bc * 0.98) {
          bc = c;
          best = &cd;
        }
      }
    if (best) L.est_cycles = bc;
  }
  for (int tier = 0; tier < 4 && !best; ++tier) {
    const int want_passes = tier < 2 ? 1 : 3, want_stages = (tier % 2 == 0) ? 3 : 2;
    for (auto& cd : cands)
      if (cd.passes == want_passes && cd.stages >= want_stages) {
        best = &cd;
        break;
      }
  }
  // fp32 tensors: convert in shared memory when a raw ring (>= 2 deep) and a
  // piece ring fit; otherwise split through HBM (conv_upd_kernel)
  const bool want_raw = in.dtype == DCONV_F32 && dout.dtype == DCONV_F32 && !(pl.has_cfg && pl.cfg.stages < 0);
  if (want_raw) {
    const Cand* rb = nullptr;
    int rbest_r = 0, rbest_s = 0;
    const int tiers[3][2] = {{3, 2}, {2, 2}, {2, 1}};
    for (int tier = 0; tier < 3 && !rb; ++tier)
      for (auto& cd : cands) {
        if (cd.passes != 1) continue;
        const int a_planes = stacked ? cb : 8;
        const UpdRawLayout rl = upd_raw_layout(cd.a_px, cd.vs, p.nb, pieces, stacked ? p.stack : 1, a_planes, 1);
        const int sp = tiers[tier][1];
        const int64_t left = static_cast<int64_t>(kSmemBudget) - static_cast<int64_t>(sp) * rl.pc_slot;
        const int rr = left > 0 ? static_cast<int>(std::min<int64_t>(kMaxStages, left / rl.raw_slot)) : 0;
        if (rr >= tiers[tier][0]) {
          rb = &cd;
          rbest_r = rr;
          rbest_s = sp;
          break;
        }
      }
    if (rb) {
      best = rb;
      L.raw = true;
      L.raw_stages = rbest_r;
      L.pc_stages = rbest_s;
      if (pl.has_cfg && pl.cfg.stages > 0) L.raw_stages = std::max(2, std::min(L.raw_stages, pl.cfg.stages));
    }
  }
  // single-tap layers: A (activations) converted straight into a TMEM ring, so only
  // the raw boxes and the dO pieces occupy shared memory
  const char* tsa_env = dev_env("DCONV_UPD_TSA");  // developer mode: tests toggle it per plan
  if (want_raw && !stacked && taps.r.size() == 1 && !(tsa_env && tsa_env[0] == '0')) {
    const int acc_w = (pieces == 3 && 3 * NT <= 256) ? 3 * NT : NT;
    const int want_vs = env_int("DCONV_UPD_TSA", 0);  // > 1: force the stage band (experiments)
    for (auto& cd : cands) {
      if (cd.passes != 1 || (want_vs > 1 && cd.vs != want_vs)) continue;
      const UpdRawLayout rl = upd_raw_layout(cd.a_px, cd.vs, p.nb, pieces, 1, 8, 1);
      const int ring = pieces * cd.vs / 2;
      const int ps = std::min(4, (512 - acc_w) / ring);
      if (ps < 2) continue;
      const int64_t left = static_cast<int64_t>(kSmemBudget) - static_cast<int64_t>(ps) * upd_ts_pc_slot(cd.vs, p.nb, pieces);
      const int rr = left > 0 ? static_cast<int>(std::min<int64_t>(kMaxStages, left / rl.raw_slot)) : 0;
      if (rr < 3) continue;
      best = &cd;
      L.raw = L.tsa = true;
      L.raw_stages = rr;
      L.pc_stages = ps;
      if (pl.has_cfg && pl.cfg.stages > 0) L.raw_stages = std::max(2, std::min(L.raw_stages, pl.cfg.stages));
      break;
    }
  }
  if (!best) fail(DCONV_ERR_PLAN_INFEASIBLE, "no weight-update tile fits shared memory / TMA box limits");
  if (L.raw) L.split_in = L.split_do = false;
  p.wsub = best->wsub;
  p.rows_ps = best->rows_ps;
  p.in_rows = best->in_rows;
  p.vs = best->vs;
  p.a_px = best->a_px;
  int stages = best->stages;
  const UpdStage layout = best->lay;
  L.passes = best->passes;
  p.stages_per_img = linear ? cdiv(P * Q, p.vs) : cdiv(P, p.rows_ps);
  if (stages < 2) fail(DCONV_ERR_PLAN_INFEASIBLE, "weight-update stage does not fit shared memory");
  if (pl.has_cfg && pl.cfg.stages > 0) stages = std::min(stages, pl.cfg.stages);
  p.stages_total = s.N * p.stages_per_img;
  if (best->pimg > 0) {  // a stage = pimg whole images (the last group may run past N: zero fill)
    p.pimg = best->pimg;
    p.img_pitch = best->rows_ps * best->wsub;
    p.stages_per_img = 1;
    p.stages_total = cdiv(s.N, p.pimg);
  }
  for (size_t t = 0; t < taps.r.size(); ++t) {
    p.tap_shift[t] = taps.r2[t] * p.wsub + taps.s2[t];
    p.tap_src[t] = taps.r[t] * s.S + taps.s[t];
  }
  for (int i = 0; i < taps.n_phases; ++i) {
    p.phase_row[i] = taps.phase_row[i];
    p.phase_col[i] = taps.phase_col[i];
  }
  for (int ph = 0; ph < taps.n_phases; ++ph)
    for (int t = 0; t < taps.phase_ntaps[ph]; ++t) p.tap_ph[taps.phase_tap0[ph] + t] = ph;
  for (size_t t = 0; t < taps.r.size(); ++t) {
    p.tap_r2[t] = taps.r2[t];
    p.tap_s2[t] = taps.s2[t];
  }
  p.n_tgroups = 0;
  if (xs > 1) {
    // cross-stacked: A slots (r, 0 / xs / 2xs ..) in groups of `stack`; N holds xs dO copies
    p.xs = xs;
    p.xs_S = s.S;
    p.tg = xs;
    int n_slots = 0;
    for (int r = 0; r < s.R; ++r)
      for (int sa = 0; sa < s.S; sa += xs) {
        p.xs_slot_r[n_slots] = r;
        p.xs_slot_s[n_slots] = sa;
        ++n_slots;
      }
    for (int t0 = 0; t0 < n_slots; t0 += p.stack) {
      p.tg_phase[p.n_tgroups] = 0;
      p.tg_tap0[p.n_tgroups] = t0;
      p.tg_ntaps[p.n_tgroups] = std::min(p.stack, n_slots - t0);
      ++p.n_tgroups;
    }
  } else if (stacked) {
    // one accumulator per CTA holding `stack` consecutive (phase-sorted) taps
    p.tg = 1;
    for (int t0 = 0; t0 < static_cast<int>(taps.r.size()); t0 += p.stack) {
      if (p.n_tgroups >= kMaxTapGroups) fail(DCONV_ERR_UNSUPPORTED, "too many tap groups");
      p.tg_phase[p.n_tgroups] = p.tap_ph[t0];
      p.tg_tap0[p.n_tgroups] = t0;
      p.tg_ntaps[p.n_tgroups] = std::min(p.stack, static_cast<int>(taps.r.size()) - t0);
      ++p.n_tgroups;
    }
  } else {
    // tap groups: per phase, <= 512 TMEM columns of accumulators. The
    // concatenated-piece MMA (3 column groups per tap) is used when every tap
    // of a phase still fits and N = 3 NT is a legal MMA width.
    L.cat = L.raw && pieces == 3 && 3 * NT <= 256 && 3 * NT * taps.taps_box <= 512;
    p.tg = std::max(1, std::min(512 / (L.cat ? 3 * NT : NT), taps.taps_box));
    // The launch is one wave of (tile, tap group, split) CTAs, so its time is the largest
    // group's: a phase's taps are spread evenly over its groups (3x3 with four accumulators
    // per CTA: 3 + 3 + 3 instead of 4 + 4 + 1, whose lone-tap CTAs staged the same operands
    // for a quarter of the MMAs)
    for (int ph = 0; ph < taps.n_phases; ++ph) {
      const int nt_ph = taps.phase_ntaps[ph], ng = cdiv(nt_ph, p.tg);
      for (int i = 0, t0 = 0; i < ng; ++i) {
        if (p.n_tgroups >= kMaxTapGroups) fail(DCONV_ERR_UNSUPPORTED, "too many tap groups");
        const int cnt = nt_ph / ng + (i < nt_ph % ng ? 1 : 0);
        p.tg_phase[p.n_tgroups] = ph;
        p.tg_tap0[p.n_tgroups] = taps.phase_tap0[ph] + t0;
        p.tg_ntaps[p.n_tgroups] = cnt;
        t0 += cnt;
        ++p.n_tgroups;
      }
    }
  }
  // split-K factor (choose_update_strategy analog, planner.cpp:54-143: the same
  // trade-off of partial-copy traffic against parallelism, for 148 SMs):
  // minimise max(MMA time over the busy SMs, HBM time of operands + partials
  // written and re-read by the reduce); one CTA per SM (smem-bound)
  const int tiles = (n_ctiles / mc) * p.n_tgroups * n_ktiles;
  const int sms = sm_count();
  const double op_bytes = (in.dtype == DCONV_BF16 ? 2.0 : 4.0) * (static_cast<double>(act_elems(in)) +
                                                                  static_cast<double>(act_elems(dout)) * (n_ctiles / mc));
  const double dw_part = 4.0 * p.n_taps * (n_ctiles * 128.0) * (n_ktiles * NT);
  const double mma_flops = 2.0 * (n_ctiles * 128.0) * (n_ktiles * NT) * p.n_taps * static_cast<double>(p.stages_total) *
                           p.vs * (pieces == 3 ? 6.0 : 1.0);
  const double sm_rate = 4.5e12;  // dense bf16 MMA FLOP/s per SM at these tile shapes (~50 % of 1332 TF / 148)
  int splits = 1;
  double best_t = 1e30;
  const int max_splits = std::max(1, std::min(cdiv(2 * sms, tiles), std::max(1, p.stages_total / 2)));
  for (int sp = 1; sp <= max_splits; ++sp) {
    const int ctas = tiles * sp;
    const int waves = cdiv(ctas, sms);
    const double t_mma = mma_flops / ctas * waves / sm_rate;
    // HBM time, also bounded by what the busy SMs can pull (~30 GB/s each through the TMA rings)
    const double bytes = op_bytes + (sp > 1 ? 2.0 : 1.0) * sp * dw_part;
    const double t_mem = std::max(bytes / 5.5e12, bytes / (std::min(ctas, sms) * 30.0e9));
    const double t = std::max(t_mma, t_mem);
    if (t < best_t * 0.98) {
      best_t = t;
      splits = sp;
    }
  }
  if (pl.has_cfg && pl.cfg.upd_splits > 0) splits = std::min(pl.cfg.upd_splits, p.stages_total);
  if (DCONV_ENV("DCONV_UPD_SPLITS")) splits = std::max(1, std::min(env_int("DCONV_UPD_SPLITS", 1), p.stages_total));
  p.splits = splits;
  // fp32-accurate: bound the accumulation chain per TMEM accumulator (the tensor
  // core truncates each fp32 accumulate; a 1-split cfg2 chain of 6272 k-steps drifted
  // to 4.8e-4 of the output RMS, 74 splits = 85 k-steps to 5e-6). Longer chains are
  // cut into periods of <= kDrainKsteps k-steps whose sums are added in fp32.
  {
    // (counted in accumulate steps into the hi*hi accumulator: one per k-step when the
    // hi*hi product has its own column group (CAT), six when all six products share one)
    constexpr int kDrainSteps = 96;
    const int steps = (p.vs / 16) * (L.cat ? 1 : 6);
    const int per_split = cdiv(p.stages_total, splits);
    p.drain = 0;
    p.drain_bufs = 1;
    if (pieces == 3 && per_split * steps > kDrainSteps) {
      p.drain = std::max(1, kDrainSteps / steps);
      const int acc_w = (L.cat ? 3 : 1) * NT;
      if (L.tsa) {
        const int ring = pieces * p.vs / 2;
        const int ps2 = std::min(4, (512 - 2 * acc_w) / ring);
        if (ps2 >= 2) {
          p.drain_bufs = 2;
          L.pc_stages = std::min(L.pc_stages, ps2);
        }
      } else if (L.raw) {
        if (2 * p.tg * acc_w <= 512) p.drain_bufs = 2;
      } else if (2 * std::max(p.tg, mc) * NT <= 512) {
        p.drain_bufs = 2;
      }
    }
  }
  p.c_pad = n_ctiles * 128;
  p.k_pad = n_ktiles * NT;
  p.partial = partial;
  L.grid = dim3(static_cast<unsigned>((n_ctiles / mc) * p.n_tgroups), static_cast<unsigned>(n_ktiles),
                static_cast<unsigned>(splits));
  L.stages = stages;
  L.smem = static_cast<size_t>(stages) * layout.bytes;
  if (L.raw) {
    const UpdRawLayout rl = upd_raw_layout(p.a_px, p.vs, p.nb, pieces, stacked ? p.stack : 1, p.cb_eff, L.raw_stages);
    L.smem = static_cast<size_t>(rl.pc_off) +
             static_cast<size_t>(L.pc_stages) * (L.tsa ? upd_ts_pc_slot(p.vs, p.nb, pieces) : rl.pc_slot);
  }
  L.ws_in = L.split_in ? align256(static_cast<size_t>(pieces) * act_elems(in) * 2) : 0;
  L.ws_do = L.split_do ? align256(static_cast<size_t>(pieces) * act_elems(dout) * 2) : 0;
  L.ws_partial = align256(static_cast<size_t>(splits) * p.n_taps * p.c_pad * p.k_pad * sizeof(float));
  if (!L.raw) {
    p.sw32 = (pieces == 1 && !L.split_in && !L.split_do && !p.half && !DCONV_ENV("DCONV_UPD_NO_SW32")) ? 1 : 0;
    // cp.async loader warps in place of the TMA box loads: opt-in experiment only
    // (DCONV_UPD_LSU=1). Measured 2-5x SLOWER than the TMA boxes on every ResNet-50
    // layer (per-chunk address arithmetic on six warps, and the loaders share the
    // MMA warp's schedulers), although a bare cp.async stream reaches ~45-60 B/clk/SM
    // (tools/probe_cpasync.cu) against the TMA's ~27 B/clk/SM for 32 B rows.
    p.lsu = (p.sw32 && p.mc == 1 && L.stages > kUpdLsuDepth && DCONV_ENV("DCONV_UPD_LSU")) ? 1 : 0;
    // linear plans over planes of 4k pixels, 32-pixel stages: 128 B rows (see UpdParams::sw32)
    if (p.sw32 && !p.lsu && p.linear && p.stack == 1 && p.vs % 32 == 0 && (in.h * in.w) % 4 == 0 &&
        (dout.h * dout.w) % 4 == 0 && !DCONV_ENV("DCONV_UPD_NO_SW128"))
      p.sw32 = 2;
  }
  // partials through TMA stores: bf16 single-period plans whose epilogue warps each own
  // 32 consecutive partial rows of one tap (staging: 16 KB of the idle operand ring)
  p.epi_tma = (!L.raw && !L.tsa && pieces == 1 && p.sw32 && !p.lsu && p.drain == 0 &&
               (p.stack == 1 || (!p.half && (16 * p.cb_eff) % 32 == 0)) && L.smem >= 16384 &&
               !DCONV_ENV("DCONV_UPD_NO_EPI_TMA"))
                  ? 1
                  : 0;
  if (!encode_maps) return L;
  encode_upd_maps(L, pl, in, dout, in_pieces, do_pieces);
  return L;
}

// operand tensor maps of a resolved weight-update launch (and the cp.async
// loader pointers of developer-mode lsu plans)
void encode_upd_maps(UpdLaunch& L, const dconv_upd_plan& pl, const dconv_act_t& in, const dconv_act_t& dout,
                     const void* in_pieces, const void* do_pieces) {
  UpdParams& p = L.p;
  const dconv_spec_t& s = pl.spec;
  const int pieces = pl.pieces;
  const int st = s.stride;
  const int cb = cdiv(s.C, 16), kb = cdiv(s.K, 16);
  const bool linear = p.linear != 0;
  // operand maps over bf16 piece tensors (piece-major planes)
  auto act_map = [&](const dconv_act_t& a, const void* data, int chans_blocks, bool is_in) {
    const int hp = a.h + 2 * a.halo_h, wp = a.w + 2 * a.halo_w;
    const uint64_t planes = static_cast<uint64_t>(is_in ? pieces : pieces) * a.n * chans_blocks;
    if (p.sw32) {  // bf16 tensors in place: 32 B pixel rows, SWIZZLE_32B (MN-major SW32 operands)
      const CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_32B;
      if (linear && p.sw32 == 2) {  // 128 B rows of four pixels, SWIZZLE_128B
        const uint64_t dims[3] = {64, static_cast<uint64_t>(a.h) * a.w / 4, planes};
        const uint64_t strides[2] = {128, static_cast<uint64_t>(a.h) * a.w * 32};
        const uint32_t box[3] = {64, static_cast<uint32_t>(p.vs / 4),
                                 static_cast<uint32_t>(is_in ? p.cb_eff * p.mc : p.nb)};
        return encode(1, 3, data, dims, strides, box, nullptr, is_in ? "upd input linear sw128" : "upd dO linear sw128",
                      CU_TENSOR_MAP_SWIZZLE_128B);
      }
      if (linear) {
        const uint64_t dims[3] = {16, static_cast<uint64_t>(a.h) * a.w, planes};
        const uint64_t strides[2] = {32, static_cast<uint64_t>(a.h) * a.w * 32};
        const uint32_t box[3] = {16, static_cast<uint32_t>(p.vs),
                                 static_cast<uint32_t>(is_in ? p.cb_eff * p.mc : p.nb)};
        return encode(1, 3, data, dims, strides, box, nullptr, is_in ? "upd input linear sw32" : "upd dO linear sw32",
                      swz);
      }
      const char* base = reinterpret_cast<const char*>(data) + (static_cast<uint64_t>(a.halo_h) * wp + a.halo_w) * 32;
      if (p.pimg > 0) {  // packed images: dims {16, w, h, images, channel blocks}, images inside the planes
        const uint64_t cbs = static_cast<uint64_t>(chans_blocks);
        const uint64_t dims5[5] = {16, static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h),
                                   static_cast<uint64_t>(a.n), cbs};
        const uint64_t plane_b = static_cast<uint64_t>(wp) * hp * 32;
        const uint64_t strides5[4] = {32, static_cast<uint64_t>(wp) * 32, plane_b * cbs, plane_b};
        const uint32_t box5[5] = {16, static_cast<uint32_t>(p.wsub), static_cast<uint32_t>(p.rows_ps),
                                  static_cast<uint32_t>(is_in ? p.pimg + 1 : p.pimg),
                                  static_cast<uint32_t>(is_in ? p.cb_eff * p.mc : p.nb)};
        return encode(1, 5, base, dims5, strides5, box5, nullptr, is_in ? "upd input packed" : "upd dO packed", swz);
      }
      const uint64_t dims[4] = {16, static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h), planes};
      const uint64_t strides3[3] = {32, static_cast<uint64_t>(wp) * 32, static_cast<uint64_t>(wp) * hp * 32};
      if (is_in) {
        const uint32_t box[4] = {16, static_cast<uint32_t>(p.wsub * st), static_cast<uint32_t>(p.in_rows * st),
                                 static_cast<uint32_t>(p.cb_eff * p.mc)};
        const uint32_t estr[4] = {1, static_cast<uint32_t>(st), static_cast<uint32_t>(st), 1};
        return encode(1, 4, base, dims, strides3, box, estr, "upd input rows sw32", swz);
      }
      const uint32_t box[4] = {16, static_cast<uint32_t>(p.wsub), static_cast<uint32_t>(p.rows_ps),
                               static_cast<uint32_t>(p.nb)};
      return encode(1, 4, base, dims, strides3, box, nullptr, "upd dO rows sw32", swz);
    }
    if (linear) {
      const uint64_t dims[4] = {8, static_cast<uint64_t>(a.h) * a.w, 2, planes};
      const uint64_t strides[3] = {32, 16, static_cast<uint64_t>(a.h) * a.w * 32};
      const uint32_t box[4] = {8, static_cast<uint32_t>(p.vs), 2, static_cast<uint32_t>(is_in ? 8 : p.nb)};
      return encode(1, 4, data, dims, strides, box, nullptr, is_in ? "upd input linear" : "upd dO linear");
    }
    const char* base = reinterpret_cast<const char*>(data) + (static_cast<uint64_t>(a.halo_h) * wp + a.halo_w) * 32;
    const uint64_t dims[5] = {8, static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h), 2, planes};
    const uint64_t strides[4] = {32, static_cast<uint64_t>(wp) * 32, 16, static_cast<uint64_t>(wp) * hp * 32};
    const uint32_t box_in[5] = {8, static_cast<uint32_t>(p.wsub * st), static_cast<uint32_t>(p.in_rows * st),
                                p.half ? 1u : 2u, static_cast<uint32_t>(p.cb_eff)};
    const uint32_t box_do[5] = {8, static_cast<uint32_t>(p.wsub), static_cast<uint32_t>(p.rows_ps), 2,
                                static_cast<uint32_t>(p.nb)};
    const uint32_t estr_in[5] = {1, static_cast<uint32_t>(st), static_cast<uint32_t>(st), 1, 1};
    return is_in ? encode(1, 5, base, dims, strides, box_in, estr_in, "upd input rows")
                 : encode(1, 5, base, dims, strides, box_do, nullptr, "upd dO rows");
  };
  // raw fp32 maps: 64 B pixel rows, SWIZZLE_64B (converters read them swizzled)
  auto raw_map = [&](const dconv_act_t& a, bool is_in) {
    const int hp = a.h + 2 * a.halo_h, wp = a.w + 2 * a.halo_w;
    const uint64_t planes = static_cast<uint64_t>(a.n) * (is_in ? cb : kb);
    const CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B;
    if (linear) {
      const uint64_t dims[3] = {16, static_cast<uint64_t>(a.h) * a.w, planes};
      const uint64_t strides[2] = {64, static_cast<uint64_t>(a.h) * a.w * 64};
      const uint32_t box[3] = {16, static_cast<uint32_t>(p.vs), static_cast<uint32_t>(is_in ? 8 : p.nb)};
      return encode(0, 3, a.data, dims, strides, box, nullptr, is_in ? "upd input linear f32" : "upd dO linear f32",
                    swz);
    }
    const char* base = reinterpret_cast<const char*>(a.data) + (static_cast<uint64_t>(a.halo_h) * wp + a.halo_w) * 64;
    const uint64_t dims[4] = {16, static_cast<uint64_t>(a.w), static_cast<uint64_t>(a.h), planes};
    const uint64_t strides[3] = {64, static_cast<uint64_t>(wp) * 64, static_cast<uint64_t>(wp) * hp * 64};
    if (is_in) {
      const uint32_t box[4] = {16, static_cast<uint32_t>(p.wsub * st), static_cast<uint32_t>(p.in_rows * st),
                               static_cast<uint32_t>(p.cb_eff)};
      const uint32_t estr[4] = {1, static_cast<uint32_t>(st), static_cast<uint32_t>(st), 1};
      return encode(0, 4, base, dims, strides, box, estr, "upd input rows f32", swz);
    }
    const uint32_t box[4] = {16, static_cast<uint32_t>(p.wsub), static_cast<uint32_t>(p.rows_ps),
                             static_cast<uint32_t>(p.nb)};
    return encode(0, 4, base, dims, strides, box, nullptr, "upd dO rows f32", swz);
  };
  if (L.raw) {
    L.map_in = raw_map(in, true);
    L.map_do = raw_map(dout, false);
    return;
  }
  if (p.lsu) {
    const int ihp = in.h + 2 * in.halo_h, iwp = in.w + 2 * in.halo_w;
    const int dhp = dout.h + 2 * dout.halo_h, dwp = dout.w + 2 * dout.halo_w;
    p.in_ptr = reinterpret_cast<const char*>(in_pieces) + (static_cast<int64_t>(in.halo_h) * iwp + in.halo_w) * 32;
    p.do_ptr = reinterpret_cast<const char*>(do_pieces) + (static_cast<int64_t>(dout.halo_h) * dwp + dout.halo_w) * 32;
    p.in_h = in.h;
    p.in_w = in.w;
    p.in_wp = iwp;
    p.in_plane = static_cast<long long>(ihp) * iwp;
    p.do_h = dout.h;
    p.do_w = dout.w;
    p.do_wp = dwp;
    p.do_plane = static_cast<long long>(dhp) * dwp;
  }
  L.map_in = act_map(in, in_pieces, cb, true);
  L.map_do = act_map(dout, do_pieces, kb, false);
}

}  // namespace

struct UpdEntry {
  UpdLaunch L;  // maps encoded for the pointers below
  const void* in_ptr = nullptr;
  const void* do_ptr = nullptr;
  bool maps = false;
  std::string desc;
};

namespace {

std::string json_upd(const UpdLaunch& L, int pieces) {
  char buf[640];
  std::snprintf(buf, sizeof(buf),
                "{\"mode\":\"%s\",\"wsub\":%d,\"rows_ps\":%d,\"vs\":%d,\"a_px\":%d,\"nb\":%d,\"tap_groups\":%d,"
                "\"tg\":%d,\"splits\":%d,\"stages\":%d,\"smem\":%zu,\"grid\":[%u,%u,%u],\"pieces\":%d,\"passes\":%d,"
                "\"smem_convert\":%d,\"raw_stages\":%d,\"pc_stages\":%d,\"cat\":%d,\"a_in_tmem\":%d,\"drain\":%d,"
                "\"drain_bufs\":%d,\"sw32\":%d,\"xs\":%d,\"pimg\":%d,\"epi_tma\":%d}",
                L.p.linear ? "linear" : "rows", L.p.wsub, L.p.rows_ps, L.p.vs, L.p.a_px, L.p.nb, L.p.n_tgroups,
                L.p.tg, L.p.splits, L.stages, L.smem, L.grid.x, L.grid.y, L.grid.z, pieces, L.passes,
                L.raw ? 1 : 0, L.raw_stages, L.pc_stages, L.cat ? 1 : 0, L.tsa ? 1 : 0, L.p.drain, L.p.drain_bufs,
                L.p.sw32, L.p.xs, L.p.pimg, L.p.epi_tma);
  return buf;
}

// the weight-update plan's resolved launch for (in, grad_out) geometry (caller holds pl->mu)
UpdEntry& upd_entry(dconv_upd_plan* pl, const dconv_act_t& in, const dconv_act_t& dout) {
  const GeoKey key = geo_key(in, dout);
  auto it = pl->cache.find(key);
  if (it != pl->cache.end()) {
    if (!g_dev_mode) return *it->second;
    delete it->second;
    pl->cache.erase(it);
  }
  auto* e = new UpdEntry();
  e->L = plan_upd(*pl, in, dout, false, nullptr, nullptr, nullptr);
  e->desc = json_upd(e->L, pl->pieces);
  pl->cache[key] = e;
  return *e;
}

void launch_split(const dconv_act_t& a, void* dst, int pieces, cudaStream_t cs) {
  const int64_t n = act_elems(a);
  if (a.dtype == DCONV_F32) {
    split_pieces_kernel<<<grid1d(n), 256, 0, cs>>>(reinterpret_cast<const float*>(a.data),
                                                   reinterpret_cast<__nv_bfloat16*>(dst), n, pieces);
  } else {
    fail(DCONV_ERR_UNSUPPORTED, "bf16 operands with fp32-accurate math");
  }
  cuda_check(cudaGetLastError(), "split_pieces");
}

}  // namespace

extern "C" {

int dconv_upd_plan_create(const dconv_spec_t* spec, const dconv_engine_config_t* cfg, int math,
                          dconv_upd_plan_t* plan) {
  dconv_upd_plan* pl = nullptr;
  const int st = guarded([&] {
    if (!spec || !plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null argument");
    validate_spec(*spec);
    pl = new dconv_upd_plan();
    pl->spec = *spec;
    if (spec->vlen != 16) {
      const dconv_spec_t s16 = spec16(*spec);
      const int rc = dconv_upd_plan_create(&s16, cfg, math, &pl->inner);
      if (rc != DCONV_OK) fail(rc, g_err);
      pl->math = math;
      pl->pieces = math_pieces(math);
      *plan = pl;
      return;
    }
    pl->math = math;
    pl->pieces = math_pieces(math);
    pl->has_cfg = cfg != nullptr;
    if (cfg) pl->cfg = *cfg;
    pl->taps = phase_taps(spec->R, spec->S, spec->stride);
    *plan = pl;
  });
  if (st != DCONV_OK && pl) {
    if (pl->inner) dconv_upd_plan_destroy(pl->inner);
    delete pl;
  }
  return st;
}

void dconv_upd_plan_destroy(dconv_upd_plan_t plan) {
  if (!plan) return;
  if (plan->inner) dconv_upd_plan_destroy(plan->inner);
  for (auto& kv : plan->cache) delete kv.second;
  delete plan;
}

static dconv_act_t default_act(const dconv_spec_t& s, bool grad, int dtype) {
  dconv_act_t a;
  std::memset(&a, 0, sizeof(a));
  a.data = reinterpret_cast<void*>(256);
  a.n = s.N;
  a.c = grad ? s.K : s.C;
  a.h = grad ? out_P(s) : s.H;
  a.w = grad ? out_Q(s) : s.W;
  a.vlen = 16;
  a.halo_h = grad ? 0 : s.pad_h;
  a.halo_w = grad ? 0 : s.pad_w;
  a.dtype = dtype;
  return a;
}

int dconv_upd_splits(dconv_upd_plan_t plan) {
  if (!plan) return -1;
  if (plan->inner) return dconv_upd_splits(plan->inner);
  int v = -1;
  guarded([&] {
    const int dt = plan->pieces == 3 ? DCONV_F32 : DCONV_BF16;
    std::lock_guard<std::mutex> lk(plan->mu);
    v = upd_entry(plan, default_act(plan->spec, false, dt), default_act(plan->spec, true, dt)).L.p.splits;
  });
  return v;
}

int dconv_upd_plan_describe(dconv_upd_plan_t plan, char* buf, size_t len) {
  if (plan && plan->inner) return dconv_upd_plan_describe(plan->inner, buf, len);
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    std::lock_guard<std::mutex> lk(plan->mu);
    copy_out(plan->last_desc ? *plan->last_desc : std::string("{\"tile\":\"chosen at first execute\"}"), buf, len);
  });
}

size_t dconv_upd_workspace_bytes(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out) {
  if (!plan || !in || !grad_out) return 0;
  if (plan->inner) {  // twin's workspace + 16-lane input (halo = pad), dO (halo 0), dW
    const dconv_spec_t& s = plan->spec;
    const dconv_act_t in16 = act_as16(*in, reinterpret_cast<void*>(256), s.pad_h, s.pad_w);
    const dconv_act_t go16 = act_as16(*grad_out, reinterpret_cast<void*>(256), 0, 0);
    const dconv_wt_t w{nullptr, s.K, s.C, s.R, s.S, 16, DCONV_F32};
    return align256(dconv_upd_workspace_bytes(plan->inner, &in16, &go16)) + act_bytes(in16) + act_bytes(go16) +
           wt_bytes(w);
  }
  size_t v = 0;
  guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    const UpdLaunch& L = upd_entry(plan, *in, *grad_out).L;
    v = L.ws_in + L.ws_do + L.ws_partial;
  });
  return v;
}

int dconv_upd_launches(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out) {
  if (!plan || !in || !grad_out) return 0;
  if (plan->inner) {
    const dconv_act_t in16 = act_as16(*in, in->data, plan->spec.pad_h, plan->spec.pad_w);
    const dconv_act_t go16 = act_as16(*grad_out, grad_out->data, 0, 0);
    return dconv_upd_launches(plan->inner, &in16, &go16) + 3;
  }
  int v = 0;
  guarded([&] {
    std::lock_guard<std::mutex> lk(plan->mu);
    const UpdLaunch& L = upd_entry(plan, *in, *grad_out).L;
    v = 1 + L.passes + (L.split_in ? 1 : 0) + (L.split_do ? 1 : 0);
  });
  return v;
}

int dconv_weight_update(dconv_upd_plan_t plan, const dconv_act_t* in, const dconv_act_t* grad_out,
                        const dconv_wt_t* grad_w, int accumulate, void* workspace, dconv_stream_t stream) {
  return guarded([&] {
    if (!plan) fail(DCONV_ERR_INVALID_ARGUMENT, "null plan");
    check_act(in, "weight_update input");
    check_act(grad_out, "weight_update grad_out");
    check_wt(grad_w, "weight_update grad_w");
    if (!workspace) fail(DCONV_ERR_INVALID_ARGUMENT, "weight_update: null workspace");
    const dconv_spec_t& s = plan->spec;
    const int P = out_P(s), Q = out_Q(s);
    // propagation.cpp:383-393
    if (in->n != s.N || in->c != s.C || in->h != s.H || in->w != s.W || in->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "weight_update: input does not match the layer spec");
    if (grad_out->n != s.N || grad_out->c != s.K || grad_out->h != P || grad_out->w != Q ||
        grad_out->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "weight_update: grad_out does not match the layer spec");
    if (grad_w->k != s.K || grad_w->c != s.C || grad_w->r != s.R || grad_w->s != s.S || grad_w->vlen != s.vlen)
      fail(DCONV_ERR_SHAPE_MISMATCH, "weight_update: grad_w does not match the layer spec");
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (plan->inner) {  // vlen != 16: re-block around the 16-lane twin
      if (in->dtype != grad_out->dtype) fail(DCONV_ERR_UNSUPPORTED, "vlen != 16: input and grad_out share one dtype");
      const dconv_act_t in16p = act_as16(*in, reinterpret_cast<void*>(256), s.pad_h, s.pad_w);
      const dconv_act_t go16p = act_as16(*grad_out, reinterpret_cast<void*>(256), 0, 0);
      char* w8 = reinterpret_cast<char*>(workspace) + align256(dconv_upd_workspace_bytes(plan->inner, &in16p, &go16p));
      const dconv_act_t in16 = act_as16(*in, w8, s.pad_h, s.pad_w);
      const dconv_act_t go16 = act_as16(*grad_out, w8 + act_bytes(in16), 0, 0);
      const dconv_wt_t dw16 = wt_as16(*grad_w, w8 + act_bytes(in16) + act_bytes(go16), grad_w->dtype);
      launch_reblock_act(*in, in16, 0, cs);
      launch_reblock_act(*grad_out, go16, 0, cs);
      const int rc = dconv_weight_update(plan->inner, &in16, &go16, &dw16, 0, workspace, stream);
      if (rc != DCONV_OK) fail(rc, g_err);
      launch_reblock_wt(dw16, *grad_w, accumulate ? 1 : 0, cs);
      return;
    }
    char* ws = reinterpret_cast<char*>(workspace);
    UpdLaunch L;
    void* in_pc = nullptr;
    void* do_pc = nullptr;
    {
      std::lock_guard<std::mutex> lk(plan->mu);
      UpdEntry& e = upd_entry(plan, *in, *grad_out);
      in_pc = e.L.split_in ? ws : in->data;
      do_pc = e.L.split_do ? ws + e.L.ws_in : grad_out->data;
      if (!e.maps || e.in_ptr != in_pc || e.do_ptr != do_pc) {
        encode_upd_maps(e.L, *plan, *in, *grad_out, in_pc, do_pc);
        e.in_ptr = in_pc;
        e.do_ptr = do_pc;
        e.maps = true;
      }
      const void* part = ws + e.L.ws_in + e.L.ws_do;
      if (e.L.p.epi_tma && e.L.part_ptr != part) {  // partial rows x k_pad fp32, 32 x 16 boxes
        const UpdParams& q = e.L.p;
        const uint64_t dims[2] = {static_cast<uint64_t>(q.k_pad),
                                  static_cast<uint64_t>(q.splits) * q.n_taps * q.c_pad};
        const uint64_t strides[1] = {static_cast<uint64_t>(q.k_pad) * 4};
        const uint32_t box[2] = {16, 32};
        e.L.map_part = encode(0, 2, part, dims, strides, box, nullptr, "upd partials", CU_TENSOR_MAP_SWIZZLE_64B);
        e.L.part_ptr = part;
      }
      L = e.L;
      plan->last_desc = &e.desc;
    }
    float* partial = reinterpret_cast<float*>(ws + L.ws_in + L.ws_do);
    L.p.partial = partial;
    L.p.dbg_mode = g_fwd_dbg_mode;
    if (L.split_in) launch_split(*in, in_pc, plan->pieces, cs);
    if (L.split_do) launch_split(*grad_out, do_pc, plan->pieces, cs);
    bool opened = false;  // profiling bracket opens right before the first conv kernel
    auto go = [&](auto kern, int a_base, int acc) {
      ensure_smem(kern, L.smem);
      if (!opened) prof_begin(2, cs), opened = true;
      kern<<<L.grid, kFwdThreads, L.smem, cs>>>(L.map_in, L.map_do, L.map_part, L.p, L.stages, a_base, acc);
      cuda_check(cudaGetLastError(), "conv_upd_kernel launch");
    };
    auto go_raw = [&](auto kern) {
      ensure_smem(kern, L.smem);
      if (!opened) prof_begin(2, cs), opened = true;
      kern<<<L.grid, (L.tsa ? kUpdTsWarps : kUpdRawWarps) * 32, L.smem, cs>>>(L.map_in, L.map_do, L.p, L.raw_stages,
                                                                             L.pc_stages);
      cuda_check(cudaGetLastError(), "conv_upd_raw_kernel launch");
    };
    if (L.tsa) {
      if (plan->pieces == 1)
        go_raw(conv_upd_ts_kernel<1, false>);
      else if (L.cat)
        go_raw(conv_upd_ts_kernel<3, true>);
      else
        go_raw(conv_upd_ts_kernel<3, false>);
    } else if (L.raw) {
      if (plan->pieces == 1)
        go_raw(conv_upd_raw_kernel<1, false>);
      else if (L.cat)
        go_raw(conv_upd_raw_kernel<3, true>);
      else
        go_raw(conv_upd_raw_kernel<3, false>);
    } else if (plan->pieces == 1) {
      go(conv_upd_kernel<1, 1>, 0, 0);
    } else if (L.passes == 1) {
      go(conv_upd_kernel<3, 3>, 0, 0);
    } else {
      go(conv_upd_kernel<1, 3>, 0, 0);
      go(conv_upd_kernel<1, 2>, 1, 1);
      go(conv_upd_kernel<1, 1>, 2, 1);
    }
    prof_end(2, cs);
    const int cb = cdiv(s.C, 16), kb = cdiv(s.K, 16);
    const int64_t total = static_cast<int64_t>(kb) * cb * s.R * s.S * 64;  // k quads
    {
      // programmatic dependent launch: the reduce waits (griddepcontrol.wait) for the
      // update kernel that precedes it on this stream, before it reads the partials
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr.val.programmaticStreamSerializationAllowed = g_prof ? 0 : 1;
      cudaLaunchConfig_t lc = {};
      // split groups per element: enough memory-level parallelism for many splits,
      // all 256 threads on distinct elements when there are few
      const int G = L.p.splits >= 24 ? kRedGroups : L.p.splits >= 8 ? 2 : 1;
      const int TX = G == 1 ? 256 : 64;  // (the group sums are exchanged through [G][64] float4)
      lc.gridDim = dim3(static_cast<unsigned>(cdiv64(total, TX)), 1, 1);
      lc.blockDim = dim3(TX, G, 1);
      lc.stream = cs;
      lc.attrs = &attr;
      lc.numAttrs = 1;
      cuda_check(cudaLaunchKernelEx(&lc, upd_reduce_kernel, static_cast<const float*>(partial), L.p.splits,
                                    s.R * s.S, L.p.c_pad, L.p.k_pad, s.C, s.K, cb, kb, grad_w->data,
                                    grad_w->dtype == DCONV_BF16 ? 1 : 0, accumulate ? 1 : 0),
                 "upd_reduce launch");
    }
    cuda_check(cudaGetLastError(), "upd_reduce launch");
  });
}

}  // extern "C"

extern "C" {

int dconv_profile(int enable) {
  g_prof = enable != 0;
  return DCONV_OK;
}

float dconv_profile_last_ms(int which) {
  if (which < 0 || which > 2 || !g_slot[which].armed) return -1.0f;
  float ms = -1.0f;
  if (cudaEventSynchronize(g_slot[which].stop) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, g_slot[which].start, g_slot[which].stop) != cudaSuccess) return -1.0f;
  return ms;
}

}  // extern "C"

extern "C" {
/* debug: point the forward kernel's per-CTA role counters at a device buffer
 * (>= 16 * #SMs int64), or null to disable */
int dconv_debug_counters(void* dev_buf) {
  g_fwd_dbg = reinterpret_cast<long long*>(dev_buf);
  return DCONV_OK;
}
/* debug: forward-kernel ablation bits (1 skip global stores, 2 skip TMEM loads); 0 in production */
int dconv_debug_mode(int mode) {
  g_fwd_dbg_mode = mode;
  return DCONV_OK;
}
}

extern "C" {

int dconv_maxpool_fwd(const dconv_act_t* in, const dconv_act_t* out, void* argmax, dconv_stream_t stream) {
  return guarded([&] {
    check_act(in, "maxpool input");
    check_act(out, "maxpool output");
    if (!argmax) fail(DCONV_ERR_INVALID_ARGUMENT, "maxpool: null argmax");
    const int P = (in->h + 2 - 3) / 2 + 1, Q = (in->w + 2 - 3) / 2 + 1;
    if (in->vlen != 16 || out->vlen != 16 || in->halo_h || in->halo_w || out->halo_h || out->halo_w ||
        out->n != in->n || out->c != in->c || out->h != P || out->w != Q || out->dtype != in->dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "maxpool: expects halo-0 vlen-16 tensors, out = (h+2-3)/2+1");
    const int planes = in->n * cdiv(in->c, 16);
    const int g = grid1d(static_cast<int64_t>(planes) * P * Q);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (in->dtype == DCONV_F32)
      maxpool_fwd_kernel<float><<<g, 256, 0, cs>>>((const float*)in->data, (float*)out->data, (uint8_t*)argmax,
                                                   planes, in->h, in->w, P, Q);
    else
      maxpool_fwd_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((const __nv_bfloat16*)in->data,
                                                           (__nv_bfloat16*)out->data, (uint8_t*)argmax, planes,
                                                           in->h, in->w, P, Q);
    cuda_check(cudaGetLastError(), "maxpool_fwd");
  });
}

}  // extern "C"

namespace {
// the 3x3 / stride 2 / pad 1 pool geometry between grad_out (pooled) and grad_in
void check_pool_pair(const dconv_act_t* grad_out, const dconv_act_t* grad_in) {
  check_act(grad_out, "maxpool grad_out");
  check_act(grad_in, "maxpool grad_in");
  const int P = (grad_in->h + 2 - 3) / 2 + 1, Q = (grad_in->w + 2 - 3) / 2 + 1;
  if (grad_in->vlen != 16 || grad_out->vlen != 16 || grad_in->halo_h || grad_in->halo_w || grad_out->halo_h ||
      grad_out->halo_w || grad_out->n != grad_in->n || grad_out->c != grad_in->c || grad_out->h != P ||
      grad_out->w != Q || grad_out->dtype != grad_in->dtype)
    fail(DCONV_ERR_SHAPE_MISMATCH, "maxpool backward: halo-0 vlen-16 tensors of one dtype, grad_out = (h+2-3)/2+1");
}
}  // namespace

extern "C" {

int dconv_maxpool_bwd(const dconv_act_t* grad_out, const void* argmax, const dconv_act_t* grad_in,
                      const void* mask, dconv_stream_t stream) {
  return guarded([&] {
    check_pool_pair(grad_out, grad_in);
    if (!argmax) fail(DCONV_ERR_INVALID_ARGUMENT, "maxpool: null argmax");
    const int planes = grad_in->n * cdiv(grad_in->c, 16);
    const int g = grid1d(static_cast<int64_t>(planes) * ((grad_in->h + 1) / 2) * ((grad_in->w + 1) / 2));
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (grad_in->dtype == DCONV_F32)
      maxpool_bwd_quad_kernel<float><<<g, 256, 0, cs>>>((const float*)grad_out->data, (const uint8_t*)argmax,
                                                        (float*)grad_in->data, (const float*)mask, planes,
                                                        grad_in->h, grad_in->w, grad_out->h, grad_out->w, nullptr);
    else
      maxpool_bwd_quad_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>(
          (const __nv_bfloat16*)grad_out->data, (const uint8_t*)argmax, (__nv_bfloat16*)grad_in->data,
          (const __nv_bfloat16*)mask, planes, grad_in->h, grad_in->w, grad_out->h, grad_out->w, nullptr);
    cuda_check(cudaGetLastError(), "maxpool_bwd");
  });
}

int dconv_subsample2(const dconv_act_t* in, const dconv_act_t* sub, int inverse, dconv_stream_t stream) {
  return guarded([&] {
    check_act(in, "subsample full-size tensor");
    check_act(sub, "subsample lattice tensor");
    if (in->vlen != 16 || sub->vlen != 16 || in->halo_h || in->halo_w || sub->halo_h || sub->halo_w ||
        sub->n != in->n || sub->c != in->c || sub->h != (in->h + 1) / 2 || sub->w != (in->w + 1) / 2 ||
        sub->dtype != in->dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "subsample2: halo-0 vlen-16 tensors of one dtype, lattice = ((h+1)/2, (w+1)/2)");
    const long long planes = static_cast<long long>(in->n) * cdiv(in->c, 16);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    const int64_t work = planes * (inverse ? static_cast<int64_t>(in->h) * in->w : static_cast<int64_t>(sub->h) * sub->w);
    const int g = grid1d(work);
    if (in->dtype == DCONV_F32) {
      if (inverse)
        unsubsample2_kernel<float><<<g, 256, 0, cs>>>((const float*)sub->data, (float*)in->data, planes, in->h, in->w,
                                                      sub->h, sub->w);
      else
        subsample2_kernel<float><<<g, 256, 0, cs>>>((const float*)in->data, (float*)sub->data, planes, in->h, in->w,
                                                    sub->h, sub->w);
    } else {
      if (inverse)
        unsubsample2_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((const __nv_bfloat16*)sub->data,
                                                              (__nv_bfloat16*)in->data, planes, in->h, in->w, sub->h,
                                                              sub->w);
      else
        subsample2_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>((const __nv_bfloat16*)in->data,
                                                            (__nv_bfloat16*)sub->data, planes, in->h, in->w, sub->h,
                                                            sub->w);
    }
    cuda_check(cudaGetLastError(), "subsample2");
  });
}

int dconv_s2d_act(const dconv_act_t* x, const dconv_act_t* xs, int pad, dconv_stream_t stream) {
  return guarded([&] {
    check_act(x, "s2d input");
    check_act(xs, "s2d output");
    if (x->vlen != 16 || xs->vlen != 16 || x->c > 4 || xs->c != 4 * x->c || x->halo_h || x->halo_w ||
        xs->halo_h || xs->halo_w || xs->n != x->n || xs->dtype != x->dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "s2d: halo-0 vlen-16 tensors, C <= 4 -> 4C channels");
    const int g = grid1d(static_cast<int64_t>(x->n) * xs->h * xs->w);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    auto go = [&](auto c_tag) {
      constexpr int Cc = decltype(c_tag)::value;
      if (x->dtype == DCONV_F32)
        s2d_act_kernel<float, Cc><<<g, 256, 0, cs>>>((const float*)x->data, (float*)xs->data, x->n, x->h, x->w,
                                                     xs->h, xs->w, pad);
      else
        s2d_act_kernel<__nv_bfloat16, Cc><<<g, 256, 0, cs>>>((const __nv_bfloat16*)x->data,
                                                             (__nv_bfloat16*)xs->data, x->n, x->h, x->w, xs->h,
                                                             xs->w, pad);
    };
    switch (x->c) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 3: go(std::integral_constant<int, 3>{}); break;
      default: go(std::integral_constant<int, 4>{}); break;
    }
    cuda_check(cudaGetLastError(), "s2d_act");
  });
}

int dconv_pack_s2d(const float* nchw, int n, int c, int h, int w, const dconv_act_t* xs, int pad,
                   dconv_stream_t stream) {
  return guarded([&] {
    check_act(xs, "pack_s2d output");
    if (!nchw) fail(DCONV_ERR_INVALID_ARGUMENT, "pack_s2d: null source");
    if (c < 1 || c > 4 || xs->vlen != 16 || xs->c != 4 * c || xs->halo_h || xs->halo_w || xs->n != n)
      fail(DCONV_ERR_SHAPE_MISMATCH, "pack_s2d: NCHW C <= 4 -> halo-0 vlen-16 tensor of 4C channels");
    const int g = grid1d(static_cast<int64_t>(n) * xs->h * xs->w);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    auto go = [&](auto c_tag) {
      constexpr int Cc = decltype(c_tag)::value;
      if (xs->dtype == DCONV_F32)
        pack_s2d_kernel<float, Cc><<<g, 256, 0, cs>>>(nchw, (float*)xs->data, n, h, w, xs->h, xs->w, pad);
      else
        pack_s2d_kernel<__nv_bfloat16, Cc><<<g, 256, 0, cs>>>(nchw, (__nv_bfloat16*)xs->data, n, h, w, xs->h, xs->w,
                                                              pad);
    };
    switch (c) {
      case 1: go(std::integral_constant<int, 1>{}); break;
      case 2: go(std::integral_constant<int, 2>{}); break;
      case 3: go(std::integral_constant<int, 3>{}); break;
      default: go(std::integral_constant<int, 4>{}); break;
    }
    cuda_check(cudaGetLastError(), "pack_s2d");
  });
}

int dconv_s2d_wt(const dconv_wt_t* w, const dconv_wt_t* w2, int inverse, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(w, "s2d weight");
    check_wt(w2, "s2d weight'");
    if (w->dtype != DCONV_F32 || w2->dtype != DCONV_F32 || w->vlen != 16 || w2->vlen != 16 || w->c > 4 ||
        w2->c != 4 * w->c || w2->k != w->k || w2->r != (w->r + 1) / 2 || w2->s != (w->s + 1) / 2)
      fail(DCONV_ERR_SHAPE_MISMATCH, "s2d weights: fp32 [K][C<=4][R][S] <-> [K][4C][ceil(R/2)][ceil(S/2)]");
    const int kb = cdiv(w->k, 16);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (!inverse)
      s2d_wt_kernel<<<grid1d(static_cast<int64_t>(kb) * w2->r * w2->s * 256), 256, 0, cs>>>(
          (const float*)w->data, (float*)w2->data, kb, w->c, w->r, w->s, w2->r, w2->s);
    else
      s2d_wt_grad_kernel<<<grid1d(static_cast<int64_t>(kb) * w->r * w->s * 256), 256, 0, cs>>>(
          (const float*)w2->data, (float*)w->data, kb, w->c, w->r, w->s, w2->r, w2->s);
    cuda_check(cudaGetLastError(), "s2d_wt");
  });
}

int dconv_maxpool_bwd_pooled_mask(const dconv_act_t* grad_out, const void* argmax, const dconv_act_t* grad_in,
                                   const dconv_act_t* pooled, dconv_stream_t stream) {
  return guarded([&] {
    check_pool_pair(grad_out, grad_in);
    check_act(pooled, "maxpool pooled mask");
    if (!argmax) fail(DCONV_ERR_INVALID_ARGUMENT, "maxpool: null argmax");
    if (pooled->n != grad_out->n || pooled->c != grad_out->c || pooled->h != grad_out->h ||
        pooled->w != grad_out->w || pooled->dtype != grad_out->dtype)
      fail(DCONV_ERR_SHAPE_MISMATCH, "maxpool: pooled mask must match grad_out");
    const int planes = grad_in->n * cdiv(grad_in->c, 16);
    const int g = grid1d(static_cast<int64_t>(planes) * ((grad_in->h + 1) / 2) * ((grad_in->w + 1) / 2));
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (grad_in->dtype == DCONV_F32)
      maxpool_bwd_quad_kernel<float><<<g, 256, 0, cs>>>((const float*)grad_out->data, (const uint8_t*)argmax,
                                                        (float*)grad_in->data, nullptr, planes, grad_in->h,
                                                        grad_in->w, grad_out->h, grad_out->w,
                                                        (const float*)pooled->data);
    else
      maxpool_bwd_quad_kernel<__nv_bfloat16><<<g, 256, 0, cs>>>(
          (const __nv_bfloat16*)grad_out->data, (const uint8_t*)argmax, (__nv_bfloat16*)grad_in->data, nullptr,
          planes, grad_in->h, grad_in->w, grad_out->h, grad_out->w, (const __nv_bfloat16*)pooled->data);
    cuda_check(cudaGetLastError(), "maxpool_bwd");
  });
}

int dconv_set_sm_budget(int sms) {
  return guarded([&] {
    if (sms < 0) fail(DCONV_ERR_INVALID_ARGUMENT, "sm budget must be >= 0 (0 = every SM)");
    g_sm_budget = sms;
  });
}

int dconv_relu_mask(const dconv_act_t* grad, const dconv_act_t* act, dconv_stream_t stream) {
  return guarded([&] {
    check_act(grad, "relu_mask grad");
    check_act(act, "relu_mask act");
    if (act_elems(*grad) != act_elems(*act) || grad->dtype != act->dtype || grad->n != act->n ||
        grad->c != act->c || grad->h != act->h || grad->w != act->w)
      fail(DCONV_ERR_SHAPE_MISMATCH, "relu_mask: grad and activation must match");
    const int64_t n = act_elems(*grad);
    cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
    if (grad->dtype == DCONV_F32)
      relu_mask_kernel<float><<<grid1d(n), 256, 0, cs>>>((float*)grad->data, (const float*)act->data, n);
    else
      relu_mask_kernel<__nv_bfloat16><<<grid1d(n), 256, 0, cs>>>((__nv_bfloat16*)grad->data,
                                                                 (const __nv_bfloat16*)act->data, n);
    cuda_check(cudaGetLastError(), "relu_mask");
  });
}

int dconv_scale_wt(const dconv_wt_t* w, float scale, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(w, "scale weight");
    if (w->dtype != DCONV_F32) fail(DCONV_ERR_UNSUPPORTED, "scale_wt: fp32 tensors");
    const int64_t n = wt_elems(*w);
    scale_kernel<<<grid1d(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>((float*)w->data, scale, n);
    cuda_check(cudaGetLastError(), "scale_wt");
  });
}

int dconv_sgd(const dconv_wt_t* w, const dconv_wt_t* g, float lr, dconv_stream_t stream) {
  return guarded([&] {
    check_wt(w, "sgd weight");
    check_wt(g, "sgd grad");
    if (w->dtype != DCONV_F32 || g->dtype != DCONV_F32 || wt_elems(*w) != wt_elems(*g))
      fail(DCONV_ERR_SHAPE_MISMATCH, "sgd: fp32 tensors of equal size required");
    const int64_t n = wt_elems(*w);
    sgd_kernel<<<grid1d(n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>((float*)w->data,
                                                                              (const float*)g->data, lr, n);
    cuda_check(cudaGetLastError(), "sgd");
  });
}

}  // extern "C"

#include "host_step.cuh"
#include "validate.cuh"
#include "plan_io.cuh"
