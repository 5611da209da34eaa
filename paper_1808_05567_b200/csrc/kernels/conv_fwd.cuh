// conv_fwd_sm100: implicit-GEMM direct convolution on NCHW16c / KCRS16c16k
// (the reference's fwd_f32_kernel + replay loop, microkernel.cpp:22-85 and
// kernel_streams.cpp:143-166, re-designed for tcgen05).
//
// GEMM view. M = 128*mb "virtual" output positions of one image (output pixel
// (p, q) is v = p*wsub + q; the wsub-Q garbage columns are computed and
// dropped), N = 16*nb output channels, K = (input block c_b, phase, tap, 16
// lanes). Each pipeline stage brings ONE input channel block (for one stride
// phase) of the tile's receptive field into shared memory; every filter tap
// then reads the same smem tile through a UMMA descriptor whose start address
// is shifted by the tap's virtual offset (r*wsub + s). Input halo rows are
// loaded once per stage, not once per tap.
//
// Operand staging. Activations arrive by ONE TMA box per stage (rows mode:
// whole sub-image rows with elementStrides = conv stride and OOB zero fill for
// the padding; linear mode: contiguous 128-pixel boxes of a halo'd plane).
// bf16 activations land directly in the canonical K-major no-swizzle layout
// ([16B chunk][pixel][16B]); fp32 activations land raw and converter warps
// rewrite them in smem as bf16 pieces (1 = cast, 3 = exact hi/mid/lo split).
// Weights are pre-laid-out bf16 pieces (layout.cuh weight_prep_kernel), one
// TMA box per piece per stage.
//
// Warp roles (384 threads): w0 activation TMA producer, w1 MMA issuer (+TMEM
// owner), w2 weight producer (fp32 path), w4..w7 epilogue, w8..w11 converters
// (fp32 activations only). Persistent over tiles with double-buffered TMEM.
//
// Numerics: pieces = 1 is bf16 x bf16 -> fp32 (TMEM). pieces = 3 splits every
// fp32 operand into hi + mid + lo bf16 (exact) and accumulates the six
// products with i + j <= 2: fp32-accurate (~2^-24 relative per product).
#pragma once
#include <cuda_bf16.h>
#include <type_traits>

#include "conv_params.h"
#include "sm100_ptx.cuh"

#ifndef DCONV_FWD_WARPS_P
#define DCONV_FWD_WARPS_P 12  // fp32 smem-staged plans: 8 role warps + 4 converters (12 warps: 168 regs, no spill)
#endif

namespace dconv_sm100 {

constexpr int kFwdThreads = 256;
constexpr int kMaxStages = 8;
constexpr int kFastTaps = 16;  // taps per weight stage issued by the unrolled MMA path
constexpr int kWarp1Iters = 8;  // single-tap plans: stages per tile from which the whole MMA warp runs the issue loop
constexpr int kConvWarp0 = 2;
constexpr int kConvThreads = 192;  // warps 2..7

__device__ __forceinline__ uint32_t pack2(__nv_bfloat16 a, __nv_bfloat16 b) {
  return static_cast<uint32_t>(__bfloat16_as_ushort(a)) | (static_cast<uint32_t>(__bfloat16_as_ushort(b)) << 16);
}

// two fp32 -> packed bf16x2, round to nearest even (one F2FP.BF16.F32.PACK_AB)
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ float lo_f(uint32_t p) { return __uint_as_float(p << 16); }
__device__ __forceinline__ float hi_f(uint32_t p) { return __uint_as_float(p & 0xFFFF0000u); }

// Exact 3-way split of 8 fp32 values into 16B bf16 rows (hi, mid, lo).
// x == hi + mid + lo for every finite normal x (8 significant bits each).
__device__ __forceinline__ void split8(const float (&x)[8], uint4& h, uint4& m, uint4& l) {
  uint32_t hh[4], mm[4], ll[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    hh[e] = cvt2(x[2 * e], x[2 * e + 1]);
    const float ra = x[2 * e] - lo_f(hh[e]), rb = x[2 * e + 1] - hi_f(hh[e]);
    mm[e] = cvt2(ra, rb);
    ll[e] = cvt2(ra - lo_f(mm[e]), rb - hi_f(mm[e]));
  }
  h = make_uint4(hh[0], hh[1], hh[2], hh[3]);
  m = make_uint4(mm[0], mm[1], mm[2], mm[3]);
  l = make_uint4(ll[0], ll[1], ll[2], ll[3]);
}

__device__ __forceinline__ uint4 cast8(const float (&x)[8]) {
  return make_uint4(cvt2(x[0], x[1]), cvt2(x[2], x[3]), cvt2(x[4], x[5]), cvt2(x[6], x[7]));
}

// 16 fp32 accumulator columns -> 16 lanes at `dst`
__device__ __forceinline__ void store16(void* dst, const float* v, int out_bf16) {
  if (out_bf16) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const float a[8] = {v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
    const float b[8] = {v[8], v[9], v[10], v[11], v[12], v[13], v[14], v[15]};
    d[0] = cast8(a);
    d[1] = cast8(b);
  } else {
    float4* d = reinterpret_cast<float4*>(dst);
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v[7]);
    d[2] = make_float4(v[8], v[9], v[10], v[11]);
    d[3] = make_float4(v[12], v[13], v[14], v[15]);
  }
}

// 16 lanes at `src` (bf16 or fp32) -> fp32
__device__ __forceinline__ void load16(const void* src, int bf16, float* v) {
  if (bf16) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    const uint4 a = s[0], b = s[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[2 * e] = __uint_as_float(w[e] << 16);
      v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  } else {
    const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 t = s[e];
      v[4 * e] = t.x;
      v[4 * e + 1] = t.y;
      v[4 * e + 2] = t.z;
      v[4 * e + 3] = t.w;
    }
  }
}

__device__ __forceinline__ void store16_zero(void* dst, int out_bf16) {
  const uint4 z = make_uint4(0, 0, 0, 0);
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = z;
  d[1] = z;
  if (!out_bf16) {
    d[2] = z;
    d[3] = z;
  }
}

// Shared-memory plan: a RAW ring (fp32 activations as landed by TMA,
// [pixel][64B]; fp32 path only) and a PIECE ring ({A bf16 pieces, W bf16
// pieces}) that the tensor core reads. The raw ring runs ahead of the piece
// ring so enough HBM bytes stay in flight while converters and MMAs work.
struct FwdSmem {
  uint32_t a_plane;  // bytes per 16B-chunk plane of the A pieces (a_px * 16)
  uint32_t raw_slot; // bytes per raw slot (a_px * 64), 0 for bf16 inputs
  uint32_t w_piece;  // bytes per weight piece
  uint32_t pc_slot;  // bytes per A-piece slot
  uint32_t w_slot;   // bytes per weight slot (all pieces)
  uint32_t w_off;    // weight ring start (after the piece ring)
  uint32_t raw_off;  // raw ring start (after the weight ring)
  uint32_t epi_off;  // epilogue staging (4 warps x 32 pixels x 64B) after the raw ring
};

// three independent rings: A pieces (MMA operand), weights (MMA operand, own
// prefetch depth so their L2 latency hides behind other stages), raw fp32
__host__ __device__ inline FwdSmem fwd_smem_layout(int a_px, int taps_box, int nb, int pieces, bool raw_f32,
                                                   int piece_stages, int w_stages) {
  FwdSmem L;
  L.a_plane = static_cast<uint32_t>(a_px) * 16u;
  L.raw_slot = raw_f32 ? ((static_cast<uint32_t>(a_px) * 64u + 1023u) & ~1023u) : 0u;
  L.w_piece = static_cast<uint32_t>(taps_box) * (2u * nb) * 256u;  // taps_box = taps per weight stage
  L.pc_slot = (static_cast<uint32_t>(pieces) * 2u * L.a_plane + 1023u) & ~1023u;
  L.w_slot = (static_cast<uint32_t>(pieces) * L.w_piece + 1023u) & ~1023u;
  L.w_off = static_cast<uint32_t>(piece_stages) * L.pc_slot;
  L.raw_off = L.w_off + static_cast<uint32_t>(w_stages) * L.w_slot;
  L.epi_off = 0;  // set by the caller: raw_off + raw_stages * raw_slot
  return L;
}
constexpr uint32_t kEpiStageBytes = 0;

// 16B chunk k of pixel j in a 64B-row buffer written by TMA with SWIZZLE_64B
// (Swizzle<2,4,3>: chunk bits [4,6) ^= row-pair bits [7,9))
__device__ __forceinline__ uint32_t sw64(uint32_t j, uint32_t k) { return j * 64u + ((k ^ ((j >> 1) & 3u)) << 4); }
// 16B chunk k of row j in a 32B-row SWIZZLE_32B buffer (Swizzle<1,4,3>: bit 4 ^= bit 7)
__device__ __forceinline__ uint32_t sw32(uint32_t j, uint32_t k) { return j * 32u + ((k ^ ((j >> 2) & 1u)) << 4); }

// optional per-CTA role counters (debug builds of the plan only): slot layout
// [0] producer wait, [1] converter wait raw, [2] converter wait slot, [3] converter busy,
// [4] MMA wait operands, [5] MMA wait accumulator, [6] epilogue wait, [7] epilogue busy, [8] total
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, long long* acc) {
  if (acc) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    *acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}
__device__ __forceinline__ void mbar_wait_bt(uint64_t* bar, uint32_t parity, long long* acc) {
  if (acc) {
    const long long t0 = clock64();
    mbar_wait_backoff(bar, parity);
    *acc += clock64() - t0;
  } else {
    mbar_wait_backoff(bar, parity);
  }
}

// position in a ring of n slots: slot index and the mbarrier phase parity of
// its current fill (no integer division on the per-stage path)
struct RingPos {
  int idx = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void adv(int n) {
    if (++idx == n) {
      idx = 0;
      ph ^= 1u;
    }
  }
};

// w0 activation producer, w1 MMA, w2 weight producer, w3 idle, w4-7 epilogue
// (one warp per TMEM lane quarter), w8-11 converters in two groups of two that
// take alternate pipeline stages
constexpr int kFwdWarps = DCONV_FWD_WARPS_P;
constexpr int kFwdThreadsP = kFwdWarps * 32;
constexpr int kEpiWarp0 = 4, kEpiWarps = 4;
constexpr int kCvtWarp0 = 8, kCvtWarps = DCONV_FWD_WARPS_P - 8;

// Persistent implicit-GEMM forward: grid = #SMs, CTA c handles tiles c, c+G, ...
// (tile = (image, virtual-row block) x output-channel tile). Two TMEM
// accumulator buffers let the epilogue of tile i overlap the mainloop of i+1.
// TS (single-tap problems, fp32 activations): the converters write the A
// pieces straight into TENSOR memory (tcgen05.st, a ring of PIECES x 8
// columns per stage after the accumulators) and the MMA reads A from TMEM —
// the A operand then costs no shared-memory bandwidth at all, which is what
// bounds the smem-staged fp32 path at small N. 16 warps: two converter groups
// of four (one warp per TMEM lane quarter) alternate stages.
constexpr int kFwdWarpsTS = 16;
constexpr uint32_t kEpiSlots = 4;  // TMA-store slabs per epilogue warp (2 KiB each)
constexpr uint32_t kEpiStagingBytes = 4u * kEpiSlots * 2048u;
constexpr int kFwdThreadsTS = kFwdWarpsTS * 32;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
// same store without a memory clobber: ordinary shared-memory loads may be
// scheduled across it (the values are in registers; tmem_st_wait orders it)
__device__ __forceinline__ void tmem_st8_nc(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// D[tmem] (+)= A[tmem] * B[smem] (A: lane = row, 8 columns = 16 packed bf16, low half = even k)
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <bool RAW_F32, int PIECES, bool TS = false>
__global__ void __launch_bounds__((TS || !RAW_F32) ? kFwdThreadsTS : kFwdThreadsP, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_out,
                    const __grid_constant__ CUtensorMap map_out2, const __grid_constant__ FwdParams p, int raw_stages,
                    int pc_stages, int w_stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t raw_full[kMaxStages], raw_empty[kMaxStages];
  __shared__ __align__(8) uint64_t pc_full[kMaxStages], pc_conv[kMaxStages], pc_empty[kMaxStages];
  __shared__ __align__(8) uint64_t w_full[kMaxStages], w_empty[kMaxStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;
  // per-phase / per-tap tables copied out of the parameter block (the hot loops
  // index them dynamically; shared memory keeps those reads off the constant cache)
  __shared__ int s_phase_row[kMaxPhases], s_phase_col[kMaxPhases], s_phase_ntaps[kMaxPhases],
      s_phase_tap0[kMaxPhases], s_tap_shift[kMaxTaps];

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  // a stage carries kc channel blocks: raw slot = kc planes, weight piece = kc x w_taps taps
  FwdSmem L = fwd_smem_layout(p.a_px * p.kc, p.w_resident ? p.cb_in : p.w_taps * p.kc, p.nb, PIECES, RAW_F32,
                              TS ? 0 : pc_stages, w_stages);
  L.epi_off = L.raw_off + static_cast<uint32_t>(raw_stages) * L.raw_slot;
  const uint32_t smem0 = smem_u32(smem);
  const int NT = 16 * p.nb;
  const int kc_stages = (p.cb_in + p.kc - 1) / p.kc;
  const int k_iters = kc_stages * p.n_phases;
  const int n_mtiles = p.mimg > 0 ? (p.n_img + p.mimg - 1) / p.mimg : p.n_img * p.tiles_per_img;
  const int n_tiles = n_mtiles * p.n_ntiles;
  // fp32-accurate mode keeps the a0*b0 products and the five correction
  // products in separate accumulators: the large sum then takes 6x fewer
  // (truncating) fp32 accumulation steps; the epilogue adds the two
  // (only long reductions need the split: short ones accumulate all six
  // products in one accumulator, halving TMEM columns and epilogue loads)
  const bool two_acc = PIECES == 3 && p.split_acc;
  const uint32_t kAccs = two_acc ? 2u : 1u;
  const uint32_t acc_cols = kAccs * static_cast<uint32_t>(p.mb * NT);
  // two converter groups alternate stages; a 1-deep ring would let the second
  // group wait on a phase two ahead (parity aliasing), so it falls back to one group
  // Two converter groups alternate stages. Each waits its piece slot first: that
  // proves every stage <= g - pc_stages was converted, hence its raw fill landed,
  // so the raw_full parity wait for g cannot be satisfied by the fill of
  // g - 2 raw_stages (TMA fills may land out of order) as long as the slot's
  // previous fill is ours (raw_stages even) or <= g - pc_stages.
  // TS plans whose tiles are one stage (output-heavy, e.g. the dual BWD of a
  // channel-expanding 1x1) give the second converter group to the epilogue
  const bool ts_epi2 = TS && p.tma_store && p.ts_epi2;
  const int cvt_groups =
      (!ts_epi2 && raw_stages >= 2 && pc_stages >= 2 && (raw_stages % 2 == 0 || raw_stages >= pc_stages)) ? 2 : 1;
  const int cvt_group_warps = TS ? 4 : kCvtWarps / cvt_groups;
  // bf16 smem-staged plans have idle converter warps: with the lean TMA-store
  // epilogue, warps 8..11 form a second epilogue group (alternate block pairs),
  // doubling the loads in flight for fused residual adds / ReLU masks
  const bool epi2 = !RAW_F32 && !TS && p.tma_store;
  // bf16 plans with the register epilogue (halo'd / strided / padded-row outputs: every
  // rows-mode layer) split each tile's (m-block, block pair) items over the same
  // groups: one warp per lane quarter is latency bound (dependent chains, no ILP)
  const bool epi_reg3 = !RAW_F32 && !TS && !p.tma_store;
  // The groups' shares of a tile's items (block pairs) are uneven when the item count is not
  // a multiple of the group count (8 pairs over 3 groups: 3, 3, 2; 4 items: 2, 1, 1), so the
  // assignment rotates by the CTA's tile counter: over three tiles every group does the same
  // work, and the double-buffered accumulators absorb the one-item skew (same values, same
  // stores: only which warp moves them changes).
  const int n_epi_groups = (epi2 || epi_reg3) ? max(1, min(3, p.epi_groups)) : ts_epi2 ? 2 : 1;  // bf16: warps 4..7, 8..11, 12..15; ts_epi2: 4..7, 12..15
  // TS: A-piece ring in TMEM after the accumulators
  const uint32_t ring_col0 = static_cast<uint32_t>(p.acc_bufs) * acc_cols;
  constexpr uint32_t kRingCols = PIECES * 8;  // per channel block
  const uint32_t ring_slot = static_cast<uint32_t>(p.kc) * kRingCols;

  uint32_t tmem_cols = 32;
  while (tmem_cols < ring_col0 + (TS ? static_cast<uint32_t>(pc_stages) * ring_slot : 0u)) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    for (int s = 0; s < raw_stages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], cvt_group_warps);
    }
    for (int s = 0; s < pc_stages; ++s) {
      mbar_init(&pc_full[s], 1);
      mbar_init(&pc_conv[s], cvt_group_warps);
      mbar_init(&pc_empty[s], 1);
    }
    const int n_wbar = p.w_resident ? kc_stages : w_stages;  // resident: one per stage group
    for (int s = 0; s < n_wbar; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kEpiWarps * n_epi_groups);
    }
    fence_barrier_init();
  }
  if (warp == 3) {
    for (int i = lane; i < kMaxTaps; i += 32) s_tap_shift[i] = p.tap_shift[i];
    if (lane < kMaxPhases) {
      s_phase_row[lane] = p.phase_row[lane];
      s_phase_col[lane] = p.phase_col[lane];
      s_phase_ntaps[lane] = p.phase_ntaps[lane];
      s_phase_tap0[lane] = p.phase_tap0[lane];
    }
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;
  long long* dbg = (kDevBuild && p.dbg) ? p.dbg + static_cast<long long>(blockIdx.x) * 16 : nullptr;
  const int dbg_mode = kDevBuild ? p.dbg_mode : 0;  // ablation bits (developer builds)
  long long t_start = clock64();
  if (dbg && threadIdx.x == 0) {
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    dbg[9] = static_cast<long long>(gt);
  }
  long long c_a = 0, c_b = 0;  // role-local counters (lane 0 / thread 0 of the role writes)

  // tile t -> (n, v0, ntile); output-channel tiles innermost so consecutive
  // CTAs share the activation tile through L2
  auto tile_coords = [&](int t, int& n, int& v0, int& ntile) {
    ntile = t % p.n_ntiles;
    const int mt = t / p.n_ntiles;
    if (p.mimg > 0) {  // multi-image tile: images [n, n + mimg), rows = (image, pixel)
      n = mt * p.mimg;
      v0 = 0;
    } else {
      n = mt / p.tiles_per_img;
      v0 = (mt % p.tiles_per_img) * 128 * p.mb;
    }
  };
  const uint32_t w_tap = (2u * p.nb) * 256u;

  if (warp == 0) {
    // ------------------------------------------------------------ activation producer
    if (lane == 0) {
      const uint32_t a_bytes = static_cast<uint32_t>(p.a_load_px) * (RAW_F32 ? 64u : 32u) * p.kc;
      uint32_t g = 0;
      RingPos rp;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int n, v0, ntile;
        tile_coords(t, n, v0, ntile);
        const int row0 = v0 / p.wsub;
        const int a_px0 = p.linear ? v0 : row0 * p.wsub;
        int cb = 0, ph = 0;
        for (int it = 0; it < k_iters; ++it, ++g, rp.adv(RAW_F32 ? raw_stages : pc_stages)) {
          if (it > 0 && ++ph == p.n_phases) {
            ph = 0;
            ++cb;
          }
          const int plane = n * p.in_cb + cb * p.kc;
          if (RAW_F32) {
            const int s = rp.idx;
            mbar_wait_t(&raw_empty[s], rp.ph ^ 1u, dbg ? &c_a : nullptr);
            if (dbg && blockIdx.x == 0 && g < 256) dbg[gridDim.x * 16 + g * 8 + 6] = clock64() - t_start;
            uint8_t* dst = smem + L.raw_off + s * L.raw_slot;
            mbar_arrive_expect_tx(&raw_full[s], a_bytes);
            if (p.mimg > 0) {
              tma_load_4d(dst, &map_a, &raw_full[s], 0, 0, cb * p.kc, n);  // box {16, hw, kc, mimg}
            } else if (p.linear) {
              for (int i = 0; i < p.lin_boxes; ++i)
                tma_load_3d(dst + i * 128 * 64, &map_a, &raw_full[s], 0, a_px0 + i * 128, plane);
            } else {
              tma_load_4d(dst, &map_a, &raw_full[s], 0, p.in_col0 + s_phase_col[ph],
                          p.in_row0 + p.stride * row0 + s_phase_row[ph], plane);
            }
          } else {
            const int s = rp.idx;
            mbar_wait_t(&pc_empty[s], rp.ph ^ 1u, dbg ? &c_a : nullptr);
            uint8_t* dst = smem + s * L.pc_slot;
            if (dbg && blockIdx.x == 0 && g < 256) dbg[gridDim.x * 16 + g * 8 + 6] = clock64() - t_start;
            if (dbg_mode & 256) {  // ablation: no activation loads
              mbar_arrive(&pc_full[s]);
              continue;
            }
            mbar_arrive_expect_tx(&pc_full[s], a_bytes);
            // bf16 pixels as SWIZZLE_32B rows: the MMA reads them in place
            if (p.img_pitch > 0) {  // packed images: one box {16, wsub, H + pad, mimg + 1, kc}
              tma_load_5d(dst, &map_a, &pc_full[s], 0, p.in_col0, p.in_row0, n, cb * p.kc);
            } else if (p.mimg > 0) {
              for (int kk = 0; kk < p.kc; ++kk)  // box {16, hw, 1, mimg} per block: rows contiguous per block
                tma_load_4d(dst + kk * p.a_px * 32, &map_a, &pc_full[s], 0, 0, cb * p.kc + kk, n);
            } else if (p.linear) {
              const int rsh = p.a_sw128 ? 2 : 0;  // 128 B rows of four pixels
              if (p.kc > 1)  // one box {16, a_px, kc}
                tma_load_3d(dst, &map_a, &pc_full[s], 0, a_px0 >> rsh, plane);
              else
                for (int i = 0; i < p.lin_boxes; ++i)
                  tma_load_3d(dst + i * 128 * 32, &map_a, &pc_full[s], 0, (a_px0 + i * 128) >> rsh, plane);
            } else {
              tma_load_4d(dst, &map_a, &pc_full[s], 0, p.in_col0 + s_phase_col[ph],
                          p.in_row0 + p.stride * row0 + s_phase_row[ph], plane);
            }
          }
        }
      }
      if (dbg) dbg[0] = c_a;
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ weight producer (own ring)
    // one weight stage = up to w_taps taps of one (c_b, phase): large filters
    // (7x7 stem) stream their taps through several small stages
    // the weight prep kernel that precedes this launch may still be running
    // (programmatic dependent launch): its output is read only after this wait
    if (lane == 0) pdl_wait_primary();
    if (lane == 0 && p.w_resident) {
      // single-tap plan whose CTA always sees the same output-channel tile:
      // the whole slice [piece][c_b][2nb][256 B] is loaded once
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wprep);
      const int ntile = blockIdx.x % p.n_ntiles;
      if (blockIdx.x < n_tiles) {
        // one barrier per stage's kc channel blocks, in stage order
        uint8_t* dst = smem + L.w_off;
        for (int ks = 0; ks < kc_stages; ++ks) {
          const int cb0 = ks * p.kc, cb1 = min(p.cb_in, cb0 + p.kc);
          mbar_arrive_expect_tx(&w_full[ks], PIECES * (cb1 - cb0) * w_tap);
          // (fp32-activation plans: prepared weights [piece][c_b][n_tile][..], see weight_prep_kernel)
          if (p.n_ntiles == 1) {  // the stage's blocks are contiguous per piece: one copy each
            for (int pc = 0; pc < PIECES; ++pc)
              bulk_load(dst + pc * L.w_piece + cb0 * w_tap,
                        wsrc + (static_cast<long long>(pc) * p.cb_in + cb0) * w_tap, (cb1 - cb0) * w_tap,
                        &w_full[ks]);
          } else {
            for (int cb = cb0; cb < cb1; ++cb)
              for (int pc = 0; pc < PIECES; ++pc)
                bulk_load(dst + pc * L.w_piece + cb * w_tap,
                          wsrc + ((static_cast<long long>(pc) * p.cb_in + cb) * p.n_ntiles + ntile) * w_tap, w_tap,
                          &w_full[ks]);
          }
        }
      }
    } else if (lane == 0) {
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wprep);
      const long long w_blk = static_cast<long long>(p.n_taps) * w_tap;
      uint32_t g = 0;
      RingPos wp;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        if (p.w_all && t != blockIdx.x) break;  // every stage has its own slot: loaded once
        int n, v0, ntile;
        tile_coords(t, n, v0, ntile);
        int cb = 0, ph = 0;
        for (int it = 0; it < k_iters; ++it) {
          if (it > 0 && ++ph == p.n_phases) {
            ph = 0;
            ++cb;
          }
          const int kc_eff = min(p.kc, p.cb_in - cb * p.kc);
          for (int t0 = 0; t0 < s_phase_ntaps[ph]; t0 += p.w_taps, ++g, wp.adv(w_stages)) {
            const int nt = min(p.w_taps, s_phase_ntaps[ph] - t0);
            const int s = wp.idx;
            mbar_wait(&w_empty[s], wp.ph ^ 1u);
            if (dbg && blockIdx.x == 0 && g < 256) p.dbg[gridDim.x * 16 + g * 8 + 7] = clock64() - t_start;
            const uint32_t w_bytes = static_cast<uint32_t>(nt) * w_tap;
            if (dbg_mode & 128) {  // ablation: no weight loads
              mbar_arrive(&w_full[s]);
              continue;
            }
            mbar_arrive_expect_tx(&w_full[s], PIECES * kc_eff * w_bytes);
            uint8_t* dst = smem + L.w_off + s * L.w_slot;
            // (bf16-activation plans: prepared weights [piece][n_tile][c_b][tap][..], see weight_prep_kernel)
            // slot layout [piece][kk][tap]: piece stride w_piece = kc * w_taps taps. A stage
            // holding every tap of its kc blocks is one contiguous run of the prepared
            // weights: one bulk copy per piece (each copy costs the issuing thread ~240
            // cycles -- four per stage paced the 1x1 layers)
            // (fp32-activation kernels keep the [piece][c_b][n_tile] layout and per-block copies:
            // their code, and timing, is left exactly as it was)
            if constexpr (!RAW_F32) {
              if (p.n_phases == 1 && nt == p.n_taps) {
                for (int pc = 0; pc < PIECES; ++pc)
                  bulk_load(dst + pc * L.w_piece,
                            wsrc + ((static_cast<long long>(pc) * p.n_ntiles + ntile) * p.cb_in + cb * p.kc) * w_blk,
                            static_cast<uint32_t>(kc_eff) * w_bytes, &w_full[s]);
              } else {
                for (int kk = 0; kk < kc_eff; ++kk)
                  for (int pc = 0; pc < PIECES; ++pc)
                    bulk_load(dst + pc * L.w_piece + kk * w_bytes,
                              wsrc + ((static_cast<long long>(pc) * p.n_ntiles + ntile) * p.cb_in + cb * p.kc + kk) *
                                         w_blk +
                                  static_cast<long long>(s_phase_tap0[ph] + t0) * w_tap,
                              w_bytes, &w_full[s]);
              }
            } else {
              for (int kk = 0; kk < kc_eff; ++kk)
                for (int pc = 0; pc < PIECES; ++pc)
                  bulk_load(dst + pc * L.w_piece + kk * w_bytes,
                            wsrc + ((static_cast<long long>(pc) * p.cb_in + cb * p.kc + kk) * p.n_ntiles + ntile) * w_blk +
                                static_cast<long long>(s_phase_tap0[ph] + t0) * w_tap,
                            w_bytes, &w_full[s]);
            }
          }
        }
      }
    }
  } else if (warp == 1 && !RAW_F32 && !TS && p.n_phases == 1 && p.w_taps == p.n_taps && !p.w_resident &&
             p.n_taps <= kFastTaps && (p.mb == 1 || p.mb == 2 || p.mb == 4)) {
    // ------------------------------------------------------------ MMA issuer, bf16 single-phase stages
    // One lane runs the whole loop: the tap shifts and descriptor high words are
    // computed once per launch, so between the last MMA of a stage and the first of
    // the next there are only the commits and the two barrier waits (the tensor
    // pipe's queue is short: issue blocks at the tensor rate, and whatever the
    // issuing thread does between stages is a bubble in the pipe).
    {  // the whole warp runs the loop (warp-uniform values); one elected lane issues each stage
      const uint32_t idesc = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(NT));
      const int nt = p.n_taps;
      uint32_t sh[kFastTaps];
#pragma unroll
      for (int i = 0; i < kFastTaps; ++i) sh[i] = i < nt ? 2u * static_cast<uint32_t>(s_tap_shift[i]) : 0u;
      const uint32_t a_hi = static_cast<uint32_t>(make_smem_desc_sw32(smem0) >> 32);
      const uint32_t b_hi = static_cast<uint32_t>(make_smem_desc(smem0, 128, 256) >> 32);
      const uint32_t a_lo0 = static_cast<uint32_t>(make_smem_desc_sw32(smem0));
      const uint32_t b_lo0 = static_cast<uint32_t>(make_smem_desc(smem0 + L.w_off, 128, 256));
      const uint32_t pc_u = L.pc_slot >> 4, w_u = L.w_slot >> 4, b_tap = w_tap >> 4;
      // KC / NTAPS > 0: compile-time channel blocks per stage and taps (every MMA of a full
      // stage is straight-line code whose operands are kernel parameters plus the stage's
      // slot bases). Measured (tools/probe_bisect.cu): the runtime-trip-count loop issued a
      // 128x128x16 MMA every ~144 cycles, the unrolled one every ~80 (floor 64), the rest
      // being the stage's barrier waits; partial stages (kc_eff < KC) take the runtime loop.
      // single-tap stages (lane 0 only): the round-1 loop shape. The lean multi-tap loop
      // below measured 10 % SLOWER on the epilogue-bound fused 1x1 layers (residual add,
      // ReLU mask), so the two stay separate
      auto run1 = [&](auto mb_c, auto kc_c, auto nt_c) {
        constexpr int MB = decltype(mb_c)::value, KC = decltype(kc_c)::value, NTAPS = decltype(nt_c)::value;
        uint32_t tl = 0, g = 0;
        RingPos pcp, wpp;
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
          int n, v0, ntile;
          tile_coords(t, n, v0, ntile);
          const int a_px0 = p.linear ? v0 : (v0 / p.wsub) * p.wsub;
          const uint32_t v_off2 = 2u * static_cast<uint32_t>(v0 - a_px0);
          const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
          const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
          mbar_wait(&acc_empty[acc], apar ^ 1u);
          tc_fence_after();
          const uint32_t d_base = tmem_base + acc * acc_cols;
          for (int it = 0; it < k_iters; ++it, pcp.adv(pc_stages), wpp.adv(w_stages), ++g) {
            long long* trace = (dbg && blockIdx.x == 0 && g < 256) ? dbg + gridDim.x * 16 + g * 8 : nullptr;
            const bool no_wait = kDevBuild && (dbg_mode & 2048);  // ablation: MMAs do not wait for operands
            if (!no_wait) mbar_wait(&pc_full[pcp.idx], pcp.ph);
            if (trace) trace[0] = clock64() - t_start;
            if ((!p.w_all || tl == 0) && !no_wait) mbar_wait(&w_full[wpp.idx], wpp.ph);
            if (trace) trace[1] = clock64() - t_start;
            tc_fence_after();
            const int kc_eff = min(p.kc, p.cb_in - it * p.kc);
            const uint32_t a_st = a_lo0 + static_cast<uint32_t>(pcp.idx) * pc_u + v_off2;
            const uint32_t b_st = b_lo0 + static_cast<uint32_t>(wpp.idx) * w_u;
            if (KC > 0 && kc_eff == KC) {
              const uint32_t acc0 = it == 0 ? 0u : 1u;
#pragma unroll
              for (int kk = 0; kk < (KC > 0 ? KC : 1); ++kk) {
                const uint32_t ak = a_st + 2u * static_cast<uint32_t>(kk * p.a_px);
                const uint32_t bk = b_st + static_cast<uint32_t>(kk * NTAPS) * b_tap;
#pragma unroll
                for (int tp = 0; tp < NTAPS; ++tp)
#pragma unroll
                  for (int mb = 0; mb < MB; ++mb)
                    mma_bf16_lo(d_base + static_cast<uint32_t>(mb * NT), ak + sh[tp] + 256u * mb, a_hi,
                                bk + static_cast<uint32_t>(tp) * b_tap, b_hi, idesc, (kk == 0 && tp == 0) ? acc0 : 1u);
              }
            } else {
              for (int kk = 0; kk < kc_eff; ++kk) {
                const uint32_t ak = a_st + 2u * static_cast<uint32_t>(kk * p.a_px);
                const uint32_t bk = b_st + ((static_cast<uint32_t>(kk * nt) * w_tap) >> 4);
                const bool first_k = it == 0 && kk == 0;
#pragma unroll
                for (int tp = 0; tp < kFastTaps; ++tp) {
                  if (tp >= nt) break;
#pragma unroll
                  for (int mb = 0; mb < MB; ++mb)
                    mma_bf16_lo(d_base + static_cast<uint32_t>(mb * NT), ak + sh[tp] + 256u * mb, a_hi,
                                bk + static_cast<uint32_t>(tp) * b_tap, b_hi, idesc, (first_k && tp == 0) ? 0u : 1u);
                }
              }
            }
            if (trace) trace[3] = clock64() - t_start;
            if (!p.w_all) mma_commit(&w_empty[wpp.idx]);
            mma_commit(&pc_empty[pcp.idx]);
            if (trace) trace[2] = clock64() - t_start;
          }
          mma_commit(&acc_full[acc]);
        }
      };
      auto run = [&](auto mb_c, auto kc_c, auto nt_c) {
        constexpr int MB = decltype(mb_c)::value, KC = decltype(kc_c)::value, NTAPS = decltype(nt_c)::value;
        // multi-tap stages (9+ MMAs each): the whole warp runs the loop and one elected lane
        // issues (warp-uniform descriptor arithmetic, measured 7-13 % on the 3x3 layers);
        // single-tap stages: lane 0 alone (the other lanes do not compete for issue slots with
        // the epilogue warps on this SM sub-partition, measured 5-10 % on fused epilogues)
        // Single-tap plans whose tiles are long reductions (>= kWarp1Iters full stages: the
        // 14x14 / 7x7 1x1 layers, MMA-issue bound) also take the whole-warp loop: on the
        // lane-0 path every MMA is a divergent-code waterfall (ELECT + 5 R2UR.BROADCAST per
        // UTCHMMA, ~80 cycles) and the stage's commits / ring bookkeeping another ~400,
        // which the 512-cycle stage of four 128x256x16 MMAs does not hide.
        constexpr bool kMulti = NTAPS > 1;
        bool warp_loop = kMulti;
        if constexpr (!kMulti && KC > 0) {
          warp_loop = p.n_phases == 1 && p.cb_in % p.kc == 0 && k_iters >= kWarp1Iters;
          if (kDevBuild && (dbg_mode & 4096)) warp_loop = p.n_phases == 1 && p.cb_in % p.kc == 0;
          if (kDevBuild && (dbg_mode & 8192)) warp_loop = false;
        }
        if (!warp_loop) {
          if (lane == 0) run1(mb_c, kc_c, nt_c);
          return;
        }
        constexpr unsigned wmask = 0xffffffffu;
        auto issuer = [&]() { return elect_one(); };
        // full stages first (compile-time MMA sequence), then the partial one (runtime loop)
        const int k_full = (KC > 0 && p.n_phases == 1) ? p.cb_in / p.kc : 0;
        uint32_t tl = 0, g = 0;
        int pci = 0, wi = 0;
        uint32_t pph = 0, wph = 0;
        // linear and multi-image tiles start their A slot at the tile's first pixel: the
        // MMA side needs no tile coordinates (no divisions between tiles)
        for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
          uint32_t v_off2 = 0;
          if (!p.linear && p.mimg == 0) {
            int n, v0, ntile;
            tile_coords(t, n, v0, ntile);
            v_off2 = 2u * static_cast<uint32_t>(v0 - (v0 / p.wsub) * p.wsub);
          }
          const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
          const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
          mbar_wait(&acc_empty[acc], apar ^ 1u);
          tc_fence_after();
          const uint32_t d_base = tmem_base + acc * acc_cols;
          const bool wait_w = !p.w_all || tl == 0;
          for (int it = 0; it < k_iters; ++it, ++g) {
            long long* trace =
                (kDevBuild && dbg && blockIdx.x == 0 && g < 256 && lane == 0) ? dbg + gridDim.x * 16 + g * 8 : nullptr;
            const bool no_wait = kDevBuild && (dbg_mode & 2048);  // ablation: MMAs do not wait for operands
            if (!no_wait) mbar_wait(&pc_full[pci], pph);
            if (trace) trace[0] = clock64() - t_start;
            if (wait_w && !no_wait) mbar_wait(&w_full[wi], wph);
            if (trace) trace[1] = clock64() - t_start;
            tc_fence_after();
            const uint32_t a_st = a_lo0 + static_cast<uint32_t>(pci) * pc_u + v_off2;
            const uint32_t b_st = b_lo0 + static_cast<uint32_t>(wi) * w_u;
            if (issuer()) {
            if (it < k_full) {
              const uint32_t acc0 = it == 0 ? 0u : 1u;
#pragma unroll
              for (int kk = 0; kk < (KC > 0 ? KC : 1); ++kk) {
                const uint32_t ak = a_st + 2u * static_cast<uint32_t>(kk * p.a_px);
                const uint32_t bk = b_st + static_cast<uint32_t>(kk * NTAPS) * b_tap;
#pragma unroll
                for (int tp = 0; tp < NTAPS; ++tp)
#pragma unroll
                  for (int mb = 0; mb < MB; ++mb)
                    mma_bf16_lo(d_base + static_cast<uint32_t>(mb * NT),
                                ak + 2u * static_cast<uint32_t>(p.tap_shift[tp]) + 256u * mb, a_hi,
                                bk + static_cast<uint32_t>(tp) * b_tap, b_hi, idesc, (kk == 0 && tp == 0) ? acc0 : 1u);
              }
            }
            if (trace) trace[3] = clock64() - t_start;
            if (!p.w_all) mma_commit(&w_empty[wi]);
            mma_commit(&pc_empty[pci]);
            if (trace) trace[2] = clock64() - t_start;
            }
            __syncwarp(wmask);
            // ring positions, branch-free
            const bool pw = ++pci == pc_stages, ww = ++wi == w_stages;
            pci = pw ? 0 : pci;
            pph ^= pw ? 1u : 0u;
            wi = ww ? 0 : wi;
            wph ^= ww ? 1u : 0u;
          }
          if (issuer()) mma_commit(&acc_full[acc]);
          __syncwarp(wmask);
        }
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I4 = std::integral_constant<int, 4>;
      using I9 = std::integral_constant<int, 9>;
      using I16 = std::integral_constant<int, 16>;
      // the ResNet-50 / Inception shapes: 1x1 (four channel blocks per stage), 3x3 and 4x4
      // (one block per stage); anything else runs the runtime-trip-count loop
      auto by_mb = [&](auto kc_c, auto nt_c) {
        if (p.mb == 1)
          run(I1{}, kc_c, nt_c);
        else if (p.mb == 2)
          run(I2{}, kc_c, nt_c);
        else
          run(I4{}, kc_c, nt_c);
      };
      if (nt == 1 && p.kc == 4)
        by_mb(I4{}, I1{});
      else if (nt == 9 && p.kc == 2)
        by_mb(I2{}, I9{});
      else if (nt == 1 && p.kc == 2)
        by_mb(I2{}, I1{});
      else if (nt == 9 && p.kc == 1)
        by_mb(I1{}, I9{});
      else if (nt == 16 && p.kc == 1)
        by_mb(I1{}, I16{});
      else
        by_mb(I0{}, I1{});
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(NT));
    uint32_t g = 0, tl = 0;
    RingPos pcp, wpp;
    uint32_t w_res_seen = 0;  // resident slice: stage groups whose weights have landed
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const int a_px0 = p.linear ? v0 : (v0 / p.wsub) * p.wsub;
      const int v_off = v0 - a_px0;
      const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
      const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
      mbar_wait_t(&acc_empty[acc], apar ^ 1u, dbg ? &c_b : nullptr);
      tc_fence_after();
      const uint32_t d_base = tmem_base + acc * acc_cols;
      int ph = -1, cbi = -1;
      for (int it = 0; it < k_iters; ++it, ++g, pcp.adv(pc_stages)) {
        const int s = pcp.idx;
        const uint32_t par = pcp.ph;
        if (++ph == p.n_phases) ph = 0;
        if (ph == 0) ++cbi;
        long long* trace = (dbg && blockIdx.x == 0 && g < 256) ? dbg + gridDim.x * 16 + g * 8 : nullptr;
        if (RAW_F32)
          mbar_wait_t(&pc_conv[s], par, dbg ? &c_a : nullptr);
        else
          mbar_wait_t(&pc_full[s], par, dbg ? &c_a : nullptr);
        if (trace && lane == 0) trace[0] = clock64() - t_start;
        const uint32_t st = smem0 + s * L.pc_slot;
        const int ntaps = s_phase_ntaps[ph];
        const int kc_eff = min(p.kc, p.cb_in - cbi * p.kc);
        const int w_kk0 = p.w_resident ? cbi * p.kc : 0;  // resident slice: channel block index
        for (int t0 = 0; t0 < ntaps; t0 += p.w_taps, wpp.adv(w_stages)) {
          const int ws = wpp.idx;
          if (!p.w_resident) {
            mbar_wait_t(&w_full[ws], wpp.ph, dbg ? &c_a : nullptr);
          } else if (static_cast<uint32_t>(cbi) >= w_res_seen) {  // first tile only
            mbar_wait(&w_full[cbi], 0);
            w_res_seen = cbi + 1;
          }
          if (trace && lane == 0) trace[1] = clock64() - t_start;
          tc_fence_after();
          const uint32_t wst = smem0 + L.w_off + ws * L.w_slot;
          const int nt = min(p.w_taps, ntaps - t0);
          if (TS && elect_one()) {
            // single tap, one m-block: straight-line issue of the stage's kc x 6 (or kc)
            // MMAs with precomputed operand addresses (the generic loop's index
            // arithmetic cost ~50 cycles per MMA on the issuing thread)
            const uint32_t w_pc = L.w_piece >> 4;  // descriptor start-address units (16 B)
            const uint64_t bd0 = make_smem_desc(wst + static_cast<uint32_t>(w_kk0) * w_tap, 128, 256);
            const uint32_t a0 = tmem_base + ring_col0 + static_cast<uint32_t>(s) * ring_slot;
            const uint32_t d_hi = d_base, d_lo = d_base + static_cast<uint32_t>(NT);
            const uint32_t d_x = two_acc ? d_lo : d_hi;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= kc_eff) break;
              const uint64_t bk = bd0 + static_cast<uint64_t>((static_cast<uint32_t>(kk) * w_tap) >> 4);
              const uint32_t ak = a0 + static_cast<uint32_t>(kk) * kRingCols;
              const bool first = it == 0 && kk == 0;
              if (dbg_mode & 8) continue;  // ablation: no MMAs
              mma_bf16_ts(d_hi, ak, bk, idesc, first ? 0u : 1u);
              if (PIECES == 3) {
                mma_bf16_ts(d_x, ak, bk + w_pc, idesc, (two_acc && first) ? 0u : 1u);
                mma_bf16_ts(d_x, ak + 8u, bk, idesc, 1u);
                mma_bf16_ts(d_x, ak, bk + 2u * w_pc, idesc, 1u);
                mma_bf16_ts(d_x, ak + 8u, bk + w_pc, idesc, 1u);
                mma_bf16_ts(d_x, ak + 16u, bk, idesc, 1u);
              }
            }
            if (!p.w_resident) mma_commit(&w_empty[ws]);
            mma_commit(&pc_empty[s]);
            if (it == k_iters - 1) mma_commit(&acc_full[acc]);
          } else if (!TS && PIECES == 1 && nt <= kFastTaps && (p.mb == 1 || p.mb == 2 || p.mb == 4) && elect_one()) {
            // single-piece multi-tap stage, fully unrolled for the tile's m-block count:
            // the stage's tap shifts are read into registers with independent loads,
            // then every MMA is one 32-bit address add away (the generic loop below
            // serialises a shared-memory load and its index arithmetic per tap: ~125
            // cycles per MMA, 2x the tensor time of a 128x128x16 MMA)
            const uint64_t a_base = RAW_F32 ? make_smem_desc(st, L.a_plane, 128) : make_smem_desc_sw32(st);
            const uint64_t b_base = make_smem_desc(wst, 128, 256);
            const uint32_t a_hi = static_cast<uint32_t>(a_base >> 32), b_hi = static_cast<uint32_t>(b_base >> 32);
            const int tap0 = s_phase_tap0[ph] + t0;
            constexpr uint32_t kRow = RAW_F32 ? 1u : 2u;  // descriptor units (16 B) per pixel row
            uint32_t sh[kFastTaps];
#pragma unroll
            for (int i = 0; i < kFastTaps; ++i) sh[i] = i < nt ? kRow * static_cast<uint32_t>(s_tap_shift[tap0 + i]) : 0u;
            const uint32_t b_tap = w_tap >> 4;
            const bool do_mma = !(dbg_mode & 8);  // ablation: no MMAs
            auto issue = [&](auto mb_c) {
              constexpr int MB = decltype(mb_c)::value;
              for (int kk = 0; kk < kc_eff; ++kk) {
                const uint32_t ak = static_cast<uint32_t>(a_base) +
                                    (RAW_F32 ? static_cast<uint32_t>(v_off) : 2u * static_cast<uint32_t>(kk * p.a_px + v_off));
                const uint32_t bk = static_cast<uint32_t>(b_base) + ((static_cast<uint32_t>(w_kk0 + kk) * nt * w_tap) >> 4);
                const bool first_k = it == 0 && t0 == 0 && kk == 0;
#pragma unroll
                for (int tp = 0; tp < kFastTaps; ++tp) {
                  if (tp >= nt) break;
#pragma unroll
                  for (int mb = 0; mb < MB; ++mb)
                    if (do_mma)
                      mma_bf16_lo(d_base + static_cast<uint32_t>(mb * NT), ak + sh[tp] + kRow * 128u * mb, a_hi,
                                  bk + static_cast<uint32_t>(tp) * b_tap, b_hi, idesc, (first_k && tp == 0) ? 0u : 1u);
                }
              }
            };
            if (p.mb == 1)
              issue(std::integral_constant<int, 1>{});
            else if (p.mb == 2)
              issue(std::integral_constant<int, 2>{});
            else
              issue(std::integral_constant<int, 4>{});
            if (trace) trace[3] = clock64() - t_start;
            if (!p.w_resident) mma_commit(&w_empty[ws]);
            if (trace) trace[4] = clock64() - t_start;
            if (t0 + p.w_taps >= ntaps) {
              mma_commit(&pc_empty[s]);
              if (it == k_iters - 1) mma_commit(&acc_full[acc]);
            }
          } else if (!TS && !(PIECES == 1 && nt <= kFastTaps && (p.mb == 1 || p.mb == 2 || p.mb == 4)) && elect_one()) {
            // operand descriptors are packed once per stage; per MMA only the 16 B-unit
            // start-address field advances (no repacking, no parameter reads)
            const uint64_t a_base = RAW_F32 ? make_smem_desc(st, L.a_plane, 128) : make_smem_desc_sw32(st);
            const uint64_t b_base = make_smem_desc(wst, 128, 256);
            const uint32_t a_pc = RAW_F32 ? (2u * L.a_plane) >> 4 : 0u, w_pc = L.w_piece >> 4;
            const int tap0 = s_phase_tap0[ph] + t0;
            for (int kk = 0; kk < kc_eff; ++kk)
              for (int tp = 0; tp < nt; ++tp) {
                const int shift = s_tap_shift[tap0 + tp];
                const uint32_t b_off = ((static_cast<uint32_t>(w_kk0 + kk) * nt + tp) * w_tap) >> 4;
                for (int mb = 0; mb < p.mb; ++mb) {
                  const uint32_t rows = static_cast<uint32_t>(v_off + mb * 128 + shift);
                  // MN-major pieces: 16 B per pixel row; SW32 K-major bf16: 32 B per pixel row
                  const uint32_t a_off = RAW_F32 ? rows : 2u * (static_cast<uint32_t>(kk * p.a_px) + rows);
                  const uint32_t d_hi = d_base + static_cast<uint32_t>(mb * NT);
                  const uint32_t d_lo = d_hi + static_cast<uint32_t>(p.mb * NT);
                  const uint32_t d_x = two_acc ? d_lo : d_hi;
                  const bool first = it == 0 && t0 == 0 && tp == 0 && kk == 0;
                  const uint64_t ad = a_base + a_off, bd = b_base + b_off;
                  if (dbg_mode & 8) continue;  // ablation: no MMAs
                  mma_bf16(d_hi, ad, bd, idesc, first ? 0u : 1u);
                  if (PIECES == 3) {  // products (ia, ib) with ia + ib <= 2
                    mma_bf16(d_x, ad, bd + w_pc, idesc, (two_acc && first) ? 0u : 1u);
                    mma_bf16(d_x, ad + a_pc, bd, idesc, 1u);
                    mma_bf16(d_x, ad, bd + 2u * w_pc, idesc, 1u);
                    mma_bf16(d_x, ad + a_pc, bd + w_pc, idesc, 1u);
                    mma_bf16(d_x, ad + 2u * a_pc, bd, idesc, 1u);
                  }
                }
              }
            if (trace) trace[3] = clock64() - t_start;
            if (!p.w_resident) mma_commit(&w_empty[ws]);
            if (trace) trace[4] = clock64() - t_start;
            if (t0 + p.w_taps >= ntaps) {
              mma_commit(&pc_empty[s]);
              if (it == k_iters - 1) mma_commit(&acc_full[acc]);
            }
          }
          __syncwarp();
          if (trace && lane == 0) trace[2] = clock64() - t_start;
        }
      }
    }
    if (dbg && lane == 0) {
      dbg[4] = c_a;
      dbg[5] = c_b;
    }
  } else if (kDevBuild && !RAW_F32 && !TS && (dbg_mode & 1024) && warp >= kEpiWarp0) {
    // ablation (developer builds): the epilogue does no work, it only hands the
    // accumulators back (warps 4..7 arrive for every epilogue group)
    if (warp < kEpiWarp0 + 4) {
      uint32_t tl = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
        const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
        const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
        mbar_wait(&acc_full[acc], apar);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0)
          for (int g = 0; g < n_epi_groups; ++g) mbar_arrive(&acc_empty[acc]);
      }
    }
  } else if (p.tma_store && ((warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) ||
                             (epi2 && warp >= kCvtWarp0 && warp < kEpiWarp0 + 4 * n_epi_groups) ||
                             (ts_epi2 && warp >= kCvtWarp0 + 4))) {
    // ------------------------------------------------------------ lean TMA-store epilogue (warps 4..7)
    // two output blocks per step: one 32-column TMEM load per accumulator, one
    // proxy fence and one bulk store of a {16 lanes, 32 pixels, 2 blocks} box
    const int qrow = (warp % 4) * 32;
    // pixel (within the warp's 32-row group) held by this lane's accumulator row: a_sw128
    // stages permute the four pixels of each 128 B row (conv_params.h)
    const int plane_px = p.a_sw128 ? (lane ^ ((lane >> 3) & 3)) : lane;
    const uint32_t esz = p.out_bf16 ? 2u : 4u;
    const uint32_t slot_bytes = 2u * 32u * 16u * esz;
    const int v_end = p.P * p.Q;  // dense output plane (wsub == Q)
    const int eg = ts_epi2 ? (warp >= kCvtWarp0 ? 1 : 0) : (warp - kEpiWarp0) / 4, n_eg = n_epi_groups;
    uint8_t* stg0 = smem + L.epi_off + (eg * 4 + warp % 4) * 2u * slot_bytes;
    // FUSED = residual add / ReLU-backward mask present: the plain variant has no
    // per-pixel addressing or extra loads in its loop (smaller, faster code)
    auto lean = [&](auto fused_tag, auto ops_tag) {
      constexpr bool FUSED = decltype(fused_tag)::value;
      constexpr bool OPS = decltype(ops_tag)::value;  // bias / ReLU present
    uint32_t n_st = 0, tl = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
      const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
      mbar_wait_t(&acc_full[acc], apar, dbg ? &c_a : nullptr);
      tc_fence_after();
      const uint32_t d_base = tmem_base + acc * acc_cols + (static_cast<uint32_t>(qrow) << 16);
      const int egr = static_cast<int>((static_cast<uint32_t>(eg) + tl) % static_cast<uint32_t>(n_eg));  // rotated: see n_epi_groups
      for (int mb = 0; mb < p.mb; ++mb) {
        for (int g0 = 2 * egr; g0 < p.nb; g0 += 2 * n_eg) {
          const int kb0 = ntile * p.nb + g0;
          if (kb0 >= p.kb_out) break;
          const bool pair = g0 + 1 < p.nb;
          uint32_t r[32], rl[32];
          tmem_ld32(d_base + static_cast<uint32_t>(mb * NT + g0 * 16), r);
          if (two_acc) tmem_ld32(d_base + static_cast<uint32_t>((p.mb + mb) * NT + g0 * 16), rl);
          tmem_ld_wait();
          uint8_t* stg = stg0 + (n_st & 1u) * slot_bytes;
          if (n_st >= 2) {  // this slot's previous store must have left smem
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j == 1 && !pair) break;
            const int kb = kb0 + j;
            float vals[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              vals[e] = two_acc ? __uint_as_float(r[16 * j + e]) + __uint_as_float(rl[16 * j + e])
                                : __uint_as_float(r[16 * j + e]);
            if (OPS && p.bias != nullptr && kb < p.kb_out) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += p.bias[kb * 16 + e];
            }
            // dense output: pixel v of plane (n, kb) at ((n*out_cb + kb)*P*Q + v)*16 lanes
            const int v = FUSED ? v0 + mb * 128 + qrow + plane_px : 0;
            const bool live = FUSED && v < v_end && kb < p.kb_out;
            const long long px_off = FUSED ? ((static_cast<long long>(n) * p.out_cb + kb) * v_end + v) * 16LL * esz : 0;
            if (FUSED && p.add != nullptr && live) {  // residual add / gradient sum
              float a[16];
              load16(reinterpret_cast<const uint8_t*>(p.add) + px_off, p.out_bf16, a);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += a[e];
            }
            if (OPS && p.relu) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = fmaxf(vals[e], 0.0f);
            }
            if (FUSED && p.mask != nullptr && live) {  // ReLU backward through the forward activation
              float m[16];
              load16(reinterpret_cast<const uint8_t*>(p.mask) + px_off, p.out_bf16, m);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = m[e] > 0.0f ? vals[e] : 0.0f;
            }
            const uint32_t row = static_cast<uint32_t>(j * 32 + plane_px);
            if (p.out_bf16) {
              const float a8[8] = {vals[0], vals[1], vals[2], vals[3], vals[4], vals[5], vals[6], vals[7]};
              const float b8[8] = {vals[8], vals[9], vals[10], vals[11], vals[12], vals[13], vals[14], vals[15]};
              *reinterpret_cast<uint4*>(stg + sw32(row, 0)) = cast8(a8);
              *reinterpret_cast<uint4*>(stg + sw32(row, 1)) = cast8(b8);
            } else {
#pragma unroll
              for (int c = 0; c < 4; ++c)
                *reinterpret_cast<float4*>(stg + sw64(row, c)) =
                    make_float4(vals[4 * c], vals[4 * c + 1], vals[4 * c + 2], vals[4 * c + 3]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            // rows past P*Q and blocks past K are clipped by the tensor bounds
            tma_store_4d(pair ? &map_out2 : &map_out, stg, 0, v0 + mb * 128 + qrow, kb0, n);
            bulk_commit_group();
          }
          ++n_st;
          (void)slot_bytes;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
    };
    // bf16 residual add / ReLU mask: the two extra operand tiles are fetched one step
    // AHEAD into registers (the first step of a tile before its accumulator wait),
    // so their HBM latency overlaps the previous step instead of stalling every
    // step (these epilogues move ~3x the bytes of their mainloop)
    // NOPS = fused operands (1: residual add OR ReLU mask, 2: both); DEPTH = steps the
    // operand loads run ahead of their use (the fused 1x1 layers are bound by these
    // loads: the forward's residual add runs two steps -- 4 KB per warp -- ahead)
    auto lean_fused_bf16 = [&](auto nops_c, auto depth_c) {  // instantiated only for the bf16-activation kernels
      constexpr int NOPS = decltype(nops_c)::value, DEPTH = decltype(depth_c)::value;
      constexpr int NB = 4 * NOPS;  // uint4 per step: (op) x (2 blocks) x (2 halves)
      uint32_t n_st = 0, tl = 0;
      const uint8_t* addp = reinterpret_cast<const uint8_t*>(p.add);
      const uint8_t* maskp = reinterpret_cast<const uint8_t*>(p.mask);
      // operand slots: [0, 4) the first operand (add if present, else mask), [4, 8) the mask when both
      const uint8_t* op0 = addp ? addp : maskp;
      int egr = eg;  // this tile's rotated group index (see n_epi_groups)
      auto fetch = [&](int n, int v0, int ntile, int s, int ng, uint4 (&b)[NB]) {
        const int mb = s / ng, g0 = 2 * egr + 2 * n_eg * (s - (s / ng) * ng);
        const int kb0 = ntile * p.nb + g0;
        const bool pair = g0 + 1 < p.nb;
        const int v = v0 + mb * 128 + qrow + plane_px;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int kb = kb0 + j;
          const bool live = v < v_end && kb < p.kb_out && (j == 0 || pair);
          const long long off = ((static_cast<long long>(n) * p.out_cb + kb) * v_end + v) * 32LL;
          const uint4 z = make_uint4(0, 0, 0, 0);
          b[2 * j] = live ? *reinterpret_cast<const uint4*>(op0 + off) : z;
          b[2 * j + 1] = live ? *reinterpret_cast<const uint4*>(op0 + off + 16) : z;
          if constexpr (NOPS == 2) {
            b[4 + 2 * j] = live ? *reinterpret_cast<const uint4*>(maskp + off) : z;
            b[4 + 2 * j + 1] = live ? *reinterpret_cast<const uint4*>(maskp + off + 16) : z;
          }
        }
      };
      auto unpack = [](const uint4& a, const uint4& b, float (&f)[16]) {
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          f[2 * e] = __uint_as_float(w[e] << 16);
          f[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
        }
      };
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
        int n, v0, ntile;
        tile_coords(t, n, v0, ntile);
        // The fused operands of this CTA's NEXT tile go to L2 now (one bulk prefetch per lane:
        // a 32-pixel slab of one channel block is 1 KB contiguous), a whole tile ahead of the
        // register fetches below, which then see L2 latency instead of HBM latency: these
        // epilogues are bound by those loads (two steps = 4 KB per warp in flight)
        // (two-operand epilogues only -- one step of register prefetch: 0.240 -> 0.227 ms on the
        // 56x56 256-channel backward-data; the one-operand ones, two steps ahead, measured
        // 2-4 % slower with it)
        if (NOPS == 2 && t + static_cast<int>(gridDim.x) < n_tiles && !(kDevBuild && (dbg_mode & 16384))) {
          int n2, v02, ntile2;
          tile_coords(t + static_cast<int>(gridDim.x), n2, v02, ntile2);
          const int egr2 = static_cast<int>((static_cast<uint32_t>(eg) + tl + 1u) % static_cast<uint32_t>(n_eg));
          // lane -> (operand, m-block, pair slot, block of the pair)
          const int op = lane >> 4, mb2 = (lane >> 3) & 1, ps = (lane >> 1) & 3, j = lane & 1;
          const int kb = ntile2 * p.nb + 2 * egr2 + 2 * n_eg * ps + j;
          const int v = v02 + mb2 * 128 + qrow;
          const uint8_t* src = op == 0 ? op0 : (NOPS == 2 ? maskp : nullptr);
          if (src != nullptr && mb2 < p.mb && 2 * egr2 + 2 * n_eg * ps + j < p.nb && kb < p.kb_out && v < v_end) {
            const int npx = min(32, v_end - v);
            l2_prefetch_bulk(src + ((static_cast<long long>(n2) * p.out_cb + kb) * v_end + v) * 32LL,
                             static_cast<uint32_t>(npx) * 32u);
          }
        }
        egr = static_cast<int>((static_cast<uint32_t>(eg) + tl) % static_cast<uint32_t>(n_eg));
        int ng = 0;  // this group's block pairs in the tile
        for (int g0 = 2 * egr; g0 < p.nb && ntile * p.nb + g0 < p.kb_out; g0 += 2 * n_eg) ++ng;
        const int total = p.mb * ng;
        uint4 buf[DEPTH + 1][NB];  // buf[0] = this step's operands, buf[d] = step + d's
#pragma unroll
        for (int d = 0; d < DEPTH; ++d)
          if (d < total) fetch(n, v0, ntile, d, ng, buf[d]);
        const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
        const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
        mbar_wait_t(&acc_full[acc], apar, dbg ? &c_a : nullptr);
        tc_fence_after();
        const uint32_t d_base = tmem_base + acc * acc_cols + (static_cast<uint32_t>(qrow) << 16);
        for (int s = 0; s < total; ++s) {
          if (s + DEPTH < total) fetch(n, v0, ntile, s + DEPTH, ng, buf[DEPTH]);
          const int mb = s / ng, g0 = 2 * egr + 2 * n_eg * (s - mb * ng);
          const int kb0 = ntile * p.nb + g0;
          const bool pair = g0 + 1 < p.nb;
          uint32_t r[32], rl[32];
          tmem_ld32(d_base + static_cast<uint32_t>(mb * NT + g0 * 16), r);
          if (two_acc) tmem_ld32(d_base + static_cast<uint32_t>((p.mb + mb) * NT + g0 * 16), rl);
          tmem_ld_wait();
          uint8_t* stg = stg0 + (n_st & 1u) * slot_bytes;
          if (n_st >= 2) {  // this slot's previous store must have left smem
            if (lane == 0) bulk_wait_group_read<1>();
            __syncwarp();
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j == 1 && !pair) break;
            const int kb = kb0 + j;
            float vals[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              vals[e] = two_acc ? __uint_as_float(r[16 * j + e]) + __uint_as_float(rl[16 * j + e])
                                : __uint_as_float(r[16 * j + e]);
            if (p.bias != nullptr && kb < p.kb_out) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += p.bias[kb * 16 + e];
            }
            if (addp) {
              float a[16];
              unpack(buf[0][2 * j], buf[0][2 * j + 1], a);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += a[e];
            }
            if (p.relu) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = fmaxf(vals[e], 0.0f);
            }
            if (maskp) {
              float m[16];
              constexpr int mo = NOPS == 2 ? 4 : 0;
              unpack(buf[0][mo + 2 * j], buf[0][mo + 2 * j + 1], m);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = m[e] > 0.0f ? vals[e] : 0.0f;
            }
            const uint32_t row = static_cast<uint32_t>(j * 32 + plane_px);
            const float a8[8] = {vals[0], vals[1], vals[2], vals[3], vals[4], vals[5], vals[6], vals[7]};
            const float b8[8] = {vals[8], vals[9], vals[10], vals[11], vals[12], vals[13], vals[14], vals[15]};
            *reinterpret_cast<uint4*>(stg + sw32(row, 0)) = cast8(a8);
            *reinterpret_cast<uint4*>(stg + sw32(row, 1)) = cast8(b8);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_4d(pair ? &map_out2 : &map_out, stg, 0, v0 + mb * 128 + qrow, kb0, n);
            bulk_commit_group();
          }
          ++n_st;
#pragma unroll
          for (int d = 0; d < DEPTH; ++d)
#pragma unroll
            for (int i = 0; i < NB; ++i) buf[d][i] = buf[d + 1][i];
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[acc]);
      }
    };
    bool done = false;
    if constexpr (!RAW_F32) {
      if ((p.add != nullptr || p.mask != nullptr) && p.out_bf16 && !(dbg_mode & 512)) {  // dbg 512: no prefetch
        if (p.add != nullptr && p.mask != nullptr)
          lean_fused_bf16(std::integral_constant<int, 2>{}, std::integral_constant<int, 1>{});
        else if (p.add != nullptr)  // residual add (forward): measured +5 % with two steps ahead
          lean_fused_bf16(std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{});
        else  // ReLU mask alone (backward-data): one step ahead measured faster
          lean_fused_bf16(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{});
        done = true;
      }
    }
    if (done) {
    } else if (p.add != nullptr || p.mask != nullptr)
      lean(std::true_type{}, std::true_type{});
    else if (p.bias != nullptr || p.relu)
      lean(std::false_type{}, std::true_type{});
    else
      lean(std::false_type{}, std::false_type{});
    if (lane == 0) bulk_wait_group0();
    if (dbg && threadIdx.x == kEpiWarp0 * 32) {
      dbg[6] = c_a;
      dbg[7] = clock64() - t_start - c_a;
    }
  } else if (TS && warp >= kCvtWarp0) {
    // ------------------------------------------------------------ TS converters (smem fp32 -> TMEM pieces)
    // group = (warp - 8) / 4 takes stages g % cvt_groups == group; a warp owns
    // TMEM lanes (warp % 4) * 32 .. +31 = A rows = pixels v_off + row
    const int grp = (warp - kCvtWarp0) / 4;
    const uint32_t q = static_cast<uint32_t>(warp % 4);
    const int row = static_cast<int>(q) * 32 + lane;
    uint32_t g = 0;
    RingPos rr, pr;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const int a_px0 = p.linear ? v0 : (v0 / p.wsub) * p.wsub;
      // raw row of this thread's pixel in channel block kk of the stage: base + kk * kstride
      uint32_t base, kstride;
      if (p.mimg > 0) {  // slot = [image][kk][pixel]
        const int hw = p.a_load_px / p.mimg;
        const int img = row / hw;
        base = img < p.mimg ? static_cast<uint32_t>(img * p.kc * hw + (row - img * hw)) : 0u;
        kstride = static_cast<uint32_t>(hw);
      } else {           // slot = [kk][pixel]
        base = static_cast<uint32_t>(v0 - a_px0 + row);
        kstride = static_cast<uint32_t>(p.a_px);
      }
      int ph = -1, cbi = -1;
      for (int it = 0; it < k_iters; ++it, ++g, rr.adv(raw_stages), pr.adv(pc_stages)) {
        if (++ph == p.n_phases) ph = 0;
        if (ph == 0) ++cbi;
        if (static_cast<int>(g & static_cast<uint32_t>(cvt_groups - 1)) != grp) continue;
        const int rs = rr.idx, ps = pr.idx;
        long long* ctr = (dbg && blockIdx.x == 0 && g < 256 && lane == 0 && q == 0) ? dbg + gridDim.x * 16 + g * 8 : nullptr;
        mbar_wait_bt(&pc_empty[ps], pr.ph ^ 1u, dbg ? &c_b : nullptr);
        if (ctr) ctr[4] = clock64() - t_start;
        mbar_wait_bt(&raw_full[rs], rr.ph, dbg ? &c_a : nullptr);
        if (ctr) ctr[3] = clock64() - t_start;
        tc_fence_after();
        const uint8_t* raw = smem + L.raw_off + rs * L.raw_slot;
        const int kc_eff = min(p.kc, p.cb_in - cbi * p.kc);
        if (!(dbg_mode & 4))
        for (int kk = 0; kk < kc_eff; ++kk) {
        const uint32_t px = base + static_cast<uint32_t>(kk) * kstride;
        float v[16];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float4 f = *reinterpret_cast<const float4*>(raw + sw64(px, k));
          v[4 * k] = f.x;
          v[4 * k + 1] = f.y;
          v[4 * k + 2] = f.z;
          v[4 * k + 3] = f.w;
        }
        const uint32_t col = tmem_base + (q * 32u << 16) + ring_col0 + static_cast<uint32_t>(ps) * ring_slot +
                             static_cast<uint32_t>(kk) * kRingCols;
        if (PIECES == 3) {
          uint32_t h[8], m[8], l[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            h[e] = cvt2(v[2 * e], v[2 * e + 1]);
            const float ra = v[2 * e] - lo_f(h[e]), rb = v[2 * e + 1] - hi_f(h[e]);
            m[e] = cvt2(ra, rb);
            l[e] = cvt2(ra - lo_f(m[e]), rb - hi_f(m[e]));
          }
          tmem_st8(col, h);
          tmem_st8(col + 8, m);
          tmem_st8(col + 16, l);
        } else {
          uint32_t h[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) h[e] = cvt2(v[2 * e], v[2 * e + 1]);
          tmem_st8(col, h);
        }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (ctr) ctr[5] = clock64() - t_start;
        if (lane == 0) {
          mbar_arrive(&raw_empty[rs]);
          mbar_arrive(&pc_conv[ps]);
        }
      }
    }
    if (dbg && threadIdx.x == kCvtWarp0 * 32) {
      dbg[1] = c_a;
      dbg[2] = c_b;
      dbg[3] = clock64() - t_start - c_a - c_b;
    }
  } else if (warp >= kCvtWarp0 && !epi_reg3) {
    // ------------------------------------------------------------ converters (smem fp32 -> bf16 pieces)
    if (RAW_F32) {
      const int grp = (warp - kCvtWarp0) / cvt_group_warps;  // this group converts stages g % cvt_groups == grp
      const int ct = threadIdx.x - (kCvtWarp0 + grp * cvt_group_warps) * 32;
      const int items = 2 * ((p.a_px + 31) / 32) * 32;  // (pixel, 16B bf16 chunk)
      uint32_t g = 0;
      RingPos rr, pr;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int it = 0; it < k_iters; ++it, ++g, rr.adv(raw_stages), pr.adv(pc_stages)) {
          if (static_cast<int>(g & static_cast<uint32_t>(cvt_groups - 1)) != grp) continue;
          const int rs = rr.idx, ps = pr.idx;
          mbar_wait_t(&pc_empty[ps], pr.ph ^ 1u, dbg ? &c_b : nullptr);  // first: see cvt_groups
          mbar_wait_t(&raw_full[rs], rr.ph, dbg ? &c_a : nullptr);
          const uint8_t* raw = smem + L.raw_off + rs * L.raw_slot;
          uint8_t* pcs = smem + ps * L.pc_slot;
          for (int i = ct; i < items; i += cvt_group_warps * 32) {
            // a warp converts one bf16 chunk c of 32 consecutive pixels: swizzled
            // reads and contiguous piece writes are both bank-conflict free
            const int c = (i >> 5) & 1, j = ((i >> 6) << 5) | (i & 31);
            if (j >= p.a_px) continue;
            const float4 a = *reinterpret_cast<const float4*>(raw + sw64(j, 2 * c));
            const float4 b = *reinterpret_cast<const float4*>(raw + sw64(j, 2 * c + 1));
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint8_t* dst = pcs + c * L.a_plane + j * 16;
            if (PIECES == 3) {
              uint4 h, m, l;
              split8(v, h, m, l);
              *reinterpret_cast<uint4*>(dst) = h;
              *reinterpret_cast<uint4*>(dst + 2 * L.a_plane) = m;
              *reinterpret_cast<uint4*>(dst + 4 * L.a_plane) = l;
            } else {
              *reinterpret_cast<uint4*>(dst) = cast8(v);
            }
          }
          fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&raw_empty[rs]);
            mbar_arrive(&pc_conv[ps]);
          }
        }
      }
      if (dbg && threadIdx.x == kCvtWarp0 * 32) {
        dbg[1] = c_a;
        dbg[2] = c_b;
        dbg[3] = clock64() - t_start - c_a - c_b;
      }
    }
  } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4 * n_epi_groups) {
    // ------------------------------------------------------------ epilogue (warps 4..7 [, 8..15])
    // warp -> TMEM lane quarter (warp % 4); group eg takes items eg, eg + n_groups, ...
    const int qrow = (warp % 4) * 32;
    const int eg = (warp - kEpiWarp0) / 4;
    const int n_pairs = (p.nb + 1) / 2;
    const int g_lo = 0, g_hi = p.nb;
    const int v_end = p.P * p.wsub;
    const int esz = p.out_bf16 ? 2 : 4;
    uint8_t* obase = reinterpret_cast<uint8_t*>(p.out);
    uint32_t tl = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const uint32_t acc = p.acc_bufs == 2 ? (tl & 1u) : 0u;
      const uint32_t apar = p.acc_bufs == 2 ? ((tl >> 1) & 1u) : (tl & 1u);
      mbar_wait_t(&acc_full[acc], apar, dbg ? &c_a : nullptr);
      tc_fence_after();
      const uint32_t d_base = tmem_base + acc * acc_cols + (static_cast<uint32_t>(qrow) << 16);
      for (int item = static_cast<int>((static_cast<uint32_t>(eg) + tl) % static_cast<uint32_t>(n_epi_groups));
           item < p.mb * n_pairs; item += n_epi_groups) {
        const int mb = item / n_pairs;
        int v = v0 + mb * 128 + qrow + lane;
        int nn = n;
        bool valid;
        if (p.mimg > 0) {  // row -> (image, pixel) of the multi-image tile (packed: at img_pitch)
          const int pitch = (!RAW_F32 && p.img_pitch > 0) ? p.img_pitch : v_end;  // (packed: bf16 plans only)
          const int img = v / pitch;
          nn = n + img;
          v -= img * pitch;
          valid = img < p.mimg && nn < p.n_img;
        } else {
          valid = v < v_end;
        }
        const int pp = v / p.wsub;
        const int qq = v - pp * p.wsub;
        valid = valid && qq < p.Q && (RAW_F32 || pp < p.P);  // (packed tiles' padding rows: bf16 plans)
        const int y = p.out_y0 + pp * p.out_scale;
        const int x = p.out_x0 + qq * p.out_scale;
        for (int g0 = 2 * (item - mb * n_pairs); g0 < ((dbg_mode & 64) ? g_lo : g_hi); g0 += 2 * n_pairs) {
          // two 16-column TMEM loads in flight, one wait
          const int ng = min(2, g_hi - g0);
          uint32_t r[2][16], rl[2][16];
          // a bf16 residual OR ReLU-mask operand (one of them: the register budget) of both
          // blocks is fetched before the TMEM loads: its HBM latency overlaps them
          const void* pre_src = (p.add != nullptr) != (p.mask != nullptr) ? (p.add ? p.add : p.mask) : nullptr;
          const bool pre_on = !RAW_F32 && p.out_bf16 && pre_src != nullptr;  // (bf16 kernels only: registers)
          // both operands (backward-data of a block's first conv on multi-image / halo'd tiles:
          // gradient sum + ReLU mask): the mask of both blocks goes through a second buffer
          const bool pre_both = !RAW_F32 && p.out_bf16 && p.add != nullptr && p.mask != nullptr;
          uint4 pre[2][2], prem[2][2];
          if (pre_both) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int kb = ntile * p.nb + g0 + k;
              const bool live = k < ng && valid && kb < p.kb_out;
              const long long off =
                  (((static_cast<long long>(nn) * p.out_cb + kb) * p.out_hp + y) * p.out_wp + x) * 32LL;
              const uint4 z = make_uint4(0, 0, 0, 0);
              const uint8_t* sa = reinterpret_cast<const uint8_t*>(p.add) + off;
              const uint8_t* sm = reinterpret_cast<const uint8_t*>(p.mask) + off;
              pre[k][0] = live ? *reinterpret_cast<const uint4*>(sa) : z;
              pre[k][1] = live ? *reinterpret_cast<const uint4*>(sa + 16) : z;
              prem[k][0] = live ? *reinterpret_cast<const uint4*>(sm) : z;
              prem[k][1] = live ? *reinterpret_cast<const uint4*>(sm + 16) : z;
            }
          }
          if (pre_on) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int kb = ntile * p.nb + g0 + k;
              const bool live = k < ng && valid && kb < p.kb_out;
              const long long off =
                  (((static_cast<long long>(nn) * p.out_cb + kb) * p.out_hp + y) * p.out_wp + x) * 32LL;
              const uint4 z = make_uint4(0, 0, 0, 0);
              const uint8_t* src = reinterpret_cast<const uint8_t*>(pre_src) + off;
              pre[k][0] = live ? *reinterpret_cast<const uint4*>(src) : z;
              pre[k][1] = live ? *reinterpret_cast<const uint4*>(src + 16) : z;
            }
          }
#pragma unroll
          for (int k = 0; k < 2; ++k)
            if (k < ng && !(dbg_mode & 2)) {
              tmem_ld16(d_base + static_cast<uint32_t>(mb * NT + (g0 + k) * 16), r[k]);
              if (two_acc) tmem_ld16(d_base + static_cast<uint32_t>((p.mb + mb) * NT + (g0 + k) * 16), rl[k]);
            }
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int kb = ntile * p.nb + g0 + k;
            if (k >= ng || !valid || kb >= p.kb_out) continue;
            float vals[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              vals[e] = two_acc ? __uint_as_float(r[k][e]) + __uint_as_float(rl[k][e]) : __uint_as_float(r[k][e]);
            // APPLY after the final reduction step (kernel_streams.cpp:96-120)
            if (p.bias != nullptr && kb < p.kb_out) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += p.bias[kb * 16 + e];
            }
            const long long plane = static_cast<long long>(nn) * p.out_cb + kb;
            const long long px_off = ((plane * p.out_hp + y) * p.out_wp + x) * 16LL * esz;
            if (p.add != nullptr) {  // residual add / gradient sum
              float a[16];
              if (pre_on)
                load16(&pre[k][0], 1, a);
              else if (pre_both)
                load16(&pre[k][0], 1, a);
              else
                load16(reinterpret_cast<const uint8_t*>(p.add) + px_off, p.out_bf16, a);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] += a[e];
            }
            if (p.relu) {
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = vals[e] > 0.0f ? vals[e] : 0.0f;
            }
            if (p.mask != nullptr) {  // ReLU backward: gradient through the forward activation
              float m[16];
              if (pre_on)
                load16(&pre[k][0], 1, m);
              else if (pre_both)
                load16(&prem[k][0], 1, m);
              else
                load16(reinterpret_cast<const uint8_t*>(p.mask) + px_off, p.out_bf16, m);
#pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = m[e] > 0.0f ? vals[e] : 0.0f;
            }
            if (!(dbg_mode & 1)) store16(obase + px_off, vals, p.out_bf16);
            if (p.out_fill) {
              // 1x1 / stride-2 backward: this lattice pixel (2y', 2x') owns the three
              // off-lattice neighbours, which are exactly zero (acceptance.cpp:106-117);
              // writing them here replaces a separate zero pass over dI
              const long long row = (plane * p.out_hp + y) * p.out_wp;
              if (x + 1 < p.fill_w_end) store16_zero(obase + (row + x + 1) * 16LL * esz, p.out_bf16);
              if (y + 1 < p.fill_h_end) {
                store16_zero(obase + (row + p.out_wp + x) * 16LL * esz, p.out_bf16);
                if (x + 1 < p.fill_w_end) store16_zero(obase + (row + p.out_wp + x + 1) * 16LL * esz, p.out_bf16);
              }
            }
            if (p.out_halo_h | p.out_halo_w) {
              // zero the halo pixels whose clamp onto the interior is this pixel
              const int dy0 = pp == 0 ? -p.out_halo_h : 0, dy1 = pp == p.P - 1 ? p.out_halo_h : 0;
              const int dx0 = qq == 0 ? -p.out_halo_w : 0, dx1 = qq == p.Q - 1 ? p.out_halo_w : 0;
              for (int dy = dy0; dy <= dy1; ++dy)
                for (int dx = dx0; dx <= dx1; ++dx)
                  if (dy != 0 || dx != 0)
                    store16_zero(obase + ((plane * p.out_hp + y + dy) * p.out_wp + x + dx) * 16LL * esz, p.out_bf16);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
    if (p.tma_store && lane == 0) bulk_wait_group0();
    if (dbg && threadIdx.x == kEpiWarp0 * 32) {
      dbg[6] = c_a;
      dbg[7] = clock64() - t_start - c_a;
    }  }
  tc_fence_before();
  __syncthreads();
  if (dbg && threadIdx.x == 0) {
    dbg[8] = clock64() - t_start;
    uint64_t gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    dbg[10] = static_cast<long long>(gt);
  }
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

}  // namespace dconv_sm100
