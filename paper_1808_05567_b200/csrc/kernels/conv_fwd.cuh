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
// Warp roles (448 threads): w0 activation TMA producer, w1 MMA issuer (+TMEM
// owner), w2 weight producer (fp32 path), w4..w7 epilogue, w8..w13 converters
// (fp32 activations only). Persistent over tiles with double-buffered TMEM.
//
// Numerics: pieces = 1 is bf16 x bf16 -> fp32 (TMEM). pieces = 3 splits every
// fp32 operand into hi + mid + lo bf16 (exact) and accumulates the six
// products with i + j <= 2: fp32-accurate (~2^-24 relative per product).
#pragma once
#include <cuda_bf16.h>

#include "conv_params.h"
#include "sm100_ptx.cuh"

namespace dconv_sm100 {

constexpr int kFwdThreads = 256;
constexpr int kMaxStages = 8;
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
  uint32_t pc_slot;  // bytes per piece slot
  uint32_t raw_off;  // raw ring starts after the piece ring
};

__host__ __device__ inline FwdSmem fwd_smem_layout(int a_px, int taps_box, int nb, int pieces, bool raw_f32,
                                                   int piece_stages) {
  FwdSmem L;
  L.a_plane = static_cast<uint32_t>(a_px) * 16u;
  L.raw_slot = raw_f32 ? ((static_cast<uint32_t>(a_px) * 64u + 1023u) & ~1023u) : 0u;
  L.w_piece = static_cast<uint32_t>(taps_box) * (2u * nb) * 256u;
  L.pc_slot = (static_cast<uint32_t>(pieces) * (2u * L.a_plane + L.w_piece) + 1023u) & ~1023u;
  L.raw_off = static_cast<uint32_t>(piece_stages) * L.pc_slot;
  return L;
}

constexpr int kFwdWarps = 14;  // w0 A/raw producer, w1 MMA, w2 W producer, w3 idle, w4-7 epilogue, w8-13 converters
constexpr int kFwdThreadsP = kFwdWarps * 32;
constexpr int kCvtWarp0 = 8, kCvtWarps = 6;

// Persistent implicit-GEMM forward: grid = #SMs, CTA c handles tiles c, c+G, ...
// (tile = (image, virtual-row block) x output-channel tile). Two TMEM
// accumulator buffers let the epilogue of tile i overlap the mainloop of i+1.
template <bool RAW_F32, int PIECES>
__global__ void __launch_bounds__(kFwdThreadsP, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ FwdParams p, int raw_stages,
                    int pc_stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t raw_full[kMaxStages], raw_empty[kMaxStages];
  __shared__ __align__(8) uint64_t pc_full[kMaxStages], pc_conv[kMaxStages], pc_empty[kMaxStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const FwdSmem L = fwd_smem_layout(p.a_px, p.taps_box, p.nb, PIECES, RAW_F32, pc_stages);
  const uint32_t smem0 = smem_u32(smem);
  const int NT = 16 * p.nb;
  const int k_iters = p.cb_in * p.n_phases;
  const int n_mtiles = p.n_img * p.tiles_per_img;
  const int n_tiles = n_mtiles * p.n_ntiles;
  const uint32_t acc_cols = static_cast<uint32_t>(p.mb * NT);

  uint32_t tmem_cols = 32;
  while (tmem_cols < 2u * acc_cols) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    for (int s = 0; s < raw_stages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], kCvtWarps);
    }
    for (int s = 0; s < pc_stages; ++s) {
      mbar_init(&pc_full[s], 1);
      mbar_init(&pc_conv[s], kCvtWarps);
      mbar_init(&pc_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  // tile t -> (n, v0, ntile); output-channel tiles innermost so consecutive
  // CTAs share the activation tile through L2
  auto tile_coords = [&](int t, int& n, int& v0, int& ntile) {
    ntile = t % p.n_ntiles;
    const int mt = t / p.n_ntiles;
    n = mt / p.tiles_per_img;
    v0 = (mt % p.tiles_per_img) * 128 * p.mb;
  };
  const uint32_t w_tap = (2u * p.nb) * 256u;

  if (warp == 0) {
    // ------------------------------------------------------------ activation producer
    if (lane == 0) {
      const uint32_t a_bytes = RAW_F32 ? static_cast<uint32_t>(p.a_px) * 64u : 2u * L.a_plane;
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int n, v0, ntile;
        tile_coords(t, n, v0, ntile);
        const int row0 = v0 / p.wsub;
        const int a_px0 = p.linear ? v0 : row0 * p.wsub;
        for (int it = 0; it < k_iters; ++it, ++g) {
          const int cb = it / p.n_phases, ph = it % p.n_phases;
          const int plane = n * p.in_cb + cb;
          if (RAW_F32) {
            const int s = g % raw_stages;
            mbar_wait(&raw_empty[s], ((g / raw_stages) & 1u) ^ 1u);
            uint8_t* dst = smem + L.raw_off + s * L.raw_slot;
            mbar_arrive_expect_tx(&raw_full[s], a_bytes);
            if (p.linear) {
              for (int i = 0; i < p.lin_boxes; ++i)
                tma_load_3d(dst + i * 128 * 64, &map_a, &raw_full[s], 0, a_px0 + i * 128, plane);
            } else {
              tma_load_4d(dst, &map_a, &raw_full[s], 0, p.in_col0 + p.phase_col[ph],
                          p.in_row0 + p.stride * row0 + p.phase_row[ph], plane);
            }
          } else {
            const int s = g % pc_stages;
            mbar_wait(&pc_empty[s], ((g / pc_stages) & 1u) ^ 1u);
            uint8_t* dst = smem + s * L.pc_slot;
            const uint32_t w_bytes = static_cast<uint32_t>(p.phase_ntaps[ph]) * w_tap;
            mbar_arrive_expect_tx(&pc_full[s], a_bytes + PIECES * w_bytes);
            if (p.linear) {
              for (int c = 0; c < 2; ++c)
                for (int i = 0; i < p.lin_boxes; ++i)
                  tma_load_4d(dst + c * L.a_plane + i * 128 * 16, &map_a, &pc_full[s], 0, a_px0 + i * 128, c, plane);
            } else {
              tma_load_5d(dst, &map_a, &pc_full[s], 0, p.in_col0 + p.phase_col[ph],
                          p.in_row0 + p.stride * row0 + p.phase_row[ph], 0, plane);
            }
            const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wprep);
            const long long w_blk = static_cast<long long>(p.n_taps) * w_tap;
            for (int pc = 0; pc < PIECES; ++pc)
              bulk_load(dst + PIECES * 2 * L.a_plane + pc * L.w_piece,
                        wsrc + ((static_cast<long long>(pc) * p.cb_in + cb) * p.n_ntiles + ntile) * w_blk +
                            static_cast<long long>(p.phase_tap0[ph]) * w_tap,
                        w_bytes, &pc_full[s]);
          }
        }
      }
    }
  } else if (warp == 2) {
    // ------------------------------------------------------------ weight producer (fp32 path)
    if (RAW_F32 && lane == 0) {
      const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(p.wprep);
      const long long w_blk = static_cast<long long>(p.n_taps) * w_tap;
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        int n, v0, ntile;
        tile_coords(t, n, v0, ntile);
        for (int it = 0; it < k_iters; ++it, ++g) {
          const int cb = it / p.n_phases, ph = it % p.n_phases;
          const int s = g % pc_stages;
          mbar_wait(&pc_empty[s], ((g / pc_stages) & 1u) ^ 1u);
          const uint32_t w_bytes = static_cast<uint32_t>(p.phase_ntaps[ph]) * w_tap;
          mbar_arrive_expect_tx(&pc_full[s], PIECES * w_bytes);
          uint8_t* dst = smem + s * L.pc_slot + PIECES * 2 * L.a_plane;
          for (int pc = 0; pc < PIECES; ++pc)
            bulk_load(dst + pc * L.w_piece,
                      wsrc + ((static_cast<long long>(pc) * p.cb_in + cb) * p.n_ntiles + ntile) * w_blk +
                          static_cast<long long>(p.phase_tap0[ph]) * w_tap,
                      w_bytes, &pc_full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(NT));
    uint32_t g = 0, tl = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const int a_px0 = p.linear ? v0 : (v0 / p.wsub) * p.wsub;
      const int v_off = v0 - a_px0;
      const uint32_t acc = tl & 1u;
      mbar_wait(&acc_empty[acc], ((tl >> 1) & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d_base = tmem_base + acc * acc_cols;
      for (int it = 0; it < k_iters; ++it, ++g) {
        const int s = g % pc_stages;
        const uint32_t par = (g / pc_stages) & 1u;
        mbar_wait(&pc_full[s], par);
        if (RAW_F32) mbar_wait(&pc_conv[s], par);
        tc_fence_after();
        const int ph = it % p.n_phases;
        const uint32_t st = smem0 + s * L.pc_slot;
        const uint32_t wst = st + PIECES * 2 * L.a_plane;
        if (elect_one()) {
          const int ntaps = p.phase_ntaps[ph];
          for (int tp = 0; tp < ntaps; ++tp) {
            const int shift = p.tap_shift[p.phase_tap0[ph] + tp];
            for (int mb = 0; mb < p.mb; ++mb) {
              const uint32_t a_off = static_cast<uint32_t>(v_off + mb * 128 + shift) * 16u;
              const uint32_t d_tmem = d_base + static_cast<uint32_t>(mb * NT);
#pragma unroll
              for (int pr = 0; pr < (PIECES == 3 ? 6 : 1); ++pr) {
                // products (ia, ib) with ia + ib <= 2
                const int ia = pr == 2 ? 1 : pr == 4 ? 1 : pr == 5 ? 2 : 0;
                const int ib = pr == 1 ? 1 : pr == 3 ? 2 : pr == 4 ? 1 : 0;
                const uint64_t ad =
                    make_smem_desc(st + static_cast<uint32_t>(ia) * 2u * L.a_plane + a_off, L.a_plane, 128);
                const uint64_t bd = make_smem_desc(wst + ib * L.w_piece + tp * w_tap, 128, 256);
                mma_bf16(d_tmem, ad, bd, idesc, (it > 0 || tp > 0 || pr > 0) ? 1u : 0u);
              }
            }
          }
          mma_commit(&pc_empty[s]);
          if (it == k_iters - 1) mma_commit(&acc_full[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= kCvtWarp0) {
    // ------------------------------------------------------------ converters (smem fp32 -> bf16 pieces)
    if (RAW_F32) {
      const int ct = threadIdx.x - kCvtWarp0 * 32;
      const int items = 2 * p.a_px;  // (pixel, 16B bf16 chunk)
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        for (int it = 0; it < k_iters; ++it, ++g) {
          const int rs = g % raw_stages, ps = g % pc_stages;
          mbar_wait(&raw_full[rs], (g / raw_stages) & 1u);
          mbar_wait(&pc_empty[ps], ((g / pc_stages) & 1u) ^ 1u);
          const uint8_t* raw = smem + L.raw_off + rs * L.raw_slot;
          uint8_t* pcs = smem + ps * L.pc_slot;
          for (int i = ct; i < items; i += kCvtWarps * 32) {
            const int j = i >> 1, c = i & 1;
            const float4 a = *reinterpret_cast<const float4*>(raw + j * 64 + c * 32);
            const float4 b = *reinterpret_cast<const float4*>(raw + j * 64 + c * 32 + 16);
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
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue (warps 4..7: TMEM lane quarters)
    const int qrow = (warp % 4) * 32;
    const int row = qrow + lane;
    const int v_end = p.P * p.wsub;
    const int esz = p.out_bf16 ? 2 : 4;
    uint8_t* obase = reinterpret_cast<uint8_t*>(p.out);
    uint32_t tl = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tl) {
      int n, v0, ntile;
      tile_coords(t, n, v0, ntile);
      const uint32_t acc = tl & 1u;
      mbar_wait(&acc_full[acc], (tl >> 1) & 1u);
      tc_fence_after();
      const uint32_t d_base = tmem_base + acc * acc_cols + (static_cast<uint32_t>(qrow) << 16);
      for (int mb = 0; mb < p.mb; ++mb) {
        const int v = v0 + mb * 128 + row;
        const int pp = v / p.wsub;
        const int qq = v - pp * p.wsub;
        const bool valid = v < v_end && qq < p.Q;
        const int y = p.out_y0 + pp * p.out_scale;
        const int x = p.out_x0 + qq * p.out_scale;
        for (int gq = 0; gq < p.nb; ++gq) {
          uint32_t r[16];
          tmem_ld16(d_base + static_cast<uint32_t>(mb * NT + gq * 16), r);
          tmem_ld_wait();
          const int kb = ntile * p.nb + gq;
          if (!valid || kb >= p.kb_out) continue;
          float vals[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) vals[e] = __uint_as_float(r[e]);
          // APPLY after the final reduction step (kernel_streams.cpp:96-120)
          if (p.bias != nullptr) {
#pragma unroll
            for (int e = 0; e < 16; ++e) vals[e] += p.bias[kb * 16 + e];
          }
          if (p.relu) {
#pragma unroll
            for (int e = 0; e < 16; ++e) vals[e] = vals[e] > 0.0f ? vals[e] : 0.0f;
          }
          const long long plane = static_cast<long long>(n) * p.out_cb + kb;
          store16(obase + ((plane * p.out_hp + y) * p.out_wp + x) * 16LL * esz, vals, p.out_bf16);
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
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

}  // namespace dconv_sm100
