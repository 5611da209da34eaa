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
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w2..w7 converters (fp32 activations only), w4..w7 epilogue.
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

// Exact 3-way split of 8 fp32 values into 16B bf16 rows (hi, mid, lo).
// x == hi + mid + lo for every finite normal x (8 significant bits each).
__device__ __forceinline__ void split8(const float (&x)[8], uint4& h, uint4& m, uint4& l) {
  uint32_t hh[4], mm[4], ll[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat16 a0 = __float2bfloat16_rn(x[2 * e]), b0 = __float2bfloat16_rn(x[2 * e + 1]);
    const float ra = x[2 * e] - __bfloat162float(a0), rb = x[2 * e + 1] - __bfloat162float(b0);
    __nv_bfloat16 a1 = __float2bfloat16_rn(ra), b1 = __float2bfloat16_rn(rb);
    __nv_bfloat16 a2 = __float2bfloat16_rn(ra - __bfloat162float(a1));
    __nv_bfloat16 b2 = __float2bfloat16_rn(rb - __bfloat162float(b1));
    hh[e] = pack2(a0, b0);
    mm[e] = pack2(a1, b1);
    ll[e] = pack2(a2, b2);
  }
  h = make_uint4(hh[0], hh[1], hh[2], hh[3]);
  m = make_uint4(mm[0], mm[1], mm[2], mm[3]);
  l = make_uint4(ll[0], ll[1], ll[2], ll[3]);
}

__device__ __forceinline__ uint4 cast8(const float (&x)[8]) {
  return make_uint4(pack2(__float2bfloat16_rn(x[0]), __float2bfloat16_rn(x[1])),
                    pack2(__float2bfloat16_rn(x[2]), __float2bfloat16_rn(x[3])),
                    pack2(__float2bfloat16_rn(x[4]), __float2bfloat16_rn(x[5])),
                    pack2(__float2bfloat16_rn(x[6]), __float2bfloat16_rn(x[7])));
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

// byte offsets of one pipeline stage: [raw fp32 A (4 planes)] [A pieces] [W pieces]
struct FwdStage {
  uint32_t a_plane;  // bytes per 16B-chunk plane (a_px * 16)
  uint32_t pc_off;   // A pieces start
  uint32_t w_off;    // weights start
  uint32_t w_piece;  // bytes per weight piece
  uint32_t bytes;    // stage stride
};

__host__ __device__ inline FwdStage fwd_stage_layout(int a_px, int taps_box, int nb, int pieces, bool raw_f32) {
  FwdStage L;
  L.a_plane = static_cast<uint32_t>(a_px) * 16u;
  L.pc_off = raw_f32 ? 4u * L.a_plane : 0u;
  L.w_off = (L.pc_off + static_cast<uint32_t>(pieces) * 2u * L.a_plane + 127u) & ~127u;
  L.w_piece = static_cast<uint32_t>(taps_box) * (2u * nb) * 256u;
  L.bytes = (L.w_off + static_cast<uint32_t>(pieces) * L.w_piece + 1023u) & ~1023u;
  return L;
}

template <bool RAW_F32, int PIECES>
__global__ void __launch_bounds__(kFwdThreads, 1)
    conv_fwd_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_w,
                    const __grid_constant__ FwdParams p, int n_stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];   // TMA bytes landed
  __shared__ __align__(8) uint64_t conv_bar[kMaxStages];   // converter pieces written
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];  // MMA done with the stage
  __shared__ __align__(8) uint64_t accum_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const FwdStage L = fwd_stage_layout(p.a_px, p.taps_box, p.nb, PIECES, RAW_F32);
  const uint32_t smem0 = smem_u32(smem);

  const int n = blockIdx.x / p.tiles_per_img;
  const int v0 = (blockIdx.x % p.tiles_per_img) * 128 * p.mb;
  const int ntile = blockIdx.y;
  const int NT = 16 * p.nb;
  const int k_iters = p.cb_in * p.n_phases;
  const int row0 = v0 / p.wsub;
  const int a_px0 = p.linear ? v0 : row0 * p.wsub;  // virtual index of smem pixel 0

  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(p.mb * NT)) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a);
    tma_prefetch_desc(&map_w);
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&conv_bar[s], kConvThreads / 32);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&accum_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      constexpr int kChunks = RAW_F32 ? 4 : 2;  // 16B chunk planes of the staged activation
      const uint32_t a_bytes = kChunks * L.a_plane;
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % n_stages;
        const uint32_t use = static_cast<uint32_t>(it / n_stages);
        mbar_wait(&empty_bar[s], (use & 1u) ^ 1u);
        const int cb = it / p.n_phases;
        const int ph = it % p.n_phases;
        uint8_t* st = smem + static_cast<uint32_t>(s) * L.bytes;
        mbar_arrive_expect_tx(&full_bar[s], a_bytes + PIECES * L.w_piece);
        const int plane = n * p.in_cb + cb;
        if (p.linear) {
          // box {e, 128 px, 1 chunk, 1 plane}
          for (int c = 0; c < kChunks; ++c)
            for (int i = 0; i < p.lin_boxes; ++i)
              tma_load_4d(st + c * L.a_plane + i * 128 * 16, &map_a, &full_bar[s], 0, a_px0 + i * 128, c, plane);
        } else {
          // box {e, wsub*stride cols, rows*stride rows, all chunks, 1 plane}
          tma_load_5d(st, &map_a, &full_bar[s], 0, p.in_col0 + p.phase_col[ph],
                      p.in_row0 + p.stride * row0 + p.phase_row[ph], 0, plane);
        }
        for (int pc = 0; pc < PIECES; ++pc)
          tma_load_5d(st + L.w_off + pc * L.w_piece, &map_w, &full_bar[s], 0, 0, 2 * p.nb * ntile,
                      p.phase_tap0[ph], pc * p.cb_in + cb);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(NT));
    const uint32_t w_tap = (2u * p.nb) * 256u;
    const int v_off = v0 - a_px0;
    for (int it = 0; it < k_iters; ++it) {
      const int s = it % n_stages;
      const uint32_t par = static_cast<uint32_t>(it / n_stages) & 1u;
      mbar_wait(&full_bar[s], par);
      if (RAW_F32) mbar_wait(&conv_bar[s], par);
      tc_fence_after();
      const int ph = it % p.n_phases;
      const uint32_t st = smem0 + static_cast<uint32_t>(s) * L.bytes;
      if (elect_one()) {
        const int ntaps = p.phase_ntaps[ph];
        for (int t = 0; t < ntaps; ++t) {
          const int shift = p.tap_shift[p.phase_tap0[ph] + t];
          for (int mb = 0; mb < p.mb; ++mb) {
            const uint32_t a_off = static_cast<uint32_t>(v_off + mb * 128 + shift) * 16u;
            const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(mb * NT);
#pragma unroll
            for (int pr = 0; pr < (PIECES == 3 ? 6 : 1); ++pr) {
              // products (ia, ib) with ia + ib <= 2
              const int ia = pr == 2 ? 1 : pr == 4 ? 1 : pr == 5 ? 2 : 0;
              const int ib = pr == 1 ? 1 : pr == 3 ? 2 : pr == 4 ? 1 : 0;
              const uint64_t ad =
                  make_smem_desc(st + L.pc_off + static_cast<uint32_t>(ia) * 2u * L.a_plane + a_off, L.a_plane, 128);
              const uint64_t bd = make_smem_desc(st + L.w_off + ib * L.w_piece + t * w_tap, 128, 256);
              mma_bf16(d_tmem, ad, bd, idesc, (it > 0 || t > 0 || pr > 0) ? 1u : 0u);
            }
          }
        }
        mma_commit(&empty_bar[s]);
        if (it == k_iters - 1) mma_commit(&accum_bar);
      }
      __syncwarp();
    }
  } else {
    if (RAW_F32) {
      // ---------------------------------------------------------- converters (smem fp32 -> bf16 pieces)
      const int ct = threadIdx.x - kConvWarp0 * 32;
      const int items = 2 * p.a_px;  // (16B bf16 chunk, pixel)
      for (int it = 0; it < k_iters; ++it) {
        const int s = it % n_stages;
        mbar_wait(&full_bar[s], static_cast<uint32_t>(it / n_stages) & 1u);
        uint8_t* st = smem + static_cast<uint32_t>(s) * L.bytes;
        for (int i = ct; i < items; i += kConvThreads) {
          const int c = i / p.a_px;
          const int j = i - c * p.a_px;
          const float4 a = *reinterpret_cast<const float4*>(st + (2 * c) * L.a_plane + j * 16);
          const float4 b = *reinterpret_cast<const float4*>(st + (2 * c + 1) * L.a_plane + j * 16);
          const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          uint8_t* dst = st + L.pc_off + c * L.a_plane + j * 16;
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
        if (lane == 0) mbar_arrive(&conv_bar[s]);
      }
    }
    if (warp >= 4) {
      // ---------------------------------------------------------- epilogue
      mbar_wait(&accum_bar, 0);
      tc_fence_after();
      const int qrow = (warp % 4) * 32;
      const int row = qrow + lane;
      const int v_end = p.P * p.wsub;
      const int esz = p.out_bf16 ? 2 : 4;
      uint8_t* obase = reinterpret_cast<uint8_t*>(p.out);
      for (int mb = 0; mb < p.mb; ++mb) {
        const int v = v0 + mb * 128 + row;
        const int pp = v / p.wsub;
        const int qq = v - pp * p.wsub;
        const bool valid = v < v_end && qq < p.Q;
        const int y = p.out_y0 + pp * p.out_scale;
        const int x = p.out_x0 + qq * p.out_scale;
        for (int g = 0; g < p.nb; ++g) {
          uint32_t r[16];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(qrow) << 16) + static_cast<uint32_t>(mb * NT + g * 16), r);
          tmem_ld_wait();
          const int kb = ntile * p.nb + g;
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
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

}  // namespace dconv_sm100
