// conv_upd_sm100: weight-gradient (UPD) as a split-K implicit GEMM
// (the reference's upd_f32_kernel + weight_update, microkernel.cpp:157-195
// and propagation.cpp:377-458).
//
// dW[tap][c][k] = sum_v I_phase[v + shift(tap)][c] * dO[v][k] over virtual
// pixels v (same virtual-row grid as the forward kernel; dO is zero on the
// garbage columns and past the last row, so they contribute nothing).
// GEMM per tap: M = 128 input channels (8 blocks), N = 16*nb output
// channels, K = virtual pixels; both operands are MN-major (channels are the
// contiguous 16B rows of NCHW16c, pixels are the K rows), which is what lets
// every tap reuse the same staged input rows through a shifted descriptor.
// A CTA owns (c-tile, k-tile, tap group, split); its stages are image row
// bands [split range); the fp32 partials go to a workspace that
// upd_reduce_kernel sums in fixed split order (COPY_REDUCE with G = splits,
// propagation.cpp:357-375) -> bitwise reproducible.
//
// Operands are bf16 (pieces = 1) or the exact hi/mid/lo bf16 split of fp32
// tensors (pieces = 3, split once in HBM by split_pieces_kernel), each staged
// by one TMA box per piece per stage straight into the canonical MN-major
// no-swizzle layout.
//
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w4..w7 epilogue (TMEM -> fp32 partials).
#pragma once
#include "conv_fwd.cuh"

namespace dconv_sm100 {

struct UpdStage {
  uint32_t a_plane, b_plane;  // bytes per 16B-chunk plane
  uint32_t a_piece, b_piece;  // bytes per operand piece (16 / 2*nb planes)
  uint32_t b_off, bytes;
};

__host__ __device__ inline UpdStage upd_stage_layout(int a_px, int vs, int nb, int pa, int pb) {
  UpdStage L;
  L.a_plane = static_cast<uint32_t>(a_px) * 16u;
  L.b_plane = static_cast<uint32_t>(vs) * 16u;
  L.a_piece = 16u * L.a_plane;
  L.b_piece = 2u * nb * L.b_plane;
  L.b_off = static_cast<uint32_t>(pa) * L.a_piece;
  L.bytes = (L.b_off + static_cast<uint32_t>(pb) * L.b_piece + 1023u) & ~1023u;
  return L;
}

// PA / PB: operand pieces staged per stage. The products (ia, ib) with
// a_base + ia + ib <= 2 are accumulated, so one launch with PA = PB = 3 (or
// PA = PB = 1 for bf16) covers everything, and when three A pieces do not
// fit in smem the host runs three passes (a_base = 0, 1, 2 with PA = 1,
// PB = 3 - a_base) that accumulate into the same partials.
template <int PA, int PB>
__global__ void __launch_bounds__(kFwdThreads, 1)
    conv_upd_kernel(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_do,
                    const __grid_constant__ UpdParams p, int n_stages, int a_base, int accumulate) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t accum_bar;
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int NT = 16 * p.nb;
  const UpdStage L = upd_stage_layout(p.a_px, p.vs, p.nb, PA, PB);
  const uint32_t smem0 = smem_u32(smem);

  // CTA coordinates: x = c-tile * n_tgroups + tap group, y = k-tile, z = split
  const int ctile = blockIdx.x / p.n_tgroups;
  const int tgrp = blockIdx.x % p.n_tgroups;
  const int ktile = blockIdx.y;
  const int split = blockIdx.z;
  const int per = (p.stages_total + p.splits - 1) / p.splits;
  const int s_begin = split * per;
  const int s_end = min(p.stages_total, s_begin + per);
  const int iters = s_end > s_begin ? s_end - s_begin : 0;
  const int ph = p.tg_phase[tgrp];
  const int tap0 = p.tg_tap0[tgrp];
  const int ntaps = p.tg_ntaps[tgrp];

  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(p.tg * NT)) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_in);
    tma_prefetch_desc(&map_do);
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full_bar[s], 1);
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
      const int in_planes = p.n_img * p.in_cb, do_planes = p.n_img * p.do_cb;
      for (int it = 0; it < iters; ++it) {
        const int s = it % n_stages;
        mbar_wait(&empty_bar[s], (static_cast<uint32_t>(it / n_stages) & 1u) ^ 1u);
        const int stage = s_begin + it;
        const int n = stage / p.stages_per_img;
        const int band = stage % p.stages_per_img;
        uint8_t* st = smem + static_cast<uint32_t>(s) * L.bytes;
        const uint32_t a_bytes =
            p.stack > 1 ? static_cast<uint32_t>(ntaps * 2 * p.cb_eff) * L.a_plane : L.a_piece;
        mbar_arrive_expect_tx(&full_bar[s], PA * a_bytes + PB * L.b_piece);
        for (int pc = 0; pc < PA; ++pc) {
          const int pa = (a_base + pc) * in_planes + n * p.in_cb + ctile * 8;
          uint8_t* a_dst = st + pc * L.a_piece;
          if (p.stack > 1) {
            // one shifted box per stacked tap: slot j = tap tap0 + j, cb_eff blocks
            for (int j = 0; j < ntaps; ++j) {
              const int tp = tap0 + j, tph = p.tap_ph[tp];
              tma_load_5d(a_dst + j * 2 * p.cb_eff * L.a_plane, &map_in, &full_bar[s], 0,
                          p.in_col0 + p.phase_col[tph] + p.stride * p.tap_s2[tp],
                          p.in_row0 + p.phase_row[tph] + p.stride * (band * p.rows_ps + p.tap_r2[tp]), 0, pa);
            }
          } else if (p.linear) {
            tma_load_4d(a_dst, &map_in, &full_bar[s], 0, band * p.vs, 0, pa);
          } else {
            tma_load_5d(a_dst, &map_in, &full_bar[s], 0, p.in_col0 + p.phase_col[ph],
                        p.in_row0 + p.stride * band * p.rows_ps + p.phase_row[ph], 0, pa);
          }
        }
        for (int pc = 0; pc < PB; ++pc) {
          const int pb = pc * do_planes + n * p.do_cb + ktile * p.nb;
          uint8_t* b_dst = st + L.b_off + pc * L.b_piece;
          if (p.linear)
            tma_load_4d(b_dst, &map_do, &full_bar[s], 0, band * p.vs, 0, pb);
          else
            tma_load_5d(b_dst, &map_do, &full_bar[s], 0, 0, band * p.rows_ps, 0, pb);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(1, 1, 1, 128, static_cast<uint32_t>(NT));
    const int ksteps = p.vs / 16;
    for (int it = 0; it < iters; ++it) {
      const int s = it % n_stages;
      mbar_wait(&full_bar[s], static_cast<uint32_t>(it / n_stages) & 1u);
      tc_fence_after();
      const uint32_t st = smem0 + static_cast<uint32_t>(s) * L.bytes;
      if (elect_one()) {
        const int n_acc = p.stack > 1 ? 1 : ntaps;  // stacked: one accumulator holds all the group's taps
        for (int t = 0; t < n_acc; ++t) {
          const int shift = p.stack > 1 ? 0 : p.tap_shift[tap0 + t];
          const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(t * NT);
          for (int ks = 0; ks < ksteps; ++ks) {
#pragma unroll
            for (int ia = 0; ia < PA; ++ia) {
#pragma unroll
              for (int ib = 0; ib < PB; ++ib) {
                if (a_base + ia + ib > 2) continue;
                // MN-major: 16B rows = 8 channels, K rows = pixels; SBO = chunk-plane stride, LBO = 8 pixels
                const uint64_t ad = make_smem_desc(
                    st + static_cast<uint32_t>(ia) * L.a_piece + static_cast<uint32_t>(ks * 16 + shift) * 16u, 128,
                    L.a_plane);
                const uint64_t bd = make_smem_desc(
                    st + L.b_off + static_cast<uint32_t>(ib) * L.b_piece + static_cast<uint32_t>(ks) * 256u, 128,
                    L.b_plane);
                mma_bf16(d_tmem, ad, bd, idesc, (it > 0 || ks > 0 || ia > 0 || ib > 0) ? 1u : 0u);
              }
            }
          }
        }
        mma_commit(&empty_bar[s]);
        if (it == iters - 1) mma_commit(&accum_bar);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue
    const int qrow = (warp % 4) * 32;
    const int c_glob = ctile * 128 + qrow + lane;
    if (iters > 0) {
      mbar_wait(&accum_bar, 0);
      tc_fence_after();
    }
    const int n_acc = p.stack > 1 ? 1 : ntaps;
    for (int t = 0; t < n_acc; ++t) {
      // stacked: TMEM row = (slot j, channel c) of tap tap0 + j
      const int slot = p.stack > 1 ? (qrow + lane) / (16 * p.cb_eff) : 0;
      const int c_row = p.stack > 1 ? (qrow + lane) % (16 * p.cb_eff) : c_glob;
      const bool row_ok = p.stack > 1 ? slot < ntaps : true;
      const int rs = p.tap_src[tap0 + (p.stack > 1 ? (row_ok ? slot : 0) : t)];
      float* dst_row =
          p.partial + ((static_cast<long long>(split) * p.n_taps + rs) * p.c_pad + c_row) * p.k_pad + ktile * NT;
      for (int g = 0; g < p.nb; ++g) {
        uint32_t r[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(qrow) << 16) + static_cast<uint32_t>(t * NT + g * 16), r);
        tmem_ld_wait();
        if (!row_ok) continue;
        float4* d = reinterpret_cast<float4*>(dst_row + g * 16);
        const bool live = iters > 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float4 v = live ? make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                        __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          if (accumulate) {
            const float4 o = d[e];
            v.x += o.x;
            v.y += o.y;
            v.z += o.z;
            v.w += o.w;
          }
          d[e] = v;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

// Fixed-order reduction of the split partials into the blocked dW
// [k_b][c_b][r][s][c][k] (tail lanes written as exact zeros).
// reduce_weight_copies analog (propagation.cpp:357-375): sum = copy0; sum += copy_g.
__global__ void upd_reduce_kernel(const float* __restrict__ partial, int splits, int n_taps, int c_pad, int k_pad, int C,
                                  int K, int cb, int kb, void* __restrict__ dw, int dw_bf16, int accumulate) {
  const long long total = static_cast<long long>(kb) * cb * n_taps * 256;
  const long long split_stride = static_cast<long long>(n_taps) * c_pad * k_pad;
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int kl = static_cast<int>(e % 16);
    const int cl = static_cast<int>((e / 16) % 16);
    const long long blk = e / 256;  // ((kbi * cb + cbi) * n_taps + rs)
    const int rs = static_cast<int>(blk % n_taps);
    const int cbi = static_cast<int>((blk / n_taps) % cb);
    const int kbi = static_cast<int>(blk / (static_cast<long long>(n_taps) * cb));
    const int c = cbi * 16 + cl, k = kbi * 16 + kl;
    float sum = 0.0f;
    if (c < C && k < K) {
      const float* src = partial + (static_cast<long long>(rs) * c_pad + c) * k_pad + k;
      sum = __ldg(src);
      // fixed index order; loads batched 8 deep for memory-level parallelism
      int sp = 1;
      for (; sp + 8 <= splits; sp += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (sp + u) * split_stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) sum += v[u];
      }
      for (; sp < splits; ++sp) sum += __ldg(src + sp * split_stride);
    }
    if (dw_bf16) {
      __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dw) + e;
      *d = __float2bfloat16_rn(accumulate ? sum + __bfloat162float(*d) : sum);
    } else {
      float* d = reinterpret_cast<float*>(dw) + e;
      *d = accumulate ? *d + sum : sum;
    }
  }
}

}  // namespace dconv_sm100
