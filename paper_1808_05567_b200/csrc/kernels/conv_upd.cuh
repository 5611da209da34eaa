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

// Accumulation periods of the fp32-accurate UPD kernels (UpdParams::drain): the
// stages [j*drain, (j+1)*drain) of a CTA accumulate in TMEM buffer j % bufs;
// when period j ends the MMA commits acc_full[buf], the drainers add the
// buffer into the CTA's fp32 partial slice (round to nearest) and arrive
// acc_drained[buf]; period j + bufs waits for that before reusing the buffer.
struct AccPeriods {
  int drain, bufs;
  __device__ __forceinline__ int period(int it) const { return drain ? it / drain : 0; }
  __device__ __forceinline__ bool starts(int it) const { return drain ? (it % drain == 0) : it == 0; }
  __device__ __forceinline__ bool ends(int it, int iters) const {
    return it == iters - 1 || (drain && (it + 1) % drain == 0);
  }
  __device__ __forceinline__ int buf(int j) const { return j % bufs; }
  __device__ __forceinline__ uint32_t par(int j) const { return static_cast<uint32_t>(j / bufs) & 1u; }
};

struct UpdStage {
  uint32_t a_plane, b_plane;  // bytes per 16B-chunk plane
  uint32_t a_piece, b_piece;  // bytes per operand piece (16 / 2*nb planes)
  uint32_t b_off, bytes;
};

__host__ __device__ inline UpdStage upd_stage_layout(int a_px, int vs, int nb, int pa, int pb, int mc = 1) {
  UpdStage L;
  L.a_plane = static_cast<uint32_t>(a_px) * 16u;
  L.b_plane = static_cast<uint32_t>(vs) * 16u;
  L.a_piece = 16u * static_cast<uint32_t>(mc) * L.a_plane;  // mc c-tiles of 8 channel blocks
  L.b_piece = 2u * nb * L.b_plane;
  L.b_off = static_cast<uint32_t>(pa) * L.a_piece;
  L.bytes = (L.b_off + static_cast<uint32_t>(pb) * L.b_piece + 1023u) & ~1023u;
  return L;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
constexpr int kUpdLoaderWarp0 = 2, kUpdLoaderWarps = 6;  // warps 2..7 stage operands (lsu plans)
constexpr int kUpdLsuDepth = 2;                          // stages in flight per loader thread

// One stage of the bf16 SW32 operand tiles by cp.async, exactly the boxes the
// TMA path loads: rows `r` of `n_rows`, `cols` pixels per row (element stride
// `st` in the source), 2 x 16 B per pixel, zero outside the interior; the
// destination [plane][row][col][32 B] with the SWIZZLE_32B XOR (bit 4 ^= bit 7).
__device__ __forceinline__ void lsu_box(uint32_t dst0, const uint8_t* src_plane0, long long plane_px, int n_planes,
                                        int n_valid, int n_rows, int cols, int row0, int col0, int st, int h, int w,
                                        int wp, int t, int nt) {
  const int chunks = 2 * cols;
  const int pairs = n_planes * n_rows;
  for (int pr = t / chunks, c = t % chunks; pr < pairs;) {
    const int pl = pr / n_rows, r = pr - pl * n_rows;
    const int rg = row0 + st * r;
    const uint8_t* rowp = src_plane0 + (static_cast<long long>(pl) * plane_px + static_cast<long long>(rg) * wp) * 32;
    const uint32_t drow = dst0 + static_cast<uint32_t>((pl * n_rows + r) * cols) * 32u;
    const bool row_ok = rg >= 0 && rg < h && pl < n_valid;  // planes past the tensor's channels: zero
    for (; c < chunks; c += nt) {
      const int col = c >> 1, cg = col0 + st * col;
      const bool ok = row_ok && cg >= 0 && cg < w;
      const uint32_t d = drow + static_cast<uint32_t>(c) * 16u;
      cp_async16(d ^ ((d >> 3) & 16u), ok ? rowp + static_cast<long long>(cg) * 32 + (c & 1) * 16 : src_plane0,
                 ok ? 16u : 0u);
    }
    // next (plane, row) pair this thread owns: advance by nt chunks overall
    c -= chunks;
    ++pr;
    while (c >= chunks && pr < pairs) {
      c -= chunks;
      ++pr;
    }
  }
}

// PA / PB: operand pieces staged per stage. The products (ia, ib) with
// a_base + ia + ib <= 2 are accumulated, so one launch with PA = PB = 3 (or
// PA = PB = 1 for bf16) covers everything, and when three A pieces do not
// fit in smem the host runs three passes (a_base = 0, 1, 2 with PA = 1,
// PB = 3 - a_base) that accumulate into the same partials.
template <int PA, int PB>
__global__ void __launch_bounds__(kFwdThreads, 1)
    conv_upd_kernel(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_do,
                    const __grid_constant__ CUtensorMap map_part, const __grid_constant__ UpdParams p, int n_stages,
                    int a_base, int accumulate) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[kMaxStages];
  __shared__ __align__(8) uint64_t empty_bar[kMaxStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_drained[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_tap_shift[kMaxTaps];  // off the constant cache in the issue loop

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 2)
    for (int i = lane; i < kMaxTaps; i += 32) s_tap_shift[i] = p.tap_shift[i];
  const int NT = 16 * p.nb;
  const int mc = p.mc > 1 ? p.mc : 1;
  // accumulation periods (fp32-accurate long chains, see AccPeriods); the bf16 paths keep drain = 0
  const AccPeriods per_acc{(PA == 1 && PB == 1) ? 0 : p.drain, p.drain_bufs > 1 ? 2 : 1};
  const int xsn = p.xs > 1 ? p.xs : 1;  // dO copies along N (cross-stacked plans)
  const UpdStage L = upd_stage_layout(p.a_px, p.vs, p.nb * xsn, PA, PB, mc);
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

  const uint32_t buf_cols = static_cast<uint32_t>(max(p.tg, mc) * NT);
  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(per_acc.bufs) * buf_cols) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_in);
    tma_prefetch_desc(&map_do);
    for (int s = 0; s < n_stages; ++s) {
      mbar_init(&full_bar[s], p.lsu ? kUpdLoaderWarps * 32 : 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_drained[b], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (PA == 1 && PB == 1 && p.lsu && warp >= kUpdLoaderWarp0 && warp < kUpdLoaderWarp0 + kUpdLoaderWarps) {
    // ------------------------------------------------------------ cp.async operand loaders
    const int t = threadIdx.x - kUpdLoaderWarp0 * 32, nt = kUpdLoaderWarps * 32;
    const uint8_t* in0 = static_cast<const uint8_t*>(p.in_ptr);
    const uint8_t* do0 = static_cast<const uint8_t*>(p.do_ptr);
    RingPos rp, fp;  // fill position, arrive position (kUpdLsuDepth behind)
    const int a_valid = p.in_cb - ctile * 8, b_valid = p.do_cb - ktile * p.nb;
    for (int it = 0; it < iters; ++it, rp.adv(n_stages)) {
      mbar_wait(&empty_bar[rp.idx], rp.ph ^ 1u);
      const int stage = s_begin + it;
      const int n = stage / p.stages_per_img;
      const int band = stage - n * p.stages_per_img;
      const uint32_t st_a = smem0 + static_cast<uint32_t>(rp.idx) * L.bytes;
      const uint8_t* in_n = in0 + (static_cast<long long>(n) * p.in_cb + ctile * 8) * p.in_plane * 32;
      const uint8_t* do_n = do0 + (static_cast<long long>(n) * p.do_cb + ktile * p.nb) * p.do_plane * 32;
      if (p.linear) {
        // dense planes: pixels [band*vs, +vs) of cb_eff (A) / nb (B) planes
        lsu_box(st_a, in_n, p.in_plane, 8, a_valid, 1, p.vs, 0, band * p.vs, 1, 1, p.in_h * p.in_w, 0, t, nt);
        lsu_box(st_a + L.b_off, do_n, p.do_plane, p.nb, b_valid, 1, p.vs, 0, band * p.vs, 1, 1, p.do_h * p.do_w, 0, t,
                nt);
      } else {
        if (p.stack > 1) {
          for (int j = 0; j < ntaps; ++j) {
            const int tp = tap0 + j, tph = p.tap_ph[tp];
            lsu_box(st_a + static_cast<uint32_t>(j * 2 * p.cb_eff) * L.a_plane, in_n, p.in_plane, p.cb_eff, a_valid,
                    p.in_rows,
                    p.wsub, p.in_row0 + p.phase_row[tph] + p.stride * (band * p.rows_ps + p.tap_r2[tp]),
                    p.in_col0 + p.phase_col[tph] + p.stride * p.tap_s2[tp], p.stride, p.in_h, p.in_w, p.in_wp, t, nt);
          }
        } else {
          lsu_box(st_a, in_n, p.in_plane, p.cb_eff, a_valid, p.in_rows, p.wsub,
                  p.in_row0 + p.stride * band * p.rows_ps + p.phase_row[ph], p.in_col0 + p.phase_col[ph], p.stride,
                  p.in_h, p.in_w, p.in_wp, t, nt);
        }
        lsu_box(st_a + L.b_off, do_n, p.do_plane, p.nb, b_valid, p.rows_ps, p.wsub, band * p.rows_ps, 0, 1, p.do_h,
                p.do_w, p.do_wp, t, nt);
      }
      cp_async_commit();
      if (it >= kUpdLsuDepth) {
        cp_async_wait<kUpdLsuDepth>();
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        mbar_arrive(&full_bar[fp.idx]);
        fp.adv(n_stages);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int it = max(0, iters - kUpdLsuDepth); it < iters; ++it) {
      mbar_arrive(&full_bar[fp.idx]);
      fp.adv(n_stages);
    }
    // warps 4..7 continue as the epilogue below
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0 && !p.lsu) {
      const int in_planes = p.n_img * p.in_cb, do_planes = p.n_img * p.do_cb;
      for (int it = 0; it < iters; ++it) {
        const int s = it % n_stages;
        mbar_wait(&empty_bar[s], (static_cast<uint32_t>(it / n_stages) & 1u) ^ 1u);
        const int stage = s_begin + it;
        const int n = stage / p.stages_per_img;
        const int band = stage % p.stages_per_img;
        uint8_t* st = smem + static_cast<uint32_t>(s) * L.bytes;
        const uint32_t a_bytes = p.stack > 1 ? static_cast<uint32_t>(ntaps * (p.half ? 1 : 2 * p.cb_eff)) * L.a_plane
                                 : p.sw32     ? static_cast<uint32_t>(2 * p.cb_eff * mc) * L.a_plane
                                              : L.a_piece;
        // dev ablation bits: 256 no operand loads, 512 no input loads, 1024 no dO loads
        const int dbl = kDevBuild ? p.dbg_mode : 0;
        if (dbl & 256) {
          mbar_arrive(&full_bar[s]);
          continue;
        }
        mbar_arrive_expect_tx(&full_bar[s], ((dbl & 512) ? 0u : PA * a_bytes) + ((dbl & 1024) ? 0u : PB * L.b_piece));
        for (int pc = 0; pc < ((dbl & 512) ? 0 : PA); ++pc) {
          const int pa = (a_base + pc) * in_planes + n * p.in_cb + ctile * 8 * mc;
          uint8_t* a_dst = st + pc * L.a_piece;
          if (p.sw32) {  // 32 B pixel rows: {16, px[, rows], planes} boxes
            if (p.xs > 1) {  // cross-stacked: slot j = the input tile shifted by (r_j, s_j)
              for (int j = 0; j < ntaps; ++j)
                tma_load_4d(a_dst + j * 2 * p.cb_eff * L.a_plane, &map_in, &full_bar[s], 0,
                            p.in_col0 + p.xs_slot_s[tap0 + j], p.in_row0 + band * p.rows_ps + p.xs_slot_r[tap0 + j],
                            pa);
            } else if (p.stack > 1) {
              for (int j = 0; j < ntaps; ++j) {
                const int tp = tap0 + j, tph = p.tap_ph[tp];
                tma_load_4d(a_dst + j * 2 * p.cb_eff * L.a_plane, &map_in, &full_bar[s], 0,
                            p.in_col0 + p.phase_col[tph] + p.stride * p.tap_s2[tp],
                            p.in_row0 + p.phase_row[tph] + p.stride * (band * p.rows_ps + p.tap_r2[tp]), pa);
              }
            } else if (p.linear) {
              tma_load_3d(a_dst, &map_in, &full_bar[s], 0, p.sw32 == 2 ? band * (p.vs / 4) : band * p.vs, pa);
            } else if (p.pimg > 0) {  // packed images: {16, wsub, H + pad, pimg + 1, planes}
              tma_load_5d(a_dst, &map_in, &full_bar[s], 0, p.in_col0, p.in_row0, n * p.pimg, ctile * 8 * mc);
            } else {
              tma_load_4d(a_dst, &map_in, &full_bar[s], 0, p.in_col0 + p.phase_col[ph],
                          p.in_row0 + p.stride * band * p.rows_ps + p.phase_row[ph], pa);
            }
          } else if (p.stack > 1) {
            // one shifted box per stacked tap: slot j = tap tap0 + j, cb_eff blocks
            for (int j = 0; j < ntaps; ++j) {
              const int tp = tap0 + j, tph = p.tap_ph[tp];
              tma_load_5d(a_dst + j * (p.half ? 1 : 2 * p.cb_eff) * L.a_plane, &map_in, &full_bar[s], 0,
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
        for (int pc = 0; pc < ((dbl & 1024) ? 0 : PB); ++pc) {
          const int pb = pc * do_planes + n * p.do_cb + ktile * p.nb;
          uint8_t* b_dst = st + L.b_off + pc * L.b_piece;
          if (p.sw32) {
            if (p.linear)
              tma_load_3d(b_dst, &map_do, &full_bar[s], 0, p.sw32 == 2 ? band * (p.vs / 4) : band * p.vs, pb);
            else if (p.pimg > 0)
              tma_load_5d(b_dst, &map_do, &full_bar[s], 0, 0, 0, n * p.pimg, ktile * p.nb);
            else
              for (int j = 0; j < xsn; ++j)  // copy j shifted right by j columns (zero fill at the left edge)
                tma_load_4d(b_dst + j * p.nb * 2 * L.b_plane, &map_do, &full_bar[s], 0, -j, band * p.rows_ps, pb);
          } else if (p.linear)
            tma_load_4d(b_dst, &map_do, &full_bar[s], 0, band * p.vs, 0, pb);
          else
            tma_load_5d(b_dst, &map_do, &full_bar[s], 0, 0, band * p.rows_ps, 0, pb);
        }
      }
    }
  } else if (warp == 1 && PA == 1 && PB == 1 && p.sw32 && (p.stack > 1 ? 1 : max(ntaps, mc)) <= kFastTaps) {
    // ------------------------------------------------------------ MMA issuer (bf16 SW32), one lane
    // shifts and descriptor words hoisted out of the stage loop; between stages
    // only the commit and the full-barrier wait (see conv_fwd_kernel)
    if (lane == 0) {
      const uint32_t idesc = make_idesc(1, 1, 1, 128, static_cast<uint32_t>(NT * xsn));  // (cross-stacked: xs dO copies)
      const int ksteps = p.vs / 16;
      // accumulators: one per tap of the group, or (single-tap, mc > 1) one per c-tile,
      // whose A rows are the next 8 channel-block planes (a_piece / mc bytes on)
      const int n_acc = p.stack > 1 ? 1 : (mc > 1 ? mc : ntaps);
      uint32_t sh[kFastTaps];
#pragma unroll
      for (int i = 0; i < kFastTaps; ++i)
        sh[i] = (i < n_acc && p.stack == 1)
                    ? (mc > 1 ? static_cast<uint32_t>(i) * ((L.a_piece / mc) >> 4)
                              : 2u * static_cast<uint32_t>(s_tap_shift[tap0 + i]))
                    : 0u;
      const uint64_t a_d = make_smem_desc_mn_sw32(smem0, 2 * L.a_plane);
      const uint64_t b_d = make_smem_desc_mn_sw32(smem0 + L.b_off, 2 * L.b_plane);
      const uint32_t a_hi = static_cast<uint32_t>(a_d >> 32), b_hi = static_cast<uint32_t>(b_d >> 32);
      const uint32_t a_lo0 = static_cast<uint32_t>(a_d), b_lo0 = static_cast<uint32_t>(b_d);
      const uint32_t slot_u = L.bytes >> 4;
      // KS / NACC > 0: compile-time k-steps per stage and accumulators (straight-line MMAs
      // whose operands are the stage's slot bases plus launch constants; see the forward
      // issuer in conv_fwd.cuh), 0: runtime trip counts
      auto run = [&](auto ks_c, auto na_c) {
        constexpr int KS = decltype(ks_c)::value, NACC = decltype(na_c)::value;
        RingPos rp;
        for (int it = 0; it < iters; ++it, rp.adv(n_stages)) {
          mbar_wait(&full_bar[rp.idx], rp.ph);
          tc_fence_after();
          const uint32_t a_s = a_lo0 + static_cast<uint32_t>(rp.idx) * slot_u;
          const uint32_t b_s = b_lo0 + static_cast<uint32_t>(rp.idx) * slot_u;
          if (kDevBuild && (p.dbg_mode & 8)) {  // dev ablation: no MMAs
          } else if (KS > 0) {
            const uint32_t acc0 = it > 0 ? 1u : 0u;
#pragma unroll
            for (int ks = 0; ks < (KS > 0 ? KS : 1); ++ks)
#pragma unroll
              for (int t = 0; t < NACC; ++t)
                mma_bf16_lo(tmem_base + static_cast<uint32_t>(t * NT), a_s + 32u * ks + sh[t], a_hi, b_s + 32u * ks,
                            b_hi, idesc, ks > 0 ? 1u : acc0);
          } else {
            for (int ks = 0; ks < ksteps; ++ks) {
#pragma unroll
              for (int t = 0; t < kFastTaps; ++t) {
                if (t >= n_acc) break;
                mma_bf16_lo(tmem_base + static_cast<uint32_t>(t * NT), a_s + 32u * ks + sh[t], a_hi, b_s + 32u * ks,
                            b_hi, idesc, (it > 0 || ks > 0) ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty_bar[rp.idx]);
        }
        if (iters > 0) mma_commit(&acc_full[0]);
      };
      using I0 = std::integral_constant<int, 0>;
      auto by_acc = [&](auto ks_c) {
        if (n_acc == 1)
          run(ks_c, std::integral_constant<int, 1>{});
        else if (n_acc == 2)
          run(ks_c, std::integral_constant<int, 2>{});
        else if (n_acc == 3)
          run(ks_c, std::integral_constant<int, 3>{});
        else if (n_acc == 4)
          run(ks_c, std::integral_constant<int, 4>{});
        else
          run(I0{}, std::integral_constant<int, 1>{});
      };
      if (ksteps == 2)
        by_acc(std::integral_constant<int, 2>{});
      else if (ksteps == 4)
        by_acc(std::integral_constant<int, 4>{});
      else if (ksteps == 8)
        by_acc(std::integral_constant<int, 8>{});
      else if (ksteps == 9)
        by_acc(std::integral_constant<int, 9>{});
      else
        run(I0{}, std::integral_constant<int, 1>{});
    }
    __syncwarp();
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = make_idesc(1, 1, 1, 128, static_cast<uint32_t>(NT * xsn));
    const int ksteps = p.vs / 16;
    for (int it = 0; it < iters; ++it) {
      const int s = it % n_stages;
      const int jp = per_acc.period(it);
      const bool p_first = per_acc.starts(it);
      if (p_first && jp >= per_acc.bufs)
        mbar_wait(&acc_drained[per_acc.buf(jp)], static_cast<uint32_t>(jp / per_acc.bufs - 1) & 1u);
      mbar_wait(&full_bar[s], static_cast<uint32_t>(it / n_stages) & 1u);
      tc_fence_after();
      const uint32_t st = smem0 + static_cast<uint32_t>(s) * L.bytes;
      const uint32_t acc0 = tmem_base + static_cast<uint32_t>(per_acc.buf(jp)) * buf_cols;
      if (elect_one()) {
        const int n_acc = p.stack > 1 ? 1 : ntaps;  // stacked: one accumulator holds all the group's taps
        // MN-major: 16B rows = 8 channels, K rows = pixels; SBO = chunk-plane stride, LBO = 8 pixels.
        // Descriptors are packed once per stage; per MMA only the start address (16 B units) advances.
        const uint64_t a0 = p.sw32 ? make_smem_desc_mn_sw32(st, 2 * L.a_plane) : make_smem_desc(st, 128, L.a_plane);
        const uint64_t b0 =
            p.sw32 ? make_smem_desc_mn_sw32(st + L.b_off, 2 * L.b_plane) : make_smem_desc(st + L.b_off, 128, L.b_plane);
        const uint32_t a_pc = L.a_piece >> 4, b_pc = L.b_piece >> 4;
        const uint32_t row_u = p.sw32 ? 2u : 1u;  // descriptor units (16 B) per pixel row
        for (int t = 0; t < n_acc; ++t) {
          const int shift = p.stack > 1 ? 0 : s_tap_shift[tap0 + t];
          const uint32_t d_tmem = acc0 + static_cast<uint32_t>(t * NT);
          for (int ks = 0; ks < ksteps; ++ks) {
            const uint64_t ak = a0 + static_cast<uint32_t>(ks * 16 + shift) * row_u;
            const uint64_t bk = b0 + static_cast<uint32_t>(ks) * 16u * row_u;
#pragma unroll
            for (int ia = 0; ia < PA; ++ia) {
#pragma unroll
              for (int ib = 0; ib < PB; ++ib) {
                if (a_base + ia + ib > 2) continue;
                mma_bf16(d_tmem, ak + static_cast<uint32_t>(ia) * a_pc, bk + static_cast<uint32_t>(ib) * b_pc, idesc,
                         (!p_first || ks > 0 || ia > 0 || ib > 0) ? 1u : 0u);
              }
            }
          }
        }
        mma_commit(&empty_bar[s]);
        if (per_acc.ends(it, iters)) mma_commit(&acc_full[per_acc.buf(jp)]);
      }
      __syncwarp();
    }
  }
  if (warp >= 4 && PA == 1 && PB == 1 && p.epi_tma && !accumulate) {
    // ---------------------------------------------------------- epilogue, TMA stores (UpdParams::epi_tma)
    // each warp stages 32 partial rows x 16 fp32 columns per store in two 2 KB slots
    // carved from the operand ring, idle once acc_full completes (every stage consumed);
    // SWIZZLE_64B: the row-per-lane float4 writes are bank-conflict free
    const int qrow = (warp % 4) * 32;
    if (iters > 0) {
      mbar_wait(&acc_full[0], 0);
      tc_fence_after();
    }
    uint8_t* stg0 = smem + (warp - 4) * 4096;
    uint32_t n_st = 0;
    const bool live = iters > 0;
    const bool no_store = (kDevBuild ? p.dbg_mode : 0) & 2048;  // dev ablation
    const int n_acc = ((kDevBuild ? p.dbg_mode : 0) & 4096) ? 0 : p.stack > 1 ? xsn : (mc > 1 ? mc : ntaps);
    for (int t = 0; t < n_acc; ++t) {
      // (host-checked: a warp's 32 TMEM rows are 32 consecutive partial rows of one tap)
      const int rows_slot = 16 * p.cb_eff;
      const int slot = p.stack > 1 ? qrow / rows_slot : 0;
      if (p.stack > 1 && slot >= ntaps) continue;
      const int sl = tap0 + slot;
      if (p.xs > 1 && p.xs_slot_s[sl] + t >= p.xs_S) continue;
      const int rs = p.xs > 1 ? p.xs_slot_r[sl] * p.xs_S + p.xs_slot_s[sl] + t
                              : p.tap_src[tap0 + (p.stack > 1 ? slot : (mc > 1 ? 0 : t))];
      const int c_row0 = p.stack > 1 ? qrow % rows_slot : (ctile * mc + (mc > 1 ? t : 0)) * 128 + qrow;
      const int row0 = (split * p.n_taps + rs) * p.c_pad + c_row0;
      for (int g = 0; g < p.nb; ++g) {
        uint32_t r[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(qrow) << 16) + static_cast<uint32_t>(t * NT + g * 16), r);
        tmem_ld_wait();
        if (no_store) continue;
        uint8_t* stg = stg0 + (n_st & 1u) * 2048u;
        if (n_st >= 2) {  // this slot's previous store must have left shared memory
          if (lane == 0) bulk_wait_group_read<1>();
          __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 v = live ? make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                              __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float4*>(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4)) = v;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&map_part, stg, ktile * NT + g * 16, row0);
          bulk_commit_group();
        }
        ++n_st;
      }
    }
    if (lane == 0) bulk_wait_group0();
    __syncwarp();
  } else if (warp >= 4) {
    // ---------------------------------------------------------- epilogue (lsu plans: after loading)
    // one pass per accumulation period: every period's buffer is added into the
    // partial slice (the first one overwrites it unless the launch accumulates)
    const int qrow = (warp % 4) * 32;
    const int n_periods = iters > 0 ? per_acc.period(iters - 1) + 1 : 1;
    for (int jd = 0; jd < n_periods; ++jd) {
      if (iters > 0) {
        mbar_wait(&acc_full[per_acc.buf(jd)], per_acc.par(jd));
        tc_fence_after();
      }
      const uint32_t acc_col0 = static_cast<uint32_t>(per_acc.buf(jd)) * buf_cols;
      const bool add_old = accumulate || jd > 0;
    // dev ablation bits: 4096 no epilogue, 2048 no partial stores
    const int n_acc = ((kDevBuild ? p.dbg_mode : 0) & 4096) ? 0 : p.stack > 1 ? xsn : (mc > 1 ? mc : ntaps);
    for (int t = 0; t < n_acc; ++t) {
      const int c_glob = (ctile * mc + (mc > 1 ? t : 0)) * 128 + qrow + lane;
      // stacked: TMEM row = (slot j, channel c) of tap tap0 + j; cross-stacked: column
      // block t of slot j is tap (r_j, s_j + t)
      const int rows_slot = p.half ? 8 : 16 * p.cb_eff;
      const int slot = p.stack > 1 ? (qrow + lane) / rows_slot : 0;
      const int c_row = p.stack > 1 ? (qrow + lane) % rows_slot : c_glob;
      const bool row_ok = p.stack > 1 ? slot < ntaps : true;
      const int sl = tap0 + (row_ok ? slot : 0);
      if (p.xs > 1 && p.xs_slot_s[sl] + t >= p.xs_S) continue;  // (no such tap: S not a multiple of xs)
      const int rs = p.xs > 1 ? p.xs_slot_r[sl] * p.xs_S + p.xs_slot_s[sl] + t
                              : p.tap_src[tap0 + (p.stack > 1 ? (row_ok ? slot : 0) : (mc > 1 ? 0 : t))];
      float* dst_row =
          p.partial + ((static_cast<long long>(split) * p.n_taps + rs) * p.c_pad + c_row) * p.k_pad + ktile * NT;
      for (int g = 0; g < p.nb; ++g) {
        uint32_t r[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(qrow) << 16) + acc_col0 + static_cast<uint32_t>(t * NT + g * 16), r);
        tmem_ld_wait();
        if (!row_ok || ((kDevBuild ? p.dbg_mode : 0) & 2048)) continue;
        float4* d = reinterpret_cast<float4*>(dst_row + g * 16);
        const bool live = iters > 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float4 v = live ? make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                        __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3]))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
          if (add_old) {
            const float4 o = d[e];
            v.x = o.x + v.x;
            v.y = o.y + v.y;
            v.z = o.z + v.z;
            v.w = o.w + v.w;
          }
          d[e] = v;
        }
      }
    }
      if (jd + 1 < n_periods) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_drained[per_acc.buf(jd)]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

// ---------------------------------------------------------------------------
// fp32 operands converted in shared memory (no HBM piece tensors).
//
// Stage = the same operand boxes as conv_upd_kernel, but TMA brings the fp32
// pixels (64 B rows, SWIZZLE_64B) into a RAW ring; converter warps split them
// into bf16 pieces (PIECES = 3: exact hi/mid/lo; 1: round to bf16) in the
// canonical MN-major layout of a PIECE ring that the MMA reads. HBM traffic
// is the fp32 tensors once; the split never round-trips through HBM.
//
// CAT (PIECES = 3 only): the three dO pieces sit consecutively along N, so
// A0 x [B0|B1|B2], A1 x [B0|B1] and A2 x B0 are three MMAs of N = 3NT, 2NT
// and NT instead of six of N = NT (half the A-operand smem reads). The
// accumulator has three column groups X | Y | Z (X = a0 b0, Y and Z collect
// the corrections); the epilogue adds them.
//
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer (+TMEM owner),
// w4..w11 converters during the main loop; w4..w7 then run the epilogue.
constexpr int kUpdRawWarps = 12;
constexpr int kUpdCvtWarp0 = 4, kUpdCvtWarps = 8;

struct UpdRawLayout {
  uint32_t a_sub;     // raw bytes of one A box (1 KiB aligned; stacked: one per tap slot)
  uint32_t a_raw;     // raw A bytes per stage
  uint32_t raw_slot;  // raw ring slot (A boxes then the dO box)
  uint32_t pc_slot;   // piece ring slot (UpdStage layout with PA = PB = pieces)
  uint32_t pc_off;    // piece ring start
};

__host__ __device__ inline UpdRawLayout upd_raw_layout(int a_px, int vs, int nb, int pieces, int a_boxes,
                                                       int a_planes_per_box, int raw_stages) {
  UpdRawLayout L;
  L.a_sub = (static_cast<uint32_t>(a_planes_per_box) * a_px * 64u + 1023u) & ~1023u;
  L.a_raw = L.a_sub * a_boxes;
  L.raw_slot = (L.a_raw + static_cast<uint32_t>(nb) * vs * 64u + 1023u) & ~1023u;
  L.pc_slot = upd_stage_layout(a_px, vs, nb, pieces, pieces).bytes;
  L.pc_off = L.raw_slot * raw_stages;
  return L;
}

// dO piece ring slot of conv_upd_ts_kernel (A lives in TMEM)
__host__ __device__ inline uint32_t upd_ts_pc_slot(int vs, int nb, int pieces) {
  return (static_cast<uint32_t>(pieces) * 2u * nb * vs * 16u + 1023u) & ~1023u;
}

// 16 B chunk k of row j of a SWIZZLE_64B box whose start is 1 KiB aligned
__device__ __forceinline__ uint32_t sw64_row(uint32_t j, uint32_t k) { return j * 64u + ((k ^ ((j >> 1) & 3u)) << 4); }


template <int PIECES, bool CAT>
__global__ void __launch_bounds__(kUpdRawWarps * 32, 1)
    conv_upd_raw_kernel(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_do,
                        const __grid_constant__ UpdParams p, int raw_stages, int pc_stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t raw_full[kMaxStages], raw_empty[kMaxStages];
  __shared__ __align__(8) uint64_t pc_full[kMaxStages], pc_empty[kMaxStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_drained[2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ int s_tap_shift[kMaxTaps];  // off the constant cache in the issue loop

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (warp == 2)
    for (int i = lane; i < kMaxTaps; i += 32) s_tap_shift[i] = p.tap_shift[i];
  const int NT = 16 * p.nb;
  const AccPeriods per_acc{p.drain, p.drain_bufs > 1 ? 2 : 1};
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
  const bool stacked = p.stack > 1;
  const int a_boxes = stacked ? ntaps : 1;
  const int a_planes = stacked ? p.cb_eff : 8;  // channel blocks per A box
  const UpdRawLayout R = upd_raw_layout(p.a_px, p.vs, p.nb, PIECES, stacked ? p.stack : 1, a_planes, raw_stages);
  const UpdStage S = upd_stage_layout(p.a_px, p.vs, p.nb, PIECES, PIECES);
  const uint32_t smem0 = smem_u32(smem);
  constexpr int kGroups = CAT ? 3 : 1;  // accumulator column groups per tap
  const int acc_w = kGroups * NT;
  const uint32_t buf_cols = static_cast<uint32_t>(p.tg * acc_w);  // one accumulation buffer

  uint32_t tmem_cols = 32;
  while (tmem_cols < static_cast<uint32_t>(per_acc.bufs) * buf_cols) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_in);
    tma_prefetch_desc(&map_do);
    for (int s = 0; s < raw_stages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], kUpdCvtWarps);
    }
    for (int s = 0; s < pc_stages; ++s) {
      mbar_init(&pc_full[s], kUpdCvtWarps);
      mbar_init(&pc_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_drained[b], 4);  // the four epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (fp32 boxes)
    if (lane == 0) {
      const uint32_t a_box_bytes = static_cast<uint32_t>(a_planes) * p.a_px * 64u;
      const uint32_t b_bytes = static_cast<uint32_t>(p.nb) * p.vs * 64u;
      for (int it = 0; it < iters; ++it) {
        const int s = it % raw_stages;
        mbar_wait(&raw_empty[s], (static_cast<uint32_t>(it / raw_stages) & 1u) ^ 1u);
        const int stage = s_begin + it;
        const int n = stage / p.stages_per_img;
        const int band = stage % p.stages_per_img;
        uint8_t* st = smem + static_cast<uint32_t>(s) * R.raw_slot;
        mbar_arrive_expect_tx(&raw_full[s], a_box_bytes * a_boxes + b_bytes);
        const int pa = n * p.in_cb + ctile * 8;
        if (stacked) {
          for (int j = 0; j < ntaps; ++j) {
            const int tp = tap0 + j, tph = p.tap_ph[tp];
            tma_load_4d(st + j * R.a_sub, &map_in, &raw_full[s], 0,
                        p.in_col0 + p.phase_col[tph] + p.stride * p.tap_s2[tp],
                        p.in_row0 + p.phase_row[tph] + p.stride * (band * p.rows_ps + p.tap_r2[tp]), pa);
          }
        } else if (p.linear) {
          tma_load_3d(st, &map_in, &raw_full[s], 0, band * p.vs, pa);
        } else {
          tma_load_4d(st, &map_in, &raw_full[s], 0, p.in_col0 + p.phase_col[ph],
                      p.in_row0 + p.stride * band * p.rows_ps + p.phase_row[ph], pa);
        }
        const int pb = n * p.do_cb + ktile * p.nb;
        if (p.linear)
          tma_load_3d(st + R.a_raw, &map_do, &raw_full[s], 0, band * p.vs, pb);
        else
          tma_load_4d(st + R.a_raw, &map_do, &raw_full[s], 0, 0, band * p.rows_ps, pb);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const int ksteps = p.vs / 16;
    for (int it = 0; it < iters; ++it) {
      const int s = it % pc_stages;
      const int jp = per_acc.period(it);
      const bool p_first = per_acc.starts(it);
      if (p_first && jp >= per_acc.bufs) {  // the buffer's previous period has been drained
        mbar_wait(&acc_drained[per_acc.buf(jp)], static_cast<uint32_t>(jp / per_acc.bufs - 1) & 1u);
      }
      mbar_wait(&pc_full[s], static_cast<uint32_t>(it / pc_stages) & 1u);
      tc_fence_after();
      const uint32_t st = smem0 + R.pc_off + static_cast<uint32_t>(s) * R.pc_slot;
      const uint32_t acc0 = tmem_base + static_cast<uint32_t>(per_acc.buf(jp)) * buf_cols;
      if (elect_one()) {
        const int n_acc = stacked ? 1 : ntaps;
        // descriptors packed once per stage; per MMA only the 16 B-unit start address advances
        const uint64_t a0 = make_smem_desc(st, 128, S.a_plane);
        const uint64_t b0 = make_smem_desc(st + S.b_off, 128, S.b_plane);
        const uint32_t a_pc = S.a_piece >> 4, b_pc = S.b_piece >> 4;
        const uint32_t id3 = make_idesc(1, 1, 1, 128, 3u * NT), id2 = make_idesc(1, 1, 1, 128, 2u * NT),
                       id1 = make_idesc(1, 1, 1, 128, static_cast<uint32_t>(NT));
        for (int t = 0; t < n_acc; ++t) {
          const int shift = stacked ? 0 : s_tap_shift[tap0 + t];
          const uint32_t d_tmem = acc0 + static_cast<uint32_t>(t * acc_w);
          for (int ks = 0; ks < (((kDevBuild ? p.dbg_mode : 0) & 8) ? 0 : ksteps); ++ks) {  // dbg 8: ablation, no MMAs
            const bool first = p_first && ks == 0;
            const uint64_t ak = a0 + static_cast<uint32_t>(ks * 16 + shift);  // 16 B per pixel row
            const uint64_t bk = b0 + static_cast<uint32_t>(ks) * 16u;          // 256 B per k-step
            if (CAT) {
              // X|Y|Z += a0 [b0|b1|b2];  Y|Z += a1 [b0|b1];  Z += a2 b0
              mma_bf16(d_tmem, ak, bk, id3, first ? 0u : 1u);
              mma_bf16(d_tmem + NT, ak + a_pc, bk, id2, 1u);
              mma_bf16(d_tmem + 2 * NT, ak + 2u * a_pc, bk, id1, 1u);
            } else {
#pragma unroll
              for (int ia = 0; ia < PIECES; ++ia)
#pragma unroll
                for (int ib = 0; ib < PIECES; ++ib) {
                  if (ia + ib > 2) continue;
                  mma_bf16(d_tmem, ak + static_cast<uint32_t>(ia) * a_pc, bk + static_cast<uint32_t>(ib) * b_pc, id1,
                           (first && ia == 0 && ib == 0) ? 0u : 1u);
                }
            }
          }
        }
        mma_commit(&pc_empty[s]);
        if (per_acc.ends(it, iters)) mma_commit(&acc_full[per_acc.buf(jp)]);
      }
      __syncwarp();
    }
  } else if (warp >= kUpdCvtWarp0) {
    // ------------------------------------------------------------ converters (fp32 raw -> bf16 pieces)
    // w4..w7 (one per TMEM lane quarter) also write the partials: after the last
    // period, and (drain > 0) at every period boundary, where they add the
    // finished accumulation buffer into the CTA's partial slice
    const bool epi_warp = warp < kUpdCvtWarp0 + 4;
    const int qrow = (warp % 4) * 32;
    auto write_partial = [&](uint32_t acc_col0, bool add_old) {
      const int c_glob = ctile * 128 + qrow + lane;
      const int n_acc = stacked ? 1 : ntaps;
      for (int t = 0; t < n_acc; ++t) {
        const int rows_slot = p.half ? 8 : 16 * p.cb_eff;
        const int slot = stacked ? (qrow + lane) / rows_slot : 0;
        const int c_row = stacked ? (qrow + lane) % rows_slot : c_glob;
        const bool row_ok = stacked ? slot < ntaps : true;
        const int rs = p.tap_src[tap0 + (stacked ? (row_ok ? slot : 0) : t)];
        float* dst_row =
            p.partial + ((static_cast<long long>(split) * p.n_taps + rs) * p.c_pad + c_row) * p.k_pad + ktile * NT;
        const uint32_t tb = tmem_base + (static_cast<uint32_t>(qrow) << 16) + acc_col0 + static_cast<uint32_t>(t * acc_w);
        for (int g = 0; g < p.nb; ++g) {
          uint32_t r[16], ry[16], rz[16];
          tmem_ld16(tb + static_cast<uint32_t>(g * 16), r);
          if (CAT) {
            tmem_ld16(tb + static_cast<uint32_t>(NT + g * 16), ry);
            tmem_ld16(tb + static_cast<uint32_t>(2 * NT + g * 16), rz);
          }
          tmem_ld_wait();
          if (!row_ok) continue;
          float4* d = reinterpret_cast<float4*>(dst_row + g * 16);
          const bool live = iters > 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float vv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int q = 4 * e + u;
              vv[u] = CAT ? __uint_as_float(r[q]) + (__uint_as_float(ry[q]) + __uint_as_float(rz[q]))
                          : __uint_as_float(r[q]);
              if (!live) vv[u] = 0.0f;
            }
            if (add_old) {
              const float4 o = d[e];
              vv[0] = o.x + vv[0];
              vv[1] = o.y + vv[1];
              vv[2] = o.z + vv[2];
              vv[3] = o.w + vv[3];
            }
            d[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
          }
        }
      }
    };
    // Work unit = one 16 B-chunk plane (8 channels) of one operand: A has
    // a_boxes * a_planes * 2 <= 16 of them, dO 2 * nb <= 32. Warp cw owns chunk
    // planes cw, cw + 8, ... of each operand for the whole kernel, so all
    // index math is hoisted out of the stage loop; a warp's lanes walk the
    // plane's pixels 32 at a time (conflict-free swizzled reads, contiguous writes).
    const int cw = warp - kUpdCvtWarp0;
    // half-block stacking: one chunk plane (channels 0..7, half 0) per tap slot
    const int a_cps = p.half ? a_boxes : a_boxes * a_planes * 2, b_cps = 2 * p.nb;
    // slots 0-1: A chunk planes cw, cw + 8; slots 2-5: dO chunk planes cw + 8 j (npx = 0: unused)
    uint32_t src_base[6], dst_base[6], piece_str[6], cp_rows0[6], cp_c0[6];
    int cp_npx[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      const bool is_a = u < 2;
      const int cp = cw + kUpdCvtWarps * (is_a ? u : u - 2);
      const bool ok = cp < (is_a ? a_cps : b_cps);
      cp_npx[u] = ok ? (is_a ? p.a_px : p.vs) : 0;
      cp_c0[u] = (is_a && p.half) ? 0u : 2u * (cp & 1);
      if (is_a) {
        const int pl = p.half ? 0 : (cp >> 1) % a_planes, box = p.half ? cp : (cp >> 1) / a_planes;
        src_base[u] = box * R.a_sub;
        cp_rows0[u] = pl * p.a_px;
        dst_base[u] = static_cast<uint32_t>(cp) * S.a_plane;
        piece_str[u] = S.a_piece;
      } else {
        src_base[u] = R.a_raw;
        cp_rows0[u] = (cp >> 1) * p.vs;
        dst_base[u] = S.b_off + static_cast<uint32_t>(cp) * S.b_plane;
        piece_str[u] = S.b_piece;
      }
    }
    int rs = 0, ps = 0;
    uint32_t rph = 0, pph = 0;
    for (int it = 0; it < iters; ++it) {
      if (epi_warp && it > 0 && per_acc.drain && per_acc.starts(it)) {
        const int jd = per_acc.period(it) - 1;  // the period that just ended
        mbar_wait(&acc_full[per_acc.buf(jd)], per_acc.par(jd));
        tc_fence_after();
        write_partial(static_cast<uint32_t>(per_acc.buf(jd)) * buf_cols, jd > 0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_drained[per_acc.buf(jd)]);
      }
      mbar_wait(&raw_full[rs], rph);
      mbar_wait(&pc_empty[ps], pph ^ 1u);
      const uint8_t* raw = smem + static_cast<uint32_t>(rs) * R.raw_slot;
      uint8_t* pcs = smem + R.pc_off + static_cast<uint32_t>(ps) * R.pc_slot;
#pragma unroll
      for (int u = 0; u < (((kDevBuild ? p.dbg_mode : 0) & 4) ? 0 : 6); ++u) {
        const uint32_t piece_stride = piece_str[u];
        const uint8_t* src0 = raw + src_base[u];
        uint8_t* dst0 = pcs + dst_base[u];
        const uint32_t row0 = cp_rows0[u];
        const uint32_t c0 = cp_c0[u];
        for (int px = lane; px < cp_npx[u]; px += 32) {
          const uint32_t row = row0 + px;
          const uint8_t* src = src0 + sw64_row(row, c0);
          const float4 a = *reinterpret_cast<const float4*>(src);
          // chunk c0 + 1 of the same row: bit 4 flips under the row's XOR pattern
          const float4 b = *reinterpret_cast<const float4*>(src0 + (sw64_row(row, c0) ^ 16u));
          const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
          uint8_t* dst = dst0 + px * 16;
          if (PIECES == 3) {
            uint4 h, m, l;
            split8(v, h, m, l);
            *reinterpret_cast<uint4*>(dst) = h;
            *reinterpret_cast<uint4*>(dst + piece_stride) = m;
            *reinterpret_cast<uint4*>(dst + 2 * piece_stride) = l;
          } else {
            *reinterpret_cast<uint4*>(dst) = cast8(v);
          }
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rs]);
        mbar_arrive(&pc_full[ps]);
      }
      if (++rs == raw_stages) {
        rs = 0;
        rph ^= 1u;
      }
      if (++ps == pc_stages) {
        ps = 0;
        pph ^= 1u;
      }
    }
    if (epi_warp) {
      // -------------------------------------------------------- epilogue (w4..w7: TMEM lane quarters)
      const int jl = iters > 0 ? per_acc.period(iters - 1) : 0;
      if (iters > 0) {
        mbar_wait(&acc_full[per_acc.buf(jl)], per_acc.par(jl));
        tc_fence_after();
      }
      if (warp == kUpdCvtWarp0 && lane == 0) pdl_launch_dependents();  // the reduce may get scheduled
      write_partial(static_cast<uint32_t>(per_acc.buf(jl)) * buf_cols, jl > 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

// ---------------------------------------------------------------------------
// Single-tap fp32 UPD with the A operand (input activations) in TENSOR memory.
// The in-smem variant above is shared-memory-bandwidth bound (TMA raw writes,
// converter reads + piece writes and the MMA's A / B reads ~170 KB per 32-pixel
// stage against ~128 B/cycle). Here a converter thread owns one TMEM lane = one
// input channel: it reads that channel's fp32 values of the stage's pixels from
// the raw box (SWIZZLE_64B, 16 lanes per 64 B row: a warp's 32 channels are two
// contiguous rows, conflict-free), splits them into bf16 pieces packed two
// pixels per column and tcgen05.st's them into a TMEM ring; the MMA reads A
// from TMEM (K = pixels along columns) and only dO pieces go through smem.
// Two converter groups of four warps (one per TMEM lane quarter) alternate
// stages; within a stage the group also converts the dO chunk planes.
// warps: w0 TMA producer, w1 MMA issuer, w4.. converter groups of four (w4..w7 then
// run the epilogue); w2, w3 idle
constexpr int kUpdTsCvtGroups = 2;  // (3 measured slower)
constexpr int kUpdTsWarps = 4 + 4 * kUpdTsCvtGroups;

template <int PIECES, bool CAT>
__global__ void __launch_bounds__(kUpdTsWarps * 32, 1)
    conv_upd_ts_kernel(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_do,
                       const __grid_constant__ UpdParams p, int raw_stages, int pc_stages) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t raw_full[kMaxStages], raw_empty[kMaxStages];
  __shared__ __align__(8) uint64_t pc_full[kMaxStages], pc_empty[kMaxStages];
  __shared__ __align__(8) uint64_t acc_full[2], acc_drained[2];
  __shared__ uint32_t tmem_base_sh;

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int NT = 16 * p.nb;
  const AccPeriods per_acc{p.drain, p.drain_bufs > 1 ? 2 : 1};
  const int ctile = blockIdx.x;  // single tap: one tap group
  const int ktile = blockIdx.y;
  const int split = blockIdx.z;
  const int per = (p.stages_total + p.splits - 1) / p.splits;
  const int s_begin = split * per;
  const int s_end = min(p.stages_total, s_begin + per);
  const int iters = s_end > s_begin ? s_end - s_begin : 0;
  // raw slot: A box (8 planes x a_px x 64 B) then the dO box; piece slot: dO pieces only
  const UpdRawLayout R = upd_raw_layout(p.a_px, p.vs, p.nb, PIECES, 1, 8, raw_stages);
  const uint32_t b_plane = static_cast<uint32_t>(p.vs) * 16u, b_piece = 2u * p.nb * b_plane;
  const uint32_t pc_slot = upd_ts_pc_slot(p.vs, p.nb, PIECES);
  const uint32_t smem0 = smem_u32(smem);
  constexpr int kGroups = CAT ? 3 : 1;
  const uint32_t acc_w = static_cast<uint32_t>(kGroups * NT);
  const uint32_t acc_all = static_cast<uint32_t>(per_acc.bufs) * acc_w;  // accumulation buffers, then the A ring
  const uint32_t a_cols = static_cast<uint32_t>(p.vs) / 2u;  // TMEM columns per piece per stage
  const uint32_t ring_slot = PIECES * a_cols;
  // converter groups take stages round-robin: same ordering argument as
  // conv_fwd_kernel's (pc_stages >= groups keeps the piece-slot parity wait
  // unambiguous); measured: all warps on every stage is slower than rotating groups
  const int cvt_groups = (raw_stages >= 2 && pc_stages >= kUpdTsCvtGroups &&
                          (raw_stages % kUpdTsCvtGroups == 0 || raw_stages >= pc_stages))
                             ? kUpdTsCvtGroups
                             : 1;
  const uint32_t cvt_arrivals = 4u;

  uint32_t tmem_cols = 32;
  while (tmem_cols < acc_all + static_cast<uint32_t>(pc_stages) * ring_slot) tmem_cols <<= 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_in);
    tma_prefetch_desc(&map_do);
    for (int s = 0; s < raw_stages; ++s) {
      mbar_init(&raw_full[s], 1);
      mbar_init(&raw_empty[s], cvt_arrivals);
    }
    for (int s = 0; s < pc_stages; ++s) {
      mbar_init(&pc_full[s], cvt_arrivals);
      mbar_init(&pc_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_drained[b], 4);  // the four epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(&tmem_base_sh, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_base_sh;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (fp32 boxes)
    if (lane == 0) {
      const uint32_t a_bytes = 8u * p.a_px * 64u, b_bytes = static_cast<uint32_t>(p.nb) * p.vs * 64u;
      for (int it = 0; it < iters; ++it) {
        const int s = it % raw_stages;
        mbar_wait(&raw_empty[s], (static_cast<uint32_t>(it / raw_stages) & 1u) ^ 1u);
        const int stage = s_begin + it;
        const int n = stage / p.stages_per_img, band = stage % p.stages_per_img;
        uint8_t* st = smem + static_cast<uint32_t>(s) * R.raw_slot;
        mbar_arrive_expect_tx(&raw_full[s], a_bytes + b_bytes);
        const int pa = n * p.in_cb + ctile * 8, pb = n * p.do_cb + ktile * p.nb;
        if (p.linear) {
          tma_load_3d(st, &map_in, &raw_full[s], 0, band * p.vs, pa);
          tma_load_3d(st + R.a_raw, &map_do, &raw_full[s], 0, band * p.vs, pb);
        } else {
          tma_load_4d(st, &map_in, &raw_full[s], 0, p.in_col0 + p.phase_col[0],
                      p.in_row0 + p.stride * band * p.rows_ps + p.phase_row[0], pa);
          tma_load_4d(st + R.a_raw, &map_do, &raw_full[s], 0, 0, band * p.rows_ps, pb);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (A from TMEM, B from smem)
    const int ksteps = p.vs / 16;
    for (int it = 0; it < iters; ++it) {
      const int s = it % pc_stages;
      const int jp = per_acc.period(it);
      const bool p_first = per_acc.starts(it);
      if (p_first && jp >= per_acc.bufs)  // the buffer's previous period has been drained
        mbar_wait(&acc_drained[per_acc.buf(jp)], static_cast<uint32_t>(jp / per_acc.bufs - 1) & 1u);
      mbar_wait(&pc_full[s], static_cast<uint32_t>(it / pc_stages) & 1u);
      tc_fence_after();
      const uint32_t st = smem0 + R.pc_off + static_cast<uint32_t>(s) * pc_slot;
      const uint32_t a_t = tmem_base + acc_all + static_cast<uint32_t>(s) * ring_slot;
      const uint32_t dacc = tmem_base + static_cast<uint32_t>(per_acc.buf(jp)) * acc_w;
      if (elect_one()) {
        // operand addresses advance by constants per k-step: no descriptor packing in the loop
        const uint64_t b0 = make_smem_desc(st, 128, b_plane);
        const uint64_t b_pc = b_piece >> 4;
        const uint32_t id3 = make_idesc(1, 0, 1, 128, 3u * NT), id2 = make_idesc(1, 0, 1, 128, 2u * NT),
                       id1 = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(NT));
        for (int ks = 0; ks < (((kDevBuild ? p.dbg_mode : 0) & 8) ? 0 : ksteps); ++ks) {  // dbg 8: ablation, no MMAs
          const bool first = p_first && ks == 0;
          const uint32_t ak = a_t + static_cast<uint32_t>(ks) * 8u;
          const uint64_t bk = b0 + static_cast<uint64_t>(ks) * 16u;  // 256 B per k-step
          if (CAT) {
            mma_bf16_ts(dacc, ak, bk, id3, first ? 0u : 1u);
            mma_bf16_ts(dacc + NT, ak + a_cols, bk, id2, 1u);
            mma_bf16_ts(dacc + 2 * NT, ak + 2u * a_cols, bk, id1, 1u);
          } else {
#pragma unroll
            for (int ia = 0; ia < PIECES; ++ia)
#pragma unroll
              for (int ib = 0; ib < PIECES; ++ib) {
                if (ia + ib > 2) continue;
                mma_bf16_ts(dacc, ak + static_cast<uint32_t>(ia) * a_cols, bk + static_cast<uint64_t>(ib) * b_pc,
                            id1, (first && ia == 0 && ib == 0) ? 0u : 1u);
              }
          }
        }
        mma_commit(&pc_empty[s]);
        if (per_acc.ends(it, iters)) mma_commit(&acc_full[per_acc.buf(jp)]);
      }
      __syncwarp();
    }
  } else if (warp >= kUpdCvtWarp0) {
    // ------------------------------------------------------------ converters
    const int grp = (warp - kUpdCvtWarp0) / 4;
    const uint32_t q = static_cast<uint32_t>(warp % 4);
    const int row = static_cast<int>(q) * 32 + lane;  // TMEM lane = input channel of the c-tile
    const int pl = row / 16, ln = row % 16;           // raw plane, lane within the 64 B row
    // a warp's lanes 0-15 / 16-31 read two planes a_px rows apart: with a_px even
    // both rows sit on the same 16 banks, so the upper half reads the pixel pair
    // in swapped order (rows of opposite parity -> disjoint bank halves)
    const uint32_t swap = ((lane >> 4) & ~p.a_px) & 1u;
    const uint32_t kq = static_cast<uint32_t>(ln >> 2), lo4 = static_cast<uint32_t>(ln & 3) * 4u;
    const uint32_t a_row0 = static_cast<uint32_t>(pl * p.a_px + p.tap_shift[0]);
    // group 0 (w4..w7, one warp per TMEM lane quarter) writes the partials: after the
    // last period and, when drain > 0, at every period boundary (adding the finished
    // buffer into the CTA's partial slice)
    const bool epi_warp = warp < kUpdCvtWarp0 + 4;
    const int qrow = (warp % 4) * 32;
    auto write_partial = [&](uint32_t acc_col0, bool add_old) {
      float* dst_row = p.partial + ((static_cast<long long>(split) * p.n_taps + p.tap_src[0]) * p.c_pad +
                                    ctile * 128 + qrow + lane) * p.k_pad + ktile * NT;
      const uint32_t tb = tmem_base + (static_cast<uint32_t>(qrow) << 16) + acc_col0;
      for (int g = 0; g < p.nb; ++g) {
        uint32_t r[16], ry[16], rz[16];
        tmem_ld16(tb + static_cast<uint32_t>(g * 16), r);
        if (CAT) {
          tmem_ld16(tb + static_cast<uint32_t>(NT + g * 16), ry);
          tmem_ld16(tb + static_cast<uint32_t>(2 * NT + g * 16), rz);
        }
        tmem_ld_wait();
        float4* d = reinterpret_cast<float4*>(dst_row + g * 16);
        const bool live = iters > 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          float vv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int qq = 4 * e + u;
            vv[u] = CAT ? __uint_as_float(r[qq]) + (__uint_as_float(ry[qq]) + __uint_as_float(rz[qq]))
                        : __uint_as_float(r[qq]);
            if (!live) vv[u] = 0.0f;
          }
          if (add_old) {
            const float4 o = d[e];
            vv[0] = o.x + vv[0];
            vv[1] = o.y + vv[1];
            vv[2] = o.z + vv[2];
            vv[3] = o.w + vv[3];
          }
          d[e] = make_float4(vv[0], vv[1], vv[2], vv[3]);
        }
      }
    };
    // dO chunk planes 0 .. 2nb-1: warp q of the group takes q, q + 4, ...
    for (int it = 0; it < iters; ++it) {
      if (epi_warp && it > 0 && per_acc.drain && per_acc.starts(it)) {
        const int jd = per_acc.period(it) - 1;  // the period that just ended
        mbar_wait_backoff(&acc_full[per_acc.buf(jd)], per_acc.par(jd));
        tc_fence_after();
        write_partial(static_cast<uint32_t>(per_acc.buf(jd)) * acc_w, jd > 0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_drained[per_acc.buf(jd)]);
      }
      if ((it % cvt_groups) != grp) continue;
      const int rs = it % raw_stages, ps = it % pc_stages;
      mbar_wait_backoff(&pc_empty[ps], (static_cast<uint32_t>(it / pc_stages) & 1u) ^ 1u);  // first: see cvt_groups
      mbar_wait_backoff(&raw_full[rs], static_cast<uint32_t>(it / raw_stages) & 1u);
      tc_fence_after();
      const uint8_t* raw = smem + static_cast<uint32_t>(rs) * R.raw_slot;
      if (!((kDevBuild ? p.dbg_mode : 0) & 4)) {
        // A: this channel's values over the stage's pixels -> pieces, 2 pixels per column
        const uint32_t col0 = tmem_base + (q * 32u << 16) + acc_all + static_cast<uint32_t>(ps) * ring_slot;
        // 16-pixel units; the next unit's values are loaded before this unit's
        // tcgen05.st so shared-memory latency overlaps the split arithmetic
        const int px_end = ((kDevBuild ? p.dbg_mode : 0) & 64) ? 0 : p.vs;
        float xa[16];
        auto load_unit = [&](int px0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const uint32_t r0 = a_row0 + static_cast<uint32_t>(px0 + 2 * e);
            xa[2 * e] = *reinterpret_cast<const float*>(raw + sw64_row(r0 + swap, kq) + lo4);
            xa[2 * e + 1] = *reinterpret_cast<const float*>(raw + sw64_row(r0 + 1u - swap, kq) + lo4);
          }
        };
        if (px_end > 0) load_unit(0);
        for (int px0 = 0; px0 < px_end; px0 += 16) {
          uint32_t h[8], m[8], l[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float va = xa[2 * e], vb = xa[2 * e + 1];
            const float x0 = swap ? vb : va, x1 = swap ? va : vb;
            h[e] = cvt2(x0, x1);
            if (PIECES == 3) {
              const float ra = x0 - lo_f(h[e]), rb = x1 - hi_f(h[e]);
              m[e] = cvt2(ra, rb);
              l[e] = cvt2(ra - lo_f(m[e]), rb - hi_f(m[e]));
            }
          }
          if (px0 + 16 < px_end) load_unit(px0 + 16);
          const uint32_t c = col0 + static_cast<uint32_t>(px0 / 2);
          tmem_st8_nc(c, h);
          if (PIECES == 3) {
            tmem_st8_nc(c + a_cols, m);
            tmem_st8_nc(c + 2 * a_cols, l);
          }
        }
        // dO: chunk planes (8 k-channels) -> MN-major pieces in smem
        uint8_t* pcs = smem + R.pc_off + static_cast<uint32_t>(ps) * pc_slot;
        for (int cp = static_cast<int>(q); cp < (((kDevBuild ? p.dbg_mode : 0) & 128) ? 0 : 2 * p.nb); cp += 4) {
          const uint32_t c0 = 2u * (cp & 1), rbase = static_cast<uint32_t>((cp >> 1) * p.vs);
          for (int px = lane; px < p.vs; px += 32) {
            const uint32_t off = sw64_row(rbase + px, c0);
            const float4 a = *reinterpret_cast<const float4*>(raw + R.a_raw + off);
            const float4 b = *reinterpret_cast<const float4*>(raw + R.a_raw + (off ^ 16u));
            const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint8_t* dst = pcs + static_cast<uint32_t>(cp) * b_plane + px * 16;
            if (PIECES == 3) {
              uint4 hh, mm, ll;
              split8(v, hh, mm, ll);
              *reinterpret_cast<uint4*>(dst) = hh;
              *reinterpret_cast<uint4*>(dst + b_piece) = mm;
              *reinterpret_cast<uint4*>(dst + 2 * b_piece) = ll;
            } else {
              *reinterpret_cast<uint4*>(dst) = cast8(v);
            }
          }
        }
      }
      tmem_st_wait();
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rs]);
        mbar_arrive(&pc_full[ps]);
      }
    }
    if (epi_warp) {
      // -------------------------------------------------------- epilogue (w4..w7: TMEM lane quarters)
      const int jl = iters > 0 ? per_acc.period(iters - 1) : 0;
      if (iters > 0) {
        mbar_wait(&acc_full[per_acc.buf(jl)], per_acc.par(jl));
        tc_fence_after();
      }
      if (warp == kUpdCvtWarp0 && lane == 0) pdl_launch_dependents();
      write_partial(static_cast<uint32_t>(per_acc.buf(jl)) * acc_w, jl > 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, tmem_cols);
}

// Fixed-order reduction of the split partials into the blocked dW
// [k_b][c_b][r][s][c][k] (tail lanes written as exact zeros).
// reduce_weight_copies analog (propagation.cpp:357-375). A thread owns four
// consecutive k of one (tap, c) partial row (16 B loads, coalesced along k; one
// 16 B / 8 B store into the dW block) and 32-bit index math; blockDim.y = G split
// groups: group y sums splits y, y + G, y + 2G, ... in increasing order, then the
// G group sums are added in group order -- the same fixed order on every run, so
// dW is bitwise reproducible.
constexpr int kRedGroups = 4;  // max split groups per element (blockDim.y)
__global__ void __launch_bounds__(256)
    upd_reduce_kernel(const float* __restrict__ partial, int splits, int n_taps, int c_pad, int k_pad, int C, int K,
                      int cb, int kb, void* __restrict__ dw, int dw_bf16, int accumulate) {
  __shared__ float4 red[kRedGroups * 64];
  pdl_wait_primary();  // launched as a programmatic dependent of the UPD kernel
  const int G = blockDim.y, TX = blockDim.x;
  const int kq = kb * 4, cw = cb * 16;  // k quads per row, c rows per tap
  const int total = n_taps * cw * kq;
  const int f = blockIdx.x * TX + threadIdx.x;
  const int y = threadIdx.y;
  const bool in_range = f < total;
  const int k = in_range ? (f % kq) * 4 : 0;
  const int rc = in_range ? f / kq : 0;
  const int c = rc % cw, rs = rc / cw;
  const bool live = in_range && c < C && k < K;
  const long long split_stride = static_cast<long long>(n_taps) * c_pad * k_pad;
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
  if (live) {
    const float4* src = reinterpret_cast<const float4*>(partial + (static_cast<long long>(rs) * c_pad + c) * k_pad + k);
    const long long st4 = split_stride / 4;
    // up to 8 independent 16 B loads in flight per thread before the (fixed-order) adds
    int sp = y;
    for (; sp + 7 * G < splits; sp += 8 * G) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (sp + u * G) * st4);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        sum.x += v[u].x;
        sum.y += v[u].y;
        sum.z += v[u].z;
        sum.w += v[u].w;
      }
    }
    for (; sp < splits; sp += G) {
      const float4 v = __ldg(src + sp * st4);
      sum.x += v.x;
      sum.y += v.y;
      sum.z += v.z;
      sum.w += v.w;
    }
  }
  if (G > 1) {
    red[y * 64 + threadIdx.x] = sum;
    __syncthreads();
    if (y != 0) return;
    sum = red[threadIdx.x];
    for (int g = 1; g < G; ++g) {
      const float4 v = red[g * 64 + threadIdx.x];
      sum.x += v.x;
      sum.y += v.y;
      sum.z += v.z;
      sum.w += v.w;
    }
  }
  if (!in_range) return;
  const bool cl_ok = c < C;
  float t[4] = {sum.x, sum.y, sum.z, sum.w};
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (!(cl_ok && k + j < K)) t[j] = 0.0f;
  const int kbi = k / 16, kl = k % 16, cbi = c / 16, cl = c % 16;
  const long long e = ((static_cast<long long>(kbi) * cb + cbi) * n_taps + rs) * 256 + cl * 16 + kl;
  if (dw_bf16) {
    __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(dw) + e;
    uint2 old = make_uint2(0u, 0u);
    if (accumulate) old = *reinterpret_cast<const uint2*>(d);
    const __nv_bfloat16* o = reinterpret_cast<const __nv_bfloat16*>(&old);
    __align__(8) __nv_bfloat16 h[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __float2bfloat16_rn(accumulate ? t[j] + __bfloat162float(o[j]) : t[j]);
    *reinterpret_cast<uint2*>(d) = *reinterpret_cast<const uint2*>(h);
  } else {
    float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(dw) + e);
    float4 v = make_float4(t[0], t[1], t[2], t[3]);
    if (accumulate) {
      const float4 o = *d;
      v.x = o.x + v.x;
      v.y = o.y + v.y;
      v.z = o.z + v.z;
      v.w = o.w + v.w;
    }
    *d = v;
  }
}

}  // namespace dconv_sm100
