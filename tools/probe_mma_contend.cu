// Probe: what slows tcgen05.mma below its floor inside the conv kernels?
// One CTA per SM; warp 0 issues MMAs (128 x N x 16, A K-major SW32, B MN-major
// no-swizzle -- the bf16 conv operands) in stages of `per_stage` MMAs with a
// commit per stage; optional concurrent activity:
//   dacc = 2      : alternate the accumulator (two m-blocks, as mb = 2)
//   epi  = 1      : warps 4..7 stream tcgen05.ld x32 over the other TMEM half
//   copy = 1      : warp 2 streams 1-D bulk copies L2 -> a separate smem region
//   ring = 1      : the MMA waits a per-stage mbarrier filled by the copy warp
//                   (the conv kernels' producer / consumer handshake)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_mma_contend probe_mma_contend.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"

using namespace dconv_sm100;

struct Cfg {
  int N, stages, per_stage, dacc, epi, copy, ring, ashift, unroll, bshift;
  uint32_t alo0, blo0, tmem0;
  int kc, a_px, nt, nosync;
  uint32_t w_tap;
};

__global__ void __launch_bounds__(256, 1) probe(Cfg c, const uint8_t* src, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t done, full[4], empty[4];
  __shared__ uint32_t tbase_sh;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (warp == 0) tmem_alloc(&tbase_sh, 512);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    stop = 0;
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_sh;
  const uint32_t s0 = smem_u32(smem);
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t idesc = make_idesc(1, 0, 1, 128, static_cast<uint32_t>(c.N));
      const uint32_t a_lo = static_cast<uint32_t>(make_smem_desc_sw32(s0));
      const uint32_t a_hi = static_cast<uint32_t>(make_smem_desc_sw32(s0) >> 32);
      const uint32_t b_lo = static_cast<uint32_t>(make_smem_desc(s0 + 32768, 128, 256));
      const uint32_t b_hi = static_cast<uint32_t>(make_smem_desc(s0 + 32768, 128, 256) >> 32);
      // descriptors from kernel parameters + the (uniform) dynamic smem base: uniform registers
      uint32_t al[8], bl[8], tb[2];
      const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        al[i] = c.alo0 + sbase + static_cast<uint32_t>(i & 7) * static_cast<uint32_t>(c.ashift);
        bl[i] = c.blo0 + sbase + static_cast<uint32_t>(i & 3) * static_cast<uint32_t>(c.bshift);
      }
      tb[0] = c.tmem0;
      tb[1] = c.tmem0 + (c.dacc == 2 ? 128u : 0u);
      uint32_t sh[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) sh[i] = i < c.nt ? 2u * static_cast<uint32_t>(i * 3) : 0u;
      const long long t0 = clock64();
      int slot = 0;
      uint32_t ph = 0;
      for (int s = 0; s < c.stages; ++s) {
        if (c.ring) {
          mbar_wait(&full[slot], ph);
          tc_fence_after();
        }
        if (c.unroll == 9) {
          // probe_mma_rate's "1x1 ring" body verbatim (A / B bases per 2-slot ring stage)
          const uint32_t a0 = s0, b0 = s0 + 65536;
          const uint32_t slot = static_cast<uint32_t>(s) & 1u;
          const uint32_t a_st = static_cast<uint32_t>(make_smem_desc_sw32(a0 + slot * 32768u));
          const uint32_t b_st = static_cast<uint32_t>(make_smem_desc(b0 + slot * 16384u, 128, 256));
#pragma unroll
          for (int i = 0; i < 8; ++i)
            mma_bf16_lo(tbase + static_cast<uint32_t>(i & 1) * 128u,
                        a_st + static_cast<uint32_t>(i >> 1) * 512u + static_cast<uint32_t>(i & 1) * 256u, a_hi,
                        b_st + static_cast<uint32_t>(i >> 1) * 256u, b_hi, idesc, 1u);
        } else if (c.unroll == 2) {
          // conv_fwd fast path shape: kk < kc (runtime), taps unrolled to 16 with a runtime break, MB = 2
          const uint32_t ak0 = c.alo0 + (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4);
          const uint32_t bk0 = c.blo0 + (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4);
          for (int kk = 0; kk < c.kc; ++kk) {
            const uint32_t ak = ak0 + 2u * static_cast<uint32_t>(kk * c.a_px);
            const uint32_t bk = bk0 + ((static_cast<uint32_t>(kk * c.nt) * c.w_tap) >> 4);
            const bool first_k = s == 0 && kk == 0;
#pragma unroll
            for (int tp = 0; tp < 16; ++tp) {
              if (tp >= c.nt) break;
#pragma unroll
              for (int mb = 0; mb < 2; ++mb)
                mma_bf16_lo(c.tmem0 + static_cast<uint32_t>(mb * 128), ak + sh[tp] + 256u * mb, a_hi,
                            bk + static_cast<uint32_t>(tp) * (c.w_tap >> 4), b_hi, idesc, (first_k && tp == 0) ? 0u : 1u);
            }
          }
        } else if (c.unroll == 5 || c.unroll == 6) {
          // uniform-friendly: per stage one A base and one B base; per MMA at most one add of a
          // compile-time immediate (or of a loop-carried uniform value) -- no tap table
          const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4;
          const uint32_t a_st = c.alo0 + sb + static_cast<uint32_t>(s & 3) * 0u;
          const uint32_t b_st = c.blo0 + sb;
          if (c.unroll == 5) {  // 1x1: KC 4 blocks of a_px rows, MB 2, N 128 (B tap = 16 groups x 256 B)
            constexpr uint32_t kBTap = (128u / 8u) * 256u / 16u;
            uint32_t ak = a_st;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk, ak += 2u * static_cast<uint32_t>(c.a_px)) {
#pragma unroll
              for (int mb = 0; mb < 2; ++mb)
                mma_bf16_lo(static_cast<uint32_t>(mb * 128), ak + 256u * mb, a_hi, b_st + kk * kBTap, b_hi, idesc,
                            (s == 0 && kk == 0) ? 0u : 1u);
            }
          } else {  // 3x3: taps (r, s2) at r * wsub + s2 pixel rows; MB 2; N 64
            constexpr uint32_t kBTap = (64u / 8u) * 256u / 16u;
            const uint32_t row2 = 2u * 58u;  // descriptor units per pixel row of the tile (wsub 58)
            uint32_t ar = a_st;
#pragma unroll
            for (int r = 0; r < 3; ++r, ar += row2) {
#pragma unroll
              for (int s2 = 0; s2 < 3; ++s2)
#pragma unroll
                for (int mb = 0; mb < 2; ++mb)
                  mma_bf16_lo(static_cast<uint32_t>(mb * 128), ar + 2u * s2 + 256u * mb, a_hi,
                              b_st + (r * 3 + s2) * kBTap, b_hi, idesc, (s == 0 && r == 0 && s2 == 0) ? 0u : 1u);
            }
          }
        } else if (c.unroll == 3 || c.unroll == 4) {
          // compile-time trip counts: 1x1 (KC 4, NT 1) or 3x3 (KC 1, NT 9), MB 2
          const uint32_t ak0 = c.alo0 + (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4);
          const uint32_t bk0 = c.blo0 + (static_cast<uint32_t>(__cvta_generic_to_shared(smem)) >> 4);
          auto body = [&](auto kc_c, auto nt_c) {
            constexpr int KC = decltype(kc_c)::value, NT = decltype(nt_c)::value;
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
              const uint32_t ak = ak0 + 2u * static_cast<uint32_t>(kk * c.a_px);
              const uint32_t bk = bk0 + ((static_cast<uint32_t>(kk * NT) * c.w_tap) >> 4);
#pragma unroll
              for (int tp = 0; tp < NT; ++tp)
#pragma unroll
                for (int mb = 0; mb < 2; ++mb)
                  mma_bf16_lo(c.tmem0 + static_cast<uint32_t>(mb * 128), ak + sh[tp] + 256u * mb, a_hi,
                              bk + static_cast<uint32_t>(tp) * (c.w_tap >> 4), b_hi, idesc,
                              (s == 0 && kk == 0 && tp == 0) ? 0u : 1u);
            }
          };
          if (c.unroll == 3)
            body(std::integral_constant<int, 4>{}, std::integral_constant<int, 1>{});
          else
            body(std::integral_constant<int, 1>{}, std::integral_constant<int, 9>{});
        } else if (c.unroll) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            mma_bf16_lo(tb[i & 1], al[i], a_hi, bl[i], b_hi, idesc, 1u);
        } else {
          for (int i = 0; i < c.per_stage; ++i) {
            const uint32_t d = tbase + (c.dacc == 2 ? static_cast<uint32_t>(i & 1) * 128u : 0u);
            mma_bf16_lo(d, a_lo + static_cast<uint32_t>(i & 7) * static_cast<uint32_t>(c.ashift), a_hi,
                        b_lo + static_cast<uint32_t>(i & 3) * static_cast<uint32_t>(c.bshift), b_hi, idesc, 1u);
          }
        }
        if (c.ring) mma_commit(&empty[slot]);
        if (++slot == 4) {
          slot = 0;
          ph ^= 1u;
        }
      }
      mma_commit(&done);
      mbar_wait(&done, 0);
      out[blockIdx.x] = clock64() - t0;
      stop = 1;
    }
    if (!c.nosync) __syncwarp();
  } else if (warp == 2) {
    if (lane == 0 && (c.copy || c.ring)) {
      int slot = 0;
      uint32_t ph = 0;
      long long off = static_cast<long long>(blockIdx.x) * 65536;
      for (int s = 0; s < (c.ring ? c.stages : 1 << 30); ++s) {
        if (!c.ring && stop) break;
        if (c.ring) mbar_wait(&empty[slot], ph ^ 1u);
        const uint32_t bytes = c.copy ? 16384u : 0u;
        mbar_arrive_expect_tx(&full[slot], bytes);
        if (c.copy) bulk_load(smem + 65536 + slot * 16384, src + (off % (64ll << 20)), bytes, &full[slot]);
        off += 16384 * 148;
        if (!c.ring) mbar_wait(&full[slot], ph);
        if (++slot == 4) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
    __syncwarp();
  } else if (warp >= 4 && c.epi) {
    uint32_t acc = 0;
    const uint32_t q = static_cast<uint32_t>((warp % 4) * 32) << 16;
    while (!stop) {
      for (int j = 0; j < 8; ++j) {
        uint32_t r[32];
        tmem_ld32(tbase + q + 256u + static_cast<uint32_t>(j) * 32u, r);
        tmem_ld_wait();
        acc += r[lane];
      }
    }
    if (acc == 12345) out[148 + blockIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  long long* d;
  uint8_t* src;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaMalloc(&src, 64 << 20);
  cudaMemset(src, 0, 64 << 20);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  Cfg cfgs[] = {
      {128, 1024, 8, 2, 0, 0, 0, 2, 9, 0},  {128, 1024, 8, 2, 0, 0, 0, 2, 5, 0}, {64, 1024, 8, 2, 0, 0, 0, 2, 9, 0},
  };
  int k = 0;
  for (Cfg& c : cfgs) c.nosync = 2 * ((k++) & 1);
  for (Cfg& c : cfgs) {
    // descriptor low words relative to the smem window start (>>4 units), TMEM column base 0
    c.alo0 = 0x10000u;            // LBO = 16 B (unused, swizzled)
    c.blo0 = (128u >> 4) << 16 | ((c.nosync & 2 ? 65536u : 32768u) >> 4);
    c.tmem0 = 0;
    // production shapes: 1x1 (kc 4, one tap) or 3x3 (kc 1, nine taps), a_px rows per block
    c.kc = c.per_stage == 8 ? 4 : 1;
    c.nt = c.per_stage == 8 ? 1 : 9;
    c.a_px = c.per_stage == 8 ? 256 : 464;
    c.w_tap = static_cast<uint32_t>(c.N / 8) * 256u;
    probe<<<148, c.epi ? 256 : 128, 160 * 1024>>>(c, src, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc = static_cast<double>(mx) / (c.stages * c.per_stage);  // unroll 2: kc * nt * 2 MMAs = per_stage
    printf("nosync %d ", c.nosync);
    printf("N %3d per_stage %d dacc %d epi %d copy %d ring %d ashift %d unroll %d bshift %d: %6.1f cyc/MMA (floor %d)\n",
           c.N, c.per_stage, c.dacc, c.epi, c.copy, c.ring, c.ashift, c.unroll, c.bshift, cyc, c.N / 2);
  }
  return 0;
}
