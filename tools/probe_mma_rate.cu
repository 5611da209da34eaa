// Probe: sustained tcgen05.mma kind::f16 issue rate (cycles per 128xNx16 MMA)
// for the operand layouts the conv kernels use, with no loads in flight:
// one CTA per SM, one elected thread issues `iters` MMAs back to back into one
// TMEM accumulator, commit + wait at the end.
//   layout 0: A K-major SWIZZLE_32B (32 B pixel rows), B K-major no-swizzle (conv weights)
//   layout 1: A K-major no-swizzle (16 B rows, LBO = plane), B as 0
//   layout 2: A K-major SWIZZLE_128B, B K-major SWIZZLE_128B (plain GEMM tiles)
//   layout 3: A in TMEM, B as 0
//   layout 4: A K-major SWIZZLE_128B, B K-major no-swizzle
//   layout 8: A and B MN-major SWIZZLE_32B (weight update: channels x pixels, LBO = block plane)
// shift = 1: the A start address moves by a pixel row per MMA (3x3 tap pattern)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_mma_rate probe_mma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"

using namespace dconv_sm100;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;  // SBO = 8 rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_ts_(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc) {
  asm volatile(
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n\t" ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc),
      "r"(idesc)
      : "memory");
}

template <int LAYOUT>
__global__ void __launch_bounds__(128, 1) probe(int N, int iters, int shift, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (warp == 0) tmem_alloc(&tbase_sh, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_sh;
  const uint32_t s0 = smem_u32(smem);
  const uint32_t a0 = s0, b0 = s0 + 64 * 1024;
  const uint32_t idesc = make_idesc(1, LAYOUT == 8 ? 1 : 0, LAYOUT == 2 ? 0 : 1, 128, static_cast<uint32_t>(N));  // conv weights: MN-major
  long long t = 0;
  if (warp == 0 && threadIdx.x == 0) {
    uint32_t alo[8], blo[8];
    uint32_t ahi = 0, bhi = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t sh = shift ? static_cast<uint32_t>(i) * 58u + (i > 4 ? 1u : 0u) : 0u;
      uint64_t ad = 0, bd;
      if (LAYOUT == 0) {
        ad = make_smem_desc_sw32(a0 + sh * 32u);
        bd = make_smem_desc(b0, 128, 256);
      } else if (LAYOUT == 1) {
        ad = make_smem_desc(a0 + sh * 16u, 128 * 64, 128);
        bd = make_smem_desc(b0, 128, 256);
      } else if (LAYOUT == 2) {
        ad = desc_sw128(a0 + sh * 128u + (i & 3) * 32u);
        bd = desc_sw128(b0 + (i & 3) * 32u);
      } else if (LAYOUT == 5) {  // conv 1x1 stage, mb = 2, kc = 4: A (kk, mb) blocks, B per kk, D per mb
        ad = make_smem_desc_sw32(a0 + static_cast<uint32_t>(i >> 1) * 8192u + static_cast<uint32_t>(i & 1) * 4096u);
        bd = make_smem_desc(b0 + static_cast<uint32_t>(i >> 1) * 4096u, 128, 256);
      } else if (LAYOUT == 8) {  // A: 8 planes of 160 px x 32 B; B: N/16 planes of 112 px x 32 B
        ad = make_smem_desc_mn_sw32(a0 + (static_cast<uint32_t>(i & 3) * 16u + (shift ? static_cast<uint32_t>(i >> 2) * 17u : 0u)) * 32u,
                                    160 * 32);
        bd = make_smem_desc_mn_sw32(b0 + static_cast<uint32_t>(i & 3) * 16u * 32u, 112 * 32);
      } else if (LAYOUT == 4) {
        ad = desc_sw128(a0 + sh * 128u + (i & 3) * 32u);
        bd = make_smem_desc(b0 + (i & 3) * 4096u, 128, 256);
      } else {
        bd = make_smem_desc(b0 + (i & 3) * 4096u, 128, 256);
      }
      alo[i] = static_cast<uint32_t>(ad);
      blo[i] = static_cast<uint32_t>(bd);
      ahi = static_cast<uint32_t>(ad >> 32);
      bhi = static_cast<uint32_t>(bd >> 32);
    }
    const long long t0 = clock64();
    if (LAYOUT == 6 || LAYOUT == 7) {
      // conv 1x1 stage (mb 2, kc 4) with the A / B bases moving through a 2-slot ring per stage;
      // LAYOUT 7: the accumulate flag of the first MMA is 0 on the first stage (runtime predicate)
      for (int it = 0; it < iters; it += 8) {
        const uint32_t slot = static_cast<uint32_t>(it >> 3) & 1u;
        const uint32_t a_st = static_cast<uint32_t>(make_smem_desc_sw32(a0 + slot * 32768u));
        const uint32_t b_st = static_cast<uint32_t>(make_smem_desc(b0 + slot * 16384u, 128, 256));
#pragma unroll
        for (int i = 0; i < 8; ++i)
          mma_bf16_lo(tbase + static_cast<uint32_t>(i & 1) * 128u,
                      a_st + static_cast<uint32_t>(i >> 1) * 512u + static_cast<uint32_t>(i & 1) * 256u, ahi,
                      b_st + static_cast<uint32_t>(i >> 1) * 256u, bhi, idesc,
                      (LAYOUT == 7 && it == 0 && i < 2) ? 0u : 1u);
      }
    }
    for (int it = 0; it < ((LAYOUT == 6 || LAYOUT == 7) ? 0 : iters); it += 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (LAYOUT == 3)
          mma_ts_(tbase, tbase + 256u + (i & 1) * 8u, (static_cast<uint64_t>(bhi) << 32) | blo[i], idesc);
        else if (LAYOUT == 5)
          mma_bf16_lo(tbase + static_cast<uint32_t>(i & 1) * 128u, alo[i], ahi, blo[i], bhi, idesc, 1u);
        else
          mma_bf16_lo(tbase, alo[i], ahi, blo[i], bhi, idesc, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    t = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int L>
void run(int N, int iters, int shift, int grid, long long* d) {
  cudaFuncSetAttribute(probe<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  probe<L><<<grid, 128, 160 * 1024>>>(N, iters, shift, d);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const char* names[] = {"A sw32 / B nosw", "A nosw16 / B nosw", "A sw128 / B sw128", "A tmem / B nosw",
                         "A sw128 / B nosw", "conv 1x1 mb2 kc4", "1x1 ring", "1x1 ring acc0", "upd A/B mn sw32"};
  const int l0 = argc > 2 ? atoi(argv[2]) : 5, l1 = argc > 3 ? atoi(argv[3]) : 8;
  for (int layout = l0; layout <= l1; ++layout)
    for (int shift = 0; shift < 2; ++shift) {
      if (layout == 3 && shift) continue;
      for (int N : {64, 128, 256}) {
        for (int grid : {1, 148}) {
          if (layout == 0) run<0>(N, iters, shift, grid, d);
          if (layout == 1) run<1>(N, iters, shift, grid, d);
          if (layout == 2) run<2>(N, iters, shift, grid, d);
          if (layout == 3) run<3>(N, iters, shift, grid, d);
          if (layout == 4) run<4>(N, iters, shift, grid, d);
          if (layout == 5) run<5>(N, iters, shift, grid, d);
          if (layout == 6) run<6>(N, iters, shift, grid, d);
          if (layout == 7) run<7>(N, iters, shift, grid, d);
          if (layout == 8) run<8>(N, iters, shift, grid, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          long long h[148];
          cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          long long mx = 0;
          for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
          const double cyc = static_cast<double>(mx) / iters;
          printf("%-20s shift %d N %3d grid %3d: %6.1f cyc/MMA (floor %d) -> %.0f%% of floor rate\n", names[layout],
                 shift, N, grid, cyc, N / 2, 100.0 * (N / 2) / cyc);
        }
      }
    }
  return 0;
}
