// Probe: pipeline signalling latencies on one SM (cycles, clock64), the numbers a
// producer / MMA-issuer ring is built on:
//   1. tcgen05.commit -> mbarrier phase seen by the committing thread (no MMA before it)
//   2. same, after one 128x256x16 bf16 MMA
//   3. same, after eight back-to-back MMAs
//   4. mbarrier.arrive by warp 0 -> phase seen by a waiting warp 1 (round trip: 1 -> 0 -> 1)
//   5. ring ping-pong: producer warp (wait empty, arrive full) / consumer warp (wait full,
//      tcgen05.commit empty, no MMAs), S slots, cycles per iteration
//   6. the same with plain mbarrier.arrive for "empty" instead of tcgen05.commit
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_latency probe_latency.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"

using namespace dconv_sm100;

constexpr int kIters = 256;

__global__ void __launch_bounds__(128, 1) probe(long long* out, int slots) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  __shared__ uint32_t tbase_sh;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc(&tbase_sh, 256);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    for (int i = 0; i < 16; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_sh;
  const uint32_t s0 = smem_u32(smem);
  const uint64_t ad = make_smem_desc_sw32(s0);
  const uint64_t bd = make_smem_desc(s0 + 32768, 128, 256);
  const uint32_t idesc = make_idesc(1, 0, 1, 128, 256);
  if (threadIdx.x == 0) {
    // 1-3: commit latency after 0 / 1 / 8 MMAs
    uint32_t ph = 0;
    for (int n_mma : {0, 1, 8}) {
      long long best = 1LL << 60, sum = 0;
      for (int r = 0; r < 64; ++r) {
        const long long t0 = clock64();
        for (int m = 0; m < n_mma; ++m) mma_bf16(tbase, ad, bd, idesc, 1u);
        mma_commit(&bar[0]);
        mbar_wait(&bar[0], ph);
        ph ^= 1u;
        const long long dt = clock64() - t0;
        best = dt < best ? dt : best;
        sum += dt;
      }
      out[blockIdx.x * 16 + (n_mma == 0 ? 0 : n_mma == 1 ? 1 : 2)] = sum / 64;
      out[blockIdx.x * 16 + 8 + (n_mma == 0 ? 0 : n_mma == 1 ? 1 : 2)] = best;
    }
  }
  __syncthreads();
  // 4: arrive -> wait round trip between warps 0 and 1
  if (warp < 2 && lane == 0) {
    long long t0 = clock64();
    for (int r = 0; r < kIters; ++r) {
      const uint32_t ph = r & 1;
      if (warp == 0) {
        mbar_arrive(&bar[1]);
        mbar_wait(&bar[2], ph);
      } else {
        mbar_wait(&bar[1], ph);
        mbar_arrive(&bar[2]);
      }
    }
    if (warp == 0) out[blockIdx.x * 16 + 3] = (clock64() - t0) / kIters;
  }
  __syncthreads();
  // 5 / 6: ring ping-pong, `slots` stages
  for (int mode = 0; mode < 2; ++mode) {
    if (warp < 2 && lane == 0) {
      const long long t0 = clock64();
      uint32_t ph = 0;
      int s = 0;
      for (int it = 0; it < kIters; ++it) {
        if (warp == 0) {  // producer
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_arrive(&full[s]);
        } else {  // consumer
          mbar_wait(&full[s], ph);
          tc_fence_after();
          if (mode == 0)
            mma_commit(&empty[s]);
          else
            mbar_arrive(&empty[s]);
        }
        if (++s == slots) {
          s = 0;
          ph ^= 1u;
        }
      }
      if (warp == 1) out[blockIdx.x * 16 + 4 + mode] = (clock64() - t0) / kIters;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // re-arm the ring: fresh barriers for the next mode
      for (int i = 0; i < 16; ++i) {
        mbar_init(&full[i], 1);
        mbar_init(&empty[i], 1);
      }
      fence_barrier_init();
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 16 * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int slots : {1, 2, 4, 7}) {
    for (int grid : {1, 148}) {
      cudaMemset(d, 0, 148 * 16 * sizeof(long long));
      probe<<<grid, 128, 64 * 1024>>>(d, slots);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[16];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("slots %d grid %3d: commit->seen (avg/best) 0 MMA %lld/%lld, 1 MMA %lld/%lld, 8 MMA %lld/%lld | "
             "arrive round trip %lld | ring/iter: commit %lld, arrive %lld cycles\n",
             slots, grid, h[0], h[8], h[1], h[9], h[2], h[10], h[3], h[4], h[5]);
    }
  }
  return 0;
}
