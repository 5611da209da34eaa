// Probe: L2 -> SMEM throughput of cp.async (LDGSTS, 16 B per thread) issued by
// W loader warps into a ring of R slots (completion through
// cp.async.mbarrier.arrive.noinc), vs the TMA box rate for 32 B rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_cpasync tools/probe_cpasync.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

constexpr size_t kSrcBytes = 24u << 20;

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// loader warps [0, W) fill slots of `slot` bytes; warp W consumes (waits full, arrives empty)
__global__ void reader(const uint8_t* src, int ring, int slot, int n_slots, int W) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) {
      mbar_init(&full[i], W * 32);
      mbar_init(&empty[i], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const size_t n_pos = kSrcBytes / slot;
  if (warp < W) {
    const int t = warp * 32 + lane;
    int s = 0;
    uint32_t ph = 0;
    size_t pos = (blockIdx.x * 7919) % n_pos;
    for (int g = 0; g < n_slots; ++g) {
      mbar_wait(&empty[s], ph ^ 1u);
      const uint8_t* base = src + pos * slot;
      const uint32_t dst = smem_u32(smem + s * slot);
      for (int o = t * 16; o < slot; o += W * 32 * 16) {
        // SW32 position of 16 B chunk o: bit 4 ^= bit 7
        const uint32_t so = o ^ ((o >> 3) & 16);
        cp16(dst + so, base + o);
      }
      cp_arrive(&full[s]);
      pos += 13;
      if (pos >= n_pos) pos -= n_pos;
      if (++s == ring) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == W && lane == 0) {
    int s = 0;
    uint32_t ph = 0;
    for (int g = 0; g < n_slots; ++g) {
      mbar_wait(&full[s], ph);
      mbar_arrive(&empty[s]);
      if (++s == ring) {
        s = 0;
        ph ^= 1;
      }
    }
  }
}

int main() {
  uint8_t* x;
  cudaMalloc(&x, kSrcBytes);
  cudaMemset(x, 1, kSrcBytes);
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n_slots = 1200;
  for (int W : {1, 2, 4, 8})
    for (int slot : {8192, 16384, 32768})
      for (int ring : {4, 6}) {
        if (ring * slot > 196 * 1024) continue;
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          reader<<<148, (W + 1) * 32, ring * slot>>>(x, ring, slot, n_slots, W);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        const double gbs = 148.0 * n_slots * slot / (best * 1e-3) / 1e9;
        printf("cp.async warps %d slot %5d ring %d: %7.1f us %6.0f GB/s %5.1f B/clk/SM %s\n", W, slot, ring,
               best * 1e3, gbs, gbs / 148 / 1.965, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
