// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (written by
// tcgen05.st 32x32b: thread = row, 8 columns = 16 packed bf16) and B in smem
// (MN-major no-swizzle, the conv weight layout). Checks the TMEM A packing and
// a non-zero A column base.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// A: [128][32] bf16 (K = 32 -> two k-steps), B: [n_group 8][k 32][8] bf16 (N = 64)
__global__ void probe(const uint16_t* ag, const uint16_t* bg, int a_col, int swap, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 8 * 32 * 8; i += blockDim.x) reinterpret_cast<uint16_t*>(smem)[i] = bg[i];
  if (warp == 0) tmem_alloc(&tbase, 256);
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int row = (warp % 4) * 32 + lane;
  for (int ks = 0; ks < 2; ++ks) {
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) {
      const uint32_t e0 = ag[row * 32 + ks * 16 + 2 * c], e1 = ag[row * 32 + ks * 16 + 2 * c + 1];
      v[c] = swap ? (e1 | (e0 << 16)) : (e0 | (e1 << 16));
    }
    tmem_st8(tbase + ((uint32_t)((warp % 4) * 32) << 16) + a_col + ks * 8, v);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0 && elect_one()) {
    for (int ks = 0; ks < 2; ++ks) {
      // B k-step ks: k rows 16*ks.. ; MN-major: LBO = 8 k rows (128 B), SBO = n-group stride (32 k * 16 B)
      const uint64_t bd = make_smem_desc(smem_u32(smem) + ks * 16 * 16, 128, 32 * 16);
      mma_ts(tbase + 128, tbase + a_col + ks * 8, bd, make_idesc(1, 0, 1, 128, 64), ks ? 1u : 0u);
    }
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  for (int g = 0; g < 4; ++g) {
    uint32_t r[16];
    tmem_ld16(tbase + ((uint32_t)((warp % 4) * 32) << 16) + 128 + g * 16, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) out[row * 64 + g * 16 + j] = __uint_as_float(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 256);
}

static uint16_t bfb(float x) {
  __nv_bfloat16 h = __float2bfloat16(x);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}

int main_check() {
  std::vector<float> A(128 * 32), B(32 * 64);  // B[k][n]
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 32; ++k) A[m * 32 + k] = (float)(((m * 5 + k * 3) % 11) - 5);
  for (int k = 0; k < 32; ++k)
    for (int n = 0; n < 64; ++n) B[k * 64 + n] = (float)(((k * 7 + n * 3) % 9) - 4);
  std::vector<uint16_t> ah(A.size()), bh(8 * 32 * 8);
  for (size_t i = 0; i < A.size(); ++i) ah[i] = bfb(A[i]);
  for (int k = 0; k < 32; ++k)
    for (int n = 0; n < 64; ++n) bh[(n / 8) * 256 + k * 8 + n % 8] = bfb(B[k * 64 + n]);
  void *ad, *bd;
  float* od;
  cudaMalloc(&ad, ah.size() * 2);
  cudaMalloc(&bd, bh.size() * 2);
  cudaMalloc(&od, 128 * 64 * 4);
  cudaMemcpy(ad, ah.data(), ah.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(bd, bh.data(), bh.size() * 2, cudaMemcpyHostToDevice);
  for (int swap = 0; swap < 2; ++swap)
    for (int a_col : {0, 64, 200}) {
      probe<<<1, 128, 8192>>>((const uint16_t*)ad, (const uint16_t*)bd, a_col, swap, od);
      const cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("swap %d a_col %d: %s\n", swap, a_col, cudaGetErrorString(e));
        return 1;
      }
      std::vector<float> D(128 * 64);
      cudaMemcpy(D.data(), od, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          double ref = 0;
          for (int k = 0; k < 32; ++k) ref += (double)A[m * 32 + k] * B[k * 64 + n];
          err = fmax(err, fabs(ref - D[m * 64 + n]));
        }
      printf("swap %d a_col %d max err %g %s\n", swap, a_col, err, err < 1e-3 ? "OK" : "WRONG");
    }
  return 0;
}

// timing: n back-to-back MMAs 128 x N x 16, A from TMEM (ts = 1) or smem (ts = 0)
__global__ void timing(int ts, int N, int n, long long* out, int st_load) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint64_t bd = make_smem_desc(smem_u32(smem), 128, 16 * 16);
    const uint64_t ad = make_smem_desc(smem_u32(smem) + 65536, 128 * 16, 128);
    const uint32_t idesc = make_idesc(1, 0, 1, 128, N);
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < n; ++i) {
        if (ts)
          mma_ts(tbase, tbase + 256 + (i % 8) * 8, bd, idesc, 1u);
        else
          mma_bf16(tbase, ad, bd, idesc, 1u);
      }
      long long ti = clock64();
      out[1] = ti - t0;
      mma_commit(&mbar);
    }
    __syncwarp();
    mbar_wait(&mbar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
  } else if (st_load && warp >= 4) {
    // concurrent tcgen05.st traffic (24 columns per 128 rows per round, like the TS converters)
    uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
    for (int i = 0; i < n * st_load / 8; ++i) {
      const uint32_t col = tbase + ((uint32_t)((warp % 4) * 32) << 16) + 384 + (i % 4) * 24;
      tmem_st8(col, v);
      tmem_st8(col + 8, v);
      tmem_st8(col + 16, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main_timing() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(timing, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int st_load : {0})
  for (int n : {4, 8, 16, 64, 2000})
  for (int N : {64, 128, 256})
    for (int ts = 0; ts < 2; ++ts) {
      timing<<<1, 256, 131072>>>(ts, N, n, d, st_load);
      cudaDeviceSynchronize();
      long long cc[2];
      cudaMemcpy(cc, d, 16, cudaMemcpyDeviceToHost);
      long long c = cc[0];
      printf("n=%d N=%d ts=%d issue %.1f cyc/MMA, total %.1f cyc/MMA\n", n, N, ts, cc[1] / (double)n, c / (double)n);
      continue;
      printf("st_load %d N=%d %s: %.1f cycles per MMA (ideal %d)\n", st_load, N, ts ? "A in TMEM" : "A in smem", c / 2000.0,
             128 * N * 16 * 2 / 8192);
    }
  return 0;
}
// MMA-warp loop model: per stage wait on a (pre-completed) mbarrier, tc fence,
// issue n MMAs, commit to another barrier; stages = 64
__global__ void loopmodel(int n_mma, int nwait, int fence, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t ready[64], done[64];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tbase, 512);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 64; ++i) {
      mbar_init(&ready[i], 1);
      mbar_init(&done[i], 1);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0)
    for (int i = 0; i < 64; ++i) mbar_arrive(&ready[i]);  // all stages ready up front
  __syncthreads();
  if (warp == 0) {
    const uint64_t bd = make_smem_desc(smem_u32(smem), 128, 16 * 16);
    const uint32_t idesc = make_idesc(1, 0, 1, 128, 64);
    long long t0 = clock64();
    for (int st = 0; st < 64; ++st) {
      for (int w = 0; w < nwait; ++w) mbar_wait(&ready[st], 0);
      if (fence) tc_fence_after();
      if (elect_one()) {
        for (int i = 0; i < n_mma; ++i) mma_ts(tbase + (i & 1) * 64, tbase + 256 + (i % 8) * 8, bd, idesc, 1u);
        mma_commit(&done[st]);
      }
      __syncwarp();
    }
    long long t1 = clock64();
    mbar_wait(&done[63], 0);
    long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

int main() {
  main_check();
  main_timing();
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(loopmodel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int n_mma : {6, 24})
    for (int nwait : {0, 1, 2})
      for (int fence : {0, 1}) {
        loopmodel<<<1, 128, 65536>>>(n_mma, nwait, fence, d);
        cudaDeviceSynchronize();
        long long c[2];
        cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
        printf("loop n_mma=%d waits=%d fence=%d: issue %.0f cyc/stage, complete %.0f cyc/stage\n", n_mma, nwait,
               fence, c[0] / 64.0, c[1] / 64.0);
      }
  return 0;
}
