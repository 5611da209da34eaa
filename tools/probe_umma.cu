// Standalone probe of the sm_100a building blocks the conv kernels rely on:
// UMMA no-swizzle descriptors (K-major and MN-major, bf16 and tf32), the tf32
// operand rounding rule, and 5-D TMA tile loads with out-of-bounds zero fill.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe_umma probe_umma.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"

using namespace dconv_sm100;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

// mode 0: bf16 A K-major [2][128][8], B MN-major [8 ngroups][16 k][8]
// mode 1: tf32 A K-major [4][128][4], B MN-major [16 ngroups][16 k][4]
// mode 2: bf16 A MN-major [16 mgroups][16 k][8], B MN-major as mode 0
// mode 3: bf16 A K-major, B K-major [2 chunks][64 n][8]
__global__ void probe_mma(int mode, const void* a_g, const void* b_g, int a_bytes, int b_bytes, float* d_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  uint8_t* sa = smem;
  uint8_t* sb = smem + 16384;
  for (int i = threadIdx.x; i < a_bytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sa)[i] = reinterpret_cast<const uint32_t*>(a_g)[i];
  for (int i = threadIdx.x; i < b_bytes / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sb)[i] = reinterpret_cast<const uint32_t*>(b_g)[i];
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc(&tmem_base, 64);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
      if (mode == 0) {
        uint64_t ad = make_smem_desc(a0, 128 * 16, 128);
        uint64_t bd = make_smem_desc(b0, 128, 256);
        mma_bf16(tbase, ad, bd, make_idesc(1, 0, 1, 128, 64), 0);
      } else if (mode == 1) {
        for (int ks = 0; ks < 2; ++ks) {
          uint64_t ad = make_smem_desc(a0 + ks * 2 * 128 * 16, 128 * 16, 128);
          uint64_t bd = make_smem_desc(b0 + ks * 128, 128, 256);
          mma_tf32(tbase, ad, bd, make_idesc(2, 0, 1, 128, 64), ks);
        }
      } else if (mode == 2) {
        uint64_t ad = make_smem_desc(a0, 128, 256);
        uint64_t bd = make_smem_desc(b0, 128, 256);
        mma_bf16(tbase, ad, bd, make_idesc(1, 1, 1, 128, 64), 0);
      } else if (mode == 3) {
        uint64_t ad = make_smem_desc(a0, 128 * 16, 128);
        uint64_t bd = make_smem_desc(b0, 64 * 16, 128);
        mma_bf16(tbase, ad, bd, make_idesc(1, 0, 0, 128, 64), 0);
      } else if (mode == 4) {
        for (int ks = 0; ks < 2; ++ks) {
          uint64_t ad = make_smem_desc(a0 + ks * 2 * 128 * 16, 128 * 16, 128);
          uint64_t bd = make_smem_desc(b0 + ks * 2 * 64 * 16, 64 * 16, 128);
          mma_tf32(tbase, ad, bd, make_idesc(2, 0, 0, 128, 64), ks);
        }
      } else if (mode == 5) {
        for (int ks = 0; ks < 2; ++ks) {
          uint64_t ad = make_smem_desc(a0 + ks * 2 * 128 * 16, 128 * 16, 128);
          uint64_t bd = make_smem_desc(b0 + ks * 2 * 64 * 16, 64 * 16, 128);
          uint32_t idesc = make_idesc(2, 0, 0, 128, 64);
          uint32_t acc = ks;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}"
                       :: "r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(0), "r"(0), "r"(0), "r"(0) : "memory");
        }
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int row = (warp % 4) * 32 + threadIdx.x % 32;
  for (int cb = 0; cb < 4; ++cb) {
    uint32_t v[16];
    tmem_ld16(tbase + ((uint32_t)((warp % 4) * 32) << 16) + cb * 16, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) d_out[row * 64 + cb * 16 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 64);
}

__global__ void probe_tma(const __grid_constant__ CUtensorMap map, uint16_t* out, int bytes, int c1, int c2,
                          int c4) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_5d(smem, &map, &bar, 0, c1, c2, 0, c4);
  }
  // bounded wait: report timeout instead of hanging
  uint32_t done = 0;
  for (int it = 0; it < 2000000 && !done; ++it) {
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  }
  if (!done) { if (threadIdx.x == 0) out[0] = 0xDEAD; return; }
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(smem)[i];
}

static float bf(float x) { return __bfloat162float(__float2bfloat16(x)); }
static uint16_t bfbits(float x) {
  __nv_bfloat16 h = __float2bfloat16(x);
  uint16_t u;
  memcpy(&u, &h, 2);
  return u;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int M = 128, N = 64, K = 16;
  std::vector<float> A(M * K), B(K * N);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) A[m * K + k] = (float)(((m * 7 + k * 3) % 17) - 8) * 0.25f;
  for (int k = 0; k < K; ++k)
    for (int n = 0; n < N; ++n) B[k * N + n] = (float)(((k * 5 + n * 11) % 13) - 6) * 0.5f;
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) ref[m * N + n] += (double)A[m * K + k] * B[k * N + n];

  void *a_d, *b_d;
  float* d_d;
  CK(cudaMalloc(&a_d, 65536));
  CK(cudaMalloc(&b_d, 65536));
  CK(cudaMalloc(&d_d, M * N * 4));
  CK(cudaFuncSetAttribute(probe_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  int fails = 0;
  for (int mode = 0; mode < 6; ++mode) {
    std::vector<uint8_t> abuf(16384, 0), bbuf(16384, 0);
    int ab = 0, bb = 0;
    if (mode == 4 || mode == 5) {
      float* a = (float*)abuf.data();
      for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) a[(k / 4) * M * 4 + m * 4 + k % 4] = A[m * K + k];
      ab = 4 * M * 16;
    } else if (mode == 0 || mode == 3) {
      uint16_t* a = (uint16_t*)abuf.data();
      for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) a[(k / 8) * M * 8 + m * 8 + k % 8] = bfbits(A[m * K + k]);
      ab = 2 * M * 16;
    } else if (mode == 1) {
      float* a = (float*)abuf.data();
      for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) a[(k / 4) * M * 4 + m * 4 + k % 4] = A[m * K + k];
      ab = 4 * M * 16;
    } else {
      uint16_t* a = (uint16_t*)abuf.data();
      for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) a[(m / 8) * 16 * 8 + k * 8 + m % 8] = bfbits(A[m * K + k]);
      ab = 2 * M * 16;
    }
    if (mode == 4 || mode == 5) {
      float* b = (float*)bbuf.data();
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) b[(k / 4) * N * 4 + n * 4 + k % 4] = B[k * N + n];
      bb = 4 * N * 16;
    } else if (mode == 0 || mode == 2) {
      uint16_t* b = (uint16_t*)bbuf.data();
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) b[(n / 8) * 16 * 8 + k * 8 + n % 8] = bfbits(B[k * N + n]);
      bb = 2 * N * 16;
    } else if (mode == 1) {
      float* b = (float*)bbuf.data();
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) b[(n / 4) * 16 * 4 + k * 4 + n % 4] = B[k * N + n];
      bb = 4 * N * 16;
    } else {
      uint16_t* b = (uint16_t*)bbuf.data();
      for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) b[(k / 8) * N * 8 + n * 8 + k % 8] = bfbits(B[k * N + n]);
      bb = 2 * N * 16;
    }
    CK(cudaMemcpy(a_d, abuf.data(), 16384, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b_d, bbuf.data(), 16384, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_d, 0, M * N * 4));
    probe_mma<<<1, 128, 65536>>>(mode, a_d, b_d, ab, bb, d_d);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(M * N);
    CK(cudaMemcpy(D.data(), d_d, M * N * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < M * N; ++i) maxerr = fmax(maxerr, fabs(D[i] - ref[i]));
    printf("mma mode %d: max abs err %.3g  D[0]=%g ref=%g D[77]=%g ref=%g -> %s\n", mode, maxerr, D[0], ref[0],
           D[77], ref[77], maxerr < 1e-3 ? "PASS" : "FAIL");
    fails += maxerr >= 1e-3;
  }

  // tf32 operand rounding: A = 1 + 2^-12 (dropped by tf32), B = 1; K=16 -> sum 16*(1+2^-12) exact
  {
    std::vector<uint8_t> abuf(16384, 0), bbuf(16384, 0);
    float* a = (float*)abuf.data();
    float* b = (float*)bbuf.data();
    const float av = 1.0f + ldexpf(1.0f, -12) + ldexpf(1.0f, -13);  // bits below tf32 mantissa: 0b11 pattern
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) a[(k / 4) * M * 4 + m * 4 + k % 4] = av;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) b[(n / 4) * 16 * 4 + k * 4 + n % 4] = 1.0f;
    CK(cudaMemcpy(a_d, abuf.data(), 16384, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(b_d, bbuf.data(), 16384, cudaMemcpyHostToDevice));
    probe_mma<<<1, 128, 65536>>>(1, a_d, b_d, 4 * M * 16, 4 * N * 16, d_d);
    CK(cudaDeviceSynchronize());
    float d0;
    CK(cudaMemcpy(&d0, d_d, 4, cudaMemcpyDeviceToHost));
    // tf32 keeps 10 mantissa bits: av truncates to 1.0, rounds to 1 + 2^-10
    printf("tf32 rounding probe: D=%.9g  trunc->%.9g round->%.9g exact->%.9g  => %s\n", d0, 16.0,
           16.0 * (1.0 + ldexp(1.0, -10)), 16.0 * av,
           d0 == 16.0f ? "TRUNCATE" : (fabs(d0 - 16.0 * (1.0 + ldexp(1.0, -10))) < 1e-6 ? "ROUND" : "OTHER"));
  }

  // TMA 5-D: tensor {8 elems, W, H, 2 chunks, planes}, box {8, Wb, Hb, 2, 1}, start (0,-1,-1,0,plane)
  {
    const int W = 5, H = 4, P = 3, Wb = 7, Hb = 6;
    std::vector<uint16_t> g(P * H * W * 16);
    for (size_t i = 0; i < g.size(); ++i) g[i] = (uint16_t)(i + 1);
    void* gd;
    uint16_t* od;
    CK(cudaMalloc(&gd, g.size() * 2));
    CK(cudaMalloc(&od, 65536));
    CK(cudaMemcpy(gd, g.data(), g.size() * 2, cudaMemcpyHostToDevice));
    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, 2, (cuuint64_t)P};
    cuuint64_t strides[4] = {32, (cuuint64_t)W * 32, 16, (cuuint64_t)H * W * 32};
    cuuint32_t box[5] = {8, (cuuint32_t)Wb, (cuuint32_t)Hb, 2, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, gd, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode result %d\n", (int)r);
    const int bytes = 2 * Hb * Wb * 16;
    CK(cudaFuncSetAttribute(probe_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    probe_tma<<<1, 128, 65536>>>(map, od, bytes, -1, -1, 1);
    CK(cudaDeviceSynchronize());
    std::vector<uint16_t> o(bytes / 2);
    CK(cudaMemcpy(o.data(), od, bytes, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int ch = 0; ch < 2; ++ch)
      for (int y = 0; y < Hb; ++y)
        for (int x = 0; x < Wb; ++x)
          for (int e = 0; e < 8; ++e) {
            const int gy = y - 1, gx = x - 1;
            uint16_t expect = 0;
            if (gy >= 0 && gy < H && gx >= 0 && gx < W) expect = g[((1 * H + gy) * W + gx) * 16 + ch * 8 + e];
            if (o[((ch * Hb + y) * Wb + x) * 8 + e] != expect) ++bad;
          }
    printf("tma 5d oob probe: %d mismatches -> %s\n", bad, bad ? "FAIL" : "PASS");
    fails += bad != 0;
  }
  // TMA elementStrides=2 on W and H: box {8, 2*Wb, 2*Hb, 2, 1}; expect Wb x Hb pixels at stride 2
  {
    const int W = 9, H = 8, P = 2, Wb = 5, Hb = 4;
    std::vector<uint16_t> g(P * H * W * 16);
    for (size_t i = 0; i < g.size(); ++i) g[i] = (uint16_t)(i + 1);
    void* gd;
    uint16_t* od;
    CK(cudaMalloc(&gd, g.size() * 2));
    CK(cudaMalloc(&od, 65536));
    CK(cudaMemset(od, 0xff, 65536));
    CK(cudaMemcpy(gd, g.data(), g.size() * 2, cudaMemcpyHostToDevice));
    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    for (int variant = 0; variant < 2; ++variant) {
      CUtensorMap map;
      cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, 2, (cuuint64_t)P};
      cuuint64_t strides[4] = {32, (cuuint64_t)W * 32, 16, (cuuint64_t)H * W * 32};
      const int bw = variant == 0 ? 2 * Wb : Wb, bh = variant == 0 ? 2 * Hb : Hb;
      cuuint32_t box[5] = {8, (cuuint32_t)bw, (cuuint32_t)bh, 2, 1};
      cuuint32_t es[5] = {1, 2, 2, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, gd, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int bytes = 2 * Hb * Wb * 16;
      fflush(stdout);
      CK(cudaMemset(od, 0xff, 65536));
      probe_tma<<<1, 128, 65536>>>(map, od, bytes, 1, -1, 1);  // start col 1, row -1
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint16_t> o(bytes / 2);
      CK(cudaMemcpy(o.data(), od, bytes, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int ch = 0; ch < 2; ++ch)
        for (int y = 0; y < Hb; ++y)
          for (int x = 0; x < Wb; ++x)
            for (int e2 = 0; e2 < 8; ++e2) {
              const int gy = -1 + 2 * y, gx = 1 + 2 * x;
              uint16_t expect = 0;
              if (gy >= 0 && gy < H && gx >= 0 && gx < W) expect = g[((1 * H + gy) * W + gx) * 16 + ch * 8 + e2];
              if (o[((ch * Hb + y) * Wb + x) * 8 + e2] != expect) ++bad;
            }
      if (o[0] == 0xDEAD) printf("variant %d TIMED OUT\n", variant);
      printf("tma elementStride variant %d (box=%d,%d) encode=%d err=%s: %d mismatches\n", variant, bw, bh, (int)r,
             cudaGetErrorString(e), bad);
    }
  }
  printf("probe done, %d failures\n", fails);
  return fails ? 2 : 0;
}
