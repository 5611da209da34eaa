// Probe: TMA SWIZZLE_32B K-major bf16 tile ([pixel][32B]) consumed by UMMA with
// the start address shifted by s pixels (s = 0..8) and base_offset variants.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// A: 256 px x 16 ch bf16 via TMA (SW32) ; B: 16(k) x 16(n) bf16 MN-major no-swizzle [2 ngroups][16 k][8]
__global__ void probe(const __grid_constant__ CUtensorMap map, const uint16_t* bg, int shift, int bomode, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  uint8_t* sa = smem;             // 256 px * 32B = 8KB
  uint8_t* sb = smem + 8192;      // 512B
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) reinterpret_cast<uint16_t*>(sb)[i] = bg[i];
  if (warp == 0) tmem_alloc(&tbase, 32);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&mbar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) { mbar_arrive_expect_tx(&bar, 8192); tma_load_3d(sa, &map, &bar, 0, 0, 0); }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp == 0 && elect_one()) {
    const uint32_t a = smem_u32(sa) + shift * 32;
    uint32_t bo = 0;
    if (bomode == 1) bo = (a >> 7) & 7;
    if (bomode == 2) bo = (a >> 5) & 7;
    if (bomode == 3) bo = ((a >> 7) & 1);
    uint64_t ad = desc_sw(a, 16, 256, 6 /*SW32*/, bo);
    uint64_t bd = make_smem_desc(smem_u32(sb), 128, 256);
    mma_bf16(tbase, ad, bd, make_idesc(1, 0, 1, 128, 16), 0);
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t v[16];
  tmem_ld16(tbase + ((uint32_t)((warp % 4) * 32) << 16), v);
  tmem_ld_wait();
  const int row = (warp % 4) * 32 + threadIdx.x % 32;
  for (int j = 0; j < 16; ++j) out[row * 16 + j] = __uint_as_float(v[j]);
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 32);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static uint16_t bfb(float x) { __nv_bfloat16 h = __float2bfloat16(x); uint16_t u; memcpy(&u, &h, 2); return u; }

// MN-major SW32: operand "A" with M = 128 channels (8 blocks x 16) and K = 16 pixels
// staged as 8 planes [block][pixel][32B] (TMA SW32 boxes), shifted by s pixels along K
__global__ void probe_mn(const __grid_constant__ CUtensorMap map, const uint16_t* bg, int shift, float* out, int lbo, int sbo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  uint8_t* sa = smem;              // 8 planes x 32 px x 32B = 8KB
  uint8_t* sb = smem + 8192;       // B: K=16 pixels x N=16, MN-major no-swizzle [2 ng][16 k][8]
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) reinterpret_cast<uint16_t*>(sb)[i] = bg[i];
  if (warp == 0) tmem_alloc(&tbase, 32);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&mbar, 1); fence_barrier_init(); }
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (threadIdx.x == 0) { mbar_arrive_expect_tx(&bar, 8192); tma_load_3d(sa, &map, &bar, 0, 0, 0); }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp == 0 && elect_one()) {
    const uint32_t a = smem_u32(sa) + shift * 32;
    uint64_t ad = desc_sw(a, lbo, sbo, 6, 0);
    uint64_t bd = make_smem_desc(smem_u32(sb), 128, 256);
    mma_bf16(tbase, ad, bd, make_idesc(1, 1, 1, 128, 16), 0);
    mma_commit(&mbar);
  }
  __syncwarp();
  mbar_wait(&mbar, 0);
  tc_fence_after();
  uint32_t v[16];
  tmem_ld16(tbase + ((uint32_t)((warp % 4) * 32) << 16), v);
  tmem_ld_wait();
  const int row = (warp % 4) * 32 + threadIdx.x % 32;
  for (int j = 0; j < 16; ++j) out[row * 16 + j] = __uint_as_float(v[j]);
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 32);
}

int main() {
  std::vector<float> A(256 * 16), B(16 * 16);
  for (int p = 0; p < 256; ++p) for (int c = 0; c < 16; ++c) A[p * 16 + c] = (float)(((p * 5 + c * 3) % 11) - 5);
  for (int k = 0; k < 16; ++k) for (int n = 0; n < 16; ++n) B[k * 16 + n] = (float)(((k * 7 + n) % 5) - 2);
  std::vector<uint16_t> ag(256 * 16), bgh(256);
  for (int i = 0; i < 256 * 16; ++i) ag[i] = bfb(A[i]);
  for (int k = 0; k < 16; ++k) for (int n = 0; n < 16; ++n) bgh[(n / 8) * 128 + k * 8 + n % 8] = bfb(B[k * 16 + n]);
  void *ad, *bd; float* od;
  cudaMalloc(&ad, ag.size() * 2); cudaMalloc(&bd, 512); cudaMalloc(&od, 128 * 16 * 4);
  cudaMemcpy(ad, ag.data(), ag.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(bd, bgh.data(), 512, cudaMemcpyHostToDevice);
  Enc enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {16, 256, 1}; cuuint64_t st[2] = {32, 8192};
  cuuint32_t box[3] = {16, 256, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ad, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (int bomode = 0; bomode < 4; ++bomode) {
    int ok = 0;
    for (int s = 0; s <= 8; ++s) {
      probe<<<1, 128, 16384>>>(map, (const uint16_t*)bd, s, bomode, od);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err\n"); return 1; }
      std::vector<float> D(128 * 16);
      cudaMemcpy(D.data(), od, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int m = 0; m < 128; ++m) for (int n = 0; n < 16; ++n) {
        double ref = 0; for (int k = 0; k < 16; ++k) ref += (double)A[(m + s) * 16 + k] * B[k * 16 + n];
        err = fmax(err, fabs(ref - D[m * 16 + n]));
      }
      ok += err < 1e-3;
      printf("bomode %d shift %d err %g\n", bomode, s, err);
    }
    printf("bomode %d: %d/9 shifts correct\n", bomode, ok);
  }
  {
    // global X[plane 8][pixel 32][16 ch]; D[c][n] = sum_{p<16} X[c/16][p+s][c%16] * B[p][n]
    std::vector<float> X(8 * 32 * 16);
    for (size_t i = 0; i < X.size(); ++i) X[i] = (float)(((i * 7) % 13) - 6);
    std::vector<uint16_t> xg(X.size());
    for (size_t i = 0; i < X.size(); ++i) xg[i] = bfb(X[i]);
    void* xd; cudaMalloc(&xd, xg.size() * 2);
    cudaMemcpy(xd, xg.data(), xg.size() * 2, cudaMemcpyHostToDevice);
    CUtensorMap m2;
    cuuint64_t d2[3] = {16, 32, 8}; cuuint64_t s2[2] = {32, 32 * 32};
    cuuint32_t b2[3] = {16, 32, 8};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, xd, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaFuncSetAttribute(probe_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    const int cand[6][2] = {{1024, 256}, {256, 1024}, {16, 1024}, {1024, 16}, {512, 256}, {256, 512}};
    for (int ci = 0; ci < 6; ++ci) {
    int ok = 0;
    for (int s = 0; s <= 8; ++s) {
      probe_mn<<<1, 128, 16384>>>(m2, (const uint16_t*)bd, s, od, cand[ci][0], cand[ci][1]);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("err mn\n"); return 1; }
      std::vector<float> D(128 * 16);
      cudaMemcpy(D.data(), od, D.size() * 4, cudaMemcpyDeviceToHost);
      double err = 0;
      for (int c = 0; c < 128; ++c) for (int n = 0; n < 16; ++n) {
        double ref = 0; for (int k = 0; k < 16; ++k) ref += (double)X[((c / 16) * 32 + k + s) * 16 + c % 16] * B[k * 16 + n];
        err = fmax(err, fabs(ref - D[c * 16 + n]));
      }
      ok += err < 1e-3;
    }
    printf("MN-major SW32 lbo %d sbo %d: %d/9 shifts correct\n", cand[ci][0], cand[ci][1], ok);
    }
  }
  return 0;
}
