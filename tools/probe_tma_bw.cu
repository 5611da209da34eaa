// Probe: HBM read throughput of TMA tile loads with the FWD kernel's box shapes
// (fp32 NCHW16c planes, 64 B pixel rows, SWIZZLE_64B) as a function of ring depth.
// One thread per CTA issues loads into an R-slot ring and re-arms a slot as soon
// as it lands (no consumer work), 148 CTAs, L2 flushed before each run.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

constexpr int kPlanes = 512, kHW = 3136, kCb = 16;  // 32 images x 16 channel blocks x 56x56

// TMA tile stores of 2 KB slabs {16 fp32, 32 px, 1 plane} from a smem ring (the lean epilogue's pattern)
__global__ void writer(const __grid_constant__ CUtensorMap map, int n_slabs_per_cta, int planes_total) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < n_slabs_per_cta; ++i) {
    const int slab = blockIdx.x + i * gridDim.x;
    const int plane = slab % planes_total, v = (slab / planes_total) * 32;
    if (i >= 4) bulk_wait_group_read<3>();
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(&map)),
                 "r"(smem_u32(smem + (i % 4) * 2048)), "r"(0), "r"(v), "r"(plane)
                 : "memory");
    bulk_commit_group();
  }
  bulk_wait_group0();
}

// plain vectorised stores for comparison
__global__ void stg_writer(float4* __restrict__ x, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    x[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

// plain vectorised loads for comparison
__global__ void ldg_reader(const float4* __restrict__ x, size_t n, float* out) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(x + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.f) out[0] = acc;
}

__device__ long long g_trace[2 * 64];
__global__ void reader(const __grid_constant__ CUtensorMap map, int ring, int box_px, int box_planes, int n_tiles,
                       int dummy) {
  const long long t0 = clock64();
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  const uint32_t slot = box_px * box_planes * 64;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
  const int tiles_per_img = (kHW + box_px - 1) / box_px;
  const int stages_per_tile = kCb / box_planes;
  int issued = 0, done = 0;
  auto issue = [&](int g) {
    const int t = blockIdx.x + (g / stages_per_tile) * gridDim.x;
    const int it = g % stages_per_tile;
    const int n = t / tiles_per_img, v0 = (t % tiles_per_img) * box_px;
    const int s = g % ring;
    mbar_arrive_expect_tx(&full[s], slot);
    tma_load_3d(smem + s * slot, &map, &full[s], 0, v0, n * kCb + it * box_planes);
    if (blockIdx.x == 0 && g < 64) g_trace[2 * g] = clock64() - t0;
  };
  const int my_tiles = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int total = my_tiles * stages_per_tile;
  for (; issued < ring && issued < total; ++issued) issue(issued);
  for (; done < total; ++done) {
    mbar_wait(&full[done % ring], (done / ring) & 1);
    if (blockIdx.x == 0 && done < 64) g_trace[2 * done + 1] = clock64() - t0;
    if (issued < total) issue(issued++);
  }
  }
  __syncthreads();  // the other warps of a 512-thread CTA idle here (FWD-kernel shape)
  (void)dummy;
}

// wide-row variant: box {W floats, rows, 4 planes}; tile = 128 pixels = 128*16/W rows
__global__ void reader_wide(const __grid_constant__ CUtensorMap map, int ring, int rows, int n_tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  const uint32_t slot = 32768;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const int tiles_per_img = (kHW + 127) / 128;
  const int stages_per_tile = kCb / 4;
  auto issue = [&](int g) {
    const int t = blockIdx.x + (g / stages_per_tile) * gridDim.x;
    const int it = g % stages_per_tile;
    const int n = t / tiles_per_img, r0 = (t % tiles_per_img) * rows;
    const int s = g % ring;
    mbar_arrive_expect_tx(&full[s], slot);
    tma_load_3d(smem + s * slot, &map, &full[s], 0, r0, n * kCb + it * 4);
  };
  const int my_tiles = (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
  const int total = my_tiles * stages_per_tile;
  int issued = 0;
  for (; issued < ring && issued < total; ++issued) issue(issued);
  for (int done = 0; done < total; ++done) {
    mbar_wait(&full[done % ring], (done / ring) & 1);
    if (issued < total) issue(issued++);
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = (size_t)kPlanes * kHW * 64;
  void* x;
  cudaMalloc(&x, bytes);
  cudaMemset(x, 0, bytes);
  if (getenv("RANDOM_X")) {  // non-zero payload (rules out any zero-data shortcut)
    std::vector<float> h(bytes / 4);
    uint32_t st = 12345u;
    for (auto& v : h) {
      st = st * 1664525u + 1013904223u;
      v = static_cast<float>(st >> 8) * (1.0f / 16777216.0f) - 0.5f;
    }
    cudaMemcpy(x, h.data(), bytes, cudaMemcpyHostToDevice);
  }
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  Enc enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  {
    float* o;
    cudaMalloc(&o, 4);
    for (int clean = 0; clean < 2; ++clean)
    for (int blocks : {148 * 4, 148 * 8}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        // clean = 1: read the flush buffer back so L2 holds clean lines (write-backs happen here, untimed)
        if (clean) ldg_reader<<<148 * 8, 512>>>((const float4*)flush, (256 << 20) / 16, o);
        cudaEventRecord(a);
        ldg_reader<<<blocks, 512>>>((const float4*)x, bytes / 16, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("ldg reader %d blocks, %s flush: %.1f us %.0f GB/s\n", blocks, clean ? "write+read" : "write", best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
  }
  {
    // write bandwidth: TMA slab stores vs plain stores, 103 MB
    CUtensorMap wmap;
    cuuint64_t dims[3] = {16, (cuuint64_t)kHW, (cuuint64_t)kPlanes};
    cuuint64_t st[2] = {64, (cuuint64_t)kHW * 64};
    cuuint32_t box[3] = {16, 32, 1}, es[3] = {1, 1, 1};
    enc(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int slabs = kPlanes * (kHW / 32);
    cudaFuncSetAttribute(writer, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    for (int ctas : {148, 296, 592}) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        ldg_reader<<<148 * 8, 512>>>((const float4*)flush, (256 << 20) / 16, (float*)flush);
        cudaEventRecord(a);
        writer<<<ctas, 32, 8192>>>(wmap, slabs / ctas, kPlanes);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("TMA slab store %d ctas: %.1f us  %.0f GB/s %s\n", ctas, best * 1e3,
             (double)slabs / ctas * ctas * 2048 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(flush, rep, 256 << 20);
      cudaEventRecord(a);
      stg_writer<<<148 * 8, 512>>>((float4*)x, bytes / 16);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("plain stores: %.1f us %.0f GB/s\n", best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  {
    // same bytes per stage, but described with wide rows: a plane's pixels are
    // contiguous, so {256 floats (16 px), hw/16, planes} boxes {W, 128*16/W, 4}
    cudaFuncSetAttribute(reader_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int wide : {256, 128, 64, 32, 16}) {
      CUtensorMap map;
      cuuint64_t dims[3] = {(cuuint64_t)wide, (cuuint64_t)kHW * 16 / wide, (cuuint64_t)kPlanes};
      cuuint64_t st[2] = {(cuuint64_t)wide * 4, (cuuint64_t)kHW * 64};
      cuuint32_t box[3] = {(cuuint32_t)wide, (cuuint32_t)(128 * 16 / wide), 4}, es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int n_tiles = 32 * ((kHW + 127) / 128);
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        ldg_reader<<<148 * 8, 512>>>((const float4*)flush, (256 << 20) / 16, (float*)flush + 1);
        cudaEventRecord(a);
        reader_wide<<<148, 32, 3 * 32768>>>(map, 3, 128 * 16 / wide, n_tiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("wide rows %d B (enc %d) box {%d,%d,4} ring 3: %.1f us %.0f GB/s %s\n", wide * 4, (int)r, wide,
             128 * 16 / wide, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  const int shapes[][2] = {{128, 2}, {128, 4}};
  float* o2;
  cudaMalloc(&o2, 4);
  for (int big = 0; big < 2; ++big)
  for (int clean = 1; clean < 2; ++clean)
  for (int ctas_per_sm : {1})
  for (auto& sh : shapes)
    for (int promo = 0; promo < 1; ++promo)
      for (int ring : {6, 3}) {
        const int box_px = sh[0], box_planes = sh[1];
        if ((size_t)ring * box_px * box_planes * 64 * ctas_per_sm > 200 * 1024) continue;
        CUtensorMap map;
        cuuint64_t dims[3] = {16, (cuuint64_t)kHW, (cuuint64_t)kPlanes};
        cuuint64_t st[2] = {64, (cuuint64_t)kHW * 64};
        cuuint32_t box[3] = {16, (cuuint32_t)box_px, (cuuint32_t)box_planes}, es[3] = {1, 1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_64B, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int n_tiles = 32 * ((kHW + box_px - 1) / box_px);
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaMemset(flush, rep, 256 << 20);
          if (clean) ldg_reader<<<148 * 8, 512>>>((const float4*)flush, (256 << 20) / 16, o2);
          cudaEventRecord(a);
          if (big)
            reader<<<148, 512, 208 * 1024>>>(map, ring, box_px, box_planes, n_tiles, 0);
          else
            reader<<<148 * ctas_per_sm, 32, ring * box_px * box_planes * 64>>>(map, ring, box_px, box_planes, n_tiles, 0);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        const cudaError_t e = cudaGetLastError();
        printf("%s%s flush ctas/SM %d box {16,%d,%d} ring %d (%zu KB in flight): %.1f us  %.0f GB/s %s\n",
               big ? "[512 thr, 208 KB] " : "", clean ? "write+read" : "write", ctas_per_sm, box_px, box_planes, ring,
               (size_t)ring * box_px * box_planes * 64 / 1024, best * 1e3, bytes / (best * 1e-3) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  {
    long long tr[128];
    cudaMemcpyFromSymbol(tr, g_trace, sizeof(tr));
    printf("last reader run, CTA 0: stage issue -> landed (cycles)\n");
    for (int i = 0; i < 24; ++i) printf("%d %lld %lld (lat %lld)\n", i, tr[2 * i], tr[2 * i + 1], tr[2 * i + 1] - tr[2 * i]);
  }
  return 0;
}
