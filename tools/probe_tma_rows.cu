// Probe: L2 -> SMEM throughput of TMA tile loads and 1-D bulk copies from an
// L2-resident 24 MB source vs box size, ring depth and the number of issuing
// warps (each with its own ring). 148 CTAs, no consumer work.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probe_tma_rows tools/probe_tma_rows.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

constexpr size_t kSrcBytes = 24u << 20;

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ int g_same;
// mode 0: tensor box {inner, rows}; mode 1: 1-D bulk copy of box_bytes. `prod` warps issue, each its own ring.
__global__ void reader(const __grid_constant__ CUtensorMap map, const uint8_t* src, int mode, int ring, int box_bytes,
                       int box_rows, int n_pos, int n_boxes, int prod) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[4][16];
  const int w = threadIdx.x / 32;
  if (threadIdx.x % 32 == 0 && w < prod) {
    for (int i = 0; i < ring; ++i) mbar_init(&full[w][i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x % 32 != 0 || w >= prod) return;
  uint8_t* base = smem + w * ring * box_bytes;
  int pos = g_same ? (w * 131) % n_pos : (blockIdx.x * 7919 + w * 131) % n_pos;
  int s_issue = 0;
  auto issue = [&]() {
    mbar_arrive_expect_tx(&full[w][s_issue], box_bytes);
    if (mode == 0)
      tma2d(base + s_issue * box_bytes, &map, &full[w][s_issue], 0, pos * box_rows);
    else
      bulk_load(base + s_issue * box_bytes, src + static_cast<size_t>(pos) * box_bytes, box_bytes, &full[w][s_issue]);
    pos += 13;
    if (pos >= n_pos) pos -= n_pos;
    if (++s_issue == ring) s_issue = 0;
  };
  const int my = n_boxes / prod;
  int issued = 0;
  for (; issued < ring && issued < my; ++issued) issue();
  int s = 0;
  uint32_t ph = 0;
  for (int done = 0; done < my; ++done) {
    mbar_wait(&full[w][s], ph);
    if (++s == ring) {
      s = 0;
      ph ^= 1;
    }
    if (issued < my) {
      issue();
      ++issued;
    }
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  uint8_t* x;
  cudaMalloc(&x, kSrcBytes);
  cudaMemset(x, 1, kSrcBytes);
  Enc enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int n_boxes = 2400;
  for (int same : {0, 1})
  for (int inner : {32, 128, 0}) {
    cudaMemcpyToSymbol(g_same, &same, 4);
    for (int box_bytes : {8192, 32768}) {
      const int rows = inner ? box_bytes / inner : 0;
      if (inner && rows > 256) continue;
      CUtensorMap map;
      const int mode = inner ? 0 : 1;
      if (inner) {
        const cuuint64_t rows_total = kSrcBytes / inner;
        cuuint64_t dims[2] = {(cuuint64_t)inner / 2, rows_total};
        cuuint64_t st[1] = {(cuuint64_t)inner};
        cuuint32_t box[2] = {(cuuint32_t)inner / 2, (cuuint32_t)rows}, es[2] = {1, 1};
        CUtensorMapSwizzle sw = inner == 16 ? CU_TENSOR_MAP_SWIZZLE_NONE : inner == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : inner == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
          printf("encode failed inner %d rows %d: %d\n", inner, rows, (int)r);
          continue;
        }
      }
      for (int prod : {4})
        for (int ring : {4}) {
          if (prod * ring * box_bytes > 196 * 1024) continue;
          float best = 1e9;
          const int n_pos = inner ? (int)(kSrcBytes / inner) / rows : (int)(kSrcBytes / box_bytes);
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            reader<<<148, 128, prod * ring * box_bytes>>>(map, x, mode, ring, box_bytes, inner ? rows : 1, n_pos,
                                                          n_boxes, prod);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          const double gbs = 148.0 * n_boxes * box_bytes / (best * 1e-3) / 1e9;
          printf("same=%d %s inner %3d box %5d prod %d ring %d: %7.1f us %6.0f GB/s %5.1f B/clk/SM  %.0f ns/box/SM %s\n",
                 same, inner ? "tma " : "bulk", inner, box_bytes, prod, ring, best * 1e3, gbs, gbs / 148 / 1.965,
                 best * 1e6 / n_boxes, cudaGetErrorString(cudaGetLastError()));
        }
    }
  }
  return 0;
}
