// Dev probe as a shared library: the TMA ring reader of tools/probe_tma_bw.cu on a
// caller-provided fp32 NCHW16c tensor, launched on the caller's stream, so it can
// be timed under exactly the conditions (allocation, flush, events) of the conv passes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include "../../paper_1808_05567_b200/csrc/kernels/sm100_ptx.cuh"
using namespace dconv_sm100;

__global__ void probe_reader(const __grid_constant__ CUtensorMap map, int ring, int n_tiles, int tiles_per_img,
                             int cb, int kc, int variant) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16];
  const uint32_t slot = 128 * 64 * kc;
  __shared__ __align__(8) uint64_t cbar;
  __shared__ uint32_t tbase;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ring; ++i) mbar_init(&full[i], 1);
    mbar_init(&cbar, 1);
    fence_barrier_init();
  }
  if (variant >= 1 && threadIdx.x / 32 == 1) tmem_alloc(&tbase, 512);
  __syncthreads();
  if (threadIdx.x / 32 == 1) {
    // variant 1: TMEM allocated only; 2: plus one tcgen05.commit (no MMA issued)
    if (variant == 2 && elect_one()) mma_commit(&cbar);
    __syncwarp();
  }
  if (threadIdx.x == 0) {
  const int stages_per_tile = cb / kc;
  auto issue = [&](int g) {
    const int t = blockIdx.x + (g / stages_per_tile) * gridDim.x;
    const int it = g % stages_per_tile;
    const int n = t / tiles_per_img, v0 = (t % tiles_per_img) * 128;
    const int s = g % ring;
    mbar_arrive_expect_tx(&full[s], slot);
    tma_load_3d(smem + s * slot, &map, &full[s], 0, v0, n * cb + it * kc);
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
  __syncwarp();
  __syncthreads();
  if (variant >= 1 && threadIdx.x / 32 == 1) tmem_dealloc(tbase, 512);
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

extern "C" int probe_read(void* x, int n, int cb, int hw, int ring, int kc, int variant, void* stream) {
  static Enc enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  }
  CUtensorMap map;
  cuuint64_t dims[3] = {16, (cuuint64_t)hw, (cuuint64_t)n * cb};
  cuuint64_t st[2] = {64, (cuuint64_t)hw * 64};
  cuuint32_t box[3] = {16, 128, (cuuint32_t)kc}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int smem = ring * 128 * 64 * kc > 120 * 1024 ? ring * 128 * 64 * kc : 120 * 1024;  // one CTA per SM
  cudaFuncSetAttribute(probe_reader, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tpi = (hw + 127) / 128;
  probe_reader<<<148, 64, smem, (cudaStream_t)stream>>>(map, ring, n * tpi, tpi, cb, kc, variant);
  return (int)cudaGetLastError();
}
