// Micro-benchmark: HBM streaming rate of the transform kernels' TMA ring
// (producer warp + consumer warps that only wait/arrive), for box / stage /
// occupancy choices.  Dev tool, not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2406_15102_b200/csrc tma_stream.cu -o tma_stream -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include "hlq_ptx.cuh"

using namespace hlq;

template <int STAGES, int CONS_WARPS>
__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, int ncol_tiles, int nrow_tiles,
                              int box_bytes, int box_cols, int box_rows, int touch) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* tiles = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * box_bytes);
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], CONS_WARPS); }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int items = ncol_tiles * nrow_tiles;
  if (warp == CONS_WARPS) {
    if (ptx::elect_one()) {
      int slot = 0; uint32_t ph = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x) {
        ptx::mbar_wait_sleep(&empty[slot], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[slot], box_bytes);
        ptx::tma_load_2d(tiles + slot * box_bytes, &map, &full[slot], (it % ncol_tiles) * box_cols,
                         (it / ncol_tiles) * box_rows);
        if (++slot == STAGES) { slot = 0; ph ^= 1; }
      }
    }
    return;
  }
  int slot = 0; uint32_t ph = 0;
  uint32_t acc = 0;
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    ptx::mbar_wait(&full[slot], ph);
    if (touch) acc += ptx::lds32(ptx::smem_u32(tiles + slot * box_bytes) + 4 * (threadIdx.x % 128));
    __syncwarp();
    if ((threadIdx.x & 31) == 0) ptx::mbar_arrive(&empty[slot]);
    if (++slot == STAGES) { slot = 0; ph ^= 1; }
  }
  if (acc == 0x12345678) printf("x");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int STAGES, int CW>
void run(void* buf, int rows, int cols, int box_cols, int box_rows, int ctas_per_sm, EncodeFn enc, int sms) {
  CUtensorMap map;
  cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
  cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  cuuint32_t es[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) { printf("encode failed\n"); return; }
  const int bb = box_cols * box_rows * 2;
  const size_t smem = size_t(STAGES) * bb + 2 * STAGES * 8;
  auto k = stream_kernel<STAGES, CW>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int nct = cols / box_cols, nrt = rows / box_rows;
  const int grid = sms * ctas_per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(a);
    k<<<grid, (CW + 1) * 32, smem>>>(map, nct, nrt, bb, box_cols, box_rows, 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (rep) best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  printf("stages %d cons_warps %d box %dx%d (%d B) ctas/sm %d : %.1f us  %.0f GB/s %s\n", STAGES, CW, box_rows,
         box_cols, bb, ctas_per_sm, best * 1e3, double(rows) * cols * 2 / (best * 1e-3) / 1e9,
         e ? cudaGetErrorString(e) : "");
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 25216, cols = 3072;  // ViT fc1 gy, bf16
  void* buf;
  cudaMalloc(&buf, size_t(rows) * cols * 2);
  cudaMemset(buf, 0, size_t(rows) * cols * 2);
  run<4, 4>(buf, rows, cols, 256, 16, 5, enc, sms);
  run<4, 4>(buf, rows, cols, 256, 16, 3, enc, sms);
  run<8, 4>(buf, rows, cols, 256, 16, 3, enc, sms);
  run<4, 4>(buf, rows, cols, 256, 32, 3, enc, sms);
  run<6, 4>(buf, rows, cols, 256, 32, 2, enc, sms);
  run<4, 8>(buf, rows, cols, 256, 32, 2, enc, sms);
  run<4, 4>(buf, rows, cols, 128, 16, 6, enc, sms);
  run<8, 4>(buf, rows, cols, 128, 16, 6, enc, sms);
  run<12, 4>(buf, rows, cols, 256, 16, 2, enc, sms);
  run<16, 4>(buf, rows, cols, 256, 16, 1, enc, sms);
  return 0;
}
