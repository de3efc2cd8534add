// tma_overlap_probe.cu -- do TMA loads issued back to back by one thread overlap? Issue n loads of `box_rows` x 128 B
// into distinct buffers, then wait for each; record the completion time of each load (globaltimer) per CTA.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"
using namespace kge::tc;
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap m, int box_rows, int n, int mode,
                                            unsigned long long* stamps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16];
  const uint32_t bytes = box_rows * 128;
  if (threadIdx.x == 0) { for (int s = 0; s < n; ++s) mbar_init(&full[s], 1); fence_mbar_init(); }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  if (mode == 0 && threadIdx.x == 0) {  // one thread issues all
    const uint64_t t0 = gt();
    for (int s = 0; s < n; ++s) {
      mbar_arrive_expect_tx(&full[s], bytes);
      tma_load_3d(smem + s * bytes, &m, &full[s], 0, (blockIdx.x * 16 + s) * box_rows, 0);
    }
    const uint64_t t1 = gt();
    for (int s = 0; s < n; ++s) { mbar_wait(&full[s], 0); stamps[blockIdx.x * 18 + 2 + s] = gt() - t0; }
    stamps[blockIdx.x * 18] = t1 - t0;
  }
  if (mode == 1 && (threadIdx.x & 31) == 0) {  // warp w issues loads s = w, w+4, ...
    const uint64_t t0 = gt();
    for (int s = w; s < n; s += 4) {
      mbar_arrive_expect_tx(&full[s], bytes);
      tma_load_3d(smem + s * bytes, &m, &full[s], 0, (blockIdx.x * 16 + s) * box_rows, 0);
    }
    for (int s = w; s < n; s += 4) { mbar_wait(&full[s], 0); stamps[blockIdx.x * 18 + 2 + s] = gt() - t0; }
  }
}
__global__ void __launch_bounds__(128, 1) k2(const __grid_constant__ CUtensorMap m, int kb, int n,
                                             unsigned long long* stamps) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16];
  const uint32_t bytes = kb * 16384;
  if (threadIdx.x == 0) { for (int s = 0; s < n; ++s) mbar_init(&full[s], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t t0 = gt();
    for (int s = 0; s < n; ++s) {
      mbar_arrive_expect_tx(&full[s], bytes);
      tma_load_3d(smem + s * bytes, &m, &full[s], 0, (blockIdx.x % 64) * 128, s * kb);
    }
    const uint64_t t1 = gt();
    for (int s = 0; s < n; ++s) { mbar_wait(&full[s], 0); stamps[blockIdx.x * 18 + 2 + s] = gt() - t0; }
    stamps[blockIdx.x * 18] = t1 - t0;
  }
}
int main() {
  const int ROWS = 1 << 18;
  float* buf; cudaMalloc(&buf, (size_t)ROWS * 128); cudaMemset(buf, 0, (size_t)ROWS * 128);
  unsigned long long* st; cudaMallocManaged(&st, 148 * 18 * 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  // 3D box {32 cols, rows, kb k-blocks} over a [rows x (32 * kbs)] matrix: one TMA instruction fetches kb k-blocks
  for (int kb : {1, 4}) {
    CUtensorMap m;
    const int R = 8192, KBS = 16;
    cuuint64_t dims[3] = {32, (cuuint64_t)R, (cuuint64_t)KBS};
    cuuint64_t strides[2] = {(cuuint64_t)KBS * 128, 128};
    cuuint32_t box[3] = {32, 128, (cuuint32_t)kb};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int n = kb == 1 ? 12 : 3;
    for (int grid : {1, 64, 148}) {
      for (int r = 0; r < 3; ++r) k2<<<grid, 128, 12 * 16384 + 1024>>>(m, kb, n, st);
      cudaDeviceSynchronize();
      printf("kb %d (box %d KB, rc %d) grid %3d issue %llu ns | completions:", kb, 16 * kb, (int)rc, grid, st[0]);
      for (int s = 0; s < n; ++s) printf(" %llu", st[2 + s]);
      unsigned long long mx = 0;
      for (int b = 0; b < grid; ++b) mx = st[b * 18 + 1 + n] > mx ? st[b * 18 + 1 + n] : mx;
      printf(" | last over CTAs %llu\n", mx);
    }
  }
  for (int box_rows : {32, 128}) {
    CUtensorMap m;
    cuuint64_t dims[3] = {32, (cuuint64_t)ROWS, 1};
    cuuint64_t strides[2] = {128, (cuuint64_t)128 * ROWS};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int mode : {0, 1}) for (int grid : {1, 64}) {
      const int n = box_rows == 32 ? 16 : 12;
      for (int r = 0; r < 3; ++r) k<<<grid, 128, n * box_rows * 128 + 1024>>>(m, box_rows, n, mode, st);
      cudaDeviceSynchronize();
      printf("box %3d rows mode %d grid %3d  issue %llu ns | completions (ns, CTA 0):", box_rows, mode, grid, st[0]);
      for (int s = 0; s < n; ++s) printf(" %llu", st[2 + s]);
      printf("\n");
    }
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
