// ingest_probe.cu -- per-SM operand ingest rate from L2 on B200: TMA (cp.async.bulk.tensor, mbarrier pipeline) vs
// plain 128-bit LDG by all threads, as a function of grid size, pipeline depth and box size. Decides how the tcgen05
// kernels are tiled (their main loops stream L2-resident operands; see profiles/r01_summary.md).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ingest_probe tools/ingest_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"

using namespace kge::tc;

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int ROWS = 8192, COLS = 32;  // 1 MB fp32 buffer, [ROWS x 32] (one 128-byte row per box row)

__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap m, int box_rows, int stages,
                                                int nload, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16];
  const uint32_t bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  float acc = 0.f;
  if (threadIdx.x == 0) {
    const int nrb = ROWS / box_rows;
    for (int i = 0; i < stages && i < nload; ++i) {
      mbar_arrive_expect_tx(&full[i], bytes);
      tma_load_3d(smem + i * bytes, &m, &full[i], 0, ((blockIdx.x * 7 + i) % nrb) * box_rows, 0);
    }
    for (int i = 0; i < nload; ++i) {
      const int s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += *reinterpret_cast<float*>(smem + s * bytes);
      const int nx = i + stages;
      if (nx < nload) {
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_3d(smem + s * bytes, &m, &full[s], 0, ((blockIdx.x * 7 + nx) % nrb) * box_rows, 0);
      }
    }
    out[blockIdx.x] = acc;
  }
}

// nprod producer threads (lane 0 of warps 0..nprod-1), each owning stages s = w, w + nprod, ...; bulk = 1 -> 1D
// cp.async.bulk of the same bytes instead of the tensor map
__global__ void __launch_bounds__(128, 1) k_tma2(const __grid_constant__ CUtensorMap m, const float* src, int box_rows,
                                                 int stages, int nload, int nprod, int bulk, int nrows, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16];
  const uint32_t bytes = box_rows * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int w = threadIdx.x >> 5;
  float acc = 0.f;
  if ((threadIdx.x & 31) == 0 && w < nprod) {
    const int nrb = nrows / box_rows;
    auto issue = [&](int s, int i) {
      mbar_arrive_expect_tx(&full[s], bytes);
      const int rb = (blockIdx.x * 7919 + i * 131) % nrb;
      if (bulk)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(smem + s * bytes)), "l"(src + (size_t)rb * box_rows * 32), "r"(bytes),
                     "r"(smem_u32(&full[s])) : "memory");
      else
        tma_load_3d(smem + s * bytes, &m, &full[s], 0, rb * box_rows, 0);
    };
    for (int s = w; s < stages && s < nload; s += nprod) issue(s, s);
    for (int i = 0; i < nload; ++i) {
      const int s = i % stages;
      if (s % nprod != w) continue;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += *reinterpret_cast<float*>(smem + s * bytes);
      const int nx = i + stages;
      if (nx < nload) issue(s, nx);
    }
    out[blockIdx.x * 4 + w] = acc;
  }
}

__global__ void __launch_bounds__(256) k_ldg(const float4* __restrict__ src, int nvec_per_cta, int unroll, float* out) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  const int nall = ROWS * COLS / 4;
  const int base = (blockIdx.x * 1931) % nall;
  for (int i = threadIdx.x; i < nvec_per_cta; i += 256 * 8) {
    float4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcg(src + (base + i + u * 256) % nall);
#pragma unroll
    for (int u = 0; u < 8; ++u) { a.x += x[u].x; a.y += x[u].y; a.z += x[u].z; a.w += x[u].w; }
  }
  if (a.x == 1234.5f) out[blockIdx.x] = a.y + a.z + a.w;
}

int main() {
  float* buf;
  cudaMalloc(&buf, ROWS * COLS * 4);
  cudaMemset(buf, 0, ROWS * COLS * 4);
  float* out;
  cudaMalloc(&out, 4096 * 4);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const size_t per_cta = 256 * 1024;  // bytes each CTA ingests
  printf("mode grid box_rows stages KB/CTA us  B/clk/SM(@1.965GHz) chipTB/s\n");
  for (int box_rows : {32, 64, 128, 256}) {
    CUtensorMap m;
    cuuint64_t dims[3] = {COLS, ROWS, 1};
    cuuint64_t strides[2] = {COLS * 4, (cuuint64_t)COLS * 4 * ROWS};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int stages : {2, 4, 8, 12}) {
      if ((size_t)stages * box_rows * 128 > 190 * 1024) continue;
      for (int grid : {32, 64, 128, 148}) {
        const int nload = (int)(per_cta / (box_rows * 128));
        const size_t smem = (size_t)stages * box_rows * 128 + 1024;
        for (int w = 0; w < 3; ++w) k_tma<<<grid, 128, smem>>>(m, box_rows, stages, nload, out);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) k_tma<<<grid, 128, smem>>>(m, box_rows, stages, nload, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = 1000.0 * ms / reps;
        printf("tma %4d %4d %3d %6zu %8.2f %8.1f %8.2f\n", grid, box_rows, stages, per_cta / 1024, us,
               per_cta / (us * 1e-6) / 1.965e9, grid * per_cta / (us * 1e-6) / 1e12);
      }
    }
  }
  {
    const int BIG = 1 << 19;  // 64 MB buffer
    float* big;
    cudaMalloc(&big, (size_t)BIG * 128);
    cudaMemset(big, 0, (size_t)BIG * 128);
    cudaFuncSetAttribute(k_tma2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    printf("tma2: grid box stages nprod bulk swz us B/clk/SM\n");
    for (int swz : {1, 0}) {
      for (int box_rows : {32, 128}) {
        CUtensorMap m;
        cuuint64_t dims[3] = {COLS, (cuuint64_t)BIG, 1};
        cuuint64_t strides[2] = {COLS * 4, (cuuint64_t)COLS * 4 * BIG};
        cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
        cuuint32_t es[3] = {1, 1, 1};
        enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, big, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int stages : {1, 4, 8}) {
          for (int nprod : {1, 4}) {
            for (int bulk : {0, 1}) {
              if (bulk && !swz) continue;
              if (nprod > stages) continue;
              const int grid = 64;
              const int nload = (int)(per_cta / (box_rows * 128));
              const size_t smem = (size_t)stages * box_rows * 128 + 1024;
              // touch: the region read is 64 x 256 KB spread over 64 MB, first run warms L2
              for (int w = 0; w < 3; ++w) k_tma2<<<grid, 128, smem>>>(m, big, box_rows, stages, nload, nprod, bulk, BIG, out);
              cudaEventRecord(e0);
              for (int r = 0; r < 20; ++r) k_tma2<<<grid, 128, smem>>>(m, big, box_rows, stages, nload, nprod, bulk, BIG, out);
              cudaEventRecord(e1);
              cudaEventSynchronize(e1);
              float ms;
              cudaEventElapsedTime(&ms, e0, e1);
              const double us = 1000.0 * ms / 20;
              printf("tma2 %4d %4d %3d %d %d %d %8.2f %8.1f\n", grid, box_rows, stages, nprod, bulk, swz, us,
                     per_cta / (us * 1e-6) / 1.965e9);
            }
          }
        }
      }
    }
  }
  for (int grid : {32, 64, 128, 148, 296}) {
    const int nvec = (int)(per_cta / 16);
    for (int w = 0; w < 3; ++w) k_ldg<<<grid, 256>>>((const float4*)buf, nvec, 8, out);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int r = 0; r < reps; ++r) k_ldg<<<grid, 256>>>((const float4*)buf, nvec, 8, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = 1000.0 * ms / reps;
    printf("ldg %4d    - 8x256 %6zu %8.2f %8.1f %8.2f\n", grid, per_cta / 1024, us,
           per_cta / (us * 1e-6) / 1.965e9, grid * per_cta / (us * 1e-6) / 1e12);
  }
  // empty-kernel launch floor
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) k_ldg<<<148, 256>>>((const float4*)buf, 0, 8, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("empty launch %.2f us\n", 1000.0 * ms / 20);
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
