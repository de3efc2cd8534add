// tc_probe.cu -- standalone check of the tcgen05 kind::tf32 building block with TMA-fed SW128 operands in the three
// operand views the negative-score kernels use (fwd: A,B K-major; dO: A K-major, B MN-major; dX: A,B MN-major).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_probe tools/tc_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"

using namespace kge::tc;

__device__ uint64_t sdesc_lt(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t lt) {
  uint64_t d = sdesc(saddr, lbo, sbo);
  d &= ~((uint64_t)7 << 61);
  d |= (uint64_t)lt << 61;
  return d;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (EncodeFn)fn;
}

// row-major [rows x cols] fp32 matrix, box {32 cols, box_rows}
static CUtensorMap make_map(EncodeFn enc, float* p, int rows, int cols, int box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 4, (cuuint64_t)rows * cols * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

// mode 0: A [128 x K] K-major, B [N x K] K-major
// mode 1: A [128 x K] K-major, B stored [K x N] (MN-major)
// mode 2: A stored [K x 128] (MN-major), B stored [K x N] (MN-major)
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                            int mode, int N, int K, float* D, uint32_t lbo, uint32_t sbo, uint32_t lt) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;                 // up to 16 KB
  uint8_t* sB = smem + 16384;         // up to 32 KB
  __shared__ uint64_t bar_full, bar_mma;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar_full, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const int nkb = K / 32;
  const uint32_t idesc = idesc_tf32(128, N, mode == 2, mode >= 1);
  for (int kb = 0; kb < nkb; ++kb) {
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      if (mode <= 1) {
        tma_load_3d(sA, &ma, &bar_full, kb * 32, 0, 0);  // 128 rows x 32 cols
        bytes += 128 * 128;
      } else {
        for (int b = 0; b < 4; ++b) tma_load_3d(sA + b * 4096, &ma, &bar_full, b * 32, kb * 32, 0);  // 32 rows
        bytes += 4 * 4096;
      }
      if (mode == 0) {
        tma_load_3d(sB, &mb, &bar_full, kb * 32, 0, 0);  // N rows x 32 cols
        bytes += N * 128;
      } else {
        for (int b = 0; b < N / 32; ++b) tma_load_3d(sB + b * 4096, &mb, &bar_full, b * 32, kb * 32, 0);
        bytes += (N / 32) * 4096;
      }
      mbar_arrive_expect_tx(&bar_full, bytes);
    }
    if (threadIdx.x == 32) {
      mbar_wait(&bar_full, kb & 1);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = mode <= 1 ? sdesc(smem_u32(sA) + kk * 32, 16, 1024) : sdesc_lt(smem_u32(sA) + kk * 1024, lbo, sbo, lt);
        uint64_t bd = mode == 0 ? sdesc(smem_u32(sB) + kk * 32, 16, 1024) : sdesc_lt(smem_u32(sB) + kk * 1024, lbo, sbo, lt);
        mma_tf32(tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
      }
      mma_commit(&bar_mma);
    }
    // everyone waits for this block's MMAs before smem is overwritten by the next TMA
    mbar_wait(&bar_mma, kb & 1);
    tc_fence_after();
    __syncthreads();
  }
  // epilogue
  const int row = warp * 32 + (threadIdx.x & 31);
  for (int c = 0; c < N; c += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
    for (int i = 0; i < 32; ++i) D[row * N + c + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  EncodeFn enc = get_encode();
  if (!enc) {
    printf("no encode fn\n");
    return 1;
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int fails = 0;
  uint32_t variants[][3] = {{4096, 512, 1}, {512, 4096, 1}, {4096, 1024, 1}, {1024, 4096, 1}, {4096, 512, 2}, {4096, 1024, 2}};
  for (int var = 0; var < 6; ++var)
  for (int mode = 1; mode < 3; ++mode) {
    const int K = 64, N = mode == 0 ? 256 : (mode == 1 ? 160 : 96);
    std::vector<float> A(128 * K), B(N * K), D(128 * N);
    srand(1 + mode);
    for (auto& x : A) x = (rand() % 2001 - 1000) / 1000.0f;
    for (auto& x : B) x = (rand() % 2001 - 1000) / 1000.0f;
    // logical A[m][k], B[n][k]; storage depends on the mode
    std::vector<float> As(A.size()), Bs(B.size());
    for (int m = 0; m < 128; ++m)
      for (int k = 0; k < K; ++k) As[mode == 2 ? k * 128 + m : m * K + k] = A[m * K + k];
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) Bs[mode == 0 ? n * K + k : k * N + n] = B[n * K + k];
    float *dA, *dB, *dD;
    cudaMalloc(&dA, As.size() * 4);
    cudaMalloc(&dB, Bs.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, As.data(), As.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bs.data(), Bs.size() * 4, cudaMemcpyHostToDevice);
    CUtensorMapSwizzle mnsw = variants[var][2] == 1 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
    CUtensorMap ma = mode == 2 ? make_map(enc, dA, K, 128, 32, mnsw) : make_map(enc, dA, 128, K, 128);
    CUtensorMap mb = mode == 0 ? make_map(enc, dB, N, K, N) : make_map(enc, dB, K, N, 32, mnsw);
    probe<<<1, 128, 64 * 1024>>>(ma, mb, mode, N, K, dD, variants[var][0], variants[var][1], variants[var][2]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 2;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < K; ++k) ref += (double)A[m * K + k] * B[n * K + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("lt %u lbo %u sbo %u mode %d (N=%d K=%d): max |err| = %.3e (max |ref| %.2f) %s\n", variants[var][2], variants[var][0], variants[var][1], mode, N, K, maxerr, maxref,
           maxerr < 2e-2 ? "OK" : "FAIL");
    fails += maxerr >= 2e-2;
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
  }
  return fails;
}
