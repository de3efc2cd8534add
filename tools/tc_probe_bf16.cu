// tc_probe_bf16.cu -- standalone check of tcgen05 kind::f16 with BF16 operands staged by TMA (SWIZZLE_128B, 64-element
// = 128-byte rows) in the three operand views of the negative-score kernels (fwd: A,B K-major; dO: A K-major,
// B MN-major; dX': A,B MN-major), over candidate (LBO, SBO) pairs of the MN-major descriptor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tc_probe_bf16 tools/tc_probe_bf16.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"

using namespace kge::tc;

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
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

// row-major [rows x cols] bf16 matrix, box {64 cols, box_rows}
static CUtensorMap make_map(EncodeFn enc, void* p, int rows, int cols, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

// K = 64 per block (one 128-byte row), 4 MMAs of K = 16
// mode 0: A [128 x K] K-major, B [N x K] K-major
// mode 1: A [128 x K] K-major, B stored [K x N] (MN-major): MN blocks of 64 at sB + b * 8192 ([64 K rows][128 B])
// mode 2: A stored [K x 128] (MN-major, 2 MN blocks), B stored [K x N] (MN-major)
__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                            int mode, int N, int K, float* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;           // 16 KB
  uint8_t* sB = smem + 16384;   // up to 32 KB
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
  const int nkb = K / 64;
  const uint32_t idesc = idesc_bf16(128, N, mode == 2, mode >= 1);
  for (int kb = 0; kb < nkb; ++kb) {
    if (threadIdx.x == 0) {
      uint32_t bytes = 0;
      if (mode <= 1) {
        tma_load_3d(sA, &ma, &bar_full, kb * 64, 0, 0);  // 128 rows x 64 cols (K-major)
        bytes += 128 * 128;
      } else {
        for (int b = 0; b < 2; ++b) tma_load_3d(sA + b * 8192, &ma, &bar_full, b * 64, kb * 64, 0);  // 64 K rows
        bytes += 2 * 8192;
      }
      if (mode == 0) {
        tma_load_3d(sB, &mb, &bar_full, kb * 64, 0, 0);  // N rows x 64 cols
        bytes += N * 128;
      } else {
        for (int b = 0; b < N / 64; ++b) tma_load_3d(sB + b * 8192, &mb, &bar_full, b * 64, kb * 64, 0);
        bytes += (N / 64) * 8192;
      }
      mbar_arrive_expect_tx(&bar_full, bytes);
    }
    if (threadIdx.x == 32) {
      mbar_wait(&bar_full, kb & 1);
      tc_fence_after();
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = mode <= 1 ? sdesc(smem_u32(sA) + kk * 32, 16, 1024) : sdesc(smem_u32(sA) + kk * 2048, lbo, sbo);
        uint64_t bd = mode == 0 ? sdesc(smem_u32(sB) + kk * 32, 16, 1024) : sdesc(smem_u32(sB) + kk * 2048, lbo, sbo);
        mma_bf16(tmem, ad, bd, idesc, (kb | kk) ? 1u : 0u);
      }
      mma_commit(&bar_mma);
    }
    mbar_wait(&bar_mma, kb & 1);
    tc_fence_after();
    __syncthreads();
  }
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

static uint16_t to_bf16(float x) {  // round to nearest even
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
  uint32_t u = (uint32_t)h << 16;
  float x;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  EncodeFn enc = get_encode();
  if (!enc) {
    printf("no encode fn\n");
    return 1;
  }
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  int fails = 0;
  const uint32_t variants[][2] = {{8192, 1024}, {1024, 8192}};
  for (int mode = 0; mode < 3; ++mode)
    for (int var = 0; var < (mode == 0 ? 1 : 2); ++var) {
      const int K = 128, N = mode == 0 ? 256 : 128;
      std::vector<float> A(128 * K), B(N * K), D(128 * N);
      srand(1 + mode);
      for (auto& x : A) x = from_bf16(to_bf16((rand() % 2001 - 1000) / 1000.0f));
      for (auto& x : B) x = from_bf16(to_bf16((rand() % 2001 - 1000) / 1000.0f));
      std::vector<uint16_t> As(A.size()), Bs(B.size());
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < K; ++k) As[mode == 2 ? k * 128 + m : m * K + k] = to_bf16(A[m * K + k]);
      for (int n = 0; n < N; ++n)
        for (int k = 0; k < K; ++k) Bs[mode == 0 ? n * K + k : k * N + n] = to_bf16(B[n * K + k]);
      void *dA, *dB;
      float* dD;
      cudaMalloc(&dA, As.size() * 2);
      cudaMalloc(&dB, Bs.size() * 2);
      cudaMalloc(&dD, D.size() * 4);
      cudaMemcpy(dA, As.data(), As.size() * 2, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, Bs.data(), Bs.size() * 2, cudaMemcpyHostToDevice);
      CUtensorMap ma = mode == 2 ? make_map(enc, dA, K, 128, 64) : make_map(enc, dA, 128, K, 128);
      CUtensorMap mb = mode == 0 ? make_map(enc, dB, N, K, N) : make_map(enc, dB, K, N, 64);
      probe<<<1, 128, 64 * 1024>>>(ma, mb, mode, N, K, dD, variants[var][0], variants[var][1]);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d var %d: CUDA error %s\n", mode, var, cudaGetErrorString(e));
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
      printf("mode %d lbo %u sbo %u (N=%d K=%d): max |err| = %.3e (max |ref| %.2f) %s\n", mode, variants[var][0],
             variants[var][1], N, K, maxerr, maxref, maxerr < 1e-3 ? "OK" : "FAIL");
      fails += maxerr >= 1e-3;
      cudaFree(dA);
      cudaFree(dB);
      cudaFree(dD);
    }
  return fails;
}
