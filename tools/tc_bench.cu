// tc_bench.cu -- timing probe of the TMA -> tcgen05 mainloop used by k_tc_fwd (32 CTAs, 4 stages, K = 416).
// Records per-CTA globaltimer stamps: start, after setup, each full-barrier pass, done.
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

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int NT = 64, STAGES = 4;

__global__ void __launch_bounds__(128, 1) bench(const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mX,
                                                int nkb, uint64_t* stamps, float* out, int mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr uint32_t A_BYTES = 128 * 128, B_BYTES = NT * 128, STAGE = A_BYTES + B_BYTES;
  __shared__ uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tbase;
  uint64_t* st = stamps + blockIdx.x * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) st[0] = gtime();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, NT);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) st[1] = gtime();
  const int i0 = (blockIdx.x % 2) * 128, j0 = ((blockIdx.x / 2) % 4) * NT, c = blockIdx.x / 8;
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
      tma_load_3d(sa, &mO, &full[s], kb * 32, i0, c);
      tma_load_3d(sa + A_BYTES, &mX, &full[s], kb * 32, j0, c);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_tf32(128, NT, false, false);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      if (kb < 40) st[2 + kb] = gtime();
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
      if (mode == 0)
        for (int kk = 0; kk < 4; ++kk)
          mma_tf32(tmem, sdesc(sa + kk * 32, 16, 1024), sdesc(sb + kk * 32, 16, 1024), idesc, (kb | kk) ? 1u : 0u);
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();
  if (threadIdx.x == 0) st[50] = gtime();
  float v[32];
  tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  out[blockIdx.x * 128 + threadIdx.x] = v[0];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, NT);
  if (threadIdx.x == 0) st[51] = gtime();
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  const int dp = 416, g = 256, k = 256, C = 4;
  float *O, *X, *out;
  uint64_t* stamps;
  cudaMalloc(&O, (size_t)C * g * dp * 4);
  cudaMalloc(&X, (size_t)C * k * dp * 4);
  cudaMalloc(&out, 64 * 128 * 4);
  cudaMalloc(&stamps, 64 * 64 * 8);
  {
    std::vector<float> hO((size_t)C * g * dp), hX((size_t)C * k * dp);
    for (auto& x : hO) x = (rand() % 2001 - 1000) / 1000.0f;
    for (auto& x : hX) x = (rand() % 2001 - 1000) / 1000.0f;
    if (getenv("ZERO")) { std::fill(hO.begin(), hO.end(), 0.f); std::fill(hX.begin(), hX.end(), 0.f); }
    cudaMemcpy(O, hO.data(), hO.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(X, hX.data(), hX.size() * 4, cudaMemcpyHostToDevice);
  }
  CUtensorMap mO, mX;
  auto mk = [&](CUtensorMap* m, float* p, int rows, int box_rows, CUtensorMapL2promotion pr) {
    cuuint64_t dims[3] = {(cuuint64_t)dp, (cuuint64_t)rows, (cuuint64_t)C};
    cuuint64_t strides[2] = {(cuuint64_t)dp * 4, (cuuint64_t)dp * 4 * rows};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode %d\n", r);
  };
  size_t smem = STAGES * (128 * 128 + NT * 128) + 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int pr = 0; pr < 2; ++pr)
    for (int mode = 0; mode < 2; ++mode) {
      mk(&mO, O, g, 128, pr ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE);
      mk(&mX, X, k, NT, pr ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        bench<<<32, 128, smem>>>(mO, mX, dp / 32, stamps, out, mode);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        if (err) {
          printf("err %s\n", cudaGetErrorString(err));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<uint64_t> h(64 * 64);
        cudaMemcpy(h.data(), stamps, h.size() * 8, cudaMemcpyDeviceToHost);
        uint64_t t0 = h[0];
        for (int b = 0; b < 32; ++b) t0 = std::min(t0, h[b * 64]);
        printf("promo %d mode %d rep %d: event %.2f us | cta0: setup %.2f us, full[0] %.2f, full[12] %.2f, done %.2f, end %.2f us\n",
               pr, mode, rep, ms * 1000, (h[1] - t0) / 1e3, (h[2] - t0) / 1e3, (h[14] - t0) / 1e3, (h[50] - t0) / 1e3,
               (h[51] - t0) / 1e3);
        if (rep == 2) {
          printf("   per-block stamps cta0 (us):");
          for (int kb = 0; kb < 13; ++kb) printf(" %.2f", (h[2 + kb] - t0) / 1e3);
          printf("\n");
        }
      }
    }
  return 0;
}
