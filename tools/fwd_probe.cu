// fwd_probe.cu -- where does the k_tc_fwd main loop spend its time? Mimics it (A = 128 x dp O tile, B = nt x dp X'
// tile, K-major SW128, kind::tf32 MMAs into TMEM) with per-k-block stamps, varying: MMA on/off, N tile, stages,
// k-blocks per TMA instruction (3D box {32, rows, kpb}: one instruction fetches kpb k-blocks), grid.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/fwd_probe tools/fwd_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
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

// maps: 4D {32 (col in k-block), rows, kblocks, chunks}, box {32, box_rows, kpb, 1}; smem per stage:
// A: kpb k-blocks of [128 rows x 128 B], B: kpb k-blocks of [nt rows x 128 B]
__global__ void __launch_bounds__(128, 1) bench(const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mX,
                                                int nkb, int nt, int stages, int kpb, int mma, uint64_t* stamps,
                                                float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t A_BYTES = 128 * 128 * kpb, B_BYTES = nt * 128 * kpb, STAGE = A_BYTES + B_BYTES;
  __shared__ uint64_t full[16], empty[16], done;
  __shared__ uint32_t tbase;
  uint64_t* st = stamps + blockIdx.x * 64;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) st[0] = gtime();
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 64);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) st[1] = gtime();
  const int ntn = 256 / nt;
  const int i0 = (blockIdx.x % 2) * 128, j0 = ((blockIdx.x / 2) % ntn) * nt, c = (blockIdx.x / (2 * ntn)) % 4;
  const int nst = (nkb + kpb - 1) / kpb;  // stages of kpb k-blocks
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < nst; ++q) {
      const int s = q % stages;
      if (q >= stages) mbar_wait(&empty[s], ((q / stages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
          ::"r"(smem_u32(sa)), "l"(&mO), "r"(smem_u32(&full[s])), "r"(0), "r"(i0), "r"(q * kpb), "r"(c) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];"
          ::"r"(smem_u32(sa + A_BYTES)), "l"(&mX), "r"(smem_u32(&full[s])), "r"(0), "r"(j0), "r"(q * kpb), "r"(c) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = idesc_tf32(128, nt, false, false);
    for (int q = 0; q < nst; ++q) {
      const int s = q % stages;
      mbar_wait(&full[s], (q / stages) & 1);
      if (q < 40) st[2 + q] = gtime();
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
      if (mma)
        for (int b = 0; b < kpb && q * kpb + b < nkb; ++b)
          for (int kk = 0; kk < 4; ++kk)
            mma_tf32(tmem, sdesc(sa + b * 16384 + kk * 32, 16, 1024), sdesc(sb + b * nt * 128 + kk * 32, 16, 1024),
                     idesc, (q | b | kk) ? 1u : 0u);
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
  if (warp == 0) tmem_dealloc(tmem, 64);
  if (threadIdx.x == 0) st[51] = gtime();
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  const int dp = 416, g = 256, k = 256, C = 4, nkb = dp / 32;
  float *O, *X, *out;
  uint64_t* stamps;
  cudaMalloc(&O, (size_t)C * g * dp * 4);
  cudaMalloc(&X, (size_t)C * k * dp * 4);
  cudaMalloc(&out, 256 * 128 * 4);
  cudaMalloc(&stamps, 256 * 64 * 8);
  cudaMemset(O, 0, (size_t)C * g * dp * 4);
  cudaMemset(X, 0, (size_t)C * k * dp * 4);
  auto mk = [&](CUtensorMap* m, float* p, int rows, int box_rows, int kpb) {
    cuuint64_t dims[4] = {32, (cuuint64_t)rows, (cuuint64_t)nkb, (cuuint64_t)C};
    cuuint64_t strides[3] = {(cuuint64_t)dp * 4, 128, (cuuint64_t)dp * 4 * rows};
    cuuint32_t box[4] = {32, (cuuint32_t)box_rows, (cuuint32_t)kpb, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode %d\n", r);
  };
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  printf("nt stages kpb mma grid | event us | cta0 setup, first full, last full, done, end (us) | max done over CTAs\n");
  struct Cfg { int nt, stages, kpb, mma, grid; };
  std::vector<Cfg> cfgs;
  for (int mma : {1, 0})
    for (int nt : {32, 64})
      for (int kpb : {1, 2, 4})
        for (int stages : {2, 4, 8}) {
          const size_t smem = (size_t)stages * (128 * 128 + nt * 128) * kpb + 1024;
          if (smem > 220 * 1024) continue;
          cfgs.push_back({nt, stages, kpb, mma, 2 * (256 / nt) * 4});
        }
  for (const Cfg& cf : cfgs) {
    CUtensorMap mO, mX;
    mk(&mO, O, g, 128, cf.kpb);
    mk(&mX, X, k, cf.nt, cf.kpb);
    const size_t smem = (size_t)cf.stages * (128 * 128 + cf.nt * 128) * cf.kpb + 1024;
    float best = 1e9;
    std::vector<uint64_t> h(256 * 64);
    for (int rep = 0; rep < 4; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      bench<<<cf.grid, 128, smem>>>(mO, mX, nkb, cf.nt, cf.stages, cf.kpb, cf.mma, stamps, out);
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      if (err) {
        printf("err %s\n", cudaGetErrorString(err));
        return 1;
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms * 1000);
      cudaMemcpy(h.data(), stamps, h.size() * 8, cudaMemcpyDeviceToHost);
    }
    uint64_t t0 = h[0];
    for (int b = 0; b < cf.grid; ++b) t0 = std::min(t0, h[b * 64]);
    uint64_t mxd = 0;
    for (int b = 0; b < cf.grid; ++b) mxd = std::max(mxd, h[b * 64 + 50]);
    const int nst = (nkb + cf.kpb - 1) / cf.kpb;
    printf("%3d %2d %d %d %3d | %6.2f | %5.2f %5.2f %5.2f %5.2f %5.2f | %5.2f\n", cf.nt, cf.stages, cf.kpb, cf.mma, cf.grid,
           best, (h[1] - t0) / 1e3, (h[2] - t0) / 1e3, (h[2 + nst - 1] - t0) / 1e3, (h[50] - t0) / 1e3,
           (h[51] - t0) / 1e3, (mxd - t0) / 1e3);
  }
  return 0;
}
