// mma_probe.cu -- cycles per tcgen05.mma (cta_group::1, M = 128, both operands in smem, K-major SW128) as a function
// of N and kind (tf32 K = 8, bf16 K = 16): R back-to-back MMAs over resident operands, timed from the first issue to
// the commit's mbarrier completion. Decides the N tile of the negative-score contraction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"

using namespace kge::tc;

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) k(int N, int kind, int R, int kspan, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t done;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += 128) reinterpret_cast<int4*>(smem)[i] = make_int4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&tbase, 512);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (kspan == 3 && threadIdx.x < 32) {
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const uint32_t id = kind == 0 ? idesc_tf32(128, N, false, false) : idesc_bf16(128, N);
    const long long t0 = clock64();
    const uint64_t a0 = sdesc(sa, 16, 1024), b0 = sdesc(sb, 16, 1024);
#pragma unroll 4
    for (int r = 0; r < R; ++r) {
      const uint64_t off = (uint64_t)((r & 3) * 2);
      uint32_t is_elected;
      asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(is_elected));
      if (is_elected) {
        if (kind == 0)
          mma_tf32(tbase, a0 + off, b0 + off, id, r ? 1u : 0u);
        else
          mma_f16(tbase, a0 + off, b0 + off, id, r ? 1u : 0u);
      }
      __syncwarp();
    }
    if (threadIdx.x == 0) mma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  if (kspan >= 5 && kspan <= 8) {  // nw = kspan - 4 issuing warps (lane 0 each), each R / nw MMAs into its own accumulator columns
    const int nw = kspan - 4, w = threadIdx.x >> 5;
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const uint32_t id = kind == 0 ? idesc_tf32(128, N, false, false) : idesc_bf16(128, N);
    __syncthreads();
    const long long t0 = clock64();
    if ((threadIdx.x & 31) == 0 && w < nw) {
      const uint64_t a0 = sdesc(sa, 16, 1024), b0 = sdesc(sb, 16, 1024);
      for (int r = 0; r < R / nw; ++r) {
        const uint64_t off = (uint64_t)((r & 3) * 2);
        if (kind == 0)
          mma_tf32(tbase + w * N, a0 + off, b0 + off, id, r ? 1u : 0u);
        else
          mma_f16(tbase + w * N, a0 + off, b0 + off, id, r ? 1u : 0u);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      mma_commit(&done);  // commit tracks this thread's MMAs only: re-wait below via a second barrier round
      mbar_wait(&done, 0);
    }
    if (w < nw && (threadIdx.x & 31) == 0 && w > 0) {}
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
  if ((kspan < 3 || kspan == 4 || kspan >= 9) && threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = sa + 128 * 128;
    const uint32_t id = kind == 0 ? idesc_tf32(128, N, false, false) : idesc_bf16(128, N);
    const long long t0 = clock64();
    if (kspan >= 9) {  // one thread, alternating over nacc = kspan - 8 accumulators (column ranges of N)
      const int nacc = kspan - 8;
      const uint64_t a0 = sdesc(sa, 16, 1024), b0 = sdesc(sb, 16, 1024);
      for (int r = 0; r < R; ++r) {
        const uint64_t off = (uint64_t)(((r / nacc) & 3) * 2);
        if (kind == 0)
          mma_tf32(tbase + (r % nacc) * N, a0 + off, b0 + off, id, r >= nacc ? 1u : 0u);
        else
          mma_f16(tbase + (r % nacc) * N, a0 + off, b0 + off, id, r >= nacc ? 1u : 0u);
      }
    } else if (kspan == 4) {  // A operand in TMEM (columns 256 + 8 * (r & 3)), B in smem
      const uint64_t b0 = sdesc(sb, 16, 1024);
#pragma unroll 4
      for (int r = 0; r < R; ++r) {
        const uint64_t off = (uint64_t)((r & 3) * 2);
        if (kind == 0)
          mma_tf32_ts(tbase, tbase + 256 + 8 * (r & 3), b0 + off, id, r ? 1u : 0u);
        else
          mma_f16_ts(tbase, tbase + 256 + 8 * (r & 3), b0 + off, id, r ? 1u : 0u);
      }
    } else if (kspan == 2) {  // descriptors built once; the loop only advances the 14-bit start address field
      const uint64_t a0 = sdesc(sa, 16, 1024), b0 = sdesc(sb, 16, 1024);
#pragma unroll 4
      for (int r = 0; r < R; ++r) {
        const uint64_t off = (uint64_t)((r & 3) * 2);  // 32 B >> 4
        if (kind == 0)
          mma_tf32(tbase, a0 + off, b0 + off, id, r ? 1u : 0u);
        else
          mma_f16(tbase, a0 + off, b0 + off, id, r ? 1u : 0u);
      }
    } else
    for (int r = 0; r < R; ++r) {
      const int kk = kspan ? (r & 3) : 0;  // K offset within the 128-byte swizzled rows (32 B per MMA)
      if (kind == 0)
        mma_tf32(tbase, sdesc(sa + kk * 32, 16, 1024), sdesc(sb + kk * 32, 16, 1024), id, r ? 1u : 0u);
      else
        mma_f16(tbase, sdesc(sa + kk * 32, 16, 1024), sdesc(sb + kk * 32, 16, 1024), id, r ? 1u : 0u);
    }
    mma_commit(&done);
    mbar_wait(&done, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tbase, 512);
}

int main() {
  long long* out;
  cudaMallocManaged(&out, 148 * 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  printf("kind N kspan grid R | cycles per MMA (CTA 0)\n");
  for (int kind : {0, 1})
    for (int N : {32, 64, 128})
      for (int kspan : {0, 10, 12, 8})
        for (int grid : {1}) {
          const int R = 256;
          for (int w = 0; w < 2; ++w) k<<<grid, 128, 64 * 1024>>>(N, kind, R, kspan, out);
          cudaDeviceSynchronize();
          printf("%s %3d %d %3d %d | %.1f\n", kind ? "bf16" : "tf32", N, kspan, grid, R, (double)out[0] / R);
        }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
