// tmem_probe.cu -- tcgen05.ld throughput: nw warps (each its own 32-lane quarter) load R x (32 lanes x 32 columns)
// of fp32 from TMEM and accumulate; cycles per warp-load and bytes per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tmem_probe tools/tmem_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2004_08532_b200/csrc/tc_ptx.cuh"
using namespace kge::tc;
__global__ void __launch_bounds__(256, 1) k(int R, int nw, int batch, long long* out, float* sink) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&tbase, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  float acc = 0.f;
  const long long t0 = clock64();
  if (warp < nw) {
    const uint32_t t = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    if (batch == 1) {
      for (int r = 0; r < R; ++r) {
        float v[32];
        tmem_ld32(t + (r & 15) * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
      }
    } else {  // 4 loads in flight before one wait
      for (int r = 0; r < R; r += 4) {
        uint32_t q[4][32];
#pragma unroll
        for (int b = 0; b < 4; ++b)
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
              "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
              : "=r"(q[b][0]), "=r"(q[b][1]), "=r"(q[b][2]), "=r"(q[b][3]), "=r"(q[b][4]), "=r"(q[b][5]), "=r"(q[b][6]),
                "=r"(q[b][7]), "=r"(q[b][8]), "=r"(q[b][9]), "=r"(q[b][10]), "=r"(q[b][11]), "=r"(q[b][12]),
                "=r"(q[b][13]), "=r"(q[b][14]), "=r"(q[b][15]), "=r"(q[b][16]), "=r"(q[b][17]), "=r"(q[b][18]),
                "=r"(q[b][19]), "=r"(q[b][20]), "=r"(q[b][21]), "=r"(q[b][22]), "=r"(q[b][23]), "=r"(q[b][24]),
                "=r"(q[b][25]), "=r"(q[b][26]), "=r"(q[b][27]), "=r"(q[b][28]), "=r"(q[b][29]), "=r"(q[b][30]),
                "=r"(q[b][31])
              : "r"(t + ((r + b) & 15) * 32));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int i = 0; i < 32; ++i) acc += __uint_as_float(q[b][i]);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  sink[blockIdx.x * 256 + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}
int main() {
  long long* out;
  float* sink;
  cudaMallocManaged(&out, 8 * 148);
  cudaMalloc(&sink, 4 * 256 * 148);
  printf("nw batch R | cycles total, cycles per warp-load (4 KB), SM bytes/cycle\n");
  for (int batch : {1, 4})
    for (int nw : {1, 4, 8}) {
      const int R = 64;
      for (int w = 0; w < 2; ++w) k<<<1, 256>>>(R, nw, batch, out, sink);
      cudaDeviceSynchronize();
      printf("%d %d %d | %lld %.1f %.1f\n", nw, batch, R, out[0], (double)out[0] / R, (double)nw * R * 4096 / out[0]);
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
