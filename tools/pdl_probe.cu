// PDL hand-over vs software grid barrier on B200 (diagnostic).
// (1) kernel A (G CTAs, each writes W floats) -> kernel B (PDL, griddepcontrol.wait): gap between A's last CTA end
//     stamp and B's first / median release.
// (2) one persistent kernel (148 CTAs, co-resident): arrival counter + spin; gap between the last arrival and the
//     release of every CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void kA(float* buf, int w, uint64_t* stamp, int trig_early, int spin_ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (trig_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float* p = buf + (size_t)blockIdx.x * w;
  for (int i = threadIdx.x; i < w; i += blockDim.x) p[i] = (float)i * 1.0001f;
  if (spin_ns) {
    const uint64_t t0 = gt();
    while (gt() - t0 < (uint64_t)spin_ns) {}
  }
  __syncthreads();
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}

// A' = update-like: spin, then every warp writes one 1600-byte row at a random (or sequential) row of a big table
__global__ void kR(float* tab, long long nrows, int random, uint64_t* stamp, int spin_ns) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t t0 = gt();
  while (gt() - t0 < (uint64_t)spin_ns) {}
  const int wg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  unsigned long long h = (unsigned long long)wg * 0x9E3779B97F4A7C15ull;
  h ^= h >> 29; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 32;
  const long long row = random ? (long long)(h % (unsigned long long)nrows) : wg;
  float* p = tab + row * 400;
  for (int i = lane; i < 100; i += 32) reinterpret_cast<float4*>(p)[i] = make_float4(1.f, 2.f, 3.f, (float)wg);
  __syncthreads();
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}

// A'' = chain member whose odd CTAs leave before griddepcontrol.wait (as k_update's CTAs without a segment start)
__global__ void kE(uint64_t* stamp, int spin_ns, int early) {
  if (early && (blockIdx.x & 1)) return;
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t t0 = gt();
  while (gt() - t0 < (uint64_t)spin_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}

// A''' = gather-like (dynamic smem limits residency), B' = fwd-like (200 KB smem, optional cluster of 2)
__global__ void kG(uint64_t* stamp, int spin_ns) {
  extern __shared__ float sm[];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint64_t t0 = gt();
  while (gt() - t0 < (uint64_t)spin_ns) {}
  sm[threadIdx.x] = 1.f;
  __syncthreads();
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}
__global__ void kF(uint64_t* stamp, uint64_t* start) {
  extern __shared__ float sm[];
  if (threadIdx.x == 0) start[blockIdx.x] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  sm[threadIdx.x] = 2.f;
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}

__global__ void kB(uint64_t* stamp, uint64_t* start) {
  if (threadIdx.x == 0) start[blockIdx.x] = gt();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) stamp[blockIdx.x] = gt();
}

__global__ void kBar(unsigned* cnt, uint64_t* arr, uint64_t* rel, int rounds) {
  for (int r = 0; r < rounds; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      arr[r * gridDim.x + blockIdx.x] = gt();
      atomicAdd(cnt, 1u);
      const unsigned want = (unsigned)(r + 1) * gridDim.x;
      while (true) {
        unsigned v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
        if (v >= want) break;
      }
      rel[r * gridDim.x + blockIdx.x] = gt();
    }
    __syncthreads();
  }
}

static void launch_pdl(void (*k)(uint64_t*, uint64_t*), int g, uint64_t* s, uint64_t* st, int pdl) {
  cudaLaunchConfig_t c = {};
  c.gridDim = g;
  c.blockDim = 256;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  c.attrs = at;
  c.numAttrs = 1;
  cudaLaunchKernelEx(&c, k, s, st);
}

int main() {
  float* buf;
  uint64_t *sa, *sb, *arr, *rel;
  unsigned* cnt;
  cudaMalloc(&buf, (size_t)512 * 65536 * 4);
  cudaMalloc(&sa, 4096 * 8);
  cudaMalloc(&sb, 4096 * 8);
  const int R = 20;
  cudaMalloc(&arr, R * 148 * 8);
  cudaMalloc(&rel, R * 148 * 8);
  cudaMalloc(&cnt, 4);
  uint64_t* sst;
  cudaMalloc(&sst, 4096 * 8);
  struct Case { int G, w, trig, spin, pdl; };
  const Case cases[] = {{148, 0, 1, 0, 1}, {148, 0, 1, 5000, 1}, {148, 0, 1, 20000, 1}, {148, 0, 0, 5000, 1},
                        {148, 0, 0, 5000, 0}, {148, 0, 1, 5000, 0}, {256, 1024, 1, 5000, 1}, {512, 1024, 1, 5000, 1},
                        {148, 8192, 1, 0, 1}, {148, 8192, 0, 0, 1}, {148, 8192, 0, 0, 0}};
  for (const Case& cs : cases) {
    const int G = cs.G;
    std::vector<double> gmin, gmed, gst;
    for (int rep = 0; rep < 20; ++rep) {
      kA<<<G, 256>>>(buf, cs.w, sa, cs.trig, cs.spin);
      launch_pdl(kB, G, sb, sst, cs.pdl);
      cudaDeviceSynchronize();
      std::vector<uint64_t> a(G), b(G), bs(G);
      cudaMemcpy(a.data(), sa, G * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), sb, G * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(bs.data(), sst, G * 8, cudaMemcpyDeviceToHost);
      const uint64_t ae = *std::max_element(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      std::sort(bs.begin(), bs.end());
      if (rep >= 5) {
        gmin.push_back(((double)b[0] - (double)ae) / 1e3);
        gmed.push_back(((double)b[G / 2] - (double)ae) / 1e3);
        gst.push_back(((double)bs[G - 1] - (double)ae) / 1e3);
      }
    }
    std::sort(gmin.begin(), gmin.end());
    std::sort(gmed.begin(), gmed.end());
    std::sort(gst.begin(), gst.end());
    printf("G=%4d W=%6d trig_early=%d spin=%5d ns pdl=%d: B release - A last end: first %.2f med %.2f us; B last start - A end %.2f us\n",
           G, cs.w, cs.trig, cs.spin, cs.pdl, gmin[gmin.size() / 2], gmed[gmed.size() / 2], gst[gst.size() / 2]);
  }
  {
    float* tab;
    const long long nrows = 20000000;  // 32 GB of 400-float rows
    if (cudaMalloc(&tab, (size_t)nrows * 1600) != cudaSuccess) { printf("no table\n"); return 1; }
    cudaMemset(tab, 0, (size_t)nrows * 1600);
    for (int random : {0, 1}) {
      for (int G : {148, 512}) {
        std::vector<double> gmed;
        for (int rep = 0; rep < 20; ++rep) {
          kR<<<G, 256>>>(tab, nrows, random, sa, 8000);
          launch_pdl(kB, G, sb, sst, 1);
          cudaDeviceSynchronize();
          std::vector<uint64_t> a(G), b(G);
          cudaMemcpy(a.data(), sa, G * 8, cudaMemcpyDeviceToHost);
          cudaMemcpy(b.data(), sb, G * 8, cudaMemcpyDeviceToHost);
          const uint64_t ae = *std::max_element(a.begin(), a.end());
          std::sort(b.begin(), b.end());
          if (rep >= 5) gmed.push_back(((double)b[G / 2] - (double)ae) / 1e3);
        }
        std::sort(gmed.begin(), gmed.end());
        printf("row writer G=%d (%d rows of 1600 B, %s): B release - A last end: med %.2f us\n", G, G * 8,
               random ? "random in 32 GB" : "sequential", gmed[gmed.size() / 2]);
      }
    }
    cudaFree(tab);
  }
  for (int early : {0, 1}) {
    const int G = 512;
    std::vector<double> gmed;
    for (int rep = 0; rep < 20; ++rep) {
      cudaMemset(sa, 0, G * 8);
      kA<<<148, 256>>>(buf, 0, sb, 1, 3000);  // a predecessor, so kE is itself a PDL secondary
      {
        cudaLaunchConfig_t c = {};
        c.gridDim = G;
        c.blockDim = 256;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        c.attrs = at;
        c.numAttrs = 1;
        cudaLaunchKernelEx(&c, kE, sa, 8000, early);
      }
      launch_pdl(kB, 256, sb, sst, 1);
      cudaDeviceSynchronize();
      std::vector<uint64_t> a(G), b(256);
      cudaMemcpy(a.data(), sa, G * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(b.data(), sb, 256 * 8, cudaMemcpyDeviceToHost);
      const uint64_t ae = *std::max_element(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      if (rep >= 5) gmed.push_back(((double)b[128] - (double)ae) / 1e3);
    }
    std::sort(gmed.begin(), gmed.end());
    printf("chain A -> E (G=512, odd CTAs leave before the wait: %d) -> B: B release - E last end: med %.2f us\n", early,
           gmed[gmed.size() / 2]);
  }
  cudaFuncSetAttribute(kG, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  cudaFuncSetAttribute(kF, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int gsm : {0, 100}) {
    for (int cl : {1, 2}) {
      std::vector<double> g0, gm, gs;
      for (int rep = 0; rep < 20; ++rep) {
        cudaLaunchConfig_t c = {};
        c.gridDim = 256;
        c.blockDim = 256;
        c.dynamicSmemBytes = (gsm ? gsm : 1) * 1024;
        cudaLaunchAttribute at[2];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        c.attrs = at;
        c.numAttrs = 1;
        kA<<<148, 256>>>(buf, 0, sb, 1, 3000);
        cudaLaunchKernelEx(&c, kG, sa, 4000);
        cudaLaunchConfig_t f = {};
        f.gridDim = 128;
        f.blockDim = 256;
        f.dynamicSmemBytes = 200 * 1024;
        at[1].id = cudaLaunchAttributeClusterDimension;
        at[1].val.clusterDim.x = cl;
        at[1].val.clusterDim.y = 1;
        at[1].val.clusterDim.z = 1;
        f.attrs = at;
        f.numAttrs = 2;
        cudaLaunchKernelEx(&f, kF, sb, sst);
        cudaDeviceSynchronize();
        std::vector<uint64_t> a(256), b(128), bs(128);
        cudaMemcpy(a.data(), sa, 256 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), sb, 128 * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(bs.data(), sst, 128 * 8, cudaMemcpyDeviceToHost);
        const uint64_t ae = *std::max_element(a.begin(), a.end());
        std::sort(b.begin(), b.end());
        std::sort(bs.begin(), bs.end());
        if (rep >= 5) {
          g0.push_back(((double)b[0] - (double)ae) / 1e3);
          gm.push_back(((double)b[64] - (double)ae) / 1e3);
          gs.push_back(((double)bs[127] - (double)ae) / 1e3);
        }
      }
      std::sort(g0.begin(), g0.end());
      std::sort(gm.begin(), gm.end());
      std::sort(gs.begin(), gs.end());
      printf("gather-like (256 CTAs, %3d KB smem) -> fwd-like (128 CTAs, 200 KB, cluster %d): release - A end: first %.2f med %.2f; last B start - A end %.2f us (err %s)\n",
             gsm, cl, g0[g0.size() / 2], gm[gm.size() / 2], gs[gs.size() / 2], cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaMemset(cnt, 0, 4);
  kBar<<<148, 256>>>(cnt, arr, rel, R);
  cudaDeviceSynchronize();
  std::vector<uint64_t> a(R * 148), r(R * 148);
  cudaMemcpy(a.data(), arr, R * 148 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(r.data(), rel, R * 148 * 8, cudaMemcpyDeviceToHost);
  std::vector<double> gl, gm;
  for (int q = 2; q < R; ++q) {
    uint64_t last = 0;
    std::vector<uint64_t> rr;
    for (int c = 0; c < 148; ++c) {
      last = std::max(last, a[q * 148 + c]);
      rr.push_back(r[q * 148 + c]);
    }
    std::sort(rr.begin(), rr.end());
    gl.push_back(((double)rr[147] - (double)last) / 1e3);
    gm.push_back(((double)rr[74] - (double)last) / 1e3);
  }
  std::sort(gl.begin(), gl.end());
  std::sort(gm.begin(), gm.end());
  printf("grid barrier (148 CTAs): release - last arrival: median CTA %.2f us, last CTA %.2f us\n", gm[gm.size() / 2],
         gl[gl.size() / 2]);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
