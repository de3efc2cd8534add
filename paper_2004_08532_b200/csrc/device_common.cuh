// device_common.cuh -- device helpers of the CUDA path (sm_100a). Independent of oracle/ (shares no code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kge {

// ---- Philox4x32-10 (reading c.1: the counter RNG the north_star names; Random123 constants) ----
constexpr uint32_t kPhiloxM0 = 0xD2511F53u, kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u, kPhiloxW1 = 0xBB67AE85u;
constexpr uint32_t kTagNeg = 1, kTagPerm = 2, kTagInit = 3, kTagDeg = 4, kTagEval = 5, kTagRepart = 6;

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += kPhiloxW0;
      k1 += kPhiloxW1;
    }
    const uint32_t hi0 = __umulhi(kPhiloxM0, c.x), lo0 = kPhiloxM0 * c.x;
    const uint32_t hi1 = __umulhi(kPhiloxM1, c.z), lo1 = kPhiloxM1 * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// ---- positive selection (reading c.2): 4-round balanced Feistel on 2^m, cycle walk ----
struct FeistelDomain {
  uint32_t half;  // m/2 bits
  uint64_t n;
};

__host__ __device__ inline FeistelDomain make_feistel_domain(uint64_t n) {
  uint32_t lg = 0;
  while ((1ull << lg) < n) ++lg;
  uint32_t m = 2 * ((lg + 1) / 2);
  if (m < 2) m = 2;
  return FeistelDomain{m / 2, n};
}

__device__ __forceinline__ uint64_t feistel_round4(uint64_t x, uint32_t half, uint32_t k0, uint32_t k1, uint32_t epoch) {
  const uint64_t mask = (1ull << half) - 1;
  uint32_t L = (uint32_t)(x >> half), R = (uint32_t)(x & mask);
#pragma unroll
  for (uint32_t i = 0; i < 4; ++i) {
    const uint4 o = philox4x32_10(make_uint4(R, i, epoch, kTagPerm), k0, k1);
    const uint32_t F = (uint32_t)(o.x & mask);
    const uint32_t nl = R;
    R = L ^ F;
    L = nl;
  }
  return ((uint64_t)L << half) | R;
}

__device__ __forceinline__ uint64_t feistel_index(FeistelDomain dom, uint32_t k0, uint32_t k1, uint32_t epoch, uint64_t p) {
  uint64_t x = feistel_round4(p, dom.half, k0, k1, epoch);
  while (x >= dom.n) x = feistel_round4(x, dom.half, k0, k1, epoch);
  return x;
}

// ---- joint negatives (reading c.3): id = mulhi64(u, N_e) ----
__device__ __forceinline__ uint32_t neg_entity(uint32_t k0, uint32_t k1, uint64_t n_ent, uint32_t step, uint32_t cg,
                                               uint32_t j) {
  const uint4 o = philox4x32_10(make_uint4(j >> 1, cg, step, kTagNeg), k0, k1);
  const uint64_t u = (j & 1u) ? (((uint64_t)o.w << 32) | o.z) : (((uint64_t)o.y << 32) | o.x);
  return (uint32_t)__umul64hi(u, n_ent);
}

// degree-based in-batch negatives: batch position of slot j < k_deg, t = mulhi64(u, B)
__device__ __forceinline__ uint32_t deg_position(uint32_t k0, uint32_t k1, uint32_t B, uint32_t step, uint32_t cg,
                                                 uint32_t j) {
  const uint4 o = philox4x32_10(make_uint4(j >> 1, cg, step, kTagDeg), k0, k1);
  const uint64_t u = (j & 1u) ? (((uint64_t)o.w << 32) | o.z) : (((uint64_t)o.y << 32) | o.x);
  return (uint32_t)__umul64hi(u, (uint64_t)B);
}

// c.4 schedule: 0 = tail, 1 = head
__device__ __forceinline__ int corrupt_mode(int corrupt, uint32_t step, uint32_t cg) {
  if (corrupt == 0) return 0;
  if (corrupt == 1) return 1;
  return (int)((step + cg) & 1u);
}

// ---- init law (reading c.6): v = bound * ((float)(int32)u * 2^-31), u = Philox(col, row_lo, row_hi^(tab<<24), INIT).x
__device__ __forceinline__ float init_value(uint32_t k0, uint32_t k1, uint32_t table, uint64_t row, uint32_t col,
                                            float bound) {
  const uint4 o = philox4x32_10(make_uint4(col, (uint32_t)row, (uint32_t)(row >> 32) ^ (table << 24), kTagInit), k0, k1);
  const float f = __int2float_rn((int32_t)o.x);
  return __fmul_rn(bound, __fmul_rn(f, 0x1p-31f));
}

// ---- diagnostics: per-CTA globaltimer stamps (slot 0 = CTA start, 1..6 = kernel-defined phases, 7 = end) ----
constexpr int kTraceCtas = 2048, kTraceSlots = 8;
__device__ __forceinline__ void trace_stamp(uint64_t* trace, int kid, int slot) {
  if (trace == nullptr || threadIdx.x != 0) return;
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (cta >= kTraceCtas) return;
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  trace[((size_t)kid * kTraceCtas + cta) * kTraceSlots + slot] = t;
}

// last warp of the CTA to finish (slot 6, atomic max over the warps' lane 0): the CTA's true end when thread 0's
// warp is not the last one (row-parallel kernels whose warps work independently)
__device__ __forceinline__ void trace_warp_end(uint64_t* trace, int kid) {
  if (trace == nullptr || (threadIdx.x & 31) != 0) return;
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (cta >= kTraceCtas) return;
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  atomicMax(reinterpret_cast<unsigned long long*>(trace + ((size_t)kid * kTraceCtas + cta) * kTraceSlots + 6),
            (unsigned long long)t);
}

// ---- programmatic dependent launch: kernels of the step are launched with PDL so the next kernel's CTAs launch and
// run their prologue while this one drains; every kernel waits for its predecessor before touching its outputs ----
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- dataflow counters (StepBuffers::flow): release by the producer CTA, acquire by the consumer ----
// producer: every thread's writes precede the caller's __syncthreads(); one thread then publishes `n` units
__device__ __forceinline__ void flow_release(uint32_t* cnt, uint32_t n) {
  __threadfence();  // cumulative: the block's writes (ordered before this thread by the barrier) become visible first
  atomicAdd(cnt, n);
}
// consumer: spin (with back-off) until *cnt >= target; a protocol bug traps after ~2 s instead of hanging
__device__ __forceinline__ void flow_acquire(const uint32_t* cnt, uint32_t target) {
  const long long t0 = clock64();
  while (true) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
    if (v >= target) break;
    __nanosleep(32);
    if (clock64() - t0 > 4000000000ll) __trap();
  }
}
// generic-proxy writes acquired above are read next by TMA (async proxy)
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// the step's loss: device ring slot + (Slot::info[2..3]) a device-visible host address, if the caller gave one
__device__ __forceinline__ void store_loss(float* ring, const int32_t* info, float L) {
  ring[info[1]] = L;
  const uint64_t dst = ((uint64_t)(uint32_t)info[3] << 32) | (uint32_t)info[2];
  if (dst) *reinterpret_cast<volatile float*>(dst) = L;
}

// ---- small helpers ----
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float log_sigmoid(float x) {  // min(x,0) - log1p(exp(-|x|))  (reading c.9)
  return fminf(x, 0.f) - log1pf(expf(-fabsf(x)));
}
__device__ __forceinline__ float sigmoid(float x) {
  if (x >= 0.f) return 1.f / (1.f + expf(-x));
  const float e = expf(x);
  return e / (1.f + e);
}

// Pairwise ranking loss (reading c.9'): the hinge m = gamma - f+ + f- of one (positive, negative)
// pair; returns max(m, 0) and sets dL/df- = [m > 0] / (B k) (subgradient 0 at the hinge), act = [m > 0]
__device__ __forceinline__ float hinge_term(float f, float fpos, float gamma, float inv_bk, float& dldf, int& act) {
  const float m = gamma - fpos + f;
  act = m > 0.f ? 1 : 0;
  dldf = act ? inv_bk : 0.f;
  return act ? m : 0.f;
}

}  // namespace kge
