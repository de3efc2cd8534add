// rank_tc.cu -- the all-entity link-prediction protocol (PAPER.md:652-665 [5.3]) on the tensor
// cores. Scoring every entity against every query is the dense contraction S = O E^T (o_q = combine(h, r) or
// combine'(r, t)), run with tcgen05 kind::tf32 for the families that are contractions: DistMult /
// ComplEx (f = o . e), TransE-L2 (f = gamma - sqrt(||o||^2 - 2 o.e + ||e||^2)) and the Table-1 RotatE (f = gamma -
// (||o||^2 - 2 o.e + ||e||^2)). Handles whose negatives run in TF32 rank with this path; the FP32 handles and TransE-L1 /
// RotatE-modulus keep the FFMA streaming kernel (k_rank, step.cu).
//
//   pass 0 (k_rank_tc<FAM, 0>): the positive's score f(q, true) for each query tile: the same kernel with the tile's
//       true-entity rows as the B operand, the diagonal of the 128 x 128 tile -- the identical MMA sequence (K blocking,
//       issuer slices, partial-sum order) and epilogue formula the candidates go through, so an entity whose row equals
//       the true entity's ties it bit-exactly (pessimistic ties, reading c.15).
//   pass 1 (k_rank_tc<FAM, 1>): CTA = (128 queries, 128 entities); S tile in TMEM (two MMA-issuing threads, private
//       accumulators added in a fixed order); each epilogue thread owns a query row and counts the entities e != true
//       with f >= f(true), skipping filtered ids with a forward-only cursor over the query's sorted filter list
//       (exact: filtered candidates are never counted); integer partial counts meet in 64-bit atomics (order-free).
#include <cuda.h>

#include <algorithm>

#include "device_common.cuh"
#include "kge_internal.h"
#include "tc_ptx.cuh"

namespace kge {

using namespace tc;

constexpr int kRtStages = 3;  // 3 x 32 KB: two CTAs per SM (TMEM 2 x 256 columns)
constexpr int kRtThreads = 256;  // warps 0-3: epilogue (query rows); warp 4 lane 0: TMA; warps 5, 6 lane 0: MMA issuers

struct RankTcArgs {
  int32_t n, nkb;          // queries, k-blocks of 32 floats over d
  int64_t n_ent;
  float gamma;
  const float* onorm;      // [n_pad] ||o_q||^2
  const float* xnorm;      // [N_e] ||e||^2 (L2 families)
  const int32_t* true_e;   // [n_pad] the positive's entity
  float* s_true;           // [n_pad] pass 0 output, pass 1 input
  const int64_t* filt_off; // [n + 1] or nullptr
  const int32_t* filt;
  unsigned long long* cnt; // [n] rank - 1 accumulators
};

template <int FAM>
__device__ __forceinline__ float rt_score(float dot, float on, float xn, float gamma) {
  if (FAM == FAM_DOT) return dot;
  const float D2 = fmaxf(on - 2.f * dot + xn, 0.f);
  return FAM == FAM_L2 ? gamma - sqrtf(D2) : gamma - D2;
}

template <int FAM, int PASS>
__global__ void __launch_bounds__(kRtThreads, 1)
    k_rank_tc(const __grid_constant__ CUtensorMap mQ, const __grid_constant__ CUtensorMap mB, RankTcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  constexpr uint32_t A_BYTES = 128 * 128, STAGE = 2 * A_BYTES;
  __shared__ uint64_t full[kRtStages], empty[kRtStages], done;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * 128;
  const int64_t e0 = PASS == 0 ? q0 : (int64_t)blockIdx.y * 128;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);
    }
    mbar_init(&done, 2);
    fence_mbar_init();
    tma_prefetch(&mQ);
    tma_prefetch(&mB);
  }
  if (warp == 0) tmem_alloc(&tbase, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 4 && lane == 0) {  // TMA producer: A = 128 query rows, B = 128 entity (pass 0: true-entity) rows
    for (int kb = 0; kb < a.nkb; ++kb) {
      const int s = kb % kRtStages;
      if (kb >= kRtStages) mbar_wait(&empty[s], ((kb / kRtStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
      tma_load_3d(sa, &mQ, &full[s], kb * 32, q0, 0);
      tma_load_3d(sa + A_BYTES, &mB, &full[s], kb * 32, (int)e0, 0);
    }
  } else if ((warp == 5 || warp == 6) && lane == 0) {  // issuers: K = 8 slices 2 qi, 2 qi + 1 of every k-block
    const int qi = warp - 5;
    const uint32_t idesc = idesc_tf32(128, 128, false, false);
    const uint32_t acc = tmem + (uint32_t)(qi * 128);
    for (int kb = 0; kb < a.nkb; ++kb) {
      const int s = kb % kRtStages;
      mbar_wait(&full[s], (kb / kRtStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int sl = 2 * qi + h2;
        mma_tf32(acc, sdesc(sa + sl * 32, 16, 1024), sdesc(sb + sl * 32, 16, 1024), idesc, (kb | h2) ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  if (warp < 4) {
    const int rl = warp * 32 + lane, q = q0 + rl;
    const bool qok = q < a.n;
    const float on = qok && FAM != FAM_DOT ? a.onorm[q] : 0.f;
    const float ft = PASS == 1 && qok ? a.s_true[q] : 0.f;
    const int32_t te = qok ? a.true_e[q] : -1;
    int64_t fc = 0, fe = 0;
    if (PASS == 1 && qok && a.filt_off) {  // the first filtered id >= e0 (binary search), then forward only
      fc = a.filt_off[q];
      fe = a.filt_off[q + 1];
      int64_t lo = fc, hi = fe;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.filt[mid] < e0) lo = mid + 1; else hi = mid;
      }
      fc = lo;
    }
    mbar_wait(&done, 0);
    tc_fence_after();
    const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
    int cnt = 0;
#pragma unroll 1
    for (int cb = 0; cb < 4; ++cb) {
      uint32_t p0[32], p1[32];
      tmem_ld32_nw(trow + cb * 32, p0);
      tmem_ld32_nw(trow + 128 + cb * 32, p1);
      tmem_wait_ld();
      if (!qok) continue;
#pragma unroll
      for (int x = 0; x < 32; ++x) {
        const int col = cb * 32 + x;
        const float dot = __uint_as_float(p0[x]) + __uint_as_float(p1[x]);
        if (PASS == 0) {
          if (col == rl) a.s_true[q] = rt_score<FAM>(dot, on, FAM == FAM_DOT ? 0.f : a.xnorm[te], a.gamma);
        } else {
          const int64_t e = e0 + col;
          if (e >= a.n_ent || e == te) continue;
          if (a.filt_off) {
            while (fc < fe && a.filt[fc] < e) ++fc;
            if (fc < fe && a.filt[fc] == e) continue;
          }
          const float f = rt_score<FAM>(dot, on, FAM == FAM_DOT ? 0.f : a.xnorm[e], a.gamma);
          cnt += f >= ft ? 1 : 0;
        }
      }
    }
    if (PASS == 1 && qok && cnt) atomicAdd(a.cnt + q, (unsigned long long)cnt);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

// ---- prep: per query o_q, ||o_q||^2, the true entity's row and id (step.cu's combine); entity norms ----
__global__ void k_ent_norms(const float* __restrict__ ent, int64_t n_ent, int d, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= n_ent) return;
  const float4* x = reinterpret_cast<const float4*>(ent + e * d);
  float s = 0.f;
  for (int v = lane; v < (d >> 2); v += 32) {
    const float4 t = x[v];
    s += t.x * t.x + t.y * t.y + t.z * t.z + t.w * t.w;
  }
  s = warp_sum(s);
  if (lane == 0) out[e] = s;
}

cudaError_t launch_rank_prep(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                             int head, float* O, float* onorm, float* T, int32_t* true_e);  // step.cu

bool rank_tc_supported(const kge_handle* h) {
  const Dims& dm = h->dims;
  return h->P == 1 && dm.x3 == 0 && h->cfg.neg_precision == KGE_PREC_TF32 && dm.model != KGE_TRANSR &&
         dm.model != KGE_RESCAL && (dm.family == FAM_DOT || dm.family == FAM_L2 || dm.family == FAM_L2SQ) &&
         dm.d % 4 == 0;
}

template <int FAM>
static cudaError_t run_rank_tc(kge_handle* h, const CUtensorMap& mQ, const CUtensorMap& mT, const CUtensorMap& mE,
                               const RankTcArgs& ra, int nqt, int net) {
  const size_t smem = (size_t)kRtStages * 2 * 128 * 128 + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_rank_tc<FAM, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_rank_tc<FAM, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_rank_tc<FAM, 0><<<dim3(nqt, 1), kRtThreads, smem, h->stream>>>(mQ, mT, ra);
  k_rank_tc<FAM, 1><<<dim3(nqt, net), kRtThreads, smem, h->stream>>>(mQ, mE, ra);
  h->launches += 2;
  return cudaGetLastError();
}

// ranks of n queries on one side with every entity as a candidate (filter CSR on the device or nullptr)
cudaError_t launch_rank_tc(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, int head,
                           const int64_t* filt_off, const int32_t* filt, int64_t* ranks) {
  const Dims& dm = h->dims;
  const int64_t n_pad = (n + 127) / 128 * 128;
  const int dp = dm.dp;
  float* O = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&O, (size_t)(2 * n_pad * dp + 2 * n_pad + dm.n_entities) * 4 + n_pad * 4,
                                  h->stream);
  if (e != cudaSuccess) return e;
  float* T = O + n_pad * dp;
  float* onorm = T + n_pad * dp;
  float* s_true = onorm + n_pad;
  float* xnorm = s_true + n_pad;
  int32_t* true_e = reinterpret_cast<int32_t*>(xnorm + dm.n_entities);
  e = cudaMemsetAsync(O, 0, (size_t)2 * n_pad * dp * 4, h->stream);  // padded rows / columns read as zero
  if (e == cudaSuccess) e = cudaMemsetAsync(ranks, 0, (size_t)n * 8, h->stream);
  if (e == cudaSuccess) e = launch_rank_prep(h, hs, rs, ts, n, head, O, onorm, T, true_e);
  if (e == cudaSuccess && dm.family != FAM_DOT) {
    k_ent_norms<<<(unsigned)((dm.n_entities * 32 + 255) / 256), 256, 0, h->stream>>>(h->ent, dm.n_entities, dm.d,
                                                                                     xnorm);
    ++h->launches;
    e = cudaGetLastError();
  }
  CUtensorMap mQ, mT, mE;
  const bool ok = e == cudaSuccess && make_map(&mQ, O, dp, (int)n_pad, 1, dp, 128, CU_TENSOR_MAP_SWIZZLE_128B) &&
                  make_map(&mT, T, dp, (int)n_pad, 1, dp, 128, CU_TENSOR_MAP_SWIZZLE_128B) &&
                  make_map(&mE, h->ent, dm.d, (int)dm.n_entities, 1, dm.d, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (e == cudaSuccess && !ok) e = cudaErrorInvalidValue;
  if (e == cudaSuccess) {
    RankTcArgs ra{(int32_t)n, (dm.d + 31) / 32, dm.n_entities, dm.gamma, onorm, xnorm, true_e, s_true, filt_off, filt,
                  reinterpret_cast<unsigned long long*>(ranks)};
    const int nqt = (int)(n_pad / 128), net = (int)((dm.n_entities + 127) / 128);
    if (dm.family == FAM_DOT) e = run_rank_tc<FAM_DOT>(h, mQ, mT, mE, ra, nqt, net);
    else if (dm.family == FAM_L2) e = run_rank_tc<FAM_L2>(h, mQ, mT, mE, ra, nqt, net);
    else e = run_rank_tc<FAM_L2SQ>(h, mQ, mT, mE, ra, nqt, net);
  }
  cudaError_t ef = cudaFreeAsync(O, h->stream);
  return e != cudaSuccess ? e : ef;
}

}  // namespace kge
