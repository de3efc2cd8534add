// tc.cu -- tcgen05 tensor-core path of the chunked negative contraction (Sec. 3.3: "converted into
// a generalized matrix multiplication") for the GEMM-shaped score families: DistMult / ComplEx (f = o . x') and
// TransE-L2 (f = gamma - sqrt(||o||^2 - 2 o.x' + ||x'||^2)). kind::tf32 on fp32 rows, fp32 accumulators in TMEM,
// operands staged by TMA through an mbarrier pipeline, one elected thread issues the MMAs.
//
//   k_tc_fwd : S_c = O_c X'_c^T (M = 128 rows of O, N = NT negatives, K = dp); fused epilogue straight from TMEM:
//              f-, logistic-loss partial, dL/dS coefficient W (reading c.9).
//   k_tc_bwd : z = 0: dO_c = W_c X'_c   (M = 128 positives, N = a quarter of dp, K = k; A K-major, B MN-major)
//              z = 1: dX'_c = W_c^T O_c (M = 128 negatives, N = a quarter of dp, K = g; A and B MN-major)
//              TransE-L2 corrections dO = rowsum(W) o - W X', dX' = colsum(W) x' - W^T O take rowsum / colsum from
//              deterministic partial sums the forward epilogue writes (fixed summation order).
// Grids are sized for parallelism (64 CTAs each at the Freebase shape): every CTA of this latency-bound step streams
// its operands at the per-SM TMA rate, so more, smaller tiles finish sooner.
// Operand formats and descriptors: tc_ptx.cuh. MN-major tf32 needs the SWIZZLE_128B_BASE32B layout (TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B; 4-row K atoms, SBO = 512 B) -- verified by tools/tc_probe.cu.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kge_internal.h"
#include "tc_ptx.cuh"

namespace kge {

using namespace tc;

struct TcState {
  CUtensorMap mO_E;          // dO epilogue operand (O rows, 4D K-major SW128), box {32, 64, 4}
  CUtensorMap mO_F;          // fwd O operand (4D {32, rows, k-blocks, chunk}): box {32, 128, 1 (cx > 1) | kFwdKpb}
  CUtensorMap mX_F;          // fwd X' operand (4D): box {32, kNT, kFwdKpb}
  CUtensorMap mW_K;          // dO operand A (K-major), box {32, 128}
  CUtensorMap mX_MN, mO_MN;  // B operands of dO / dX' (MN-major, 128B_ATOM_32B), box {32, 32}
  CUtensorMap mW_MN;         // A operand of dX' (MN-major), box {32, 32}
  CUtensorMap mX_E;          // dX' epilogue operand (X' rows, 4D K-major SW128), box {32, 64, 4}
  float4* xbuf = nullptr;    // split-K exchange of the backward pairs (L2-resident scratch)
  CUtensorMap mG_S, mR_S, mD_S;
  CUtensorMap mG_S1, mG_L1;  // lag = 1: the same maps over the second (odd-step) Gocc buffer
  CUtensorMap mG_L;          // fused chain: gx rows of Gocc (written by k_gather), box {32, 64}
  // BF16 path (KGE_PREC_BF16): the same operand views over the bf16 copies, 64-element (128-byte) k-blocks
  CUtensorMap mO_F16, mX_F16, mW_K16, mW_MN16, mX_MN16, mO_MN16;
  // 3xTF32 path (KGE_PREC_3XTF32): the contraction maps above point at the hi parts, these at the lo parts
  CUtensorMap mO_Fl, mX_Fl, mW_Kl, mW_MNl, mX_MNl, mO_MNl;
  int fwd_cx = 1;  // backward TMA-store targets: Gocc, Grel, dO (SW128), box {32, 32}
  bool ok = false;
};

constexpr int kNT = 32;         // negatives per forward CTA
constexpr int kIssuers = 4;     // MMA-issuing threads per CTA (one per K = 8 slice of a 32-float k-block)
constexpr int kFwdKpb = 4;      // forward: k-blocks (32 floats of K) per pipeline stage = per TMA instruction
constexpr int kFwdStages = 2;   // forward stages of kFwdKpb k-blocks (A 64 KB + B 16 KB each)
constexpr int kBwdKpb = 2;      // backward: k-blocks per stage (one 4D box per operand)
constexpr int kBwdStages = 2;   // stages of kBwdKpb k-blocks: each split-K half (K = 128) is exactly two
constexpr int kNSplit = 4;      // column ranges of dp per backward tile
constexpr int kThreads = (8 + 4) * 32;  // backward: warps 0-7 = finalise (they alone run the prologue loads, so no
                                       // role thread waits at a reconvergence point behind a load), lane 0 of warps
                                       // 8-11 = the kIssuers MMA issuers, the first of them also the TMA producer
static_assert(kIssuers == 4, "the epilogues add exactly four partial accumulators");
constexpr int kFwdThreads = 256;  // forward: 8 epilogue warps (two per TMEM lane quarter, 16 negatives each) so the
                                  // transcendental chains of the loss epilogue have latency hiding

struct TcArgs {
  Dims dm;
  int32_t dp, kp;
  const float* O;
  const float* X;
  const float* onorm;
  const float* xnorm;
  float* W;
  float* lneg;
  float* dO;
  float* Gocc;
  float* rowsum_part;  // [B x nrp]   partial sums of W over the forward CTA's 32 negatives
  float* colsum_part;  // [C*k x ncp] partial sums of W over the forward CTA's 128 positives
  int32_t nrp, ncp;
  // fused positive chain rule (TransE-L2): the dO epilogue adds the positive-score gradient and applies the chain rule
  // through o = h + r / t - r itself, writing Gocc (H, T rows) and Grel instead of dO; CTA 0 reduces the loss
  int32_t fuse;
  Slot s;
  EntRows ent;
  const float* wpos;
  const float* pstat;
  const float* lpos;
  float* Grel;
  float* loss;
  int32_t* flags;
  int32_t n_neg_parts;
  float inv_bk;    // 1 / (B k), the dL/df- scale (reading c.9)
  float4* xbuf;    // backward split-K exchange scratch
  uint32_t* flow;  // dataflow counters (StepBuffers::flow)
  int32_t fwd_per_chunk;  // forward CTAs per chunk (the backward's target on flow[C + c])
  int32_t fwd_cx;  // forward cluster size along x: the CTAs of one 128-positive tile share its O tile by TMA multicast
  float* fdbg;     // KGE_OPT_CAPTURE_NEG: [B x k] negative pair scores, or nullptr
  int32_t* pcnt;   // pairwise ranking loss: active hinges per positive (StepBuffers::pcnt)
  uint16_t* W16;   // BF16 path: the forward writes dL/dS here (bf16, pitch kp16) instead of W
  int32_t dp16, kp16;
  float* W_hi;     // 3xTF32 path: dL/dS split into tf32 hi + lo (pitch kp) instead of W
  float* W_lo;
};

// f+ from the positive's pair statistic (k_gather's pstat), as the FFMA path's pair_score_from
template <int FAM>
__device__ __forceinline__ float pair_score_from_tc(float stat, float gamma) {
  return FAM == FAM_DOT ? stat : (FAM == FAM_L2 ? gamma - sqrtf(stat) : gamma - stat);
}

// families scored through the expansion ||o - x||^2 = ||o||^2 - 2 o.x + ||x||^2 (reading c.8): TransE-L2 (f = gamma -
// sqrt) and the Table-1 squared RotatE (f = gamma - ||o - x||^2 on the [re | im] rows, o = h e^{i theta} / t e^{-i theta})
template <int FAM>
__host__ __device__ constexpr bool expands() { return FAM == FAM_L2 || FAM == FAM_L2SQ; }

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return (uint8_t*)(((uintptr_t)p + 1023) & ~(uintptr_t)1023);
}

__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr, uint32_t lbo) {
  // SWIZZLE_128B_BASE32B (layout type 1), SBO = 512 B between 4-row K atoms
  uint64_t d = sdesc(saddr, lbo, 512);
  d &= ~((uint64_t)7 << 61);
  d |= (uint64_t)1 << 61;
  return d;
}

// ------------------------------------------------------------------------------------------------
// forward
// ------------------------------------------------------------------------------------------------
// BF: BF16 operands (kind::f16, k-blocks of 64 elements = the same 128-byte rows as the TF32 k-blocks of 32), W out
// in bf16
// X3: 3xTF32 split precision (KGE_PREC_3XTF32): every operand x = hi + lo with hi = x with the low 13 mantissa bits
// cleared (exactly a tf32 value) and lo = x - hi (exact); S = O_hi X_hi^T + O_hi X_lo^T + O_lo X_hi^T accumulated in
// fp32 TMEM -- the dropped O_lo X_lo^T term is ~2^-22 relative, FP32-level accuracy on the tensor cores. A stage
// holds the hi and the lo operands of half as many k-blocks (the same shared-memory footprint).
template <int FAM, bool BF, bool X3 = false>
__global__ void __launch_bounds__(kFwdThreads, 1)
    k_tc_fwd(const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mX,
             const __grid_constant__ CUtensorMap mOl, const __grid_constant__ CUtensorMap mXl, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr int KPB = X3 ? kFwdKpb / 2 : kFwdKpb;  // k-blocks per stage
  constexpr uint32_t A_KB = 128 * 128, B_KB = kNT * 128;  // one k-block of A (O rows) / B (X' rows)
  constexpr uint32_t A_BYTES = KPB * A_KB, HALF = KPB * (A_KB + B_KB), STAGE = (X3 ? 2 : 1) * HALF;
  constexpr int kHalf = kNT / 2;  // columns this CTA finalises
  __shared__ uint64_t full[kFwdStages], empty[kFwdStages], done;
  __shared__ uint32_t tbase;
  __shared__ float s_xn[kHalf];
  __shared__ float s_red[8];
  __shared__ float s_col[4][kHalf];
  __shared__ float s_rs[2][128];
  float* xch = reinterpret_cast<float*>(smem + kFwdStages * STAGE);  // [128 rows][kHalf]: the peer's partial sums
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // Split-K pair: the CTAs x = 2 t + ks (t = 32-negative tile) share the tile, ks = 0 / 1 contracting the first /
  // second half of the k-blocks; after the main loop each sends the other half of its 32 columns of partial sums
  // to the peer through distributed shared memory, and finalises kHalf columns (the sum is always P0 + P1).
  // Cluster = cxn tiles x 2 halves: the CTAs with the same ks share one O operand, CTA (ntl, ks) loading k-block ntl
  // of every stage and multicasting it (cxn = kFwdKpb) -- a stage is refilled once all of them released it.
  const int cxn = a.fwd_cx, cl = 2 * cxn;
  const uint32_t crank = cluster_ctarank();
  const int ks = (int)(crank & 1), ntl = (int)(crank >> 1);
  const uint16_t mmask = (uint16_t)(cxn > 1 ? (0x55u << ks) & ((1u << cl) - 1) : 0);  // same-ks CTAs
  const int c = blockIdx.z, i0 = blockIdx.y * 128, t = blockIdx.x >> 1, j0 = t * kNT;
  const int nkb = BF ? a.dp16 / 64 : a.dp / 32, kh = (nkb + 1) / 2;
  const int kb0 = ks ? kh : 0, kb1 = ks ? nkb : kh;
  const int nst = (kb1 - kb0 + KPB - 1) / KPB;
  const int jf0 = j0 + ks * kHalf;  // first column this CTA finalises
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kIssuers * cxn);
    }
    mbar_init(&done, kIssuers);
    fence_mbar_init();
    tma_prefetch(&mO);
    tma_prefetch(&mX);
  }
  if (warp == 0) tmem_alloc(&tbase, kIssuers * kNT);
  if (a.flow) {
    // dataflow (KGE_FLOW=1): this chunk's g + k rows (O, X', norms) are final once k_gather published them -- no
    // wait for the whole gather grid; the thread that acquires is also the TMA producer (proxy fence before its loads)
    pdl_trigger();
    if (threadIdx.x == 0) {
      flow_acquire(&a.flow[c], (uint32_t)(dm.g + dm.k));
      fence_proxy_async_global();
    }
  } else {
    pdl_wait();  // predecessor (gather) complete: O, X', norms are final
    pdl_trigger();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync();  // every CTA's barriers are initialised before any multicast or DSMEM store lands
  const uint32_t tmem = tbase;
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 1);

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int q = 0; q < nst; ++q) {
      const int s = q % kFwdStages;
      if (q >= kFwdStages) mbar_wait(&empty[s], ((q / kFwdStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      // a box always delivers its full size (out-of-range rows / k-blocks are zero-filled); with multicast only the
      // k-blocks of this half that exist are loaded (one box each)
      const int kq = kb0 + q * KPB, nk = min(KPB, kb1 - kq);
      mbar_arrive_expect_tx(&full[s], (cxn > 1 ? nk * A_KB + KPB * B_KB : STAGE));
      if (cxn > 1) {
        if (ntl < nk) tma_load_4d_mc(sa + ntl * A_KB, &mO, &full[s], 0, i0, kq + ntl, c, mmask);
      } else {
        tma_load_4d(sa, &mO, &full[s], 0, i0, kq, c);
      }
      tma_load_4d(sa + A_BYTES, &mX, &full[s], 0, j0, kq, c);
      if (X3) {  // the lo halves of the same k-blocks
        tma_load_4d(sa + HALF, &mOl, &full[s], 0, i0, kq, c);
        tma_load_4d(sa + HALF + A_BYTES, &mXl, &full[s], 0, j0, kq, c);
      }
    }
  } else if (warp >= 8 - kIssuers && lane == 0) {
    // MMA issuers: a single thread issues one tcgen05.mma per ~130 cycles whatever N is (measured, tools/mma_probe.cu),
    // so the K = 8 slices of each k-block are dealt to kIssuers threads, issuer q accumulating slice q of every
    // k-block into its own TMEM columns [q * kNT, (q + 1) * kNT); the epilogue adds the partials in a fixed order
    const int q = warp - (8 - kIssuers);
    const uint32_t idesc = BF ? idesc_bf16(128, kNT, false, false) : idesc_tf32(128, kNT, false, false);
    const uint32_t acc = tmem + (uint32_t)(q * kNT);
    for (int st = 0; st < nst; ++st) {
      const int s = st % kFwdStages;
      mbar_wait(&full[s], (st / kFwdStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
      const int nk = min(KPB, kb1 - (kb0 + st * KPB));
      for (int b = 0; b < nk; ++b) {
        // slice q of the k-block: K = 8 tf32 or 16 bf16 = 32 bytes into each 128-byte row
        const uint64_t ad = sdesc(sa + b * A_KB + q * 32, 16, 1024), bd = sdesc(sb + b * B_KB + q * 32, 16, 1024);
        if (BF) {
          mma_bf16(acc, ad, bd, idesc, (st | b) ? 1u : 0u);
        } else {
          mma_tf32(acc, ad, bd, idesc, (st | b) ? 1u : 0u);
          if (X3) {  // + hi x lo + lo x hi
            mma_tf32(acc, ad, sdesc(sb + HALF + b * B_KB + q * 32, 16, 1024), idesc, 1u);
            mma_tf32(acc, sdesc(sa + HALF + b * A_KB + q * 32, 16, 1024), bd, idesc, 1u);
          }
        }
      }
      if (cxn > 1)
        mma_commit_mc(&empty[s], mmask);
      else
        mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  // epilogue: thread <-> row i (TMEM lane 32*(warp%4) + lane); warp/4 = hf picks 8 of the kHalf finalised columns
  // and 8 of the kHalf columns sent to the peer
  const int lg = warp & 3, hf = warp >> 2;
  const int rl = lg * 32 + lane, i = i0 + rl;
  const bool iok = i < dm.g;
  const float on = iok && expands<FAM>() ? a.onorm[(int64_t)c * dm.g + i] : 0.f;  // loaded while the MMAs run
  const bool pairwise = dm.loss == KGE_LOSS_PAIRWISE;
  const float fpos = iok && pairwise ? pair_score_from_tc<FAM>(a.pstat[(int64_t)c * dm.g + i], dm.gamma) : 0.f;
  if (threadIdx.x < kHalf) {
    const int jj = jf0 + threadIdx.x;
    s_xn[threadIdx.x] = expands<FAM>() && jj < dm.k ? a.xnorm[(int64_t)c * dm.k + jj] : 0.f;
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 2);
  // own partial sums of the kept (kc) and sent (sc) column groups: ((p0 + p1) + p2) + p3
  const int kc = ks * kHalf + hf * 8, sc = (1 - ks) * kHalf + hf * 8;
  float v[8], w[8];
  if (nst > 0) {
    const uint32_t tl = tmem + ((uint32_t)(lg * 32) << 16);
    uint32_t pv[kIssuers][8], pw[kIssuers][8];  // all eight loads in flight, one wait
#pragma unroll
    for (int q = 0; q < kIssuers; ++q) {
      tmem_ld8_nw(tl + q * kNT + kc, pv[q]);
      tmem_ld8_nw(tl + q * kNT + sc, pw[q]);
    }
    tmem_wait_ld();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v[u] = __uint_as_float(pv[0][u]);
      w[u] = __uint_as_float(pw[0][u]);
    }
#pragma unroll
    for (int q = 1; q < kIssuers; ++q)
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[u] += __uint_as_float(pv[q][u]);
        w[u] += __uint_as_float(pw[q][u]);
      }
  } else {
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = w[u] = 0.f;
  }
  {  // send: the peer's xch[row][hf * 8 ..] (its kept columns are our sent ones)
    const uint32_t dst = mapa_shared(smem_u32(xch + rl * kHalf + hf * 8), crank ^ 1u);
    st_cluster_v4(dst, w[0], w[1], w[2], w[3]);
    st_cluster_v4(dst + 16, w[4], w[5], w[6], w[7]);
  }
  cluster_sync();  // release our stores / acquire the peer's
  {
    const float4 x0 = *reinterpret_cast<const float4*>(xch + rl * kHalf + hf * 8);
    const float4 x1 = *reinterpret_cast<const float4*>(xch + rl * kHalf + hf * 8 + 4);
    const float xp[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ks == 0 ? v[u] + xp[u] : xp[u] + v[u];  // always P0 + P1
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 3);
  const float inv_bk = a.inv_bk;
  float lsum = 0.f, rsum = 0.f, lprod = 1.f;
  int nact = 0;
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const int j = jf0 + hf * 8 + jj;
    float coef = 0.f;
    if (iok && j < dm.k) {
      float f, rD = 1.f;
      if (FAM == FAM_DOT) {
        f = v[jj];
      } else if (FAM == FAM_L2) {  // TransE-L2 by expansion, clamped at 0 before the root (reading c.8)
        const float D2 = fmaxf(on - 2.f * v[jj] + s_xn[hf * 8 + jj], 0.f);
        rD = fminf(rsqrtf(D2), 1e12f);
        f = dm.gamma - D2 * rD;
      } else {  // RotatE (Table 1, squared) by expansion: f = gamma - D^2, df/do = -2 (o - x)
        const float D2 = fmaxf(on - 2.f * v[jj] + s_xn[hf * 8 + jj], 0.f);
        rD = 2.f;
        f = dm.gamma - D2;
      }
      if (a.fdbg) a.fdbg[((int64_t)c * dm.g + i) * dm.k + j] = f;
      // e = exp(-|f|): sigma(f) = f>=0 ? 1/(1+e) : e/(1+e);  -log sigma(-f) = max(f,0) + log1p(e). Three MUFU ops
      // per element (rsqrt, ex2, rcp): the log1p terms are summed as one log of their product (each factor in (1, 2],
      // 8 factors: no overflow; relative error ~8 ulp of the product, far inside the TC path's 2e-3)
      float dLdf;
      if (pairwise) {  // reading c.9': hinge gamma - f+ + f-
        int act;
        lsum += hinge_term(f, fpos, dm.gamma, inv_bk, dLdf, act);
        nact += act;
      } else {
        const float e = __expf(-fabsf(f));
        float r1;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(1.f + e));
        lsum += fmaxf(f, 0.f);
        lprod *= 1.f + e;
        dLdf = (f >= 0.f ? r1 : e * r1) * inv_bk;
      }
      coef = FAM == FAM_DOT ? dLdf : -dLdf * rD;
    }
    v[jj] = coef;
    rsum += coef;
  }
  lsum += __logf(lprod);
  if (nact) atomicAdd(&a.pcnt[(int64_t)c * dm.g + i], nact);  // integer: exact in any order
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 4);
  if (iok && X3) {  // dL/dS split hi + lo for the 3xTF32 backward GEMMs
    float* hrow = a.W_hi + ((int64_t)c * dm.g + i) * a.kp + jf0 + hf * 8;
    float* lrow = a.W_lo + ((int64_t)c * dm.g + i) * a.kp + jf0 + hf * 8;
#pragma unroll
    for (int jj = 0; jj < 8; ++jj)
      if (jf0 + hf * 8 + jj < dm.k) {
        const float hi = __uint_as_float(__float_as_uint(v[jj]) & 0xFFFFE000u);
        hrow[jj] = hi;
        lrow[jj] = v[jj] - hi;
      }
  } else if (iok && BF) {  // dL/dS in bf16 for the backward GEMMs (the pads beyond k stay zero)
    uint16_t* wrow = a.W16 + ((int64_t)c * dm.g + i) * a.kp16 + jf0 + hf * 8;
    if (jf0 + hf * 8 + 8 <= dm.k) {
      uint4 u;
      __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]), p1 = __floats2bfloat162_rn(v[2], v[3]);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(v[4], v[5]), p3 = __floats2bfloat162_rn(v[6], v[7]);
      u.x = *reinterpret_cast<uint32_t*>(&p0);
      u.y = *reinterpret_cast<uint32_t*>(&p1);
      u.z = *reinterpret_cast<uint32_t*>(&p2);
      u.w = *reinterpret_cast<uint32_t*>(&p3);
      *reinterpret_cast<uint4*>(wrow) = u;
    } else {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (jf0 + hf * 8 + jj < dm.k) {
          const __nv_bfloat16 b16 = __float2bfloat16_rn(v[jj]);
          wrow[jj] = *reinterpret_cast<const uint16_t*>(&b16);
        }
    }
  } else if (iok) {
    float* wrow = a.W + ((int64_t)c * dm.g + i) * a.kp + jf0 + hf * 8;
    if (jf0 + hf * 8 + 8 <= dm.k && (a.kp & 3) == 0) {
      float4* dst = reinterpret_cast<float4*>(wrow);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)  // static indices keep v[] in registers
        if (jf0 + hf * 8 + jj < dm.k) wrow[jj] = v[jj];
    }
  }
  if (expands<FAM>()) {
    s_rs[hf][rl] = rsum;
    // column sums over this warp's 32 rows for its 8 columns: transposing butterfly (fixed order) over the low 3
    // lane bits, then the four 8-lane groups are added; lane l (< 8) ends with column l
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) {
#pragma unroll
      for (int q = 0; q < off; ++q) {
        const bool upper = (lane & off) != 0;
        const float send = upper ? v[q] : v[q + off];
        const float keep = upper ? v[q + off] : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 8);
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
    if (lane < 8) s_col[lg][hf * 8 + lane] = v[0];
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 5);
  lsum = warp_sum(lsum);
  if (lane == 0) s_red[warp] = lsum;
  tc_fence_before();
  __syncthreads();
  if (expands<FAM>()) {
    if (threadIdx.x < 128 && i0 + (int)threadIdx.x < dm.g)  // one row-sum partial per (row, half tile): 16 columns
      a.rowsum_part[((int64_t)c * dm.g + i0 + threadIdx.x) * a.nrp + blockIdx.x] =
          s_rs[0][threadIdx.x] + s_rs[1][threadIdx.x];
    if (threadIdx.x >= 128 && threadIdx.x < 128 + kHalf && jf0 + (int)threadIdx.x - 128 < dm.k) {
      const int u = threadIdx.x - 128;
      a.colsum_part[((int64_t)c * dm.k + jf0 + u) * a.ncp + blockIdx.y] =
          ((s_col[0][u] + s_col[1][u]) + s_col[2][u]) + s_col[3][u];
    }
  }
  if (threadIdx.x == 0) {
    float tt = 0.f;
    for (int w8 = 0; w8 < 8; ++w8) tt += s_red[w8];
    a.lneg[((int64_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tt;
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 6);
  __syncthreads();
  if (a.flow && threadIdx.x == 0) flow_release(&a.flow[dm.C + c], 1u);  // W, row / column partials and lneg
  if (cxn > 1) cluster_sync();  // no CTA leaves while a peer's MMA commit may still arrive on its barriers
  if (warp == 0) tmem_dealloc(tmem, kIssuers * kNT);
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 7);
}

// ------------------------------------------------------------------------------------------------
// backward: z = 0 -> dO tile (128 positives of chunk y), z = 1 -> dX' tile (128 negatives of chunk y);
// blockIdx.x = 2 (row tile * kNSplit + column part) + ks. Split-K pair (cluster of 2): ks = 0 / 1 contracts the first /
// second half of K; each CTA then hands the peer the 64 rows the peer finalises (through L2, coalesced float4 columns)
// and finalises its own 64 rows of the 128 x (nb * 32) tile -- the sum is always P0 + P1.
// ------------------------------------------------------------------------------------------------
// Columns of backward part p (of kNSplit), in 32-column units: the TF32 path cuts the dp / 32 column blocks of the
// rows, the BF16 path the dp16 / 64 blocks of 64 columns (two 32-column units each; TMA boxes and MN-major atoms are
// 64 bf16 wide) -- the TMEM columns and the finalise keep 32-column units either way
template <bool BF>
__device__ __forceinline__ void bwd_part(const TcArgs& a, int p, int& b0, int& nb) {
  if (BF) {
    const int n64 = a.dp16 / 64;
    const int c0 = p * n64 / kNSplit, c1 = (p + 1) * n64 / kNSplit;
    b0 = 2 * c0;
    nb = 2 * (c1 - c0);
  } else {
    const int n32 = a.dp / 32;
    b0 = p * n32 / kNSplit;
    nb = (p + 1) * n32 / kNSplit - b0;
  }
}

template <int FAM, bool BF, bool X3 = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_bwd(const __grid_constant__ CUtensorMap mW_K, const __grid_constant__ CUtensorMap mW_MN,
             const __grid_constant__ CUtensorMap mX_MN, const __grid_constant__ CUtensorMap mO_MN,
             const __grid_constant__ CUtensorMap mO_E, const __grid_constant__ CUtensorMap mX_E,
             const __grid_constant__ CUtensorMap mG_S, const __grid_constant__ CUtensorMap mR_S,
             const __grid_constant__ CUtensorMap mD_S, const __grid_constant__ CUtensorMap mG_L,
             const __grid_constant__ CUtensorMap mW_Kl, const __grid_constant__ CUtensorMap mW_MNl,
             const __grid_constant__ CUtensorMap mX_MNl, const __grid_constant__ CUtensorMap mO_MNl, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  __shared__ uint64_t full[kBwdStages], empty[kBwdStages], done, selfbar;
  __shared__ uint32_t tbase;
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool pass_x = blockIdx.z == 1;
  const int ks = blockIdx.x & 1, tp = blockIdx.x >> 1;
  const int c = blockIdx.y, part = tp % kNSplit, r0 = (tp / kNSplit) * 128;
  const int nrows = pass_x ? dm.k : dm.g;
  int b0, nb;  // this CTA's 32-column blocks
  bwd_part<BF>(a, part, b0, nb);
  if (r0 >= nrows || nb == 0 || b0 * 32 >= dm.d) {  // uniform per CTA pair, before any barrier / TMEM use
    pdl_trigger();
    return;
  }
  const int nk = pass_x ? dm.g : dm.k;  // contraction length
  constexpr int KB = BF ? 64 : 32;      // contraction rows per k-block (one 128-byte row of the K-major operand)
  const int nkb = (nk + KB - 1) / KB, kh = (nkb + 1) / 2;
  const int kb0 = ks ? kh : 0, kb1 = ks ? nkb : kh;
  constexpr int KPB = X3 ? kBwdKpb / 2 : kBwdKpb;  // k-blocks per stage (3xTF32: hi and lo of half as many)
  const int nst = (kb1 - kb0 + KPB - 1) / KPB;
  constexpr uint32_t A_BYTES = KPB * 16384, B_BYTES = KPB * 4 * 4096, HALF = A_BYTES + B_BYTES;
  constexpr uint32_t STAGE = (X3 ? 2 : 1) * HALF;
  // bytes between MN blocks (32 tf32 / 64 bf16 columns) of an MN-major stage operand
  constexpr uint32_t KROWS_B = KPB * KB * 128;
  // shared memory: [stages][self: this CTA's 64 finalised rows x 4 column blocks of O (dO) / X' (dX'), SW128]
  // after the main loop the stage area holds xown ([32 float4 columns][64 rows]) and the TMA-store staging
  uint8_t* self_smem = smem + kBwdStages * STAGE;
  float4* xown = reinterpret_cast<float4*>(smem);
  uint8_t* stg = smem + 32768 + warp * 12288;  // 3 tiles x 4 KB per warp
  const int rfin0 = ks * 64;                    // first tile row this CTA finalises
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kIssuers);
    }
    mbar_init(&done, kIssuers);
    mbar_init(&selfbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, kIssuers * 128);
  if (a.flow) {  // dataflow: W and the row / column partials of chunk c are final once its forward CTAs published them
    pdl_trigger();
    if (threadIdx.x == 0) flow_acquire(&a.flow[dm.C + c], (uint32_t)a.fwd_per_chunk);
  } else {
    pdl_wait();  // predecessor (forward) complete: W and the row / column partial sums are final
    pdl_trigger();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 1);

  // ---- finalise prologue, issued before the main loop so its global loads (row / column partial sums of W, the
  // positive's scale and the uncorrupted entity row) overlap the MMAs: warp w finalises rows rfin0 + 32 (w / 4) +
  // lane of column block w % 4 ----
  const int b = warp & 3, fr = (warp >> 2) * 32 + lane;
  const int rl = rfin0 + fr, r = r0 + rl;
  const bool rok = r < nrows;
  const int d = dm.d;
  const bool fuse = FAM == FAM_L2 && a.fuse && !pass_x;
  const int e0 = (b0 + b) * 32;
  const bool bok = warp < 8 && b < nb && e0 < d;
  // The loads are issued by every thread except the TMA producer and the MMA issuers, which run their loops first
  // and load afterwards; the additions happen at finalise time so nothing here waits on a load.
  const bool role = warp >= 8;
  float4 cpart[4];  // rowsum(W) partials (nrp = 16 -> 4 float4) for dO, colsum(W) partials (ncp) for dX'
  const int pi = c * dm.g + r;
  int mode = 0;
  auto prologue = [&]() {
#pragma unroll
    for (int q = 0; q < 4; ++q) cpart[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (expands<FAM>() && rok && bok) {
      const int np = pass_x ? a.ncp : a.nrp;
      const float* pp = pass_x ? a.colsum_part + ((int64_t)c * dm.k + r) * a.ncp
                               : a.rowsum_part + ((int64_t)c * dm.g + r) * a.nrp;
      if (np == 16) {
#pragma unroll
        for (int q = 0; q < 4; ++q) cpart[q] = __ldcg(reinterpret_cast<const float4*>(pp) + q);
      } else {
        float t = 0.f;
        for (int q = 0; q < np; ++q) t += pp[q];
        cpart[0].x = t;
      }
    }
    mode = fuse ? a.s.mode[c] : 0;
  };
  if (!role) prologue();

  int loss_part = 0;  // the loss is reduced by the first CTA of (row tile 0, chunk 0) that has columns to process
  for (;; ++loss_part) {
    int lb0, lnb;
    bwd_part<BF>(a, loss_part, lb0, lnb);
    if (loss_part + 1 >= kNSplit || (lnb > 0 && lb0 * 32 < d)) break;
  }
  if (fuse && tp == loss_part && ks == 0 && blockIdx.y == 0 && warp == 1) {
    // deterministic loss (reading c.9): fixed lane assignment and order, identical to the unfused k_chain; it needs
    // every chunk's forward partials
    if (a.flow && lane == 0)
      for (int cc = 0; cc < dm.C; ++cc) flow_acquire(&a.flow[dm.C + cc], (uint32_t)a.fwd_per_chunk);
    __syncwarp();
    float sp = 0.f, sn = 0.f;
    for (int i = lane; i < dm.B; i += 32) sp += a.lpos[i];
    for (int q = lane; q < a.n_neg_parts; q += 32) sn += a.lneg[q];
    sp = warp_sum(sp);
    sn = warp_sum(sn);
    if (lane == 0) {
      const float L = sp / (float)dm.B + sn / ((float)dm.B * (float)dm.k);
      store_loss(a.loss, a.s.info, L);
      const bool bad = !isfinite(L);
      a.flags[2 + (a.s.info[0] & 1)] = bad ? 1 : 0;
      if (bad) a.flags[0] = 1;
    }
  }
  if (warp >= 8 && lane == 0) {
    // MMA issuers (see k_tc_fwd): issuer q takes the K = 8 slice q of every k-block into TMEM columns [128 q, +nb*32).
    // Issuer 0 is also the TMA producer (one box per operand per stage), keeping kBwdStages stages in flight: it only
    // ever waits for a stage its own previous MMAs already released, so the shared thread cannot deadlock.
    const int q = warp - 8;
    int issued = 0;
    auto produce = [&](int upto) {
      for (; issued < upto && issued < nst; ++issued) {
        const int s = issued % kBwdStages;
        if (issued >= kBwdStages) mbar_wait(&empty[s], ((issued / kBwdStages) - 1) & 1);
        uint8_t* sa = smem + s * STAGE;
        uint8_t* sb = sa + A_BYTES;
        const int kq = kb0 + issued * KPB;
        mbar_arrive_expect_tx(&full[s], STAGE);
        // TF32: blocks of 32 columns (4 per box); BF16: of 64 (2 per box) -- the same 128-byte rows
        if (!pass_x)
          tma_load_4d(sa, &mW_K, &full[s], 0, r0, kq, c);  // W[rows, k-blocks kq..]: [kb][128 rows][128 B]
        else
          tma_load_4d(sa, &mW_MN, &full[s], 0, kq * KB, r0 / KB, c);  // W^T: [j-blocks][K rows][128 B]
        tma_load_4d(sb, pass_x ? &mO_MN : &mX_MN, &full[s], 0, kq * KB, BF ? b0 / 2 : b0, c);  // [col blocks][K rows]
        if (X3) {  // the lo halves
          if (!pass_x)
            tma_load_4d(sa + HALF, &mW_Kl, &full[s], 0, r0, kq, c);
          else
            tma_load_4d(sa + HALF, &mW_MNl, &full[s], 0, kq * KB, r0 / KB, c);
          tma_load_4d(sb + HALF, pass_x ? &mO_MNl : &mX_MNl, &full[s], 0, kq * KB, b0, c);
        }
      }
    };
    if (q == 0) {
      fence_proxy_async_global();  // the forward's W (acquired by thread 0 before the barrier) is read by TMA
      produce(kBwdStages);
      if (expands<FAM>()) {
        const bool fz = FAM == FAM_L2 && a.fuse && !pass_x;
        mbar_arrive_expect_tx(&selfbar, (fz ? 8 : 4) * 8192);
        tma_load_4d(self_smem, pass_x ? &mX_E : &mO_E, &selfbar, 0, r0 + rfin0, b0, c);
        if (fz) {  // gx rows of the uncorrupted entities (written by k_gather): [4 col blocks][64 rows][128 B]
          const int orow = (a.s.mode[c] == 0 ? dm.B : 0) + c * dm.g + r0 + rfin0;
          for (int bb = 0; bb < 4; ++bb) tma_load_3d(self_smem + (4 + bb) * 8192, &mG_L, &selfbar, (b0 + bb) * 32, orow, 0);
        }
      }
    }
    const uint32_t idesc = BF ? idesc_bf16(128, nb * 32, pass_x, true) : idesc_tf32(128, nb * 32, pass_x, true);
    const uint32_t acc = tmem + (uint32_t)(q * 128);
    for (int st = 0; st < nst; ++st) {
      const int s = st % kBwdStages;
      if (q == 0 && st > 0) produce(st + kBwdStages);  // stage st + S - 1 needs stage st - 1 released
      mbar_wait(&full[s], (st / kBwdStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
      const int nkq = min(KPB, kb1 - (kb0 + st * KPB));
      for (int b = 0; b < nkq; ++b) {
        if (BF) {  // K slice q = 16 rows: 2048 B into an MN-major operand, 32 B into a K-major row
          const uint32_t koff = (uint32_t)(b * 64 + q * 16) * 128;
          const uint64_t ad = pass_x ? sdesc(sa + koff, KROWS_B, 1024) : sdesc(sa + b * 16384 + q * 32, 16, 1024);
          mma_bf16(acc, ad, sdesc(sb + koff, KROWS_B, 1024), idesc, (st | b) ? 1u : 0u);
        } else {
          const uint32_t koff = (uint32_t)(b * 32 + q * 8) * 128;  // K rows of an MN-major operand
          const uint64_t ad = pass_x ? sdesc_mn(sa + koff, KROWS_B) : sdesc(sa + b * 16384 + q * 32, 16, 1024);
          const uint64_t bd = sdesc_mn(sb + koff, KROWS_B);
          mma_tf32(acc, ad, bd, idesc, (st | b) ? 1u : 0u);
          if (X3) {  // + hi x lo + lo x hi
            const uint64_t al = pass_x ? sdesc_mn(sa + HALF + koff, KROWS_B)
                                       : sdesc(sa + HALF + b * 16384 + q * 32, 16, 1024);
            mma_tf32(acc, ad, sdesc_mn(sb + HALF + koff, KROWS_B), idesc, 1u);
            mma_tf32(acc, al, bd, idesc, 1u);
          }
        }
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  // ---- partial sums out of TMEM: warp w reads lane quarter w % 4, column blocks 2 (w / 4) + {0, 1} ----
  const int pair = tp + (gridDim.x >> 1) * (c + gridDim.y * blockIdx.z);
  float4* xsend = a.xbuf + ((int64_t)pair * 2 + ks) * (32 * 64);  // [32 float4 columns][64 rows] for the peer
  const float4* xpeer = a.xbuf + ((int64_t)pair * 2 + (1 - ks)) * (32 * 64);
  mbar_wait(&done, 0);
  tc_fence_after();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 2);
  if (warp < 8) {
    const int lq = warp & 3, rl = lq * 32 + lane;
    const bool mine = (rl >> 6) == ks;
    const int fr = rl & 63;
    const uint32_t trow = tmem + ((uint32_t)(lq * 32) << 16);
#pragma unroll
    for (int bb = 0; bb < 2; ++bb) {
      const int b = (warp >> 2) * 2 + bb;
      if (b >= nb) break;
      float v[32];
      if (nst > 0) {  // ((p0 + p1) + p2) + p3: fixed order, deterministic; two loads in flight per wait
        uint32_t pa[32], pb[32];
        tmem_ld32_nw(trow + b * 32, pa);
        tmem_ld32_nw(trow + 128 + b * 32, pb);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = __uint_as_float(pa[u]) + __uint_as_float(pb[u]);
        tmem_ld32_nw(trow + 256 + b * 32, pa);
        tmem_ld32_nw(trow + 384 + b * 32, pb);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = (v[u] + __uint_as_float(pa[u])) + __uint_as_float(pb[u]);
      } else {
#pragma unroll
        for (int u = 0; u < 32; ++u) v[u] = 0.f;
      }
      float4* dst = mine ? xown : xsend;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        dst[(b * 8 + u) * 64 + fr] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();  // xown complete
  cluster_sync();   // release xsend (global, cluster scope) / acquire the peer's
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 3);

  // ---- finalise ----
  if (bok) {
    // correction factor: the rowsum / colsum partials of W added in a fixed order
    float corr = cpart[0].x;
    if (expands<FAM>() && (pass_x ? a.ncp : a.nrp) == 16) {
      corr = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) corr = (((corr + cpart[q].x) + cpart[q].y) + cpart[q].z) + cpart[q].w;
    }
    // output tiles of these 32 rows: t = 0 the primary (dO | dX' | fused: gradient of the combined entity),
    // fused only: t = 1 gradient of the other entity, t = 2 relation gradient. Full 32-row warps stage each
    // 32 x 32 tile in shared memory in the SW128 layout and TMA-store it; a ragged warp stores its valid rows directly.
    const int wrow0 = r0 + rfin0 + (warp >> 2) * 32;
    const bool wtma = wrow0 + 32 <= nrows;
    const int ne = min(32, d - e0);
    int trow0[3];
    trow0[0] = pass_x ? 2 * dm.B + c * dm.k + wrow0 : (fuse && mode == 1 ? dm.B : 0) + c * dm.g + wrow0;
    trow0[1] = (mode == 0 ? dm.B : 0) + c * dm.g + wrow0;
    trow0[2] = c * dm.g + wrow0;
    float* gdst[3];
    gdst[0] = pass_x ? a.Gocc + ((int64_t)2 * dm.B + (int64_t)c * dm.k + r) * d
                     : fuse ? a.Gocc + ((int64_t)(mode == 0 ? 0 : dm.B) + pi) * d : a.dO + (int64_t)pi * d;
    gdst[1] = a.Gocc + ((int64_t)(mode == 0 ? dm.B : 0) + pi) * d;
    gdst[2] = a.Grel + (int64_t)pi * dm.drel;
    const float rsign = mode == 0 ? 1.f : -1.f;
    if (expands<FAM>()) mbar_wait(&selfbar, 0);
    if (rok) {
      const uint8_t* rowp = self_smem + b * 8192 + fr * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 po = xown[(b * 8 + u) * 64 + fr];
        const float4 pp = __ldcg(xpeer + (b * 8 + u) * 64 + fr);
        float4 t0 = ks == 0 ? make_float4(po.x + pp.x, po.y + pp.y, po.z + pp.z, po.w + pp.w)
                            : make_float4(pp.x + po.x, pp.y + po.y, pp.z + po.z, pp.w + po.w);
        float4 t1, t2;
        if (expands<FAM>()) {  // dO = rowsum o - W X' ; dX' = colsum x' - W^T O  (coef = -dL/df / D | -2 dL/df)
          const float4 sv = *reinterpret_cast<const float4*>(rowp + ((u ^ (fr & 7)) << 4));
          t0 = make_float4(corr * sv.x - t0.x, corr * sv.y - t0.y, corr * sv.z - t0.z, corr * sv.w - t0.w);
          if (fuse) {
            // go = dO + w+ df/do, gx = w+ df/dx; f = gamma - ||o - x||: go = dO - s u, gx = s u (u = o - x, s = w+/D)
            // tail (o = h + r): gH = go, gR = go, gT = gx ; head (o = t - r): gT = go, gR = -go, gH = gx.
            // gx was written to the uncorrupted entity's occurrence row by k_gather (fuse_pos); read it back (L2)
            t1 = *reinterpret_cast<const float4*>(rowp + 4 * 8192 + ((u ^ (fr & 7)) << 4));
            t0 = make_float4(-t1.x + t0.x, -t1.y + t0.y, -t1.z + t0.z, -t1.w + t0.w);
            t2 = make_float4(rsign * t0.x, rsign * t0.y, rsign * t0.z, rsign * t0.w);
          }
        }
        if (wtma) {
          const int off = lane * 128 + ((u ^ (lane & 7)) << 4);
          *reinterpret_cast<float4*>(stg + off) = t0;
          if (fuse) *reinterpret_cast<float4*>(stg + 8192 + off) = t2;
        } else if (4 * u < ne) {
          reinterpret_cast<float4*>(gdst[0] + e0)[u] = t0;
          if (fuse) reinterpret_cast<float4*>(gdst[2] + e0)[u] = t2;
        }
      }
    }
    trace_stamp(dm.trace, KGE_K_NEG_BWD, 4);
    if (wtma) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(pass_x || fuse ? &mG_S : &mD_S, stg, e0, trow0[0], 0);
        if (fuse) tma_store_3d(&mR_S, stg + 8192, e0, trow0[2], 0);
        bulk_commit();
        bulk_wait_all();
      }
    }
  }
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 5);
  tc_fence_before();
  __syncthreads();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 6);
  if (warp == 0) tmem_dealloc(tmem, kIssuers * 128);
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 7);
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
    else
      cudaGetLastError();
  }
  return fn;
}

// 3D map over a [chunks x rows x cols] fp32 buffer with row pitch `pitch` floats; box {32, box_rows, 1}
bool make_map(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows,
                     CUtensorMapSwizzle sw) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)chunks};
  cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)pitch * 4 * rows};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4D map over a [chunks x rows x cols] fp32 buffer seen as {32 (col in k-block), rows, k-blocks, chunks}: one box of
// {32, box_rows, box_kb} lands as box_kb consecutive [box_rows x 128 B] SW128 k-block tiles
static bool make_map4(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows,
                      int box_kb, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {32, (cuuint64_t)rows, (cuuint64_t)(cols / 32), (cuuint64_t)chunks};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 4, 128, (cuuint64_t)pitch * 4 * rows};
  cuuint32_t box[4] = {32, (cuuint32_t)box_rows, (cuuint32_t)box_kb, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The 4D view with ceil(cols / 32) k-blocks (a ragged last block reads past the row end into the next row: only for
// operands whose columns are an M or N dimension of the MMA, where those lanes land in discarded outputs -- and the
// buffer needs 128 bytes of slack after its last row)
bool make_map4c(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows, int box_kb,
                CUtensorMapSwizzle sw) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {32, (cuuint64_t)rows, (cuuint64_t)((cols + 31) / 32), (cuuint64_t)chunks};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 4, 128, (cuuint64_t)pitch * 4 * rows};
  cuuint32_t box[4] = {32, (cuuint32_t)box_rows, (cuuint32_t)box_kb, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The same 4D view over a [chunks x rows x cols] bf16 buffer: {64 (col in k-block), rows, k-blocks, chunks}
static bool make_map4_16(CUtensorMap* m, const uint16_t* base, int cols, int rows, int chunks, int pitch, int box_rows,
                         int box_kb) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64), (cuuint64_t)chunks};
  cuuint64_t strides[3] = {(cuuint64_t)pitch * 2, 128, (cuuint64_t)pitch * 2 * rows};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, (cuuint32_t)box_kb, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)base, dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static size_t fwd_smem() { return (size_t)kFwdStages * kFwdKpb * (128 * 128 + kNT * 128) + 128 * (kNT / 2) * 4 + 1024; }
static size_t bwd_smem(int dp) {
  (void)dp;
  return (size_t)kBwdStages * kBwdKpb * (16384 + 4 * 4096) + 8 * 8192 + 1024;
}

bool tc_init(kge_handle* h) {
  const Dims& dm = h->dims;
  // DistMult / ComplEx (dot), TransE-L2 and the Table-1 squared RotatE (expansion); TransE-L1 and the RotatE
  // modulus variant are not contractions and stay on the FFMA path (north_star)
  if (!(dm.family == FAM_DOT || dm.family == FAM_L2 || (dm.family == FAM_L2SQ && dm.model == KGE_ROTATE))) return false;
  if (h->dp > 512 || bwd_smem(h->dp) > 227 * 1024 || (dm.dp / 32 + kNSplit - 1) / kNSplit > 4 || h->kp % 32)
    return false;
  if (dm.bf16 && (2 * ((dm.dp16 / 64 + kNSplit - 1) / kNSplit) > 4 || !h->buf.O16)) return false;
  if (dm.x3 && !h->buf.O_hi) return false;
  TcState* st = new TcState();
  const StepBuffers& b = h->buf;
  bool ok = true;
  const int fx = (dm.k + kNT - 1) / kNT;
  // O multicast across cxn = kFwdKpb tiles (clusters of 8 CTAs) is off by default: measured on the Freebase step, the
  // 8-CTA clusters wait for room in one GPC while the gather kernel drains, which costs more than the L2 reads saved
  // (37.3 vs 42.8 us per step); KGE_FWD_MC=1 turns it on for experiments
  st->fwd_cx = getenv("KGE_FWD_MC") && fx % kFwdKpb == 0 && !dm.x3 ? kFwdKpb : 1;
  ok &= make_map4(&st->mO_F, b.O, h->dp, dm.g, dm.C, h->dp, 128, st->fwd_cx > 1 ? 1 : kFwdKpb);
  ok &= make_map4(&st->mX_F, b.X, h->dp, dm.k, dm.C, h->dp, kNT, kFwdKpb);
  // backward operands (4D {32, rows, 32-column blocks, chunk}): W K-major (dO's A), W / X' / O MN-major with K = rows
  // (dX''s A and both B operands), and the epilogue rows of O / X' (64 finalised rows x 4 column blocks)
  const CUtensorMapSwizzle mn = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
  ok &= make_map4(&st->mW_K, b.W, h->kp, dm.g, dm.C, h->kp, 128, kBwdKpb);
  ok &= make_map4(&st->mW_MN, b.W, h->kp, dm.g, dm.C, h->kp, 32 * kBwdKpb, 4, mn);
  ok &= make_map4(&st->mX_MN, b.X, h->dp, dm.k, dm.C, h->dp, 32 * kBwdKpb, 4, mn);
  ok &= make_map4(&st->mO_MN, b.O, h->dp, dm.g, dm.C, h->dp, 32 * kBwdKpb, 4, mn);
  ok &= make_map4(&st->mO_E, b.O, h->dp, dm.g, dm.C, h->dp, 64, 4);
  ok &= make_map4(&st->mX_E, b.X, h->dp, dm.k, dm.C, h->dp, 64, 4);
  ok &= make_map(&st->mG_S, b.Gocc, dm.d, 2 * dm.B + dm.C * dm.k, 1, dm.d, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mR_S, b.Grel, dm.drel, dm.B, 1, dm.drel, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mD_S, b.dO, dm.d, dm.B, 1, dm.d, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mG_L, b.Gocc, dm.d, 2 * dm.B + dm.C * dm.k, 1, dm.d, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mG_S1, h->gocc2[1], dm.d, 2 * dm.B + dm.C * dm.k, 1, dm.d, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mG_L1, h->gocc2[1], dm.d, 2 * dm.B + dm.C * dm.k, 1, dm.d, 64, CU_TENSOR_MAP_SWIZZLE_128B);
  if (dm.bf16) {  // BF16 operands: the contraction maps point at the bf16 copies (the epilogue maps stay fp32)
    ok &= make_map4_16(&st->mO_F, b.O16, dm.dp16, dm.g, dm.C, dm.dp16, 128, st->fwd_cx > 1 ? 1 : kFwdKpb);
    ok &= make_map4_16(&st->mX_F, b.X16, dm.dp16, dm.k, dm.C, dm.dp16, kNT, kFwdKpb);
    ok &= make_map4_16(&st->mW_K, b.W16, dm.kp16, dm.g, dm.C, dm.kp16, 128, kBwdKpb);
    ok &= make_map4_16(&st->mW_MN, b.W16, dm.kp16, dm.g, dm.C, dm.kp16, 64 * kBwdKpb, 2);
    ok &= make_map4_16(&st->mX_MN, b.X16, dm.dp16, dm.k, dm.C, dm.dp16, 64 * kBwdKpb, 2);
    ok &= make_map4_16(&st->mO_MN, b.O16, dm.dp16, dm.g, dm.C, dm.dp16, 64 * kBwdKpb, 2);
  }
  if (dm.x3) {  // 3xTF32: hi and lo parts, half as many k-blocks per stage (k_tc_fwd / k_tc_bwd X3)
    const int kf = kFwdKpb / 2, kb = kBwdKpb / 2;
    ok &= make_map4(&st->mO_F, b.O_hi, h->dp, dm.g, dm.C, h->dp, 128, kf);
    ok &= make_map4(&st->mO_Fl, b.O_lo, h->dp, dm.g, dm.C, h->dp, 128, kf);
    ok &= make_map4(&st->mX_F, b.X_hi, h->dp, dm.k, dm.C, h->dp, kNT, kf);
    ok &= make_map4(&st->mX_Fl, b.X_lo, h->dp, dm.k, dm.C, h->dp, kNT, kf);
    ok &= make_map4(&st->mW_K, b.W_hi, h->kp, dm.g, dm.C, h->kp, 128, kb);
    ok &= make_map4(&st->mW_Kl, b.W_lo, h->kp, dm.g, dm.C, h->kp, 128, kb);
    ok &= make_map4(&st->mW_MN, b.W_hi, h->kp, dm.g, dm.C, h->kp, 32 * kb, 4, mn);
    ok &= make_map4(&st->mW_MNl, b.W_lo, h->kp, dm.g, dm.C, h->kp, 32 * kb, 4, mn);
    ok &= make_map4(&st->mX_MN, b.X_hi, h->dp, dm.k, dm.C, h->dp, 32 * kb, 4, mn);
    ok &= make_map4(&st->mX_MNl, b.X_lo, h->dp, dm.k, dm.C, h->dp, 32 * kb, 4, mn);
    ok &= make_map4(&st->mO_MN, b.O_hi, h->dp, dm.g, dm.C, h->dp, 32 * kb, 4, mn);
    ok &= make_map4(&st->mO_MNl, b.O_lo, h->dp, dm.g, dm.C, h->dp, 32 * kb, 4, mn);
  } else {  // unused parameters of the other instantiations
    st->mO_Fl = st->mO_F;
    st->mX_Fl = st->mX_F;
    st->mW_Kl = st->mW_K;
    st->mW_MNl = st->mW_MN;
    st->mX_MNl = st->mX_MN;
    st->mO_MNl = st->mO_MN;
  }
  if (!ok) {
    delete st;
    return false;
  }
  cudaError_t e = cudaSuccess;
  auto attrs = [&](auto fwd, auto bwd) {
    e = cudaFuncSetAttribute(fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem(h->dp));
  };
  if (dm.x3) {
    if (dm.family == FAM_DOT)
      attrs(k_tc_fwd<FAM_DOT, false, true>, k_tc_bwd<FAM_DOT, false, true>);
    else if (dm.family == FAM_L2)
      attrs(k_tc_fwd<FAM_L2, false, true>, k_tc_bwd<FAM_L2, false, true>);
    else
      attrs(k_tc_fwd<FAM_L2SQ, false, true>, k_tc_bwd<FAM_L2SQ, false, true>);
  } else if (dm.bf16) {
    if (dm.family == FAM_DOT)
      attrs(k_tc_fwd<FAM_DOT, true>, k_tc_bwd<FAM_DOT, true>);
    else if (dm.family == FAM_L2)
      attrs(k_tc_fwd<FAM_L2, true>, k_tc_bwd<FAM_L2, true>);
    else
      attrs(k_tc_fwd<FAM_L2SQ, true>, k_tc_bwd<FAM_L2SQ, true>);
  } else {
    if (dm.family == FAM_DOT)
      attrs(k_tc_fwd<FAM_DOT, false>, k_tc_bwd<FAM_DOT, false>);
    else if (dm.family == FAM_L2)
      attrs(k_tc_fwd<FAM_L2, false>, k_tc_bwd<FAM_L2, false>);
    else
      attrs(k_tc_fwd<FAM_L2SQ, false>, k_tc_bwd<FAM_L2SQ, false>);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete st;
    return false;
  }
  {
    const int tiles = (std::max(dm.g, dm.k) + 127) / 128;
    const size_t pairs = (size_t)tiles * kNSplit * dm.C * 2;
    if (cudaMalloc(&st->xbuf, pairs * 2 * 32 * 64 * sizeof(float4)) != cudaSuccess) {
      cudaGetLastError();
      delete st;
      return false;
    }
  }
  st->ok = true;
  h->tc = st;
  return true;
}

void tc_destroy(kge_handle* h) {
  if (h->tc && static_cast<TcState*>(h->tc)->xbuf) cudaFree(static_cast<TcState*>(h->tc)->xbuf);
  delete static_cast<TcState*>(h->tc);
  h->tc = nullptr;
}

bool tc_supported(const kge_handle* h) { return h->tc && static_cast<const TcState*>(h->tc)->ok; }

int32_t tc_neg_parts(const kge_handle* h) {
  const Dims& dm = h->dims;
  return dm.C * ((dm.g + 127) / 128) * ((dm.k + kNT - 1) / kNT) * 2;  // one loss partial per split-K half
}

// Chunk-level dataflow between k_gather -> k_tc_fwd -> k_tc_bwd (StepBuffers::flow) instead of whole-grid PDL waits.
// Off by default: measured on the Freebase step it was slower (34.6 vs 30.9 us): the consumers' CTAs cannot become
// resident next to the gather's (register file full) and the counters add a barrier + atomics per CTA.
bool tc_flow() {
  static const bool on = getenv("KGE_FLOW") != nullptr;
  return on;
}

// the positive's gradient is fused into the TransE-L2 backward under the logistic loss (dL/df+ known at the gather);
// the pairwise loss needs the forward's hinge counts first, so it takes k_chain
bool tc_fuses_chain(const kge_handle* h) {
  return h->dims.model == KGE_TRANSE_L2 && h->dims.loss == KGE_LOSS_LOGISTIC;
}

cudaError_t launch_tc_neg(kge_handle* h, const Slot& s) {
  const Dims& dm = h->dims;
  const TcState* st = static_cast<const TcState*>(h->tc);
  TcArgs a{dm, h->dp, h->kp, h->buf.O, h->buf.X, h->buf.onorm, h->buf.xnorm, h->buf.W, h->buf.lneg, h->buf.dO,
           h->buf.Gocc, h->buf.rowsumW, h->buf.colsumW, 2 * ((dm.k + kNT - 1) / kNT), (dm.g + 127) / 128,
           tc_fuses_chain(h) ? 1 : 0, s, h->rows, h->buf.wpos, h->buf.pstat, h->buf.lpos, h->buf.Grel,
           h->buf.loss, h->buf.flags, h->n_neg_parts, 1.f / ((float)dm.B * (float)dm.k), st->xbuf, tc_flow() ? h->buf.flow : nullptr,
           2 * ((dm.k + kNT - 1) / kNT) * ((dm.g + 127) / 128), st->fwd_cx, h->buf.fdbg, h->buf.pcnt, h->buf.W16,
           dm.dp16, dm.kp16, h->buf.W_hi, h->buf.W_lo};
  dim3 gf(2 * ((dm.k + kNT - 1) / kNT), (dm.g + 127) / 128, dm.C);  // x = 2 tile + split-K half
  const int tiles = (std::max(dm.g, dm.k) + 127) / 128;
  dim3 gb(2 * tiles * kNSplit, dm.C, 2);  // x = 2 (row tile * kNSplit + column part) + split-K half
  const bool odd = h->buf.Gocc != h->gocc2[0];  // lag = 1: odd steps write the second Gocc buffer
  auto run = [&](auto fwd, auto bwd) -> cudaError_t {
    launch_begin(h, KGE_K_NEG_FWD);
    launch_pdl_cluster(fwd, gf, kFwdThreads, fwd_smem(), h->stream, 2 * st->fwd_cx, st->mO_F, st->mX_F, st->mO_Fl,
                       st->mX_Fl, a);
    launch_end(h, KGE_K_NEG_FWD);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    launch_begin(h, KGE_K_NEG_BWD);
    launch_pdl_cluster(bwd, gb, kThreads, bwd_smem(h->dp), h->stream, 2, st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN,
                       st->mO_E, st->mX_E, odd ? st->mG_S1 : st->mG_S, st->mR_S, st->mD_S, odd ? st->mG_L1 : st->mG_L,
                       st->mW_Kl, st->mW_MNl, st->mX_MNl, st->mO_MNl, a);
    launch_end(h, KGE_K_NEG_BWD);
    return cudaGetLastError();
  };
  if (dm.x3) {
    if (dm.family == FAM_DOT) return run(k_tc_fwd<FAM_DOT, false, true>, k_tc_bwd<FAM_DOT, false, true>);
    if (dm.family == FAM_L2) return run(k_tc_fwd<FAM_L2, false, true>, k_tc_bwd<FAM_L2, false, true>);
    return run(k_tc_fwd<FAM_L2SQ, false, true>, k_tc_bwd<FAM_L2SQ, false, true>);
  }
  if (dm.bf16) {
    if (dm.family == FAM_DOT) return run(k_tc_fwd<FAM_DOT, true>, k_tc_bwd<FAM_DOT, true>);
    if (dm.family == FAM_L2) return run(k_tc_fwd<FAM_L2, true>, k_tc_bwd<FAM_L2, true>);
    return run(k_tc_fwd<FAM_L2SQ, true>, k_tc_bwd<FAM_L2SQ, true>);
  }
  if (dm.family == FAM_DOT) return run(k_tc_fwd<FAM_DOT, false>, k_tc_bwd<FAM_DOT, false>);
  if (dm.family == FAM_L2) return run(k_tc_fwd<FAM_L2, false>, k_tc_bwd<FAM_L2, false>);
  return run(k_tc_fwd<FAM_L2SQ, false>, k_tc_bwd<FAM_L2SQ, false>);
}

}  // namespace kge
