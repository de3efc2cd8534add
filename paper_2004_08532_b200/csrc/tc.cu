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

#include "device_common.cuh"
#include "kge_internal.h"
#include "tc_ptx.cuh"

namespace kge {

using namespace tc;

struct TcState {
  CUtensorMap mO_K, mX_K;    // O (K-major, SW128), box {32, 128}; fwd X' operand, box {32, NT}
  CUtensorMap mO_F;          // fwd O operand: box {32, 128 / fwd_cx} (this CTA's multicast slice)
  CUtensorMap mW_K;          // dO operand A (K-major), box {32, 128}
  CUtensorMap mX_MN, mO_MN;  // B operands of dO / dX' (MN-major, 128B_ATOM_32B), box {32, 32}
  CUtensorMap mW_MN;         // A operand of dX' (MN-major), box {32, 32}
  CUtensorMap mX_E;          // dX' epilogue operand (X' rows, K-major SW128), box {32, 128}
  CUtensorMap mG_S, mR_S, mD_S;
  int fwd_cx = 1;  // backward TMA-store targets: Gocc, Grel, dO (SW128), box {32, 32}
  bool ok = false;
};

constexpr int kNT = 32;         // negatives per forward CTA
constexpr int kFwdStages = 8;
constexpr int kBwdStages = 5;
constexpr int kNSplit = 4;      // column ranges of dp per backward tile
constexpr uint32_t kBwdStaging = 4 * 24576;  // backward epilogue store staging (reuses the pipeline stages)
constexpr int kThreads = 128;   // 4 warps: warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer; all 4 = epilogue
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
  int32_t loss_slot, n_neg_parts;
  int32_t fwd_cx;  // forward cluster size along x: the CTAs of one 128-positive tile share its O tile by TMA multicast
};

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
template <int FAM>
__global__ void __launch_bounds__(kFwdThreads, 1)
    k_tc_fwd(const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mX, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr uint32_t A_BYTES = 128 * 128, B_BYTES = kNT * 128, STAGE = A_BYTES + B_BYTES;
  __shared__ uint64_t full[kFwdStages], empty[kFwdStages], done;
  __shared__ uint32_t tbase;
  __shared__ float s_xn[kNT];
  __shared__ float s_red[8];
  __shared__ float s_col[4][kNT];
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.z, i0 = blockIdx.y * 128, j0 = blockIdx.x * kNT;
  const int nkb = a.dp / 32;
  // cluster of cx CTAs along x (same positives, different negatives): CTA `crank` loads rows [crank*128/cx, +128/cx)
  // of each O k-block and multicasts them; a stage is refilled only after all cx CTAs' MMAs released it
  const int cx = a.fwd_cx;
  const uint32_t crank = cx > 1 ? cluster_ctarank() : 0;
  const uint16_t cmask = (uint16_t)((1u << cx) - 1);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cx);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
    tma_prefetch(&mO);
    tma_prefetch(&mX);
  }
  if (warp == 0) tmem_alloc(&tbase, 32);
  pdl_wait();  // predecessor (gather) complete: O, X', norms are final
  pdl_trigger();
  if (threadIdx.x < kNT) {
    const int jj = j0 + threadIdx.x;
    s_xn[threadIdx.x] = jj < dm.k ? a.xnorm[(int64_t)c * dm.k + jj] : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (cx > 1) cluster_sync();  // every CTA's barriers are initialised before any multicast lands
  const uint32_t tmem = tbase;
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 1);

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kFwdStages;
      if (kb >= kFwdStages) mbar_wait(&empty[s], ((kb / kFwdStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
      if (cx > 1)
        tma_load_3d_mc(sa + crank * (A_BYTES / cx), &mO, &full[s], kb * 32, i0 + (int)crank * (128 / cx), c, cmask);
      else
        tma_load_3d(sa, &mO, &full[s], kb * 32, i0, c);
      tma_load_3d(sa + A_BYTES, &mX, &full[s], kb * 32, j0, c);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = idesc_tf32(128, kNT, false, false);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kFwdStages;
      mbar_wait(&full[s], (kb / kFwdStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32(tmem, sdesc(sa + kk * 32, 16, 1024), sdesc(sb + kk * 32, 16, 1024), idesc, (kb | kk) ? 1u : 0u);
      if (cx > 1)
        mma_commit_mc(&empty[s], cmask);
      else
        mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  // epilogue: thread <-> row i (TMEM lane 32*(warp%4) + lane); warp/4 picks 16 of the CTA's 32 negatives
  const int lg = warp & 3, hf = warp >> 2;
  const int i = i0 + lg * 32 + lane;
  const bool iok = i < dm.g;
  const float on = iok && FAM == FAM_L2 ? a.onorm[(int64_t)c * dm.g + i] : 0.f;  // loaded while the MMAs run
  mbar_wait(&done, 0);
  tc_fence_after();
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 2);
  const float inv_bk = 1.f / ((float)dm.B * (float)dm.k);
  float v[16];
  tmem_ld16(tmem + ((uint32_t)(lg * 32) << 16) + hf * 16, v);
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 3);
  float lsum = 0.f, rsum = 0.f;
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const int j = j0 + hf * 16 + jj;
    float coef = 0.f;
    if (iok && j < dm.k) {
      float f, rD = 1.f;
      if (FAM == FAM_DOT) {
        f = v[jj];
      } else {  // TransE-L2 by expansion, clamped at 0 before the root (reading c.8)
        const float D2 = fmaxf(on - 2.f * v[jj] + s_xn[hf * 16 + jj], 0.f);
        rD = fminf(rsqrtf(D2), 1e12f);
        f = dm.gamma - D2 * rD;
      }
      // e = exp(-|f|): sigma(f) = f>=0 ? 1/(1+e) : e/(1+e);  -log sigma(-f) = max(f,0) + log1p(e)
      const float e = __expf(-fabsf(f));
      const float r1 = __fdividef(1.f, 1.f + e);
      lsum += fmaxf(f, 0.f) + __logf(1.f + e);
      const float dLdf = (f >= 0.f ? r1 : e * r1) * inv_bk;
      coef = FAM == FAM_DOT ? dLdf : -dLdf * rD;
    }
    v[jj] = coef;
    rsum += coef;
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 4);
  if (iok) {
    float* wrow = a.W + ((int64_t)c * dm.g + i) * a.kp + j0 + hf * 16;
    if (j0 + hf * 16 + 16 <= dm.k && (a.kp & 3) == 0) {
      float4* dst = reinterpret_cast<float4*>(wrow);
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    } else {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)  // static indices keep v[] in registers
        if (j0 + hf * 16 + jj < dm.k) wrow[jj] = v[jj];
    }
    if (FAM == FAM_L2) a.rowsum_part[((int64_t)c * dm.g + i) * a.nrp + 2 * blockIdx.x + hf] = rsum;
  }
  if (FAM == FAM_L2) {
    // column sums over this warp's 32 rows for its 16 columns: transposing butterfly (fixed order) over the low 4
    // lane bits, then the two 16-lane halves are added; lane l (< 16) ends with column l
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) {
#pragma unroll
      for (int q = 0; q < off; ++q) {
        const bool upper = (lane & off) != 0;
        const float send = upper ? v[q] : v[q + off];
        const float keep = upper ? v[q + off] : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
      }
    }
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], 16);
    if (lane < 16) s_col[lg][hf * 16 + lane] = v[0];
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 5);
  lsum = warp_sum(lsum);
  if (lane == 0) s_red[warp] = lsum;
  tc_fence_before();
  __syncthreads();
  if (FAM == FAM_L2 && threadIdx.x < kNT && j0 + (int)threadIdx.x < dm.k)
    a.colsum_part[((int64_t)c * dm.k + j0 + threadIdx.x) * a.ncp + blockIdx.y] =
        ((s_col[0][threadIdx.x] + s_col[1][threadIdx.x]) + s_col[2][threadIdx.x]) + s_col[3][threadIdx.x];
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += s_red[w];
    a.lneg[((int64_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 6);
  if (cx > 1) cluster_sync();  // no CTA leaves while a peer's MMA commit may still arrive on its barriers
  if (warp == 0) tmem_dealloc(tmem, 32);
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 7);
}

// ------------------------------------------------------------------------------------------------
// backward: z = 0 -> dO tile (128 positives of chunk y), z = 1 -> dX' tile (128 negatives of chunk y);
// blockIdx.x = (row tile, column part)
// ------------------------------------------------------------------------------------------------
template <int FAM>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_bwd(const __grid_constant__ CUtensorMap mW_K, const __grid_constant__ CUtensorMap mW_MN,
             const __grid_constant__ CUtensorMap mX_MN, const __grid_constant__ CUtensorMap mO_MN,
             const __grid_constant__ CUtensorMap mO_E, const __grid_constant__ CUtensorMap mX_E,
             const __grid_constant__ CUtensorMap mG_S, const __grid_constant__ CUtensorMap mR_S,
             const __grid_constant__ CUtensorMap mD_S, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  __shared__ uint64_t full[kBwdStages], empty[kBwdStages], done, selfbar;
  __shared__ uint32_t tbase;
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool pass_x = blockIdx.z == 1;
  const int c = blockIdx.y, part = blockIdx.x % kNSplit, r0 = (blockIdx.x / kNSplit) * 128;
  const int nrows = pass_x ? dm.k : dm.g;
  const int nb_all = a.dp / 32;
  const int b0 = part * nb_all / kNSplit, b1 = (part + 1) * nb_all / kNSplit;  // this CTA's column blocks
  const int nb = b1 - b0;
  if (r0 >= nrows || nb == 0 || b0 * 32 >= dm.d) {  // uniform per CTA, before any barrier / TMEM use
    pdl_trigger();
    return;
  }
  const int nk = pass_x ? dm.g : dm.k;  // contraction length
  const int nkb = (nk + 31) / 32;
  const uint32_t A_BYTES = 128 * 128, STAGE = A_BYTES + (uint32_t)nb * 4096;
  // epilogue operand (L2): this CTA's rows x column blocks of O (dO) or X' (dX'), TMA'd at the start so the load
  // overlaps the main loop; block b at self_smem + b * 16 KB, 128-byte rows, 16-byte chunks swizzled by (row % 8)
  uint8_t* self_smem = smem + max(kBwdStages * STAGE, kBwdStaging);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    mbar_init(&selfbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, 128);
  pdl_wait();  // predecessor (forward) complete: W and the row / column partial sums are final
  pdl_trigger();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 1);

  if (warp == 0 && lane == 0) {  // TMA producer
    if (FAM == FAM_L2) {
      mbar_arrive_expect_tx(&selfbar, (uint32_t)nb * 16384);
      for (int b = 0; b < nb; ++b)
        tma_load_3d(self_smem + b * 16384, pass_x ? &mX_E : &mO_E, &selfbar, (b0 + b) * 32, r0, c);
    }
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kBwdStages;
      if (kb >= kBwdStages) mbar_wait(&empty[s], ((kb / kBwdStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      mbar_arrive_expect_tx(&full[s], STAGE);
      if (!pass_x) {
        tma_load_3d(sa, &mW_K, &full[s], kb * 32, r0, c);  // W[i0.., j-block]
        for (int b = 0; b < nb; ++b) tma_load_3d(sb + b * 4096, &mX_MN, &full[s], (b0 + b) * 32, kb * 32, c);
      } else {
        for (int b = 0; b < 4; ++b) tma_load_3d(sa + b * 4096, &mW_MN, &full[s], r0 + b * 32, kb * 32, c);
        for (int b = 0; b < nb; ++b) tma_load_3d(sb + b * 4096, &mO_MN, &full[s], (b0 + b) * 32, kb * 32, c);
      }
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    const uint32_t idesc = idesc_tf32(128, nb * 32, pass_x, true);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kBwdStages;
      mbar_wait(&full[s], (kb / kBwdStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = pass_x ? sdesc_mn(sa + kk * 1024, 4096) : sdesc(sa + kk * 32, 16, 1024);
        mma_tf32(tmem, ad, sdesc_mn(sb + kk * 1024, 4096), idesc, (kb | kk) ? 1u : 0u);
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  // epilogue prologue while the MMAs run: row r (TMEM lane 32*warp + lane) and its correction factor,
  // rowsum(W) for dO, colsum(W) for dX' -- partials summed in a fixed order
  const int r = r0 + warp * 32 + lane;
  const bool rok = r < nrows;
  const int d = dm.d;
  float corr = 0.f;
  if (FAM == FAM_L2 && rok) {
    if (!pass_x) {
      const float* rp = a.rowsum_part + ((int64_t)c * dm.g + r) * a.nrp;
      for (int q = 0; q < a.nrp; ++q) corr += rp[q];
    } else {
      const float* cp = a.colsum_part + ((int64_t)c * dm.k + r) * a.ncp;
      for (int q = 0; q < a.ncp; ++q) corr += cp[q];
    }
  }
  const bool fuse = FAM == FAM_L2 && a.fuse && !pass_x;
  int loss_part = 0;  // the loss is reduced by the first CTA of (row tile 0, chunk 0) that has columns to process
  while (loss_part + 1 < kNSplit && ((loss_part + 1) * nb_all / kNSplit == loss_part * nb_all / kNSplit ||
                                     loss_part * nb_all / kNSplit * 32 >= d))
    ++loss_part;
  if (fuse && blockIdx.x == loss_part && blockIdx.y == 0 && warp == 3) {
    // deterministic loss (reading c.9): fixed lane assignment and order, identical to the unfused k_chain
    float sp = 0.f, sn = 0.f;
    for (int i = lane; i < dm.B; i += 32) sp += a.lpos[i];
    for (int q = lane; q < a.n_neg_parts; q += 32) sn += a.lneg[q];
    sp = warp_sum(sp);
    sn = warp_sum(sn);
    if (lane == 0) {
      const float L = sp / (float)dm.B + sn / ((float)dm.B * (float)dm.k);
      a.loss[a.loss_slot] = L;
      const bool bad = !isfinite(L);
      a.flags[1] = bad ? 1 : 0;
      if (bad) a.flags[0] = 1;
    }
  }
  // fused chain: positive i of this row; x = the uncorrupted "other" entity row (t for tail mode, h for head mode),
  // prefetched for all column blocks while the MMAs run
  const int pi = c * dm.g + r;
  const int mode = fuse ? a.s.mode[c] : 0;
  float pscale = 0.f;
  float4 xr[4][8];
  if (fuse && rok) {
    pscale = a.wpos[pi] / fmaxf(sqrtf(a.pstat[pi]), 1e-12f);
    const float* xrow = a.ent.row(mode == 0 ? a.s.pt[pi] : a.s.ph[pi]);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int e0 = (b0 + b) * 32;
      if (b < nb && e0 < d) {
        const float4* x4 = reinterpret_cast<const float4*>(xrow + e0);
#pragma unroll
        for (int u = 0; u < 8; ++u) xr[b][u] = 4 * u < d - e0 ? __ldg(x4 + u) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  // output tiles of this warp's 32 rows: t = 0 the primary (dO | dX' | fused: gradient of the combined entity),
  // fused only: t = 1 gradient of the other entity, t = 2 relation gradient. Full 32-row warps stage each
  // 32 x 32 tile in (free) pipeline shared memory in the SW128 layout and TMA-store it (coalesced, asynchronous);
  // a ragged warp (chunk shorter than its rows) stores its valid rows directly.
  const int wrow0 = r0 + warp * 32;
  const bool wtma = wrow0 + 32 <= nrows;
  const int ntile = fuse ? 3 : 1;
  const CUtensorMap* tmap0 = pass_x || fuse ? &mG_S : &mD_S;
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
  uint8_t* stg = smem + warp * 24576;  // 2 buffers x 3 tiles x 4 KB per warp (the MMAs are done with this memory)
  mbar_wait(&done, 0);
  tc_fence_after();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 2);
  if (FAM == FAM_L2) mbar_wait(&selfbar, 0);
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 3);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  const int rl = warp * 32 + lane;  // row within the tile
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    if (b >= nb) break;
    const int e0 = (b0 + b) * 32;
    float v[32];
    tmem_ld32(trow + b * 32, v);
    if (e0 >= d) continue;
    const int ne = min(32, d - e0);
    uint8_t* buf = stg + (b & 1) * 12288;
    if (wtma && b >= 2) {  // the buffer written two blocks ago must have been read by its TMA store
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
    }
    if (rok) {
      const uint8_t* rowp = self_smem + b * 16384 + rl * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float4 t0 = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]), t1, t2;
        if (FAM == FAM_L2) {  // dO = rowsum o - W X' ; dX' = colsum x' - W^T O  (coef = -dL/df / D)
          const float4 sv = *reinterpret_cast<const float4*>(rowp + ((u ^ (rl & 7)) << 4));
          t0 = make_float4(corr * sv.x - t0.x, corr * sv.y - t0.y, corr * sv.z - t0.z, corr * sv.w - t0.w);
          if (fuse) {
            // go = dO + w+ df/do, gx = w+ df/dx; f = gamma - ||o - x||: go = dO - s u, gx = s u (u = o - x, s = w+/D)
            // tail (o = h + r): gH = go, gR = go, gT = gx ; head (o = t - r): gT = go, gR = -go, gH = gx
            const float4 xv = xr[b][u];
            t1 = make_float4(pscale * (sv.x - xv.x), pscale * (sv.y - xv.y), pscale * (sv.z - xv.z),
                             pscale * (sv.w - xv.w));
            t0 = make_float4(-t1.x + t0.x, -t1.y + t0.y, -t1.z + t0.z, -t1.w + t0.w);
            t2 = make_float4(rsign * t0.x, rsign * t0.y, rsign * t0.z, rsign * t0.w);
          }
        }
        if (wtma) {
          const int off = lane * 128 + ((u ^ (lane & 7)) << 4);
          *reinterpret_cast<float4*>(buf + off) = t0;
          if (fuse) {
            *reinterpret_cast<float4*>(buf + 4096 + off) = t1;
            *reinterpret_cast<float4*>(buf + 8192 + off) = t2;
          }
        } else if (4 * u < ne) {
          reinterpret_cast<float4*>(gdst[0] + e0)[u] = t0;
          if (fuse) {
            reinterpret_cast<float4*>(gdst[1] + e0)[u] = t1;
            reinterpret_cast<float4*>(gdst[2] + e0)[u] = t2;
          }
        }
      }
    }
    if (wtma) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(tmap0, buf, e0, trow0[0], 0);
        if (ntile > 1) {
          tma_store_3d(&mG_S, buf + 4096, e0, trow0[1], 0);
          tma_store_3d(&mR_S, buf + 8192, e0, trow0[2], 0);
        }
        bulk_commit();
      }
    }
    if (b == 0) trace_stamp(dm.trace, KGE_K_NEG_BWD, 4);
  }
  if (wtma && lane == 0) bulk_wait_all();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 5);
  tc_fence_before();
  __syncthreads();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 6);
  if (warp == 0) tmem_dealloc(tmem, 128);
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
static bool make_map(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows,
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

static size_t fwd_smem() { return (size_t)kFwdStages * (128 * 128 + kNT * 128) + 1024; }
static size_t bwd_smem(int dp) {
  const int nb_max = (dp / 32 + kNSplit - 1) / kNSplit;
  return std::max((size_t)kBwdStages * (128 * 128 + (size_t)nb_max * 4096), (size_t)kBwdStaging) +
         (size_t)nb_max * 16384 + 1024;
}

bool tc_init(kge_handle* h) {
  const Dims& dm = h->dims;
  if (!(dm.family == FAM_DOT || dm.family == FAM_L2)) return false;
  if (h->dp > 512 || bwd_smem(h->dp) > 227 * 1024) return false;
  TcState* st = new TcState();
  const StepBuffers& b = h->buf;
  bool ok = true;
  const int fx = (dm.k + kNT - 1) / kNT;
  st->fwd_cx = fx % 8 == 0 ? 8 : fx % 4 == 0 ? 4 : fx % 2 == 0 ? 2 : 1;
  ok &= make_map(&st->mO_K, b.O, h->dp, dm.g, dm.C, h->dp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mO_F, b.O, h->dp, dm.g, dm.C, h->dp, 128 / st->fwd_cx, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mX_K, b.X, h->dp, dm.k, dm.C, h->dp, kNT, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mW_K, b.W, dm.k, dm.g, dm.C, h->kp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mX_MN, b.X, h->dp, dm.k, dm.C, h->dp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mO_MN, b.O, h->dp, dm.g, dm.C, h->dp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mW_MN, b.W, dm.k, dm.g, dm.C, h->kp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mX_E, b.X, h->dp, dm.k, dm.C, h->dp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mG_S, b.Gocc, dm.d, 2 * dm.B + dm.C * dm.k, 1, dm.d, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mR_S, b.Grel, dm.drel, dm.B, 1, dm.drel, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mD_S, b.dO, dm.d, dm.B, 1, dm.d, 32, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!ok) {
    delete st;
    return false;
  }
  cudaError_t e = cudaSuccess;
  if (dm.family == FAM_DOT) {
    e = cudaFuncSetAttribute(k_tc_fwd<FAM_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_tc_bwd<FAM_DOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem(h->dp));
  } else {
    e = cudaFuncSetAttribute(k_tc_fwd<FAM_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_tc_bwd<FAM_L2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bwd_smem(h->dp));
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete st;
    return false;
  }
  st->ok = true;
  h->tc = st;
  return true;
}

void tc_destroy(kge_handle* h) {
  delete static_cast<TcState*>(h->tc);
  h->tc = nullptr;
}

bool tc_supported(const kge_handle* h) { return h->tc && static_cast<const TcState*>(h->tc)->ok; }

int32_t tc_neg_parts(const kge_handle* h) {
  const Dims& dm = h->dims;
  return dm.C * ((dm.g + 127) / 128) * ((dm.k + kNT - 1) / kNT);
}

bool tc_fuses_chain(const kge_handle* h) { return h->dims.model == KGE_TRANSE_L2; }

cudaError_t launch_tc_neg(kge_handle* h, const Slot& s, int32_t loss_slot) {
  const Dims& dm = h->dims;
  const TcState* st = static_cast<const TcState*>(h->tc);
  TcArgs a{dm, h->dp, h->kp, h->buf.O, h->buf.X, h->buf.onorm, h->buf.xnorm, h->buf.W, h->buf.lneg, h->buf.dO,
           h->buf.Gocc, h->buf.rowsumW, h->buf.colsumW, 2 * ((dm.k + kNT - 1) / kNT), (dm.g + 127) / 128,
           tc_fuses_chain(h) ? 1 : 0, s, h->rows, h->buf.wpos, h->buf.pstat, h->buf.lpos, h->buf.Grel,
           h->buf.loss, h->buf.flags, loss_slot, h->n_neg_parts, st->fwd_cx};
  dim3 gf((dm.k + kNT - 1) / kNT, (dm.g + 127) / 128, dm.C);
  const int tiles = (std::max(dm.g, dm.k) + 127) / 128;
  dim3 gb(tiles * kNSplit, dm.C, 2);
  launch_begin(h, KGE_K_NEG_FWD);
  if (dm.family == FAM_DOT)
    launch_pdl_cluster(k_tc_fwd<FAM_DOT>, gf, kFwdThreads, fwd_smem(), h->stream, st->fwd_cx, st->mO_F, st->mX_K, a);
  else
    launch_pdl_cluster(k_tc_fwd<FAM_L2>, gf, kFwdThreads, fwd_smem(), h->stream, st->fwd_cx, st->mO_F, st->mX_K, a);
  launch_end(h, KGE_K_NEG_FWD);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_begin(h, KGE_K_NEG_BWD);
  if (dm.family == FAM_DOT)
    launch_pdl(k_tc_bwd<FAM_DOT>, gb, kThreads, bwd_smem(h->dp), h->stream, st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN,
               st->mO_K, st->mX_E, st->mG_S, st->mR_S, st->mD_S, a);
  else
    launch_pdl(k_tc_bwd<FAM_L2>, gb, kThreads, bwd_smem(h->dp), h->stream, st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN,
               st->mO_K, st->mX_E, st->mG_S, st->mR_S, st->mD_S, a);
  launch_end(h, KGE_K_NEG_BWD);
  return cudaGetLastError();
}

}  // namespace kge
