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
  CUtensorMap mO_K, mX_K;    // fwd operands (K-major, SW128), boxes {32, 128 | NT}
  CUtensorMap mW_K;          // dO operand A (K-major), box {32, 128}
  CUtensorMap mX_MN, mO_MN;  // B operands of dO / dX' (MN-major, 128B_ATOM_32B), box {32, 32}
  CUtensorMap mW_MN;         // A operand of dX' (MN-major), box {32, 32}
  CUtensorMap mX_E;          // dX' epilogue operand (X' rows, K-major SW128), box {32, 128}
  bool ok = false;
};

constexpr int kNT = 32;         // negatives per forward CTA
constexpr int kFwdStages = 4;
constexpr int kBwdStages = 4;
constexpr int kNSplit = 4;      // column ranges of dp per backward tile
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
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
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
  const uint32_t tmem = tbase;
  trace_stamp(dm.trace, KGE_K_NEG_FWD, 1);

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kFwdStages;
      if (kb >= kFwdStages) mbar_wait(&empty[s], ((kb / kFwdStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      mbar_arrive_expect_tx(&full[s], STAGE);
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
             const __grid_constant__ CUtensorMap mO_E, const __grid_constant__ CUtensorMap mX_E, TcArgs a) {
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
  uint8_t* self_smem = smem + kBwdStages * STAGE;
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
  mbar_wait(&done, 0);
  tc_fence_after();
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 2);
  if (FAM == FAM_L2) mbar_wait(&selfbar, 0);
  trace_stamp(dm.trace, KGE_K_NEG_BWD, 3);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  float* dst = pass_x ? a.Gocc + ((int64_t)2 * dm.B + (int64_t)c * dm.k + r) * d : a.dO + ((int64_t)c * dm.g + r) * d;
  const int rl = warp * 32 + lane;  // row within the tile
#pragma unroll 1
  for (int b = 0; b < nb; ++b) {
    const int e0 = (b0 + b) * 32;
    float v[32];
    tmem_ld32(trow + b * 32, v);
    if (!rok || e0 >= d) continue;
    const int ne = min(32, d - e0);
    if (FAM == FAM_L2) {  // dO = rowsum o - W X' ; dX' = colsum x' - W^T O  (coef = -dL/df / D)
      const uint8_t* rowp = self_smem + b * 16384 + rl * 128;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float4 sv = *reinterpret_cast<const float4*>(rowp + ((u ^ (rl & 7)) << 4));
        v[4 * u] = corr * sv.x - v[4 * u];
        v[4 * u + 1] = corr * sv.y - v[4 * u + 1];
        v[4 * u + 2] = corr * sv.z - v[4 * u + 2];
        v[4 * u + 3] = corr * sv.w - v[4 * u + 3];
      }
    }
    if (ne == 32) {
      float4* o4 = reinterpret_cast<float4*>(dst + e0);
#pragma unroll
      for (int u = 0; u < 8; ++u) o4[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    } else {
#pragma unroll
      for (int u = 0; u < 32; ++u)  // static indices keep v[] in registers
        if (u < ne) dst[e0 + u] = v[u];
    }
    if (b == 0) trace_stamp(dm.trace, KGE_K_NEG_BWD, 4);
  }
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
  return (size_t)kBwdStages * (128 * 128 + (size_t)nb_max * 4096) + (size_t)nb_max * 16384 + 1024;
}

bool tc_init(kge_handle* h) {
  const Dims& dm = h->dims;
  if (!(dm.family == FAM_DOT || dm.family == FAM_L2)) return false;
  if (h->dp > 512 || bwd_smem(h->dp) > 227 * 1024) return false;
  TcState* st = new TcState();
  const StepBuffers& b = h->buf;
  bool ok = true;
  ok &= make_map(&st->mO_K, b.O, h->dp, dm.g, dm.C, h->dp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mX_K, b.X, h->dp, dm.k, dm.C, h->dp, kNT, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mW_K, b.W, dm.k, dm.g, dm.C, h->kp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  ok &= make_map(&st->mX_MN, b.X, h->dp, dm.k, dm.C, h->dp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mO_MN, b.O, h->dp, dm.g, dm.C, h->dp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mW_MN, b.W, dm.k, dm.g, dm.C, h->kp, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  ok &= make_map(&st->mX_E, b.X, h->dp, dm.k, dm.C, h->dp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
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

cudaError_t launch_tc_neg(kge_handle* h, const Slot& s) {
  (void)s;
  const Dims& dm = h->dims;
  const TcState* st = static_cast<const TcState*>(h->tc);
  TcArgs a{dm, h->dp, h->kp, h->buf.O, h->buf.X, h->buf.onorm, h->buf.xnorm, h->buf.W, h->buf.lneg, h->buf.dO,
           h->buf.Gocc, h->buf.rowsumW, h->buf.colsumW, 2 * ((dm.k + kNT - 1) / kNT), (dm.g + 127) / 128};
  dim3 gf((dm.k + kNT - 1) / kNT, (dm.g + 127) / 128, dm.C);
  const int tiles = (std::max(dm.g, dm.k) + 127) / 128;
  dim3 gb(tiles * kNSplit, dm.C, 2);
  launch_begin(h, KGE_K_NEG_FWD);
  if (dm.family == FAM_DOT)
    launch_pdl(k_tc_fwd<FAM_DOT>, gf, kFwdThreads, fwd_smem(), h->stream, st->mO_K, st->mX_K, a);
  else
    launch_pdl(k_tc_fwd<FAM_L2>, gf, kFwdThreads, fwd_smem(), h->stream, st->mO_K, st->mX_K, a);
  launch_end(h, KGE_K_NEG_FWD);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_begin(h, KGE_K_NEG_BWD);
  if (dm.family == FAM_DOT)
    launch_pdl(k_tc_bwd<FAM_DOT>, gb, kThreads, bwd_smem(h->dp), h->stream, st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN,
               st->mO_K, st->mX_E, a);
  else
    launch_pdl(k_tc_bwd<FAM_L2>, gb, kThreads, bwd_smem(h->dp), h->stream, st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN,
               st->mO_K, st->mX_E, a);
  launch_end(h, KGE_K_NEG_BWD);
  return cudaGetLastError();
}

}  // namespace kge
