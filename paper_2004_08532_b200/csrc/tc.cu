// tc.cu -- tcgen05 tensor-core path of the chunked negative contraction (Sec. 3.3: "converted into
// a generalized matrix multiplication") for the GEMM-shaped score families: DistMult / ComplEx (f = o . x') and
// TransE-L2 (f = gamma - sqrt(||o||^2 - 2 o.x' + ||x'||^2)). kind::tf32 on fp32 rows, fp32 accumulators in TMEM,
// operands staged by TMA through an mbarrier pipeline, one elected thread issues the MMAs.
//
//   k_tc_fwd : S_c = O_c X'_c^T (M = 128 rows of O, N = NT negatives, K = dp); fused epilogue straight from TMEM:
//              f-, logistic-loss partial, dL/dS coefficient W (reading c.9).
//   k_tc_bwd : z = 0: dO_c = W_c X'_c   (M = 128 positives, N = dp, K = k; A K-major, B MN-major)
//              z = 1: dX'_c = W_c^T O_c (M = 128 negatives, N = dp, K = g; A and B MN-major)
//              The L2 corrections rowsum(W) o and colsum(W) x' come out of the same MMAs: O carries a ones column at
//              d and X' a ones column at d+1 (zero elsewhere in the padding), so TMEM column d+1 of dO is rowsum(W)
//              and column d of dX' is colsum(W), while the forward product sees 1*0 + 0*1 there.
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
  bool ok = false;
};

constexpr int kNT = 64;         // negatives per forward CTA
constexpr int kFwdStages = 4;
constexpr int kBwdStages = 3;
constexpr int kThreads = 256;  // 8 warps: warp 0 lane 0 = TMA, warp 1 lane 0 = MMA; all 8 run the epilogue
// (warps w and w+4 read the same 32 TMEM lanes, different column halves)

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
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_fwd(const __grid_constant__ CUtensorMap mO, const __grid_constant__ CUtensorMap mX, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  constexpr uint32_t A_BYTES = 128 * 128, B_BYTES = kNT * 128, STAGE = A_BYTES + B_BYTES;
  __shared__ uint64_t full[kFwdStages], empty[kFwdStages], done;
  __shared__ uint32_t tbase;
  __shared__ float s_xn[kNT];
  __shared__ float s_red[8];
  const Dims& dm = a.dm;
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
  if (warp == 0) tmem_alloc(&tbase, kNT);
  for (int j = threadIdx.x; j < kNT; j += kThreads) {
    const int jj = j0 + j;
    s_xn[j] = jj < dm.k ? a.xnorm[(int64_t)c * dm.k + jj] : 0.f;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;

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
  mbar_wait(&done, 0);
  tc_fence_after();

  // epilogue: thread <-> row i (TMEM lane 32*(warp%4) + lane); warp/4 selects the column half
  const int lg = warp & 3, half = warp >> 2;
  const int i = i0 + lg * 32 + lane;
  const bool iok = i < dm.g;
  const float on = iok && FAM == FAM_L2 ? a.onorm[(int64_t)c * dm.g + i] : 0.f;
  const float inv_bk = 1.f / ((float)dm.B * (float)dm.k);
  float lsum = 0.f;
  float* wrow = a.W + ((int64_t)c * dm.g + i) * a.kp;
#pragma unroll 1
  for (int q = half * (kNT / 2); q < (half + 1) * (kNT / 2); q += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + q, v);
#pragma unroll
    for (int jj = 0; jj < 32; ++jj) {
      const int j = j0 + q + jj;
      float coef = 0.f;
      if (iok && j < dm.k) {
        float f, D = 1.f;
        if (FAM == FAM_DOT) {
          f = v[jj];
        } else {  // TransE-L2 by expansion, clamped at 0 before the root (reading c.8)
          D = sqrtf(fmaxf(on - 2.f * v[jj] + s_xn[q + jj], 0.f));
          f = dm.gamma - D;
        }
        // one exp serves both: e = exp(-|f|); sigma(f) = f>=0 ? 1/(1+e) : e/(1+e); -log sigma(-f) = max(f,0)+log1p(e)
        const float e = expf(-fabsf(f));
        const float r1 = 1.f / (1.f + e);
        const float sig = f >= 0.f ? r1 : e * r1;
        lsum += fmaxf(f, 0.f) + log1pf(e);
        const float dLdf = sig * inv_bk;
        coef = FAM == FAM_DOT ? dLdf : -dLdf / fmaxf(D, 1e-12f);
      }
      v[jj] = coef;
    }
    if (iok) {
      if (j0 + q + 32 <= dm.k && (a.kp & 3) == 0) {
        float4* dst = reinterpret_cast<float4*>(wrow + j0 + q);
#pragma unroll
        for (int u = 0; u < 8; ++u) dst[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
      } else {
        for (int jj = 0; jj < 32 && j0 + q + jj < dm.k; ++jj) wrow[j0 + q + jj] = v[jj];
      }
    }
  }
  lsum = warp_sum(lsum);
  if (lane == 0) s_red[warp] = lsum;
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += s_red[w];
    a.lneg[((int64_t)c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
  }
  if (warp == 0) tmem_dealloc(tmem, kNT);
}

// ------------------------------------------------------------------------------------------------
// backward: z = 0 -> dO tile (128 positives of chunk y), z = 1 -> dX' tile (128 negatives of chunk y)
// ------------------------------------------------------------------------------------------------
template <int FAM>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_bwd(const __grid_constant__ CUtensorMap mW_K, const __grid_constant__ CUtensorMap mW_MN,
             const __grid_constant__ CUtensorMap mX_MN, const __grid_constant__ CUtensorMap mO_MN, TcArgs a,
             uint32_t tmem_cols) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  __shared__ uint64_t full[kBwdStages], empty[kBwdStages], done;
  __shared__ uint32_t tbase;
  const Dims& dm = a.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool pass_x = blockIdx.z == 1;
  const int c = blockIdx.y, r0 = blockIdx.x * 128;  // output rows: i (dO) or j (dX')
  const int nrows = pass_x ? dm.k : dm.g;
  if (r0 >= nrows) return;  // uniform per CTA, before any barrier / TMEM use
  const int nk = pass_x ? dm.g : dm.k;  // contraction length
  const int nkb = (nk + 31) / 32;
  const int nb = a.dp / 32;  // column blocks of the MN-major B operand
  const uint32_t A_BYTES = 128 * 128, B_BYTES = (uint32_t)nb * 4096, STAGE = A_BYTES + B_BYTES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBwdStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&done, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&tbase, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kBwdStages;
      if (kb >= kBwdStages) mbar_wait(&empty[s], ((kb / kBwdStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      uint8_t* sb = sa + A_BYTES;
      mbar_arrive_expect_tx(&full[s], STAGE);
      if (!pass_x) {
        tma_load_3d(sa, &mW_K, &full[s], kb * 32, r0, c);                       // W[i0.., j-block]
        for (int b = 0; b < nb; ++b) tma_load_3d(sb + b * 4096, &mX_MN, &full[s], b * 32, kb * 32, c);  // X'[j-blk, :]
      } else {
        for (int b = 0; b < 4; ++b) tma_load_3d(sa + b * 4096, &mW_MN, &full[s], r0 + b * 32, kb * 32, c);  // W[i-blk, j0..]
        for (int b = 0; b < nb; ++b) tma_load_3d(sb + b * 4096, &mO_MN, &full[s], b * 32, kb * 32, c);      // O[i-blk, :]
      }
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kBwdStages;
      mbar_wait(&full[s], (kb / kBwdStages) & 1);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = pass_x ? sdesc_mn(sa + kk * 1024, 4096) : sdesc(sa + kk * 32, 16, 1024);
        for (int n0 = 0; n0 < a.dp; n0 += 256) {
          const int nn = min(256, a.dp - n0);
          const uint64_t bd = sdesc_mn(sb + (n0 / 32) * 4096 + kk * 1024, 4096);
          mma_tf32(tmem + n0, ad, bd, idesc_tf32(128, nn, pass_x, true), (kb | kk) ? 1u : 0u);
        }
      }
      mma_commit(&empty[s]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();

  // epilogue: thread <-> output row r (TMEM lane 32*(warp%4) + lane); warp/4 selects half of the column chunks
  const int lg = warp & 3, half = warp >> 2;
  const int r = r0 + lg * 32 + lane;
  const bool rok = r < nrows;
  const uint32_t trow = tmem + ((uint32_t)(lg * 32) << 16);
  const int d = dm.d;
  float corr = 0.f;  // rowsum(W) (dO) or colsum(W) (dX'), read from the ones column
  if (FAM == FAM_L2) {
    const int cc = pass_x ? d : d + 1;
    float v[32];
    tmem_ld32(trow + (cc & ~31), v);
    corr = v[cc & 31];
  }
  const float* self = pass_x ? a.X + ((int64_t)c * dm.k + r) * a.dp : a.O + ((int64_t)c * dm.g + r) * a.dp;
  float* dst = pass_x ? a.Gocc + ((int64_t)2 * dm.B + (int64_t)c * dm.k + r) * d : a.dO + ((int64_t)c * dm.g + r) * d;
  const int nch = (d + 31) / 32, ch0 = half ? (nch + 1) / 2 : 0, ch1 = half ? nch : (nch + 1) / 2;
#pragma unroll 1
  for (int ch = ch0; ch < ch1; ++ch) {
    const int e0 = ch * 32;
    float v[32];
    tmem_ld32(trow + e0, v);
    if (!rok) continue;
    const int ne = min(32, d - e0);
    if (FAM == FAM_L2) {  // dO = rowsum o - W X' ; dX' = colsum x' - W^T O  (coef = -dL/df / D); self pitch dp
      const float4* s4 = reinterpret_cast<const float4*>(self + e0);
      float4 sv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) sv[u] = s4[u];  // dp >= d + 2 keeps this in bounds
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        v[4 * u] = corr * sv[u].x - v[4 * u];
        v[4 * u + 1] = corr * sv[u].y - v[4 * u + 1];
        v[4 * u + 2] = corr * sv[u].z - v[4 * u + 2];
        v[4 * u + 3] = corr * sv[u].w - v[4 * u + 3];
      }
    }
    if (ne == 32) {
      float4* o4 = reinterpret_cast<float4*>(dst + e0);
#pragma unroll
      for (int u = 0; u < 8; ++u) o4[u] = make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
    } else {
      for (int u = 0; u < ne; ++u) dst[e0 + u] = v[u];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, tmem_cols);
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
static size_t bwd_smem(int dp) { return (size_t)kBwdStages * (128 * 128 + (size_t)(dp / 32) * 4096) + 1024; }

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
           h->buf.Gocc};
  dim3 gf((dm.k + kNT - 1) / kNT, (dm.g + 127) / 128, dm.C);
  const int tiles = (std::max(dm.g, dm.k) + 127) / 128;
  dim3 gb(tiles, dm.C, 2);
  uint32_t tcols = 32;
  while ((int)tcols < h->dp) tcols <<= 1;
  launch_begin(h, KGE_K_NEG_FWD);
  if (dm.family == FAM_DOT)
    k_tc_fwd<FAM_DOT><<<gf, kThreads, fwd_smem(), h->stream>>>(st->mO_K, st->mX_K, a);
  else
    k_tc_fwd<FAM_L2><<<gf, kThreads, fwd_smem(), h->stream>>>(st->mO_K, st->mX_K, a);
  launch_end(h, KGE_K_NEG_FWD);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_begin(h, KGE_K_NEG_BWD);
  if (dm.family == FAM_DOT)
    k_tc_bwd<FAM_DOT><<<gb, kThreads, bwd_smem(h->dp), h->stream>>>(st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN, a, tcols);
  else
    k_tc_bwd<FAM_L2><<<gb, kThreads, bwd_smem(h->dp), h->stream>>>(st->mW_K, st->mW_MN, st->mX_MN, st->mO_MN, a, tcols);
  launch_end(h, KGE_K_NEG_BWD);
  return cudaGetLastError();
}

}  // namespace kge
