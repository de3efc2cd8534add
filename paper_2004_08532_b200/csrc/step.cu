// step.cu -- steps (2)-(4) of the mini-batch loop (Sec. 3.1) on the device, FP32 path.
//
//   k_gather     : per positive i, o_i = combine(h_i, r_i) (tail) / combine'(r_i, t_i) (head) -- "o is computed as
//                  before because there are only b pairs" -- and f+_i = pair(o_i, t_i | h_i);
//                  per negative slot, the gathered row x'_j. One warp per row, 128-bit coalesced row access.
//   k_neg_fwd    : per chunk, S = pair(O_c, X'_c) for all g x k pairs ("converted into a
//                  generalized matrix multiplication"), shared-memory tiled, 4x4 register micro-tiles, FFMA;
//                  fused epilogue: f-, logistic loss and dL/dS.
//   k_neg_bwd    : dO = sum_j W_ij dpair/do, dX' = sum_i W_ij dpair/dx' (the transpose contractions), same tiling.
//   k_chain      : per positive: positive-score gradient + chain rule of dO through combine -> per-occurrence grads;
//                  one extra CTA reduces the loss in a fixed order (deterministic) and flags non-finite steps.
//   k_update     : per unique row: segmented sum of its occurrence gradients in sorted-occurrence order (no float
//                  atomics) fused with the sparse row-wise Adagrad update (reading c.11).
// The tensor-core variant of k_neg_fwd / k_neg_bwd for the GEMM-shaped families lives in tc.cu.
#include <algorithm>

#include <cuda_bf16.h>

#include "device_common.cuh"
#include "kge_internal.h"

namespace kge {

// 3xTF32 split (KGE_PREC_3XTF32): hi = x with the low 13 mantissa bits cleared (a tf32 value), lo = x - hi (exact)
__device__ __forceinline__ void st_split4(float* hi_row, float* lo_row, int q, float4 v) {
  const float4 h = make_float4(__uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u),
                               __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u));
  reinterpret_cast<float4*>(hi_row)[q] = h;
  reinterpret_cast<float4*>(lo_row)[q] = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
}

// BF16 operand copies (KGE_PREC_BF16): float4 -> 4 bf16 (round to nearest even) stored as 8 bytes at element 4 q of
// a bf16 row; returns the squared norm of the ROUNDED values (the tcgen05 expansion ||o||^2 - 2 o.x + ||x||^2 then
// measures the distance of the rounded rows exactly up to fp32 accumulation)
__device__ __forceinline__ float st_bf16x4(uint16_t* row, int q, float4 v) {
  const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  uint2 u;
  u.x = *reinterpret_cast<const uint32_t*>(&a);
  u.y = *reinterpret_cast<const uint32_t*>(&b);
  reinterpret_cast<uint2*>(row)[q] = u;
  return fa.x * fa.x + fa.y * fa.y + fb.x * fb.x + fb.y * fb.y;
}

// ------------------------------------------------------------------------------------------------
// row helpers (one warp per row, float4 lanes)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float4 ld4(const float* p, int v) { return reinterpret_cast<const float4*>(p)[v]; }
__device__ __forceinline__ void st4(float* p, int v, float4 x) { reinterpret_cast<float4*>(p)[v] = x; }

#define F4MAP(out, a, b, expr)            \
  do {                                    \
    { float A = a.x, Bv = b.x; out.x = expr; } \
    { float A = a.y, Bv = b.y; out.y = expr; } \
    { float A = a.z, Bv = b.z; out.z = expr; } \
    { float A = a.w, Bv = b.w; out.w = expr; } \
  } while (0)

__device__ __forceinline__ bool is_complex_model(int model) { return model == KGE_COMPLEX || model == KGE_ROTATE; }

// o = combine(h, r) (mode 0, tail corruption) or combine'(r, t) (mode 1, head corruption); reading c.8 table.
// While writing o it accumulates (per lane) the pair statistic of o against `other` (family `fam`, see pair_partial)
// and ||o||^2, so callers need no second pass over o.
__device__ void combine_row(int model, int mode, const float* __restrict__ h, const float* __restrict__ r,
                            const float* __restrict__ t, float* __restrict__ o, int d, int lane,
                            const float* __restrict__ other, int fam, float& stat, float& onorm) {
  stat = 0.f;
  onorm = 0.f;
  if (!is_complex_model(model)) {
    const int d4 = d >> 2;
    for (int v = lane; v < d4; v += 32) {
      const float4 rv = ld4(r, v);
      float4 ov;
      if (model == KGE_DISTMULT) {
        const float4 xv = mode == 0 ? ld4(h, v) : ld4(t, v);
        F4MAP(ov, xv, rv, A * Bv);
      } else {  // TransE: h + r | t - r
        if (mode == 0) {
          const float4 hv = ld4(h, v);
          F4MAP(ov, hv, rv, A + Bv);
        } else {
          const float4 tv = ld4(t, v);
          F4MAP(ov, tv, rv, A - Bv);
        }
      }
      st4(o, v, ov);
      const float4 xv = ld4(other, v);
      onorm += ov.x * ov.x + ov.y * ov.y + ov.z * ov.z + ov.w * ov.w;
      if (fam == FAM_DOT) {
        stat += ov.x * xv.x + ov.y * xv.y + ov.z * xv.z + ov.w * xv.w;
      } else if (fam == FAM_L1) {
        stat += fabsf(ov.x - xv.x) + fabsf(ov.y - xv.y) + fabsf(ov.z - xv.z) + fabsf(ov.w - xv.w);
      } else {
        float4 u;
        F4MAP(u, ov, xv, A - Bv);
        stat += u.x * u.x + u.y * u.y + u.z * u.z + u.w * u.w;
      }
    }
    return;
  }
  const int n4 = d >> 3;
  for (int v = lane; v < n4; v += 32) {
    const float4 xr = mode == 0 ? ld4(h, v) : ld4(t, v);
    const float4 xi = mode == 0 ? ld4(h, v + n4) : ld4(t, v + n4);
    float4 orr, oi;
    float cr[4], ci[4];
    if (model == KGE_COMPLEX) {
      const float4 rr = ld4(r, v), ri = ld4(r, v + n4);
      cr[0] = rr.x; cr[1] = rr.y; cr[2] = rr.z; cr[3] = rr.w;
      ci[0] = ri.x; ci[1] = ri.y; ci[2] = ri.z; ci[3] = ri.w;
    } else {  // RotatE: r = e^{i theta}; head mode uses e^{-i theta}
      const float4 th = ld4(r, v);
      const float tt[4] = {th.x, th.y, th.z, th.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) sincosf(tt[u], &ci[u], &cr[u]);
    }
    const float a[4] = {xr.x, xr.y, xr.z, xr.w}, b[4] = {xi.x, xi.y, xi.z, xi.w};
    float outr[4], outi[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (model == KGE_COMPLEX) {
        if (mode == 0) {  // h * r
          outr[u] = a[u] * cr[u] - b[u] * ci[u];
          outi[u] = a[u] * ci[u] + b[u] * cr[u];
        } else {  // conj-side: [rr tr + ri ti | rr ti - ri tr]
          outr[u] = cr[u] * a[u] + ci[u] * b[u];
          outi[u] = cr[u] * b[u] - ci[u] * a[u];
        }
      } else {
        if (mode == 0) {  // h e^{i theta}
          outr[u] = a[u] * cr[u] - b[u] * ci[u];
          outi[u] = a[u] * ci[u] + b[u] * cr[u];
        } else {  // t e^{-i theta}
          outr[u] = a[u] * cr[u] + b[u] * ci[u];
          outi[u] = -a[u] * ci[u] + b[u] * cr[u];
        }
      }
    }
    orr = make_float4(outr[0], outr[1], outr[2], outr[3]);
    oi = make_float4(outi[0], outi[1], outi[2], outi[3]);
    st4(o, v, orr);
    st4(o, v + n4, oi);
    const float4 xr4 = ld4(other, v), xi4 = ld4(other, v + n4);
    const float xr_[4] = {xr4.x, xr4.y, xr4.z, xr4.w}, xi_[4] = {xi4.x, xi4.y, xi4.z, xi4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      onorm += outr[u] * outr[u] + outi[u] * outi[u];
      const float ur = outr[u] - xr_[u], ui = outi[u] - xi_[u];
      if (fam == FAM_DOT)
        stat += outr[u] * xr_[u] + outi[u] * xi_[u];
      else if (fam == FAM_CMOD)
        stat += sqrtf(ur * ur + ui * ui);
      else if (fam == FAM_L1)
        stat += fabsf(ur) + fabsf(ui);
      else
        stat += ur * ur + ui * ui;
    }
  }
}

// per-lane partial of the pair statistic: DOT sum o.x ; L2/L2SQ sum (o-x)^2 ; L1 sum |o-x| ; CMOD sum |z_c|
__device__ float pair_partial(int fam, const float* __restrict__ o, const float* __restrict__ x, int d, int lane) {
  float acc = 0.f;
  if (fam == FAM_CMOD) {
    const int n4 = d >> 3;
    for (int v = lane; v < n4; v += 32) {
      const float4 orr = ld4(o, v), oi = ld4(o, v + n4), xr = ld4(x, v), xi = ld4(x, v + n4);
      float4 ur, ui;
      F4MAP(ur, orr, xr, A - Bv);
      F4MAP(ui, oi, xi, A - Bv);
      acc += sqrtf(ur.x * ur.x + ui.x * ui.x) + sqrtf(ur.y * ur.y + ui.y * ui.y) +
             sqrtf(ur.z * ur.z + ui.z * ui.z) + sqrtf(ur.w * ur.w + ui.w * ui.w);
    }
    return acc;
  }
  const int d4 = d >> 2;
  for (int v = lane; v < d4; v += 32) {
    const float4 ov = ld4(o, v), xv = ld4(x, v);
    if (fam == FAM_DOT) {
      acc += ov.x * xv.x + ov.y * xv.y + ov.z * xv.z + ov.w * xv.w;
    } else if (fam == FAM_L1) {
      acc += fabsf(ov.x - xv.x) + fabsf(ov.y - xv.y) + fabsf(ov.z - xv.z) + fabsf(ov.w - xv.w);
    } else {
      float4 u;
      F4MAP(u, ov, xv, A - Bv);
      acc += u.x * u.x + u.y * u.y + u.z * u.z + u.w * u.w;
    }
  }
  return acc;
}

// f from the pair statistic (Table 1 + margin, reading Q7)
__device__ __forceinline__ float pair_score_from(int fam, float stat, float gamma) {
  switch (fam) {
    case FAM_DOT: return stat;
    case FAM_L2: return gamma - sqrtf(stat);
    default: return gamma - stat;
  }
}

// ------------------------------------------------------------------------------------------------
// k_gather: positives (o, f+, dL/df+) and negative rows
// ------------------------------------------------------------------------------------------------
struct GatherArgs {
  Dims dm;
  Slot s;
  EntRows ent;
  const float* rel;
  StepBuffers b;
  int32_t first_row;  // B: negatives only (TransR handles its positives in transr.cu)
  int32_t fuse_pos;   // TransE-L2 on the tcgen05 path: also write the positive-score gradient of the uncorrupted
                      // entity, gx = w+ (o - x) / ||o - x||, into its occurrence row of Gocc (read back by k_tc_bwd)
  uint32_t* flow;     // tcgen05 path: publish rows done per chunk (StepBuffers::flow), else nullptr
};

// Register-staged rows: every lane issues all of its row loads before any arithmetic or store, so a warp has its whole
// row in flight at once (the per-iteration loop otherwise serialises on load latency, since the stores to O / X'
// may alias the next iteration's loads as far as the compiler knows). V = float4 per lane (d <= 128 * V).
template <int V>
struct Row4 {
  float4 v[V];
  __device__ __forceinline__ void load(const float* __restrict__ p, int lane, int n4) {
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int q = lane + 32 * m;
      v[m] = q < n4 ? ld4(p, q) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
};

__device__ __forceinline__ void f4_to(const float4& a, float* x) {
  x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
}

template <int V>
__device__ __forceinline__ void combine_stage(int model, int mode, const float* __restrict__ h, const float* __restrict__ r,
                                              const float* __restrict__ t, const float* __restrict__ other,
                                              float* __restrict__ o, int d, int lane, int fam, float& stat, float& onorm) {
  stat = 0.f;
  onorm = 0.f;
  if (!is_complex_model(model)) {
    const int d4 = d >> 2;
    Row4<V> X, R, Y;
    X.load(mode == 0 ? h : t, lane, d4);
    R.load(r, lane, d4);
    Y.load(other, lane, d4);
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int q = lane + 32 * m;
      if (q >= d4) continue;
      float xv[4], rv[4], yv[4], ov[4];
      f4_to(X.v[m], xv);
      f4_to(R.v[m], rv);
      f4_to(Y.v[m], yv);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ov[u] = model == KGE_DISTMULT ? xv[u] * rv[u] : (mode == 0 ? xv[u] + rv[u] : xv[u] - rv[u]);
        onorm += ov[u] * ov[u];
        const float df = ov[u] - yv[u];
        stat += fam == FAM_DOT ? ov[u] * yv[u] : (fam == FAM_L1 ? fabsf(df) : df * df);
      }
      st4(o, q, make_float4(ov[0], ov[1], ov[2], ov[3]));
    }
    return;
  }
  const int n4 = d >> 3;
  const float* e = mode == 0 ? h : t;
  Row4<V> A, Bm, R1, R2, XR, XI;
  A.load(e, lane, n4);
  Bm.load(e + 4 * n4, lane, n4);
  R1.load(r, lane, n4);
  if (model == KGE_COMPLEX) R2.load(r + 4 * n4, lane, n4);
  XR.load(other, lane, n4);
  XI.load(other + 4 * n4, lane, n4);
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int q = lane + 32 * m;
    if (q >= n4) continue;
    float a[4], b[4], c1[4], c2[4], xr[4], xi[4], outr[4], outi[4];
    f4_to(A.v[m], a);
    f4_to(Bm.v[m], b);
    f4_to(R1.v[m], c1);
    f4_to(XR.v[m], xr);
    f4_to(XI.v[m], xi);
    if (model == KGE_COMPLEX) {
      f4_to(R2.v[m], c2);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float sn, cs;
        sincosf(c1[u], &sn, &cs);
        c1[u] = cs;
        c2[u] = sn;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      // c1 = Re r (or cos theta), c2 = Im r (or sin theta)
      if (mode == 0) {  // h * r
        outr[u] = a[u] * c1[u] - b[u] * c2[u];
        outi[u] = a[u] * c2[u] + b[u] * c1[u];
      } else {          // ComplEx: [rr tr + ri ti | rr ti - ri tr];  RotatE: t e^{-i theta} (same formula)
        outr[u] = c1[u] * a[u] + c2[u] * b[u];
        outi[u] = c1[u] * b[u] - c2[u] * a[u];
      }
      onorm += outr[u] * outr[u] + outi[u] * outi[u];
      const float ur = outr[u] - xr[u], ui = outi[u] - xi[u];
      if (fam == FAM_DOT)
        stat += outr[u] * xr[u] + outi[u] * xi[u];
      else if (fam == FAM_CMOD)
        stat += sqrtf(ur * ur + ui * ui);
      else if (fam == FAM_L1)
        stat += fabsf(ur) + fabsf(ui);
      else
        stat += ur * ur + ui * ui;
    }
    st4(o, q, make_float4(outr[0], outr[1], outr[2], outr[3]));
    st4(o, q + n4, make_float4(outi[0], outi[1], outi[2], outi[3]));
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_gather(GatherArgs a) {
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_GATHER, 0);
  pdl_wait();
  pdl_trigger();
  trace_stamp(dm.trace, KGE_K_GATHER, 1);
  const int lane = threadIdx.x & 31;
  const int row = a.first_row + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int n_neg = dm.C * dm.k;
  if (row < dm.B && a.fuse_pos) {
    // TransE-L2 (tail: o = h + r, x = t; head: o = t - r, x = h): o, its norm and pair statistic as below, plus
    // gx = s (o - x), s = w+ / max(||o - x||, 1e-12) -- the positive term of the uncorrupted entity's gradient
    // (reading c.10) -- written to that entity's occurrence row (t: B + i in tail mode, h: i in head mode)
    const int i = row, mode = a.s.mode[i / dm.g];
    const float* e = a.ent.row(mode == 0 ? a.s.ph[i] : a.s.pt[i]);
    const float* x = a.ent.row(mode == 0 ? a.s.pt[i] : a.s.ph[i]);
    const float* r = a.rel + (int64_t)a.s.pr[i] * dm.drel;
    float* o = a.b.O + (int64_t)i * dm.dp;
    const int d4 = dm.d >> 2;
    Row4<V> X, R, Y;
    X.load(e, lane, d4);
    R.load(r, lane, d4);
    Y.load(x, lane, d4);
    float stat = 0.f, on = 0.f;
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int q = lane + 32 * m;
      if (q >= d4) continue;
      float xv[4], rv[4], yv[4], ov[4];
      f4_to(X.v[m], xv);
      f4_to(R.v[m], rv);
      f4_to(Y.v[m], yv);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ov[u] = mode == 0 ? xv[u] + rv[u] : xv[u] - rv[u];
        on += ov[u] * ov[u];
        const float df = ov[u] - yv[u];
        stat += df * df;
      }
      const float4 o4 = make_float4(ov[0], ov[1], ov[2], ov[3]);
      st4(o, q, o4);
      X.v[m] = o4;  // keep o for the gradient below
    }
    if (a.b.O_hi) {  // 3xTF32 split of o
#pragma unroll
      for (int m = 0; m < V; ++m)
        if (lane + 32 * m < d4)
          st_split4(a.b.O_hi + (int64_t)i * dm.dp, a.b.O_lo + (int64_t)i * dm.dp, lane + 32 * m, X.v[m]);
    }
    if (a.b.O16) {  // BF16 copy of o; the expansion uses the norm of the rounded row
      on = 0.f;
      uint16_t* o16 = a.b.O16 + (int64_t)i * dm.dp16;
#pragma unroll
      for (int m = 0; m < V; ++m)
        if (lane + 32 * m < d4) on += st_bf16x4(o16, lane + 32 * m, X.v[m]);
    }
    stat = warp_sum(stat);
    on = warp_sum(on);
    const float f = pair_score_from(dm.family, stat, dm.gamma);
    const float wp = -sigmoid(-f) / (float)dm.B;  // dL/df+ (reading c.9)
    if (lane == 0) {
      a.b.pstat[i] = stat;
      a.b.wpos[i] = wp;
      a.b.lpos[i] = -log_sigmoid(f);
      a.b.onorm[i] = on;
    }
    const float ps = wp / fmaxf(sqrtf(stat), 1e-12f);
    float* gx = a.b.Gocc + ((int64_t)(mode == 0 ? dm.B : 0) + i) * dm.d;
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int q = lane + 32 * m;
      if (q >= d4) continue;
      const float4 ov = X.v[m], yv = Y.v[m];
      st4(gx, q, make_float4(ps * (ov.x - yv.x), ps * (ov.y - yv.y), ps * (ov.z - yv.z), ps * (ov.w - yv.w)));
    }
  } else if (row < dm.B) {
    const int i = row, mode = a.s.mode[i / dm.g];
    const float* h = a.ent.row(a.s.ph[i]);
    const float* t = a.ent.row(a.s.pt[i]);
    const float* r = a.rel + (int64_t)a.s.pr[i] * dm.drel;
    float* o = a.b.O + (int64_t)i * dm.dp;
    float stat, on;
    combine_stage<V>(dm.model, mode, h, r, t, mode == 0 ? t : h, o, dm.d, lane, dm.family, stat, on);
    if (a.b.O_hi) {  // 3xTF32 split of o (read back after the warp's stores)
      __syncwarp();
      for (int q = lane; q < (dm.d >> 2); q += 32)
        st_split4(a.b.O_hi + (int64_t)i * dm.dp, a.b.O_lo + (int64_t)i * dm.dp, q, ld4(o, q));
    }
    if (a.b.O16) {  // BF16 copy of o (this lane's own stores, read back), norm of the rounded row
      __syncwarp();
      on = 0.f;
      uint16_t* o16 = a.b.O16 + (int64_t)i * dm.dp16;
      for (int q = lane; q < (dm.d >> 2); q += 32) on += st_bf16x4(o16, q, ld4(o, q));
    }
    stat = warp_sum(stat);
    on = warp_sum(on);
    if (lane == 0) {
      a.b.pstat[i] = stat;
      const float f = pair_score_from(dm.family, stat, dm.gamma);
      if (dm.loss == KGE_LOSS_PAIRWISE) {  // the positive's terms come from its hinges (forward epilogues, k_chain)
        a.b.wpos[i] = 0.f;
        a.b.lpos[i] = 0.f;
        a.b.pcnt[i] = 0;
      } else {
        a.b.wpos[i] = -sigmoid(-f) / (float)dm.B;  // dL/df+ (reading c.9)
        a.b.lpos[i] = -log_sigmoid(f);
      }
      a.b.onorm[i] = on;
    }
  } else if (row < dm.B + n_neg) {
    const int q = row - dm.B;
    const int d4 = dm.d >> 2;
    Row4<V> Xr;
    Xr.load(a.ent.row(a.s.neg[q]), lane, d4);
    float* X = a.b.X + (int64_t)q * dm.dp;
    uint16_t* x16 = a.b.X16 ? a.b.X16 + (int64_t)q * dm.dp16 : nullptr;
    float acc = 0.f;
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int v = lane + 32 * m;
      if (v < d4) {
        const float4 xv = Xr.v[m];
        st4(X, v, xv);
        if (a.b.X_hi) st_split4(a.b.X_hi + (int64_t)q * dm.dp, a.b.X_lo + (int64_t)q * dm.dp, v, xv);
        if (x16)
          acc += st_bf16x4(x16, v, xv);  // BF16 copy; the norm of the rounded row
        else
          acc += xv.x * xv.x + xv.y * xv.y + xv.z * xv.z + xv.w * xv.w;
      }
    }
    acc = warp_sum(acc);
    if (lane == 0) a.b.xnorm[q] = acc;
  }
  if (dm.trace) __threadfence();  // diagnostics: the warp's stores performed before its end stamp
  trace_warp_end(dm.trace, KGE_K_GATHER);
  if (a.flow) {  // rows of each chunk done: k_tc_fwd starts a chunk as soon as its g + k rows are here
    __shared__ int s_chunk[8];
    if (lane == 0)
      s_chunk[threadIdx.x >> 5] = row < dm.B ? row / dm.g : (row < dm.B + n_neg ? (row - dm.B) / dm.k : -1);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      int c0 = -1;
      uint32_t n = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        const int cw = s_chunk[w];
        if (cw != c0) {
          if (c0 >= 0) atomicAdd(&a.flow[c0], n);
          c0 = cw;
          n = 0;
        }
        if (cw >= 0) ++n;
      }
      if (c0 >= 0) atomicAdd(&a.flow[c0], n);
    }
  }
  trace_stamp(dm.trace, KGE_K_GATHER, 7);
  if (dm.trace && blockIdx.x == 0) {
    // diagnostics: the previous step's k_update end (max over its CTAs' end stamps, not yet overwritten by this
    // step's) into CTA 0's slot 2 -- the gap to this step's release (slot 1) is the inter-step PDL hand-over
    // (slot 3: the last k_update CTA start, early-leaving CTAs included)
    __shared__ unsigned long long s_mx, s_m0;
    if (threadIdx.x == 0) s_mx = s_m0 = 0;
    __syncthreads();
    unsigned long long mx = 0, m0 = 0;
    for (int c = threadIdx.x; c < kTraceCtas; c += blockDim.x) {
      mx = max(mx, (unsigned long long)dm.trace[((size_t)KGE_K_UPDATE * kTraceCtas + c) * kTraceSlots + 6]);
      m0 = max(m0, (unsigned long long)dm.trace[((size_t)KGE_K_UPDATE * kTraceCtas + c) * kTraceSlots + 0]);
    }
    atomicMax(&s_mx, mx);
    atomicMax(&s_m0, m0);
    __syncthreads();
    if (threadIdx.x == 0) {
      dm.trace[((size_t)KGE_K_GATHER * kTraceCtas) * kTraceSlots + 2] = s_mx;
      dm.trace[((size_t)KGE_K_GATHER * kTraceCtas) * kTraceSlots + 3] = s_m0;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// k_neg_fwd (FFMA): S_c = pair(O_c, X'_c), 64x64 tiles, K-chunks of 32 floats, 4x4 micro-tiles
// ------------------------------------------------------------------------------------------------
constexpr int TM = 64, TN = 64, TK = 32, TPAD = 4;

// Blackwell 2-wide FP32 (FADD2 / FFMA2 on a register pair; a scalar operand is broadcast for free): the FFMA
// kernels process output columns in pairs for the families whose per-element work is add / fma only
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

struct NegArgs {
  Dims dm;
  StepBuffers b;
  float* Gocc;  // dX' destination (occurrence rows 2B + q)
  float4* part;  // split-K partial tiles [tile][ks][4][256 threads] (float4), L2-resident scratch
  int32_t* cnt;  // [tiles] arrival counters (zero between launches: the last CTA of a tile resets its counter)
  int32_t ks;    // split-K factor of this launch
};

// Register-staged tile loader: a [64 rows x 32 k] tile of a row-major [rows x d] matrix is fetched as 2 float4 per
// thread into registers (next chunk in flight while the current one is computed) and stored transposed into smem
// T[k][row]. CMOD: k-chunk = 16 real parts from column kc and 16 imaginary parts from column d/2 + kc.
template <bool CPLX>
struct TileRegs {
  float4 x[2];
  __device__ __forceinline__ void load(const float* __restrict__ base, int row0, int nrows, int kc, int d, int pitch) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = threadIdx.x + q * 256;
      const int r = idx / (TK / 4), v = idx % (TK / 4);
      x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (CPLX) {
        const int half = d >> 1;
        const int cc = kc + (v & 3) * 4;  // complex index
        const int col = (v < 4) ? cc : half + cc;
        if (row0 + r < nrows && cc < half) x[q] = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)(row0 + r) * pitch + col));
      } else {
        const int col = kc + v * 4;
        if (row0 + r < nrows && col < d) x[q] = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)(row0 + r) * pitch + col));
      }
    }
  }
  __device__ __forceinline__ void store(float (*T)[TM + TPAD]) const {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = threadIdx.x + q * 256;
      const int r = idx / (TK / 4), v = idx % (TK / 4);
      T[v * 4 + 0][r] = x[q].x;
      T[v * 4 + 1][r] = x[q].y;
      T[v * 4 + 2][r] = x[q].z;
      T[v * 4 + 3][r] = x[q].w;
    }
  }
};

// Deterministic split-K: every CTA of a tile parks its 16 per-thread partial sums, the last to arrive adds all
// ks partials in ks order (the result does not depend on arrival order) and runs the epilogue. Returns false for the
// CTAs that leave. acc is overwritten with the full sum in the returning CTA.
__device__ __forceinline__ bool splitk_reduce(float (&acc)[4][4], float4* __restrict__ part, int32_t* cnt, int tile,
                                              int ks, int nks) {
  if (nks == 1) return true;
  __shared__ int s_last;
  float4* mine = part + ((int64_t)tile * nks + ks) * 4 * 256;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
    mine[ii * 256 + threadIdx.x] = make_float4(acc[ii][0], acc[ii][1], acc[ii][2], acc[ii][3]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&cnt[tile], 1) == nks - 1;
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
#pragma unroll
  for (int ii = 0; ii < 4; ++ii)
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = 0.f;
  for (int q = 0; q < nks; ++q) {
    const float4* pq = part + ((int64_t)tile * nks + q) * 4 * 256;
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const float4 v = __ldcg(pq + ii * 256 + threadIdx.x);
      acc[ii][0] += v.x;
      acc[ii][1] += v.y;
      acc[ii][2] += v.z;
      acc[ii][3] += v.w;
    }
  }
  if (threadIdx.x == 0) cnt[tile] = 0;  // ready for the next launch
  return true;
}

template <int FAM>
__global__ void __launch_bounds__(256, 2) k_neg_fwd(NegArgs a) {
  constexpr bool CPLX = FAM == FAM_CMOD;
  const Dims& dm = a.dm;
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float As[TK][TM + TPAD];
  __shared__ __align__(16) float Bs[TK][TN + TPAD];
  __shared__ float red[8];
  const int nks = a.ks, c = blockIdx.z / nks, ks = blockIdx.z % nks;
  const int i0 = blockIdx.y * TM, j0 = blockIdx.x * TN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* Oc = a.b.O + (int64_t)c * dm.g * dm.dp;
  const float* Xc = a.b.X + (int64_t)c * dm.k * dm.dp;
  float acc[4][4] = {};
  uint64_t acc2[4][2] = {};  // packed accumulators (DOT / L2 / L2SQ)
  const int kend = CPLX ? (dm.d >> 1) : dm.d;
  const int kstep = CPLX ? TK / 2 : TK;
  const int nch = (kend + kstep - 1) / kstep, per = (nch + nks - 1) / nks;
  const int ch0 = min(nch, ks * per), ch1 = min(nch, ch0 + per);
  TileRegs<CPLX> ra, rb;
  if (ch0 < ch1) {
    ra.load(Oc, i0, dm.g, ch0 * kstep, dm.d, dm.dp);
    rb.load(Xc, j0, dm.k, ch0 * kstep, dm.d, dm.dp);
  }
  for (int ch = ch0; ch < ch1; ++ch) {
    ra.store(As);
    rb.store(Bs);
    __syncthreads();
    if (ch + 1 < ch1) {  // next chunk's loads in flight during this chunk's arithmetic
      ra.load(Oc, i0, dm.g, (ch + 1) * kstep, dm.d, dm.dp);
      rb.load(Xc, j0, dm.k, (ch + 1) * kstep, dm.d, dm.dp);
    }
    if (CPLX) {
#pragma unroll 4
      for (int e = 0; e < TK / 2; ++e) {
        const float4 ar = *reinterpret_cast<const float4*>(&As[e][ty * 4]);
        const float4 ai = *reinterpret_cast<const float4*>(&As[e + TK / 2][ty * 4]);
        const float4 br = *reinterpret_cast<const float4*>(&Bs[e][tx * 4]);
        const float4 bi = *reinterpret_cast<const float4*>(&Bs[e + TK / 2][tx * 4]);
        const float arr[4] = {ar.x, ar.y, ar.z, ar.w}, aii[4] = {ai.x, ai.y, ai.z, ai.w};
        const float brr[4] = {br.x, br.y, br.z, br.w}, bii[4] = {bi.x, bi.y, bi.z, bi.w};
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const float ur = arr[ii] - brr[jj], ui = aii[ii] - bii[jj];
            acc[ii][jj] += sqrtf(ur * ur + ui * ui);
          }
      }
    } else if (FAM == FAM_L1) {
#pragma unroll 8
      for (int e = 0; e < TK; ++e) {
        const float4 av = *reinterpret_cast<const float4*>(&As[e][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[e][tx * 4]);
        const float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[ii][jj] += fabsf(ar[ii] - br[jj]);
      }
    } else {  // DOT / L2 / L2SQ on packed column pairs (same operations and order as the scalar form)
#pragma unroll 8
      for (int e = 0; e < TK; ++e) {
        const float4 av = *reinterpret_cast<const float4*>(&As[e][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[e][tx * 4]);
        const float ar[4] = {av.x, av.y, av.z, av.w};
        const uint64_t b01 = pk2(bv.x, bv.y), b23 = pk2(bv.z, bv.w);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const uint64_t a2 = pk2(ar[ii], ar[ii]);
          if (FAM == FAM_DOT) {
            acc2[ii][0] = fma2(a2, b01, acc2[ii][0]);
            acc2[ii][1] = fma2(a2, b23, acc2[ii][1]);
          } else {
            const uint64_t u0 = sub2(a2, b01), u1 = sub2(a2, b23);
            acc2[ii][0] = fma2(u0, u0, acc2[ii][0]);
            acc2[ii][1] = fma2(u1, u1, acc2[ii][1]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (!CPLX && FAM != FAM_L1) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      upk2(acc2[ii][0], acc[ii][0], acc[ii][1]);
      upk2(acc2[ii][1], acc[ii][2], acc[ii][3]);
    }
  }
  const int tile = (c * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (!splitk_reduce(acc, a.part, a.cnt, tile, ks, nks)) return;
  // epilogue: f-, dL/dS coefficient, loss partial
  const float inv_bk = 1.f / ((float)dm.B * (float)dm.k);
  const bool pairwise = dm.loss == KGE_LOSS_PAIRWISE;
  float lsum = 0.f;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int i = i0 + ty * 4 + ii;
    const float fpos = pairwise && i < dm.g ? pair_score_from(FAM, a.b.pstat[(int64_t)c * dm.g + i], dm.gamma) : 0.f;
    int nact = 0;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = j0 + tx * 4 + jj;
      if (i < dm.g && j < dm.k) {
        const float st = acc[ii][jj];
        float f, coef, dLdf, lterm;
        f = pair_score_from(FAM, st, dm.gamma);
        if (pairwise) {
          int act;
          lterm = hinge_term(f, fpos, dm.gamma, inv_bk, dLdf, act);
          nact += act;
        } else {
          dLdf = sigmoid(f) * inv_bk;
          lterm = -log_sigmoid(-f);
        }
        if (FAM == FAM_DOT) {
          coef = dLdf;
        } else if (FAM == FAM_L2) {
          coef = -dLdf / fmaxf(sqrtf(st), 1e-12f);
        } else if (FAM == FAM_L2SQ) {
          coef = -2.f * dLdf;
        } else {
          coef = -dLdf;
        }
        a.b.W[((int64_t)c * dm.g + i) * dm.kp + j] = coef;
        if (a.b.fdbg) a.b.fdbg[((int64_t)c * dm.g + i) * dm.k + j] = f;  // KGE_OPT_CAPTURE_NEG
        lsum += lterm;
      }
    }
    if (nact) atomicAdd(&a.b.pcnt[(int64_t)c * dm.g + i], nact);  // integer: exact in any order
  }
  lsum = warp_sum(lsum);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += red[w];
    a.b.lneg[tile] = sum;
  }
}

// ------------------------------------------------------------------------------------------------
// k_neg_bwd (FFMA): blockIdx.z < C -> dO tiles of chunk z ; blockIdx.z >= C -> dX' tiles of chunk z - C.
//   dO[i][e]  = sum_j W_ij phi_o(o_ie, x_je)      phi_o: DOT x ; L2/L2SQ (o-x) ; L1 sgn(o-x) ; CMOD (o-x)/|z|
//   dX'[j][e] = sum_i W_ij phi_x(o_ie, x_je)      phi_x: DOT o ; others -phi_o
// Columns of a tile: 64 floats (CMOD: 32 complex elements -> re and im halves).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ float sgnf(float u) { return u > 0.f ? 1.f : (u < 0.f ? -1.f : 0.f); }

template <int FAM>
__global__ void __launch_bounds__(256, 2) k_neg_bwd(NegArgs a) {
  constexpr bool CPLX = FAM == FAM_CMOD;
  const Dims& dm = a.dm;
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float Ws[TK][TM + TPAD];  // [K index][row index of the output]
  __shared__ __align__(16) float Vs[TK][TN + TPAD];  // [K index][column]  (CPLX: re cols 0..31, im cols 32..63)
  const int nks = a.ks, zz = blockIdx.z / nks, ks = blockIdx.z % nks;
  const bool pass_x = zz >= dm.C;
  const int c = pass_x ? zz - dm.C : zz;
  const int nrows = pass_x ? dm.k : dm.g;        // output rows: j (dX') or i (dO)
  const int nk = pass_x ? dm.g : dm.k;           // contraction: i or j
  const int r0 = blockIdx.y * TM;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int half = dm.d >> 1;
  const float* Oc = a.b.O + (int64_t)c * dm.g * dm.dp;
  const float* Xc = a.b.X + (int64_t)c * dm.k * dm.dp;
  const float* Wc = a.b.W + (int64_t)c * dm.g * dm.kp;
  const float* Self = pass_x ? Xc : Oc;   // the matrix whose rows are the output rows
  const float* Other = pass_x ? Oc : Xc;  // streamed over the contraction index
  // output columns of this thread
  int col[4];
  bool colok[4];
  const int cb = blockIdx.x * (CPLX ? TN / 2 : TN);
#pragma unroll
  for (int ee = 0; ee < 4; ++ee) {
    if (CPLX) {
      const int cc = cb + (tx & 7) * 4 + ee;  // complex index
      col[ee] = cc;
      colok[ee] = cc < half;
    } else {
      col[ee] = cb + tx * 4 + ee;
      colok[ee] = col[ee] < dm.d;
    }
  }
  const bool imag_lane = CPLX && tx >= 8;  // CPLX: tx<8 own re columns, tx>=8 own the matching im columns
  // own values (self rows x own columns); CPLX needs both parts of own complex entries
  float sv[4][4], si[4][4];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int rr = r0 + ty * 4 + ii;
#pragma unroll
    for (int ee = 0; ee < 4; ++ee) {
      const bool ok = rr < nrows && colok[ee];
      if (CPLX) {
        sv[ii][ee] = ok ? Self[(int64_t)rr * dm.dp + col[ee]] : 0.f;
        si[ii][ee] = ok ? Self[(int64_t)rr * dm.dp + half + col[ee]] : 0.f;
      } else {
        sv[ii][ee] = ok ? Self[(int64_t)rr * dm.dp + col[ee]] : 0.f;
        si[ii][ee] = 0.f;
      }
    }
  }
  // register-staged tiles (2 float4 of W and 2 of V per thread), the next chunk in flight during the arithmetic.
  // W chunk: 32 contraction x 64 output rows. dX' reads W[k][row] (rows contiguous); dO reads W[row][k] (k
  // contiguous): each float4 then runs along k and is transposed on the smem store.
  float4 wr[2], vr[2];
  auto load = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = threadIdx.x + q * 256;  // 512 float4 per operand tile
      float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
      if (pass_x) {  // kk = idx / 16, rows 4 * (idx % 16) .. +3
        const int kk = idx >> 4, rq = (idx & 15) * 4, kidx = k0 + kk;
        if (kidx < nk && r0 + rq < nrows) w = __ldcg(reinterpret_cast<const float4*>(Wc + (int64_t)kidx * dm.kp + r0 + rq));
      } else {       // row = idx / 8, k 4 * (idx % 8) .. +3
        const int rr = idx >> 3, kq = (idx & 7) * 4, kidx = k0 + kq;
        if (kidx < nk && r0 + rr < nrows) w = __ldcg(reinterpret_cast<const float4*>(Wc + (int64_t)(r0 + rr) * dm.kp + kidx));
      }
      wr[q] = w;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      const int kk = idx >> 4, cq = (idx & 15) * 4, kidx = k0 + kk;  // Vs[kk][cq .. cq+3]
      if (kidx < nk) {
        if (CPLX) {
          const int cc = cb + (cq & 31);
          if (cc < half) v = __ldcg(reinterpret_cast<const float4*>(Other + (int64_t)kidx * dm.dp + (cq < 32 ? cc : half + cc)));
        } else {
          const int gcol = cb + cq;
          if (gcol < dm.d) v = __ldcg(reinterpret_cast<const float4*>(Other + (int64_t)kidx * dm.dp + gcol));
        }
      }
      vr[q] = v;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int idx = threadIdx.x + q * 256;
      if (pass_x) {
        const int kk = idx >> 4, rq = (idx & 15) * 4;
        *reinterpret_cast<float4*>(&Ws[kk][rq]) = wr[q];
      } else {
        const int rr = idx >> 3, kq = (idx & 7) * 4;
        Ws[kq + 0][rr] = wr[q].x;
        Ws[kq + 1][rr] = wr[q].y;
        Ws[kq + 2][rr] = wr[q].z;
        Ws[kq + 3][rr] = wr[q].w;
      }
      const int kk = idx >> 4, cq = (idx & 15) * 4;
      *reinterpret_cast<float4*>(&Vs[kk][cq]) = vr[q];
    }
  };
  float acc[4][4] = {};
  uint64_t acc2[4][2] = {}, sv2[4][2];
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    sv2[ii][0] = pk2(sv[ii][0], sv[ii][1]);
    sv2[ii][1] = pk2(sv[ii][2], sv[ii][3]);
  }
  const int nch = (nk + TK - 1) / TK, per = (nch + nks - 1) / nks;
  const int ch0 = min(nch, ks * per), ch1 = min(nch, ch0 + per);
  if (ch0 < ch1) load(ch0 * TK);
  for (int ch = ch0; ch < ch1; ++ch) {
    store();
    __syncthreads();
    if (ch + 1 < ch1) load((ch + 1) * TK);
#pragma unroll 4
    for (int kk = 0; kk < TK; ++kk) {
      const float4 wv = *reinterpret_cast<const float4*>(&Ws[kk][ty * 4]);
      const float w[4] = {wv.x, wv.y, wv.z, wv.w};
      float ov[4], oi[4];
      if (CPLX) {
        const int cl = (tx & 7) * 4;
        const float4 a_ = *reinterpret_cast<const float4*>(&Vs[kk][cl]);
        const float4 b_ = *reinterpret_cast<const float4*>(&Vs[kk][32 + cl]);
        ov[0] = a_.x; ov[1] = a_.y; ov[2] = a_.z; ov[3] = a_.w;
        oi[0] = b_.x; oi[1] = b_.y; oi[2] = b_.z; oi[3] = b_.w;
      } else {
        const float4 a_ = *reinterpret_cast<const float4*>(&Vs[kk][tx * 4]);
        ov[0] = a_.x; ov[1] = a_.y; ov[2] = a_.z; ov[3] = a_.w;
        oi[0] = oi[1] = oi[2] = oi[3] = 0.f;
      }
      if (!CPLX && FAM != FAM_L1) {  // DOT / L2 / L2SQ on packed column pairs (same operations and order)
        const uint64_t o01 = pk2(ov[0], ov[1]), o23 = pk2(ov[2], ov[3]);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
          const uint64_t w2 = pk2(w[ii], w[ii]);
          if (FAM == FAM_DOT) {
            acc2[ii][0] = fma2(w2, o01, acc2[ii][0]);
            acc2[ii][1] = fma2(w2, o23, acc2[ii][1]);
          } else {  // u = self - other
            acc2[ii][0] = fma2(w2, sub2(sv2[ii][0], o01), acc2[ii][0]);
            acc2[ii][1] = fma2(w2, sub2(sv2[ii][1], o23), acc2[ii][1]);
          }
        }
      } else {
#pragma unroll
      for (int ii = 0; ii < 4; ++ii)
#pragma unroll
        for (int ee = 0; ee < 4; ++ee) {
          // o = (pass_x ? other : self), x = (pass_x ? self : other)
          const float s_ = sv[ii][ee], t_ = ov[ee];
          if (FAM == FAM_DOT) {
            acc[ii][ee] = fmaf(w[ii], t_, acc[ii][ee]);
          } else if (FAM == FAM_L1) {
            // dO: w sgn(o - x) with o = self; dX': -w sgn(o - x) = w sgn(x - o) with x = self -- both are
            // w sgn(self - other), sgn(0) = 0 (reading c.10), formed as (s > t) - (s < t) (one FSET each): no
            // per-element selects on the pass (the same exact +-1 / 0 factors as before)
            const float sg = (s_ > t_ ? 1.f : 0.f) - (s_ < t_ ? 1.f : 0.f);
            acc[ii][ee] = fmaf(w[ii], sg, acc[ii][ee]);
          } else if (FAM == FAM_CMOD) {
            // dO: w (o - x) / |o - x|, dX': -w (o - x) / |o - x| = w (x - o) / |x - o|: both w (self - other) / |.|
            // (x - o == -(o - x) exactly), so no per-element selects on the pass
            const float ur = s_ - t_, ui = si[ii][ee] - oi[ee];
            const float inv = 1.f / fmaxf(sqrtf(ur * ur + ui * ui), 1e-12f);
            const float comp = imag_lane ? ui : ur;
            acc[ii][ee] = fmaf(w[ii], comp * inv, acc[ii][ee]);
          } else {  // L2, L2SQ: phi_o = o - x
            const float u = s_ - t_;  // self - other: = (o - x) for dO, = (x - o) = -phi_o for dX'
            acc[ii][ee] = fmaf(w[ii], u, acc[ii][ee]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (!CPLX && FAM != FAM_L1) {
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      upk2(acc2[ii][0], acc[ii][0], acc[ii][1]);
      upk2(acc2[ii][1], acc[ii][2], acc[ii][3]);
    }
  }
  const int tile = (zz * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  if (!splitk_reduce(acc, a.part, a.cnt, tile, ks, nks)) return;
  // store
  float* dst = pass_x ? a.Gocc + ((int64_t)2 * dm.B + (int64_t)c * dm.k) * dm.d : a.b.dO + (int64_t)c * dm.g * dm.d;
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int rr = r0 + ty * 4 + ii;
    if (rr >= nrows) continue;
#pragma unroll
    for (int ee = 0; ee < 4; ++ee) {
      if (!colok[ee]) continue;
      const int gcol = CPLX ? (imag_lane ? half + col[ee] : col[ee]) : col[ee];
      dst[(int64_t)rr * dm.d + gcol] = acc[ii][ee];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// k_chain: per positive, total d/do and d/d(other) = dO (negatives) + w+ * dpair(o, other), then the chain rule of
// combine -> per-occurrence gradients Gocc[i] (head row), Gocc[B+i] (tail row), Grel[i]. Last CTA: loss.
// ------------------------------------------------------------------------------------------------
struct ChainArgs {
  Dims dm;
  Slot s;
  EntRows ent;
  const float* rel;
  StepBuffers b;
  int32_t n_neg_parts;
};

__device__ __forceinline__ void dpair(int fam, float o, float x, float scale, float& go, float& gx) {
  // derivative of the pair score f w.r.t. o and x, times scale (scale folds 1/D for L2)
  switch (fam) {
    case FAM_DOT: go = scale * x; gx = scale * o; return;
    case FAM_L1: { const float s = sgnf(o - x); go = -scale * s; gx = scale * s; return; }
    case FAM_L2: { const float u = o - x; go = -scale * u; gx = scale * u; return; }
    default: { const float u = o - x; go = -2.f * scale * u; gx = 2.f * scale * u; return; }  // L2SQ
  }
}

template <int V>
__global__ void __launch_bounds__(256) k_chain(ChainArgs a) {
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_CHAIN, 0);
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == gridDim.x - 1) {
    // deterministic loss: fixed lane assignment, fixed warp order (reading c.9 normalisation)
    if (threadIdx.x < 32) {
      float sp = 0.f, sn = 0.f;
      for (int i = lane; i < dm.B; i += 32) sp += a.b.lpos[i];
      for (int q = lane; q < a.n_neg_parts; q += 32) sn += a.b.lneg[q];
      sp = warp_sum(sp);
      sn = warp_sum(sn);
      if (lane == 0) {
        const float L = sp / (float)dm.B + sn / ((float)dm.B * (float)dm.k);
        store_loss(a.b.loss, a.s.info, L);
        const bool bad = !isfinite(L);
        a.b.flags[2 + (a.s.info[0] & 1)] = bad ? 1 : 0;
        if (bad) a.b.flags[0] = 1;
      }
    }
    return;
  }
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= dm.B) return;
  const int mode = a.s.mode[i / dm.g];
  const float* h = a.ent.row(a.s.ph[i]);
  const float* t = a.ent.row(a.s.pt[i]);
  const float* r = a.rel + (int64_t)a.s.pr[i] * dm.drel;
  const float* o = a.b.O + (int64_t)i * dm.dp;
  const float* dO = a.b.dO + (int64_t)i * dm.d;
  const float* other = mode == 0 ? t : h;
  const float* ent_c = mode == 0 ? h : t;  // the combined entity side
  float* gH = a.b.Gocc + (int64_t)i * dm.d;
  float* gT = a.b.Gocc + (int64_t)(dm.B + i) * dm.d;
  float* gR = a.b.Grel + (int64_t)i * dm.drel;
  float* gOther = mode == 0 ? gT : gH;
  float* gC = mode == 0 ? gH : gT;
  // dL/df+: logistic from the gather; pairwise = -(active hinges of positive i) / (B k) (reading c.9')
  const float wp = dm.loss == KGE_LOSS_PAIRWISE ? -(float)a.b.pcnt[i] * (1.f / ((float)dm.B * (float)dm.k))
                                                : a.b.wpos[i];
  const float scale = dm.family == FAM_L2 ? wp / fmaxf(sqrtf(a.b.pstat[i]), 1e-12f) : wp;
  const int model = dm.model;
  if (!is_complex_model(model)) {
    const int d4 = dm.d >> 2;
    Row4<V> Ov, Xv, Dv, Rv, Ev;
    Ov.load(o, lane, d4);
    Xv.load(other, lane, d4);
    Dv.load(dO, lane, d4);
    if (model == KGE_DISTMULT) {
      Rv.load(r, lane, d4);
      Ev.load(ent_c, lane, d4);
    }
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int v = lane + 32 * m;
      if (v >= d4) continue;
      float oo[4], xx[4], dd[4], go[4], gx[4];
      f4_to(Ov.v[m], oo);
      f4_to(Xv.v[m], xx);
      f4_to(Dv.v[m], dd);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        dpair(dm.family, oo[u], xx[u], scale, go[u], gx[u]);
        go[u] += dd[u];
      }
      st4(gOther, v, make_float4(gx[0], gx[1], gx[2], gx[3]));
      float4 gc, gr;
      if (model == KGE_DISTMULT) {  // tail o = h*r: dh = go*r, dr = go*h ; head o = r*t: dt = go*r, dr = go*t
        const float4 rv = Rv.v[m], ev = Ev.v[m];
        gc = make_float4(go[0] * rv.x, go[1] * rv.y, go[2] * rv.z, go[3] * rv.w);
        gr = make_float4(go[0] * ev.x, go[1] * ev.y, go[2] * ev.z, go[3] * ev.w);
      } else {  // TransE: tail o = h + r ; head o = t - r
        gc = make_float4(go[0], go[1], go[2], go[3]);
        gr = mode == 0 ? gc : make_float4(-go[0], -go[1], -go[2], -go[3]);
      }
      st4(gC, v, gc);
      st4(gR, v, gr);
    }
    return;
  }
  // complex models: lanes own complex element groups (re at v, im at v + n4)
  const int n4 = dm.d >> 3;
  Row4<V> OR, OI, XR, XI, DR, DI, ER, EI, R1, R2;
  OR.load(o, lane, n4);
  OI.load(o + 4 * n4, lane, n4);
  XR.load(other, lane, n4);
  XI.load(other + 4 * n4, lane, n4);
  DR.load(dO, lane, n4);
  DI.load(dO + 4 * n4, lane, n4);
  ER.load(ent_c, lane, n4);
  EI.load(ent_c + 4 * n4, lane, n4);
  R1.load(r, lane, n4);
  if (model == KGE_COMPLEX) R2.load(r + 4 * n4, lane, n4);
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int v = lane + 32 * m;
    if (v >= n4) continue;
    float o_r[4], o_i[4], x_r[4], x_i[4], d_r[4], d_i[4], e_r[4], e_i[4], rr_[4], ri_[4];
    f4_to(OR.v[m], o_r);
    f4_to(OI.v[m], o_i);
    f4_to(XR.v[m], x_r);
    f4_to(XI.v[m], x_i);
    f4_to(DR.v[m], d_r);
    f4_to(DI.v[m], d_i);
    f4_to(ER.v[m], e_r);
    f4_to(EI.v[m], e_i);
    if (model == KGE_COMPLEX) {
      f4_to(R1.v[m], rr_);
      f4_to(R2.v[m], ri_);
    } else {
      float th[4];
      f4_to(R1.v[m], th);
#pragma unroll
      for (int u = 0; u < 4; ++u) sincosf(th[u], &ri_[u], &rr_[u]);  // (cos, sin)
    }
    float gxr[4], gxi[4], ger[4], gei[4], grr[4], gri[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float gor, goi;
      if (dm.family == FAM_CMOD) {
        const float ur = o_r[u] - x_r[u], ui = o_i[u] - x_i[u];
        const float inv = scale / fmaxf(sqrtf(ur * ur + ui * ui), 1e-12f);
        gor = -inv * ur;
        goi = -inv * ui;
        gxr[u] = inv * ur;
        gxi[u] = inv * ui;
      } else {
        dpair(dm.family, o_r[u], x_r[u], scale, gor, gxr[u]);
        dpair(dm.family, o_i[u], x_i[u], scale, goi, gxi[u]);
      }
      gor += d_r[u];
      goi += d_i[u];
      const float c = rr_[u], sn = ri_[u], ea = e_r[u], eb = e_i[u];
      if (model == KGE_COMPLEX) {
        if (mode == 0) {  // o = (a c - b s, a s + b c) with r = c + i s
          ger[u] = gor * c + goi * sn;
          gei[u] = -gor * sn + goi * c;
          grr[u] = gor * ea + goi * eb;
          gri[u] = -gor * eb + goi * ea;
        } else {  // o = (c a + s b, c b - s a) with t = a + i b
          ger[u] = gor * c - goi * sn;
          gei[u] = gor * sn + goi * c;
          grr[u] = gor * ea + goi * eb;
          gri[u] = gor * eb - goi * ea;
        }
      } else {  // RotatE, r = e^{i theta}
        if (mode == 0) {  // o = (a c - b s, a s + b c)
          ger[u] = gor * c + goi * sn;
          gei[u] = -gor * sn + goi * c;
          grr[u] = gor * (-ea * sn - eb * c) + goi * (ea * c - eb * sn);
        } else {  // o = (a c + b s, -a s + b c)
          ger[u] = gor * c - goi * sn;
          gei[u] = gor * sn + goi * c;
          grr[u] = gor * (-ea * sn + eb * c) + goi * (-ea * c - eb * sn);
        }
        gri[u] = 0.f;
      }
    }
    st4(gOther, v, make_float4(gxr[0], gxr[1], gxr[2], gxr[3]));
    st4(gOther, v + n4, make_float4(gxi[0], gxi[1], gxi[2], gxi[3]));
    st4(gC, v, make_float4(ger[0], ger[1], ger[2], ger[3]));
    st4(gC, v + n4, make_float4(gei[0], gei[1], gei[2], gei[3]));
    st4(gR, v, make_float4(grr[0], grr[1], grr[2], grr[3]));
    if (model == KGE_COMPLEX) st4(gR, v + n4, make_float4(gri[0], gri[1], gri[2], gri[3]));
  }
}

// ------------------------------------------------------------------------------------------------
// k_update: segmented reduce (sorted occurrence order) fused with sparse row-wise Adagrad (reading c.11)
//   state += mean_j G_j^2 ; row -= lr * G / sqrt(state + eps)
// ------------------------------------------------------------------------------------------------
struct UpdateArgs {
  Dims dm;
  Slot s;
  float* ent;
  float* ent_st;
  float* rel;
  float* rel_st;
  StepBuffers b;
  float* gu;                   // P > 1: per-unique entity gradient sums go here (the owner applies Adagrad)
  const int32_t* split_index;  // P > 1: relation -> index among split relations, -1 if not split
  float* grel_split;           // P > 1: per-rank sums of split relations
  int32_t* seg_cnt;            // [B + n_occ] per-unique-row segment arrival counters (zero between steps)
  int32_t pos_lo, pos_hi;      // positions handled: [0, B) relations, [B, B + n_occ) entities (lag = 1 splits them)
  const Slot* next;            // device slot of the next step (P == 1), or nullptr: its entity rows are prefetched
  int32_t stg_rows;            // V <= 4: rows per warp staged in dynamic shared memory (pitch w4 float4)
};

// Row accumulator: V float4 per lane.
template <int V>
struct RowAcc {
  float4 g[V];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int m = 0; m < V; ++m) g[m] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __device__ __forceinline__ void add(const float4& x, int m) {
    g[m].x += x.x; g[m].y += x.y; g[m].z += x.z; g[m].w += x.w;
  }
};

// Adagrad on one row given its summed gradient (reading c.11): state += mean(G^2); row -= lr G / sqrt(state + eps).
// row_v / st0 were prefetched before the segment sum.
template <int V>
__device__ __forceinline__ void adagrad_row(float* __restrict__ row, float* __restrict__ st, const RowAcc<V>& acc,
                                            float4 (&row_v)[V], float st0, int w4, int w, float lr, float eps,
                                            int lane) {
  float sq = 0.f;
#pragma unroll
  for (int m = 0; m < V; ++m)
    if (lane + 32 * m < w4)
      sq += acc.g[m].x * acc.g[m].x + acc.g[m].y * acc.g[m].y + acc.g[m].z * acc.g[m].z + acc.g[m].w * acc.g[m].w;
  sq = warp_sum(sq);
  const float s = st0 + sq / (float)w;
  if (lane == 0) *st = s;
  const float step = lr / sqrtf(s + eps);
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int v = lane + 32 * m;
    if (v < w4) {
      float4 x = row_v[m];
      x.x -= step * acc.g[m].x; x.y -= step * acc.g[m].y; x.z -= step * acc.g[m].z; x.w -= step * acc.g[m].w;
      st4(row, v, x);
    }
  }
}

template <int V>
__device__ __forceinline__ void prefetch_row(const float* __restrict__ row, float4 (&row_v)[V], int w4, int lane) {
#pragma unroll
  for (int m = 0; m < V; ++m) {
    const int v = lane + 32 * m;
    row_v[m] = v < w4 ? ld4(row, v) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// One warp per SEGMENT: the sorted occurrence list of each unique row is cut into segments of kSeg consecutive
// positions; the warp whose position starts a segment sums that segment in occurrence order. A row with one segment is
// updated by that warp directly. A row with several (hub relations carry ~10% of a Zipf batch) parks each segment sum
// in the gradient row of the segment's first occurrence (read by no other warp), bumps a per-row arrival counter, and
// the last arriver adds the segment sums in segment order (deterministic: the association is fixed, no float
// atomics) and applies Adagrad. Warps: [B relation positions][n_occ entity positions]; relation warps first.
// Everything not produced by the backward pass (sample-slot indices, current rows and Adagrad state -- written by
// kernels that completed before the forward pass started) is loaded before griddepcontrol.wait.
constexpr int kSeg = 8;
constexpr int kStgBytes = 56 * 1024;  // k_update (V <= 4): staging budget per CTA (4 CTAs per SM)

__device__ __forceinline__ void cpa16(float4* dst, const float4* src) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <int V>
__global__ void __launch_bounds__(256, V >= 8 ? 1 : 4) k_update(UpdateArgs a) {
  const Dims& dm = a.dm;
  trace_stamp(dm.trace, KGE_K_UPDATE, 0);
  const int lane = threadIdx.x & 31;
  const int gw = a.pos_lo + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const bool rel = gw < dm.B;
  const int p = rel ? gw : gw - dm.B;
  const int npos = rel ? dm.B : dm.n_occ;
  const int32_t* occ_sorted = rel ? a.s.rel_occ : a.s.ent_occ;
  const int32_t* off = rel ? a.s.rel_off : a.s.ent_off;
  float* G = rel ? a.b.Grel : a.b.Gocc;
  const int w = rel ? dm.drel : dm.d, w4 = w >> 2;
  bool live = p < npos && gw < a.pos_hi;
  int u = 0, r0 = 0, r1 = 0;
  if (live) {
    u = (rel ? a.s.rel_inv : a.s.ent_inv)[occ_sorted[p]];
    r0 = off[u];
    r1 = off[u + 1];
    live = (p - r0) % kSeg == 0;
  }
  if (a.next) {
    // warm L2 and the TLBs with the next step's entity rows while this step's backward still runs: its gather follows
    // this kernel and otherwise pays the page walks of random rows in a 137 GB table (the rows this update writes
    // stay coherent in L2). One 128-byte line per thread.
    const Slot nx = *a.next;
    const int lines = (dm.d * 4 + 127) / 128;
    const int n = dm.n_occ * lines;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
      const int o = q / lines, l = q - o * lines;
      const int32_t e = o < dm.B ? nx.ph[o] : (o < 2 * dm.B ? nx.pt[o - dm.B] : nx.neg[o - 2 * dm.B]);
      if (e >= 0 && e < dm.n_entities)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.ent + (int64_t)e * dm.d + l * 32));
    }
  }
  if (__syncthreads_or(live) == 0) return;  // no segment starts in this CTA: leave before the wait
  if (!live) return;
  const int n = min(kSeg, r1 - p);  // this segment: positions [p, p + n)
  const int oj = lane < n ? occ_sorted[p + lane] : 0;
  const int nseg = (r1 - r0 + kSeg - 1) / kSeg;
  const int32_t id = (rel ? a.s.rel_uniq : a.s.ent_uniq)[u];
  float* row;
  float* st;
  bool plain_sum;  // write the sum (P > 1 entity sum for the owner / split-relation rank sum) instead of Adagrad
  if (rel) {
    const int sidx = a.split_index ? a.split_index[id] : -1;
    plain_sum = sidx >= 0;
    row = plain_sum ? a.grel_split + (int64_t)sidx * w : a.rel + (int64_t)id * w;
    st = a.rel_st + id;
  } else {
    plain_sum = a.gu != nullptr;
    row = plain_sum ? a.gu + (int64_t)u * w : a.ent + (int64_t)id * w;
    st = a.ent_st + id;
  }
  if (!plain_sum) {  // warm L2 with the row and its state (HBM latency off the critical path; no registers held)
    if (lane * 32 < w + 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + min(lane * 32, w - 1)));
    if (lane == 31) asm volatile("prefetch.global.L2 [%0];" ::"l"(st));
  }
  pdl_wait();
  pdl_trigger();
  if (a.pos_lo == 0 && blockIdx.x == 0 && threadIdx.x < 2 * dm.C) a.b.flow[threadIdx.x] = 0u;  // consumers done
  trace_stamp(dm.trace, KGE_K_UPDATE, 1);
  if (a.b.flags[2 + (a.s.info[0] & 1)]) return;  // non-finite loss: skip this step's update (KGE_ENONFINITE)
  RowAcc<V> acc;
  acc.zero();
  // V <= 4: the rows of stg_rows occurrences at a time are copied into this warp's shared-memory staging area by
  // cp.async (no registers held, so more rows are in flight than the 64-register budget allows) and added in
  // occurrence order -- the same additions as the register path. <= 56 KB per CTA keeps 4 CTAs per SM (one wave).
  extern __shared__ float4 stg_dyn[];  // [warps][stg_rows][w4]
  auto staged_sum = [&](int nrows, auto rowptr) {  // acc += rows 0..nrows-1 (rowptr(q): const float* of row q)
    const int ns = a.stg_rows;
    float4* my = stg_dyn + (int64_t)(threadIdx.x >> 5) * ns * w4;
    for (int j = 0; j < nrows; j += ns) {
      const int nb = min(ns, nrows - j);
      for (int q = 0; q < nb; ++q) {
        const float4* src = reinterpret_cast<const float4*>(rowptr(j + q));
#pragma unroll
        for (int m = 0; m < V; ++m)
          if (lane + 32 * m < w4) cpa16(my + q * w4 + lane + 32 * m, src + lane + 32 * m);
      }
      cpa_wait_all();  // a lane reads back only what it copied
      for (int q = 0; q < nb; ++q)
#pragma unroll
        for (int m = 0; m < V; ++m)
          if (lane + 32 * m < w4) acc.add(my[q * w4 + lane + 32 * m], m);
    }
  };
  // loads of UNR occurrences in flight, additions in occurrence order; V = 4 (d <= 512) keeps two in flight so the
  // kernel fits 4 CTAs (32 warps) per SM: the whole grid (B + n_occ warps) is resident in one wave
  constexpr int UNR = V >= 4 ? 2 : 4;
  if (V <= 4) {
    staged_sum(n, [&](int q) { return G + (int64_t)__shfl_sync(0xffffffffu, oj, q & 31) * w; });
  } else
  for (int j = 0; j < n; j += UNR) {
    float4 x[UNR][V];
#pragma unroll
    for (int q = 0; q < UNR; ++q) {
      const int o = __shfl_sync(0xffffffffu, oj, (j + q) & 31);
      const float* src = j + q < n ? G + (int64_t)o * w : nullptr;
#pragma unroll
      for (int m = 0; m < V; ++m) {
        const int v = lane + 32 * m;
        x[q][m] = (src && v < w4) ? ld4(src, v) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int q = 0; q < UNR; ++q)
#pragma unroll
      for (int m = 0; m < V; ++m) acc.add(x[q][m], m);
  }
  trace_stamp(dm.trace, KGE_K_UPDATE, 2);
  if (nseg > 1) {
    float* home = G + (int64_t)__shfl_sync(0xffffffffu, oj, 0) * w;
#pragma unroll
    for (int m = 0; m < V; ++m)
      if (lane + 32 * m < w4) st4(home, lane + 32 * m, acc.g[m]);
    __threadfence();
    int32_t* cnt = a.seg_cnt + (rel ? 0 : dm.B) + u;
    int last = 0;
    if (lane == 0) last = atomicAdd(cnt, 1) == nseg - 1;
    if (!__shfl_sync(0xffffffffu, last, 0)) {
      trace_warp_end(dm.trace, KGE_K_UPDATE);
      return;
    }
    __threadfence();
    if (lane == 0) *cnt = 0;  // ready for the next step
    acc.zero();
    constexpr int UNR2 = V >= 4 ? 2 : 4;
    for (int b0 = 0; b0 < nseg; b0 += 32) {
      // the home rows of up to 32 segments in one round trip (lane q: segment b0 + q), then the sums in segment order
      const int hq = b0 + lane < nseg ? occ_sorted[r0 + (b0 + lane) * kSeg] : 0;
      const int nq = min(32, nseg - b0);
      if (V <= 4) {
        staged_sum(nq, [&](int q) { return G + (int64_t)__shfl_sync(0xffffffffu, hq, q & 31) * w; });
        continue;
      }
      for (int q0 = 0; q0 < nq; q0 += UNR2) {
        float4 x[UNR2][V];
#pragma unroll
        for (int q = 0; q < UNR2; ++q) {
          const int hrow = __shfl_sync(0xffffffffu, hq, (q0 + q) & 31);
          const float* src = q0 + q < nq ? G + (int64_t)hrow * w : nullptr;
#pragma unroll
          for (int m = 0; m < V; ++m) {
            const int v = lane + 32 * m;
            x[q][m] = (src && v < w4) ? __ldcg(reinterpret_cast<const float4*>(src) + v) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int q = 0; q < UNR2; ++q)
#pragma unroll
          for (int m = 0; m < V; ++m) acc.add(x[q][m], m);
      }
    }
  }
  if (plain_sum) {
#pragma unroll
    for (int m = 0; m < V; ++m)
      if (lane + 32 * m < w4) st4(row, lane + 32 * m, acc.g[m]);
    trace_warp_end(dm.trace, KGE_K_UPDATE);
    return;
  }
  float4 row_v[V];
  prefetch_row<V>(row, row_v, w4, lane);
  const float st0 = *st;
  adagrad_row<V>(row, st, acc, row_v, st0, w4, w, dm.lr, dm.eps, lane);
  trace_warp_end(dm.trace, KGE_K_UPDATE);
  trace_stamp(dm.trace, KGE_K_UPDATE, 7);
}

// ------------------------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------------------------
// split-K factor: enough CTAs for ~2 per SM (the kernels are latency bound at one), at least 2 chunks per split
static int ffma_splits(int tiles, int nchunks) {
  int ks = 1;
  while (ks < 8 && tiles * ks * 2 <= 2 * 148 && nchunks >= 4 * ks) ks *= 2;
  return ks;
}

template <int FAM>
static void launch_neg(kge_handle* h, const NegArgs& na0) {
  const Dims& dm = h->dims;
  NegArgs na = na0;
  na.part = h->ffma_part;
  na.cnt = h->ffma_cnt;
  const int kend = FAM == FAM_CMOD ? dm.d / 2 : dm.d, kstep = FAM == FAM_CMOD ? TK / 2 : TK;
  dim3 gf((dm.k + TN - 1) / TN, (dm.g + TM - 1) / TM, dm.C);
  na.ks = std::min(h->ffma_ks_force ? h->ffma_ks_force : ffma_splits(gf.x * gf.y * gf.z, (kend + kstep - 1) / kstep),
                   h->ffma_ks_max);
  gf.z *= na.ks;
  launch_begin(h, KGE_K_NEG_FWD);
  launch_pdl(k_neg_fwd<FAM>, gf, 256, 0, h->stream, na);
  launch_end(h, KGE_K_NEG_FWD);
  const int cols_per_tile = FAM == FAM_CMOD ? TN / 2 : TN;
  const int ncols = FAM == FAM_CMOD ? dm.d / 2 : dm.d;
  dim3 gb((ncols + cols_per_tile - 1) / cols_per_tile, (std::max(dm.g, dm.k) + TM - 1) / TM, 2 * dm.C);
  na.ks = std::min(h->ffma_ks_force ? h->ffma_ks_force
                                   : ffma_splits(gb.x * gb.y * gb.z, (std::min(dm.g, dm.k) + TK - 1) / TK),
                   h->ffma_ks_max);
  gb.z *= na.ks;
  launch_begin(h, KGE_K_NEG_BWD);
  launch_pdl(k_neg_bwd<FAM>, gb, 256, 0, h->stream, na);
  launch_end(h, KGE_K_NEG_BWD);
}


static int row_v(int d) {  // float4 per lane for a d-float row
  const int d4 = d / 4;
  return d4 <= 32 ? 1 : (d4 <= 64 ? 2 : (d4 <= 128 ? 4 : 8));
}

// warps per CTA of the row-parallel kernels (k_gather, k_update). 8 (default) measured faster than 4 on the Freebase
// step (33.6 vs 33.2 M pos/s) although 4 spreads the row warps over all 148 SMs; KGE_ROW_WARPS=4 for experiments
static int row_warps() {
  static const int w = getenv("KGE_ROW_WARPS") && atoi(getenv("KGE_ROW_WARPS")) == 4 ? 4 : 8;
  return w;
}

static void launch_gather_v(kge_handle* h, const GatherArgs& ga, int rows) {
  const int wpc = row_warps();
  const unsigned grid = (rows + wpc - 1) / wpc;
  switch (row_v(h->dims.d)) {
    case 1: launch_pdl(k_gather<1>, grid, 32 * wpc, 0, h->stream, ga); break;
    case 2: launch_pdl(k_gather<2>, grid, 32 * wpc, 0, h->stream, ga); break;
    case 4: launch_pdl(k_gather<4>, grid, 32 * wpc, 0, h->stream, ga); break;
    default: launch_pdl(k_gather<8>, grid, 32 * wpc, 0, h->stream, ga); break;
  }
}

cudaError_t launch_gather_neg(kge_handle* h, const Slot& s) {
  const Dims& dm = h->dims;
  GatherArgs ga{dm, s, h->rows, h->rel, h->buf, dm.B, 0, nullptr};
  const int rows = dm.C * dm.k;
  launch_gather_v(h, ga, rows);
  return cudaGetLastError();
}

// KGE_NO_PREFETCH=1: k_update does not warm L2 / the TLBs with the next step's entity rows (experiments)
static bool no_row_prefetch() {
  static const bool off = getenv("KGE_NO_PREFETCH") != nullptr;
  return off;
}

cudaError_t launch_update_range(kge_handle* h, const Slot& s, int lo, int hi, cudaStream_t st, float* gocc) {
  const Dims& dm = h->dims;
  StepBuffers b = h->buf;
  b.Gocc = gocc;
  UpdateArgs ua{dm, s, h->ent, h->ent_st, h->rel, h->rel_st, b, h->P > 1 ? h->dist.gu : nullptr,
                h->P > 1 ? h->dist.split_index : nullptr, h->dist.grel_split, h->seg_cnt, lo, hi,
                lo == 0 && h->P == 1 && !no_row_prefetch() ? h->next_slot : nullptr};
  const int wpc = row_warps();
  const int grid = (hi - lo + wpc - 1) / wpc;
  if (grid <= 0) return cudaSuccess;
  const int w4 = std::max(dm.d, dm.drel) / 4;
  // staged rows per warp: as many (<= kSeg) as the per-CTA budget holds at this row width
  ua.stg_rows = std::max(1, std::min(kSeg, kStgBytes / (wpc * w4 * 16)));
  const size_t stg = (size_t)wpc * ua.stg_rows * w4 * 16;
  cudaStream_t main = h->stream;
  h->stream = st;  // the profiler brackets the launch on the stream it runs on
  launch_begin(h, KGE_K_UPDATE);
  if (w4 <= 32)
    launch_pdl(k_update<1>, grid, 32 * wpc, stg, st, ua);
  else if (w4 <= 64)
    launch_pdl(k_update<2>, grid, 32 * wpc, stg, st, ua);
  else if (w4 <= 128)
    launch_pdl(k_update<4>, grid, 32 * wpc, stg, st, ua);
  else
    launch_pdl(k_update<8>, grid, 32 * wpc, 0, st, ua);
  launch_end(h, KGE_K_UPDATE);
  h->stream = main;
  return cudaGetLastError();
}

// lag = 0: every table; lag = 1: relations only -- the entity positions of this step are applied by the next step
// (api.cu, reading c.12)
cudaError_t launch_update(kge_handle* h, const Slot& s) {
  const Dims& dm = h->dims;
  // (P > 1: the entity positions only form this rank's per-unique sums here, which the exchange needs now; the owner's
  // Adagrad step is what lag = 1 holds back, dist.cu)
  return launch_update_range(h, s, 0, h->cfg.lag == 1 && h->P == 1 ? dm.B : dm.B + dm.n_occ, h->stream,
                             h->buf.Gocc);
}

// the dot family's chunked negatives and their backward (RESCAL after its per-positive matrix-vector products)
cudaError_t launch_dot_negatives(kge_handle* h, const Slot& s) {
  if (tc_supported(h)) return launch_tc_neg(h, s);
  NegArgs na{h->dims, h->buf, h->buf.Gocc, nullptr, nullptr, 1};
  launch_neg<FAM_DOT>(h, na);
  return cudaGetLastError();
}

cudaError_t launch_step(kge_handle* h, const Slot& s, int64_t step) {
  const Dims& dm = h->dims;
  if (dm.model == KGE_TRANSR) return launch_transr_step(h, s, step);
  if (dm.model == KGE_RESCAL) return launch_rescal_step(h, s, step);
  const bool tc = tc_supported(h);
  GatherArgs ga{dm, s, h->rows, h->rel, h->buf, 0, tc && tc_fuses_chain(h) ? 1 : 0, tc && tc_flow() ? h->buf.flow : nullptr};
  const int rows = dm.B + dm.C * dm.k;
  launch_begin(h, KGE_K_GATHER);
  launch_gather_v(h, ga, rows);
  launch_end(h, KGE_K_GATHER);
  // lag = 1: the held-back entity update of the previous step may start once this step no longer reads the entity
  // table -- after the gather on the fused tcgen05 path, after the chain rule otherwise
  const bool fused_tc = tc && tc_fuses_chain(h);
  if (h->cfg.lag == 1 && fused_tc) {
    cudaError_t e = cudaEventRecord(h->ev_eread, h->stream);
    if (e != cudaSuccess) return e;
  }

  NegArgs na{dm, h->buf, h->buf.Gocc, nullptr, nullptr, 1};
  if (tc) {
    cudaError_t e = launch_tc_neg(h, s);
    if (e != cudaSuccess) return e;
    if (tc_fuses_chain(h)) return launch_update(h, s);  // chain rule + loss done in the backward epilogue
  } else {
    switch (dm.family) {
      case FAM_DOT: launch_neg<FAM_DOT>(h, na); break;
      case FAM_L2: launch_neg<FAM_L2>(h, na); break;
      case FAM_L2SQ: launch_neg<FAM_L2SQ>(h, na); break;
      case FAM_L1: launch_neg<FAM_L1>(h, na); break;
      case FAM_CMOD: launch_neg<FAM_CMOD>(h, na); break;
    }
  }
  ChainArgs ca{dm, s, h->rows, h->rel, h->buf, h->n_neg_parts};
  launch_begin(h, KGE_K_CHAIN);
  const unsigned cgrid = (dm.B + 7) / 8 + 1;
  switch (row_v(dm.d)) {
    case 1: launch_pdl(k_chain<1>, cgrid, 256, 0, h->stream, ca); break;
    case 2: launch_pdl(k_chain<2>, cgrid, 256, 0, h->stream, ca); break;
    case 4: launch_pdl(k_chain<4>, cgrid, 256, 0, h->stream, ca); break;
    default: launch_pdl(k_chain<8>, cgrid, 256, 0, h->stream, ca); break;
  }
  launch_end(h, KGE_K_CHAIN);
  if (h->cfg.lag == 1) {
    cudaError_t e = cudaEventRecord(h->ev_eread, h->stream);
    if (e != cudaSuccess) return e;
  }

  return launch_update(h, s);
}

// ---- kge_score: f(h, r, t) per triple (tail-mode decomposition: f = pair(combine(h, r), t)) ----
struct ScoreArgs {
  Dims dm;
  EntRows ent;
  const float* rel;
  const int32_t* hs;
  const int32_t* rs;
  const int32_t* ts;
  int64_t n;
  float* o_scratch;  // [n x d]
  float* out;
};

__global__ void __launch_bounds__(256) k_score(ScoreArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= a.n) return;
  const Dims& dm = a.dm;
  const float* h = a.ent.row(a.hs[i]);
  const float* t = a.ent.row(a.ts[i]);
  const float* r = a.rel + (int64_t)a.rs[i] * dm.drel;
  float* o = a.o_scratch + i * dm.dp;
  float st, on;
  combine_row(dm.model, 0, h, r, t, o, dm.d, lane, t, dm.family, st, on);
  st = warp_sum(st);
  if (lane == 0) a.out[i] = pair_score_from(dm.family, st, dm.gamma);
}

cudaError_t launch_transr_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                                float* out);  // transr.cu
cudaError_t launch_rescal_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                                float* out);  // rescal.cu

// ------------------------------------------------------------------------------------------------
// k_rank: link-prediction rank of the true entity among all entities (raw setting), one CTA per test triple
// ------------------------------------------------------------------------------------------------
struct RankArgs {
  Dims dm;
  EntRows ent;
  const float* rel;
  const int32_t* hs;
  const int32_t* rs;
  const int32_t* ts;
  int32_t head;      // 0: candidates replace the tail, 1: the head
  const int64_t* cand_off;  // [n+1] or NULL (every entity is a candidate)
  const int32_t* cand;
  const int64_t* filt_off;  // [n+1] or NULL (raw); distinct ids, only with cand_off == NULL
  const int32_t* filt;
  int64_t* ranks;
  int32_t nsplit;  // entity-range splits (blockIdx.y) of the all-entity protocol; > 1: ranks zeroed, partial counts added
};

// per-float4 increment of the pair statistic (one expression shared by every rank path, so equal rows give
// bit-equal scores and ties are decided identically)
__device__ __forceinline__ float stat4(int fam, const float4 ov, const float4 xv) {
  if (fam == FAM_DOT) return ov.x * xv.x + ov.y * xv.y + ov.z * xv.z + ov.w * xv.w;
  if (fam == FAM_L1) return fabsf(ov.x - xv.x) + fabsf(ov.y - xv.y) + fabsf(ov.z - xv.z) + fabsf(ov.w - xv.w);
  const float a = ov.x - xv.x, b = ov.y - xv.y, c = ov.z - xv.z, e = ov.w - xv.w;
  return a * a + b * b + c * c + e * e;
}

__device__ __forceinline__ float cmod1(const float* o, const float* x, int c, int hlf) {
  const float ur = o[c] - x[c], ui = o[c + hlf] - x[c + hlf];
  return sqrtf(ur * ur + ui * ui);
}

// the same statistic of one entity row against QB query rows o_q = osm + q*dp: the row is read once for all queries.
// Not inlined: the positive's own score and every candidate's come out of this one compiled body, so a candidate
// whose row equals the positive's ties it bit-exactly (pessimistic ties, reading c.15)
template <int QB>
__device__ __noinline__ void pair_stat_rows(int fam, const float* osm, int dp, const float* __restrict__ x, int d,
                                               int lane, float (&st)[QB]) {
#pragma unroll
  for (int q = 0; q < QB; ++q) st[q] = 0.f;
  if (fam == FAM_CMOD) {
    for (int c = lane; c < (d >> 1); c += 32) {
#pragma unroll
      for (int q = 0; q < QB; ++q) st[q] += cmod1(osm + q * dp, x, c, d >> 1);
    }
  } else {
    for (int v = lane; v < (d >> 2); v += 32) {
      const float4 xv = ld4(x, v);
#pragma unroll
      for (int q = 0; q < QB; ++q) st[q] += stat4(fam, reinterpret_cast<const float4*>(osm + q * dp)[v], xv);
    }
  }
#pragma unroll
  for (int q = 0; q < QB; ++q) st[q] = warp_sum(st[q]);
}

// One CTA ranks QB queries of one corrupted side (QB > 1 only with every entity as the candidate set): warp q builds
// o_q = combine(h, r) (tail) | combine'(r, t) (head) in shared memory and the positive's score through the same
// arithmetic as every candidate; the 8 warps then stream the candidate rows, each row scored against all QB queries.
// With every entity as the candidate set the entity range is split over blockIdx.y (a few thousand queries alone
// would not fill 148 SMs); split 0 also handles the filter list and adds the 1; partial counts meet in integer
// atomics (exact, order-free).
template <int QB>
__global__ void __launch_bounds__(256) k_rank(RankArgs a, int64_t n) {
  extern __shared__ __align__(16) float osm[];  // QB x dp floats
  __shared__ float s_true[QB];
  __shared__ int64_t s_tid[QB];
  __shared__ int s_cnt[8][QB];
  const Dims& dm = a.dm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * QB;
  const int nq = (int)(n - i0 < QB ? n - i0 : (int64_t)QB);
  const int mode = a.head ? 1 : 0;
  if (warp < nq) {
    const int64_t i = i0 + warp;
    const float* h = a.ent.row(a.hs[i]);
    const float* t = a.ent.row(a.ts[i]);
    const float* r = a.rel + (int64_t)a.rs[i] * dm.drel;
    float st, on;
    combine_row(dm.model, mode, h, r, t, osm + warp * dm.dp, dm.d, lane, mode == 0 ? t : h, dm.family, st, on);
  }
  __syncthreads();  // every o_q is in shared memory
  if (warp < nq) {  // the positive's score through the candidates' arithmetic
    const int64_t i = i0 + warp;
    float sp[QB];
    pair_stat_rows<QB>(dm.family, osm, dm.dp, a.ent.row(mode == 0 ? a.ts[i] : a.hs[i]), dm.d, lane, sp);
    float mine = sp[0];
#pragma unroll
    for (int q = 1; q < QB; ++q)
      if (q == warp) mine = sp[q];
    if (lane == 0) {
      s_true[warp] = pair_score_from(dm.family, mine, dm.gamma);
      s_tid[warp] = mode == 0 ? a.ts[i] : a.hs[i];
    }
  }
  __syncthreads();
  // pessimistic ties (reading c.15): every candidate other than the true entity scoring >= f(true) ranks above it
  int cnt[QB];
#pragma unroll
  for (int q = 0; q < QB; ++q) cnt[q] = 0;
  int64_t lo = 0, hi = dm.n_entities;
  if (a.cand_off) lo = a.cand_off[i0], hi = a.cand_off[i0 + 1];  // QB == 1
  const int split = blockIdx.y;
  if (gridDim.y > 1) {
    const int64_t per = (hi + gridDim.y - 1) / gridDim.y;
    lo = per * split;
    hi = min(hi, lo + per);
  }
  // filtered protocol: a known triple among the candidates is skipped, never scored -- each warp walks its queries'
  // sorted filter lists with a cursor that only moves forward (its candidates ascend), so the filter decision does
  // not depend on a second evaluation of the score
  int64_t fc[QB], fe[QB];
#pragma unroll
  for (int q = 0; q < QB; ++q) {
    fc[q] = fe[q] = 0;
    if (a.filt_off && q < nq) {
      fc[q] = a.filt_off[i0 + q];
      fe[q] = a.filt_off[i0 + q + 1];
      while (fc[q] < fe[q] && a.filt[fc[q]] < lo + warp) ++fc[q];
    }
  }
  for (int64_t j = lo + warp; j < hi; j += 8) {
    const int64_t e = a.cand_off ? (int64_t)a.cand[j] : j;
    if (e < 0) continue;  // a sampled slot that belongs to the other corrupted side
    float st[QB];
    pair_stat_rows<QB>(dm.family, osm, dm.dp, a.ent.row(e), dm.d, lane, st);
#pragma unroll
    for (int q = 0; q < QB; ++q) {
      bool skip = q >= nq || e == s_tid[q];
      if (a.filt_off && q < nq) {
        while (fc[q] < fe[q] && a.filt[fc[q]] < e) ++fc[q];
        skip |= fc[q] < fe[q] && a.filt[fc[q]] == e;
      }
      if (!skip) cnt[q] += pair_score_from(dm.family, st[q], dm.gamma) >= s_true[q] ? 1 : 0;
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < QB; ++q) s_cnt[warp][q] = cnt[q];
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    int64_t c = 0;
    for (int w = 0; w < 8; ++w) c += s_cnt[w][threadIdx.x];
    if (gridDim.y == 1)
      a.ranks[i0 + threadIdx.x] = 1 + c;
    else  // two's-complement wrap makes a negative partial (filter subtraction) exact
      atomicAdd(reinterpret_cast<unsigned long long*>(a.ranks + i0 + threadIdx.x),
                (unsigned long long)(c + (split == 0 ? 1 : 0)));
  }
}

// tcgen05 ranking prep (rank_tc.cu): per query (warp) o_q = combine(h, r) | combine'(r, t) into O (pitch dp),
// ||o_q||^2, the true entity's row into T and its id
__global__ void k_rank_prep(Dims dm, EntRows ent, const float* rel, const int32_t* hs, const int32_t* rs,
                            const int32_t* ts, int64_t n, int head, float* O, float* onorm, float* T, int32_t* true_e) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= n) return;
  const float* h = ent.row(hs[q]);
  const float* t = ent.row(ts[q]);
  const float* r = rel + (int64_t)rs[q] * dm.drel;
  const float* x = head ? h : t;
  float st, on;
  combine_row(dm.model, head, h, r, t, O + q * dm.dp, dm.d, lane, x, dm.family, st, on);
  on = warp_sum(on);
  for (int v = lane; v < (dm.d >> 2); v += 32) st4(T + q * dm.dp, v, ld4(x, v));
  if (lane == 0) {
    onorm[q] = on;
    true_e[q] = head ? hs[q] : ts[q];
  }
}

cudaError_t launch_rank_prep(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                             int head, float* O, float* onorm, float* T, int32_t* true_e) {
  if (n == 0) return cudaSuccess;
  k_rank_prep<<<(unsigned)((n * 32 + 255) / 256), 256, 0, h->stream>>>(h->dims, h->rows, h->rel, hs, rs, ts, n, head, O,
                                                                       onorm, T, true_e);
  ++h->launches;
  return cudaGetLastError();
}

// Second-protocol candidates (reading c.15'): slot j of query i draws u from Philox(ctr=(j/2,
// lo32(i), hi32(i), EVAL), key = eval seed); uniform slots: an entity (both sides: a (side, entity) pair) uniform;
// degree slots: a uniform endpoint of the graph's triples (both sides: and a side bit). Writes the entity into the
// list of its side and -1 into the other's (both = 0: side 0 only).
__global__ void k_eval_cand(int64_t n, int32_t m, int32_t n_uniform, int32_t both, uint32_t k0, uint32_t k1,
                            int64_t n_ent, int64_t n_trip, const int32_t* __restrict__ th,
                            const int32_t* __restrict__ tt, int32_t* __restrict__ cand_t, int32_t* __restrict__ cand_h) {
  const int64_t total = n * m;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / m;
    const int32_t j = (int32_t)(q - i * m);
    const uint4 o = philox4x32_10(make_uint4((uint32_t)j >> 1, (uint32_t)i, (uint32_t)((uint64_t)i >> 32), kTagEval),
                                  k0, k1);
    const uint64_t u = (j & 1) ? (((uint64_t)o.w << 32) | o.z) : (((uint64_t)o.y << 32) | o.x);
    const uint64_t range = j < n_uniform ? (uint64_t)n_ent * (both ? 2u : 1u) : (uint64_t)n_trip * (both ? 4u : 2u);
    uint64_t p = __umul64hi(u, range);
    int side = 0;
    if (both) {
      side = (int)(p & 1u);
      p >>= 1;
    }
    int32_t e;
    if (j < n_uniform) {
      e = (int32_t)p;
    } else {
      const int64_t tq = (int64_t)(p >> 1);
      e = (p & 1u) ? tt[tq] : th[tq];
    }
    cand_t[q] = side == 0 ? e : -1;
    if (cand_h) cand_h[q] = side == 1 ? e : -1;
  }
}

cudaError_t launch_eval_cand(kge_handle* h, int64_t n, int32_t n_uniform, int32_t n_degree, int32_t both,
                             uint64_t seed, int32_t* cand_t, int32_t* cand_h) {
  const int64_t total = n * (int64_t)(n_uniform + n_degree);
  const unsigned grid = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (total == 0) return cudaSuccess;
  k_eval_cand<<<grid, 256, 0, h->stream>>>(n, n_uniform + n_degree, n_uniform, both, (uint32_t)seed,
                                          (uint32_t)(seed >> 32), h->dims.n_entities, h->n_triples, h->th, h->tt,
                                          cand_t, cand_h);
  ++h->launches;
  return cudaGetLastError();
}

cudaError_t launch_rank(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, int head,
                        const int64_t* cand_off, const int32_t* cand, const int64_t* filt_off, const int32_t* filt,
                        int64_t* ranks) {
  RankArgs ra{h->dims, h->rows, h->rel, hs, rs, ts, head, cand_off, cand, filt_off, filt, ranks, 1};
  static const int qb_env = getenv("KGE_RANK_QB") ? atoi(getenv("KGE_RANK_QB")) : 8;
  if (cand_off || qb_env == 1) {
    k_rank<1><<<(unsigned)n, 256, (size_t)h->dims.dp * 4, h->stream>>>(ra, n);
  } else {
    // at least 4 splits (ncu kernel times, FB15k-sized table, d=400: 2000 queries 5.77 -> 3.56 ms TransE-L2, 4.80 ->
    // 3.15 ms DistMult; 20000 queries 33.2 -> 31.4 / 30.1 -> 26.6 ms: shorter CTAs trim the last wave), more when the
    // queries alone give fewer than ~4 CTAs per SM; each split streams at least 512 entity rows
    const int64_t nb = (n + 7) / 8;
    static const int split_env = getenv("KGE_RANK_SPLIT") ? atoi(getenv("KGE_RANK_SPLIT")) : 0;
    int64_t S = split_env > 0 ? split_env : std::max<int64_t>(4, (4 * 148 + nb - 1) / nb);
    S = std::max<int64_t>(1, std::min<int64_t>({S, h->dims.n_entities / 512, 65535}));
    ra.nsplit = (int32_t)S;
    if (S > 1) {
      cudaError_t e = cudaMemsetAsync(ranks, 0, (size_t)n * sizeof(int64_t), h->stream);
      if (e != cudaSuccess) return e;
    }
    k_rank<8><<<dim3((unsigned)nb, (unsigned)S), 256, (size_t)8 * h->dims.dp * 4, h->stream>>>(ra, n);
  }
  ++h->launches;
  return cudaGetLastError();
}

cudaError_t launch_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, float* out) {
  if (h->dims.model == KGE_TRANSR) return launch_transr_score(h, hs, rs, ts, n, out);
  if (h->dims.model == KGE_RESCAL) return launch_rescal_score(h, hs, rs, ts, n, out);
  // scratch: reuse the X buffer in chunks of its capacity
  const int64_t cap = (int64_t)h->dims.C * h->dims.k;
  for (int64_t b = 0; b < n; b += cap) {
    const int64_t m = std::min(cap, n - b);
    ScoreArgs sa{h->dims, h->rows, h->rel, hs + b, rs + b, ts + b, m, h->buf.X, out + b};
    k_score<<<(unsigned)((m + 7) / 8), 256, 0, h->stream>>>(sa);
    ++h->launches;
  }
  return cudaGetLastError();
}

// ---- row get / set ----
__global__ void k_rows(float* __restrict__ tab, int32_t w, const int32_t* __restrict__ ids, int64_t n,
                       float* __restrict__ buf, int write) {
  const int64_t total = n * w;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / w, c = q - i * w;
    float* p = tab + (int64_t)ids[i] * w + c;
    if (write)
      *p = buf[q];
    else
      buf[q] = *p;
  }
}

cudaError_t launch_rows(kge_handle* h, float* tab, int32_t w, const int32_t* ids, int64_t n, float* buf, bool write) {
  if (n == 0) return cudaSuccess;
  const int64_t total = n * w;
  int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_rows<<<blocks, 256, 0, h->stream>>>(tab, w, ids, n, buf, write ? 1 : 0);
  ++h->launches;
  return cudaGetLastError();
}

// Force-load every kernel of this file at init: with CUDA's lazy module loading, the first launch of a kernel may wait
// for running kernels -- a deadlock when a peer's device barrier is spinning (multi-rank emulation on one device).
template <typename F>
static void preload(F f, cudaError_t& e) {
  cudaFuncAttributes at;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void*)f);
}

cudaError_t step_preload() {
  cudaError_t e = cudaSuccess;
  preload(k_gather<1>, e);
  preload(k_gather<2>, e);
  preload(k_gather<4>, e);
  preload(k_gather<8>, e);
  preload(k_chain<1>, e);
  preload(k_chain<2>, e);
  preload(k_chain<4>, e);
  preload(k_chain<8>, e);
  preload(k_score, e);
  preload(k_rows, e);
  preload(k_update<1>, e);
  preload(k_update<2>, e);
  preload(k_update<4>, e);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_update<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStgBytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_update<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStgBytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_update<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStgBytes);
  preload(k_update<8>, e);
  preload(k_neg_fwd<FAM_DOT>, e);
  preload(k_neg_fwd<FAM_L2>, e);
  preload(k_neg_fwd<FAM_L2SQ>, e);
  preload(k_neg_fwd<FAM_L1>, e);
  preload(k_neg_fwd<FAM_CMOD>, e);
  preload(k_neg_bwd<FAM_DOT>, e);
  preload(k_neg_bwd<FAM_L2>, e);
  preload(k_neg_bwd<FAM_L2SQ>, e);
  preload(k_neg_bwd<FAM_L1>, e);
  preload(k_neg_bwd<FAM_CMOD>, e);
  return e;
}

}  // namespace kge
