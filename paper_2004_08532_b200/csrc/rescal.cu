// rescal.cu -- RESCAL (Table 1: f(h, r, t) = h^T M_r t, M_r a d x d matrix per relation; SURVEY 8(f)
// item 4) on the chunked negative path. The decomposition of PAPER.md:429-435 holds with
//   tail corruption: o_i = M_r^T h_i  and  f(h_i, r_i, x'_j) = o_i . x'_j
//   head corruption: o_i = M_r t_i    and  f(x'_j, r_i, t_i) = x'_j . o_i
// so after the per-positive matrix-vector product the negatives are the dot family's g x k contraction (FFMA tiles
// or tcgen05, step.cu / tc.cu) unchanged. Kernels here:
//   k_rc_pos   : CTA per positive -- o_i (fixed summation order), ||o||^2, f+ = o . (t | h), dL/df+ and the loss term
//   k_rc_chain : CTA per relation-sorted position p (+ one CTA for the loss) -- g = dO + w+ df+/do, then
//                tail: dh = M g, dt = w+ o, dM += h g^T ;  head: dt = M^T g, dh = w+ o, dM += g t^T
//                (per-occurrence rows into Gocc; the outer-product factors into the relation-sorted U / V rows)
//   k_rc_dm    : per unique relation u, dM_u = sum over its occurrences (ascending position) of U_p V_p^T
// then the entity rows take the shared segmented-sum + Adagrad update (step.cu) and M_r the projection update
// (transr.cu: one Adagrad state per matrix, split relations exchanged when P > 1). RESCAL has no relation vector.
#include <algorithm>

#include "device_common.cuh"
#include "kge_internal.h"

namespace kge {

struct RcArgs {
  Dims dm;
  Slot s;
  EntRows ent;
  const float* M;  // [N_r x d x d]
  StepBuffers b;
  float* U;        // [B x d] left factors of dM, relation-sorted position p
  float* V;        // [B x d] right factors
  float* dM;       // [B x d x d] per unique relation
  int32_t n_neg_parts;
};

// o = M^T x (tail: thread per output column b, rows streamed) or M x (head: warp per output row a)
__device__ void rc_matvec(const float* __restrict__ M, const float* __restrict__ x_sm, float* __restrict__ o_sm, int d,
                          bool transpose) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (transpose) {
    for (int b = threadIdx.x; b < d; b += blockDim.x) {
      float acc = 0.f;
      for (int a = 0; a < d; ++a) acc = fmaf(x_sm[a], M[(int64_t)a * d + b], acc);
      o_sm[b] = acc;
    }
  } else {
    for (int a = warp; a < d; a += nw) {
      float acc = 0.f;
      for (int b = lane; b < d; b += 32) acc = fmaf(M[(int64_t)a * d + b], x_sm[b], acc);
      acc = warp_sum(acc);
      if (lane == 0) o_sm[a] = acc;
    }
  }
}

__global__ void __launch_bounds__(256) k_rc_pos(RcArgs a) {
  const Dims& dm = a.dm;
  extern __shared__ float sm[];
  float* xs = sm;        // the combined entity row (h tail, t head)
  float* os = sm + dm.d; // o
  __shared__ float red[8][2];
  const int i = blockIdx.x, d = dm.d, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mode = a.s.mode[i / dm.g];
  const float* x = a.ent.row(mode == 0 ? a.s.ph[i] : a.s.pt[i]);
  const float* other = a.ent.row(mode == 0 ? a.s.pt[i] : a.s.ph[i]);
  const float* M = a.M + (int64_t)a.s.pr[i] * d * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) xs[e] = x[e];
  __syncthreads();
  rc_matvec(M, xs, os, d, mode == 0);
  __syncthreads();
  float st = 0.f, on = 0.f;
  float* o = a.b.O + (int64_t)i * dm.dp;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const float v = os[e];
    o[e] = v;
    on = fmaf(v, v, on);
    st = fmaf(v, other[e], st);
  }
  st = warp_sum(st);
  on = warp_sum(on);
  if (lane == 0) {
    red[warp][0] = st;
    red[warp][1] = on;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f, n = 0.f;
    for (int w = 0; w < 8; ++w) {
      s += red[w][0];
      n += red[w][1];
    }
    a.b.pstat[i] = s;  // f+ = o . other (dot family)
    a.b.onorm[i] = n;
    if (dm.loss == KGE_LOSS_PAIRWISE) {
      a.b.wpos[i] = 0.f;
      a.b.lpos[i] = 0.f;
      a.b.pcnt[i] = 0;
    } else {
      a.b.wpos[i] = -sigmoid(-s) / (float)dm.B;  // dL/df+ (reading c.9)
      a.b.lpos[i] = -log_sigmoid(s);
    }
  }
}

__global__ void __launch_bounds__(256) k_rc_chain(RcArgs a) {
  const Dims& dm = a.dm;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == gridDim.x - 1) {  // the step's loss, fixed order (as k_chain)
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
  extern __shared__ float sm[];
  const int d = dm.d;
  float* gs = sm;  // g = dO + w+ other
  const int p = blockIdx.x, i = a.s.rel_occ[p];
  const int mode = a.s.mode[i / dm.g];
  const float w = dm.loss == KGE_LOSS_PAIRWISE ? -(float)a.b.pcnt[i] * (1.f / ((float)dm.B * (float)dm.k))
                                               : a.b.wpos[i];  // dL/df+ (reading c.9 / c.9')
  const float* hrow = a.ent.row(a.s.ph[i]);
  const float* trow = a.ent.row(a.s.pt[i]);
  const float* other = mode == 0 ? trow : hrow;
  const float* o = a.b.O + (int64_t)i * dm.dp;
  const float* dO = a.b.dO + (int64_t)i * d;
  const float* M = a.M + (int64_t)a.s.pr[i] * d * d;
  float* gH = a.b.Gocc + (int64_t)i * d;
  float* gT = a.b.Gocc + (int64_t)(dm.B + i) * d;
  float* U = a.U + (int64_t)p * d;
  float* V = a.V + (int64_t)p * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const float g = fmaf(w, other[e], dO[e]);  // dL/do: negatives' dO plus the positive's w+ d(o . other)/do
    gs[e] = g;
    if (mode == 0) {  // o = M^T h, f+ = o . t: dt = w+ o; dM = h g^T
      gT[e] = w * o[e];
      U[e] = hrow[e];
      V[e] = g;
    } else {          // o = M t, f+ = h . o: dh = w+ o; dM = g t^T
      gH[e] = w * o[e];
      U[e] = g;
      V[e] = trow[e];
    }
  }
  __syncthreads();
  // the combined entity: tail dh = M g ; head dt = M^T g (same matrix-vector body as the forward)
  float* outs = sm + d;
  rc_matvec(M, gs, outs, d, mode == 1);
  __syncthreads();
  float* gC = mode == 0 ? gH : gT;
  for (int e = threadIdx.x; e < d; e += blockDim.x) gC[e] = outs[e];
}

// dM_u = sum over the occurrences p of unique relation u (ascending relation-sorted position) of U_p V_p^T; CTA =
// (u, 8-row tile of dM), thread per column
__global__ void __launch_bounds__(256) k_rc_dm(RcArgs a) {
  const Dims& dm = a.dm;
  const int u = blockIdx.x;
  if (u >= *a.s.rel_n) return;
  const int d = dm.d, a0 = blockIdx.y * 8;
  const int p0 = a.s.rel_off[u], p1 = a.s.rel_off[u + 1];
  float* G = a.dM + (int64_t)u * d * d;
  for (int b = threadIdx.x; b < d; b += blockDim.x) {
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.f;
    for (int p = p0; p < p1; ++p) {
      const float vb = a.V[(int64_t)p * d + b];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (a0 + q < d) acc[q] = fmaf(a.U[(int64_t)p * d + a0 + q], vb, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (a0 + q < d) G[(int64_t)(a0 + q) * d + b] = acc[q];
  }
}

// kge_score: f = h^T M_r t per triple (CTA per triple, the forward's matrix-vector body)
__global__ void __launch_bounds__(256) k_rc_score(Dims dm, EntRows ent, const float* M, const int32_t* hs,
                                                  const int32_t* rs, const int32_t* ts, float* out) {
  extern __shared__ float sm[];
  float* xs = sm;
  float* os = sm + dm.d;
  __shared__ float red[8];
  const int i = blockIdx.x, d = dm.d, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* h = ent.row(hs[i]);
  const float* t = ent.row(ts[i]);
  for (int e = threadIdx.x; e < d; e += blockDim.x) xs[e] = h[e];
  __syncthreads();
  rc_matvec(M + (int64_t)rs[i] * d * d, xs, os, d, true);  // o = M^T h, f = o . t (the tail decomposition)
  __syncthreads();
  float st = 0.f;
  for (int e = threadIdx.x; e < d; e += blockDim.x) st = fmaf(os[e], t[e], st);
  st = warp_sum(st);
  if (lane == 0) red[warp] = st;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w];
    out[i] = s;
  }
}

cudaError_t launch_gather_neg(kge_handle* h, const Slot& s);                                         // step.cu
cudaError_t launch_dot_negatives(kge_handle* h, const Slot& s);                                      // step.cu
cudaError_t launch_update_range(kge_handle* h, const Slot& s, int lo, int hi, cudaStream_t st, float* gocc);
cudaError_t launch_proj_update(kge_handle* h, const Slot& s);                                        // transr.cu

cudaError_t launch_rescal_step(kge_handle* h, const Slot& s, int64_t step) {
  (void)step;
  const Dims& dm = h->dims;
  RcArgs a{dm, s, h->rows, h->proj, h->buf, h->tr_buf.U, h->tr_buf.H, h->tr_buf.dM, h->n_neg_parts};
  const size_t smem = 2 * (size_t)dm.d * sizeof(float);
  launch_begin(h, KGE_K_GATHER);
  k_rc_pos<<<dm.B, 256, smem, h->stream>>>(a);
  cudaError_t e = launch_gather_neg(h, s);
  launch_end(h, KGE_K_GATHER);
  if (e != cudaSuccess) return e;
  e = launch_dot_negatives(h, s);  // S = O X'^T and its backward: FFMA tiles or tcgen05 (dot family)
  if (e != cudaSuccess) return e;
  launch_begin(h, KGE_K_CHAIN);
  k_rc_chain<<<dm.B + 1, 256, smem, h->stream>>>(a);
  k_rc_dm<<<dim3(dm.B, (dm.d + 7) / 8), 256, 0, h->stream>>>(a);
  launch_end(h, KGE_K_CHAIN);
  h->launches += 3;
  e = launch_update_range(h, s, dm.B, dm.B + dm.n_occ, h->stream, h->buf.Gocc);  // entity rows (no relation vector)
  if (e != cudaSuccess) return e;
  return launch_proj_update(h, s);
}

cudaError_t launch_rescal_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                                float* out) {
  for (int64_t b = 0; b < n; b += 65535) {
    const int64_t m = std::min<int64_t>(65535, n - b);
    k_rc_score<<<(unsigned)m, 256, 2 * (size_t)h->dims.d * sizeof(float), h->stream>>>(h->dims, h->rows, h->proj,
                                                                                       hs + b, rs + b, ts + b, out + b);
    ++h->launches;
  }
  return cudaGetLastError();
}

bool rescal_init(kge_handle* h) {
  const int smem = 2 * h->dims.d * (int)sizeof(float);
  bool ok = cudaFuncSetAttribute(k_rc_pos, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_rc_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  ok = ok && cudaFuncSetAttribute(k_rc_score, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
  if (!ok) cudaGetLastError();
  return ok;
}

}  // namespace kge
