// transr.cu -- the TransR step (Table 1: f = gamma - ||M_r h + r - M_r t||_2^2; M_r is d x d).
//
// TransR is "d times more computationally expensive than TransE" because every negative must be
// projected by the relation of each positive it is scored against. With joint negatives the
// projections are shared by all positives of a chunk that carry the same relation, so the step is organised around
// groups (relation u, chunk c) = the runs of the relation-sorted occurrence list (reading c.5) that fall in one chunk:
//
//   k_tr_groups : (1 CTA) group table from the relation dedup segments: per group (u, c, positions); per chunk the
//                 ordered list of its groups; per unique relation the range of its groups.
//   k_tr_pos    : per positive (relation-sorted order): Mh, Mt, p = Mh + r - Mt, f+ = gamma - ||p||^2, o = Mh + r (tail)
//                 or Mt - r (head)  [the decomposition of PAPER.md:429-435 with q_j = M x'_j]
//   k_tr_gemm<0>: QX_g = X'_c M_u^T                                     (per group, k x d x d)
//   k_tr_score  : per group: f_ij = gamma - ||o_i - QX_g[j]||^2, loss partial, dO_i, dQ_g (sums in fixed order)
//   k_tr_gemm<1>: P_g = dQ_g M_u  (dL/dx'_j = M_u^T dq_j)              (per group)
//   k_tr_reduce : dX'_c = sum over the chunk's groups, in group order, of P_g -> per-occurrence rows (no atomics)
//   k_tr_chain  : per positive: gMh, gMt, dr; dh = M^T gMh, dt = M^T gMt; rows for the dM outer products; loss CTA
//   k_tr_gemm<2>: dM_u = sum_g dQ_g^T X'_c + sum_{i in u} (gMh_i h_i^T + gMt_i t_i^T)   (per unique relation)
//   k_tr_proj   : Adagrad on M_u with one state per matrix (reading c.11, w = d*d)
// FP32 FFMA (64x64 tiles, 4x4 micro-tiles) on the FP32 path; on the TF32 negatives path the three grouped GEMMs run on
// tcgen05 (k_tr_tc<0> / k_tr_tc<1> / k_tr_dm_tc, two MMA-issuing threads with private TMEM accumulators).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"
#include "kge_internal.h"
#include "tc_ptx.cuh"

namespace kge {

struct TrArgs {
  Dims dm;
  Slot s;
  EntRows ent;  // entity rows: the local table, or (P > 1) the owner's shard over peer memory
  const float* rel;
  float* proj;
  float* proj_st;
  StepBuffers b;
  TrBuffers t;
  int32_t n_neg_parts;
  const int32_t* split_index;  // P > 1: relation -> index among split relations (-1 if not split), else nullptr
  float* gproj_split;          // P > 1: this rank's sums of the split relations' M_r gradients
};

// ------------------------------------------------------------------------------------------------
// group table
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_tr_groups(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  __shared__ int warp_tot[32];
  __shared__ int s_total;
  const int B = dm.B, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (B + blockDim.x - 1) / blockDim.x;
  const int b0 = min(B, tid * per), b1 = min(B, b0 + per);
  auto key_u = [&](int p) { return a.s.rel_inv[a.s.rel_occ[p]]; };
  auto key_c = [&](int p) { return a.s.rel_occ[p] / dm.g; };
  auto is_new = [&](int p) { return p == 0 || key_u(p) != key_u(p - 1) || key_c(p) != key_c(p - 1); };
  auto scan = [&](int v) {  // block exclusive scan, total in s_total
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;
      if (lane == 31) s_total = t;
    }
    __syncthreads();
    const int r = (wid ? warp_tot[wid - 1] : 0) + x - v;
    __syncthreads();
    return r;
  };
  int cnt = 0;
  for (int p = b0; p < b1; ++p) cnt += is_new(p);
  int gid = scan(cnt) - 1;
  const int n_groups = s_total;
  for (int p = b0; p < b1; ++p) {
    if (is_new(p)) {
      ++gid;
      T.grp_u[gid] = key_u(p);
      T.grp_c[gid] = key_c(p);
      T.grp_p0[gid] = p;
    }
  }
  __syncthreads();
  for (int q = tid; q < n_groups; q += blockDim.x) T.grp_p1[q] = q + 1 < n_groups ? T.grp_p0[q + 1] : B;
  // per unique relation: first group (groups are sorted by (u, c))
  const int n_rel = *a.s.rel_n;
  for (int q = tid; q < n_groups; q += blockDim.x)
    if (q == 0 || T.grp_u[q] != T.grp_u[q - 1]) T.rg_off[T.grp_u[q]] = q;
  if (tid == 0) {
    T.rg_off[n_rel] = n_groups;
    *T.n_groups = n_groups;
  }
  // per chunk: its groups in increasing group id (stable), via one scan per chunk
  __syncthreads();
  const int per_g = (n_groups + blockDim.x - 1) / blockDim.x;
  const int g0 = min(n_groups, tid * per_g), g1 = min(n_groups, g0 + per_g);
  int base = 0;
  for (int c = 0; c < dm.C; ++c) {
    int cc = 0;
    for (int q = g0; q < g1; ++q) cc += T.grp_c[q] == c;
    int pos = scan(cc);
    const int tot = s_total;
    for (int q = g0; q < g1; ++q)
      if (T.grp_c[q] == c) {
        T.grp_lc[q] = pos;  // index of the group within its chunk (QX slot of the chunk-wise projections)
        T.cg_list[base + pos++] = q;
      }
    if (tid == 0) T.cg_off[c] = base;
    base += tot;
  }
  if (tid == 0) T.cg_off[dm.C] = base;
  // per unique relation: its first row in the padded U / H layout (2 n_u rows rounded up to 32), a contiguous run of
  // relations per thread
  __syncthreads();
  const int per_u = (n_rel + blockDim.x - 1) / blockDim.x;
  const int u0 = min(n_rel, tid * per_u), u1 = min(n_rel, u0 + per_u);
  auto padded = [&](int u) { return (2 * (a.s.rel_off[u + 1] - a.s.rel_off[u]) + 31) / 32 * 32; };
  int tot_u = 0;
  for (int u = u0; u < u1; ++u) tot_u += padded(u);
  int po = scan(tot_u);
  for (int u = u0; u < u1; ++u) {
    T.pad_off[u] = po;
    po += padded(u);
  }
  if (tid == 0) T.pad_off[n_rel] = s_total;
  // k_tr_mv work items: each relation's positions cut into runs of 8 (uniform items, so a hub relation is spread
  // over many CTAs)
  auto nitems = [&](int u) { return (a.s.rel_off[u + 1] - a.s.rel_off[u] + 7) / 8; };
  int tot_i = 0;
  for (int u = u0; u < u1; ++u) tot_i += nitems(u);
  int io = scan(tot_i);
  for (int u = u0; u < u1; ++u)
    for (int q = 0; q < nitems(u); ++q, ++io) {
      T.item_u[io] = u;
      T.item_p[io] = a.s.rel_off[u] + 8 * q;
    }
  if (tid == 0) *T.n_items = s_total;
  // k_tr_score work items: each group's positions cut into slices of kTrSlice (a hub group is spread over many CTAs);
  // the slices of a group with several get consecutive slots for their dQ partials
  // Items follow the chunk-ordered group list (cg_list), so each chunk's items are one range [si_off[c], si_off[c+1]).
  __syncthreads();
  auto nsl = [&](int q) { return (T.grp_p1[q] - T.grp_p0[q] + kTrSlice - 1) / kTrSlice; };
  int tot_s = 0, tot_m = 0;
  for (int l = g0; l < g1; ++l) {
    const int q = T.cg_list[l];
    tot_s += nsl(q);
    tot_m += nsl(q) > 1 ? nsl(q) : 0;
  }
  int so = scan(tot_s);
  const int n_s = s_total;
  int mo = scan(tot_m);
  for (int l = g0; l < g1; ++l) {
    const int q = T.cg_list[l], ns = nsl(q);
    for (int c = 0; c < dm.C; ++c)
      if (T.cg_off[c] == l) T.si_off[c] = so;  // (a chunk has >= 1 group, so every cg_off[c] < n_groups is hit)
    T.ms_off[q] = ns > 1 ? mo : -1;
    if (ns > 1) mo += ns;
    for (int t = 0; t < ns; ++t, ++so) {
      T.sitem_g[so] = q;
      T.sitem_p[so] = T.grp_p0[q] + t * kTrSlice;
    }
  }
  if (tid == 0) {
    *T.n_sitems = n_s;
    T.si_off[dm.C] = n_s;
  }
  // k_tr_dm_tc order: unique relations by descending group count (<= C; stable), so the CTAs with the most k-blocks
  // start in the first wave instead of forming the kernel's tail
  int rbase = 0;
  for (int ng = dm.C; ng >= 1; --ng) {
    int cc = 0;
    for (int u = u0; u < u1; ++u) cc += T.rg_off[u + 1] - T.rg_off[u] == ng;
    int pos = scan(cc);
    const int tot = s_total;
    for (int u = u0; u < u1; ++u)
      if (T.rg_off[u + 1] - T.rg_off[u] == ng) T.rel_order[rbase + pos++] = u;
    rbase += tot;
  }
}

// ------------------------------------------------------------------------------------------------
// batched projections: CTA (block of 32 output coordinates x0.., y) takes the work items y, y + gridDim.y, ... of
// k_tr_groups (a run of <= 8 positions of one relation u): the 32 x d slab of M_u is staged in shared memory and applied
// to the item's 16 vectors -- M_u is read once per 8 positives instead of once per positive, and a hub relation's
// positions are spread over many CTAs.
//   BWD = 0: Mh_i = M_u h_i, Mt_i = M_u t_i  -> U rows urow, urow + 1 (slab[x][kk] = M[x0 + x][kk])
//   BWD = 1: dh_i = M_u^T gMh_i, dt_i = M_u^T gMt_i (U rows, k_tr_chain) -> occurrence rows i, B + i
//            (slab[x][kk] = M[kk][x0 + x])
// urow = pad_off[u] + 2 (p - rel_off[u]) is the relation-sorted padded layout of k_tr_groups. Thread = (x = tid / 8,
// part q = tid % 8): partial sums over kk = q, q + 8, ..., added over the 8 lanes of x by a butterfly (every lane gets
// the same bits; fixed order).
// ------------------------------------------------------------------------------------------------
static size_t tr_mv_smem(int d) { return (size_t)2 * (32 * (d + 4) + 16 * d) * sizeof(float); }

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(sa), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async16(float4* dst, const float4* src, bool valid) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int BWD>
__global__ void __launch_bounds__(256) k_tr_mv(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  extern __shared__ float sm[];
  // slab pitch: d + 1 for the transposed (4-byte) copies of BWD (conflict-free column writes), d + 4 for FWD so its
  // rows stay 16-byte aligned for 16-byte copies
  const int d = dm.d, lda = BWD ? d + 1 : d + 4, x0 = blockIdx.x * 32, d4 = d >> 2;
  const int buf_floats = 32 * lda + 16 * d;  // per buffer: slab [32][lda], then vectors [16][d]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_items = *a.t.n_items;
  // items it = blockIdx.y, + gridDim.y, ... through two shared-memory buffers: the cp.async copies of item i + 1 are
  // in flight while item i is computed (zero-filled where out of range; warp w: slab rows / vectors w, w + 8, ...,
  // lanes along the contiguous dimension)
  auto stage = [&](int it, float* buf) {
    const int u = a.t.item_u[it], pb = a.t.item_p[it];
    const int pr0 = a.s.rel_off[u], np = min(8, a.s.rel_off[u + 1] - pb);
    const float* M = a.proj + (int64_t)a.s.rel_uniq[u] * d * d;
    float* slab = buf;
    float* vec = buf + 32 * lda;
    if (BWD) {  // slab[xx][kk] = M[kk][x0 + xx]
      const bool ok = x0 + lane < d;
      for (int kk = warp; kk < d; kk += 8) cp_async4(slab + lane * lda + kk, M + (int64_t)kk * d + (ok ? x0 + lane : 0), ok);
    } else {  // slab[xx][kk] = M[x0 + xx][kk], 16-byte copies
      for (int xx = warp; xx < 32; xx += 8) {
        const bool ok = x0 + xx < d;
        const float4* row = reinterpret_cast<const float4*>(M + (int64_t)(ok ? x0 + xx : 0) * d);
        for (int c = lane; c < d4; c += 32) cp_async16(reinterpret_cast<float4*>(slab + xx * lda) + c, row + c, ok);
      }
    }
    const int p = pb + warp;  // vectors 2 warp, 2 warp + 1 (BWD: the gMh / gMt rows of U; else h / t)
    const bool ok = warp < np;
    const float* src0 = M;
    const float* src1 = M;
    if (ok) {
      if (BWD) {
        src0 = a.t.U + (a.t.pad_off[u] + 2 * (int64_t)(p - pr0)) * d;
        src1 = src0 + d;
      } else {
        const int i = a.s.rel_occ[p];
        src0 = a.ent.row(a.s.ph[i]);
        src1 = a.ent.row(a.s.pt[i]);
      }
    }
    for (int c = lane; c < d4; c += 32) {  // 16-byte copies (rows of d floats, d % 4 == 0)
      cp_async16(reinterpret_cast<float4*>(vec + (2 * warp) * d) + c, reinterpret_cast<const float4*>(src0) + (ok ? c : 0), ok);
      cp_async16(reinterpret_cast<float4*>(vec + (2 * warp + 1) * d) + c, reinterpret_cast<const float4*>(src1) + (ok ? c : 0),
                 ok);
    }
  };
  int cur = 0;
  if ((int)blockIdx.y < n_items) stage(blockIdx.y, sm);
  cp_async_commit();
  for (int it = blockIdx.y; it < n_items; it += gridDim.y) {
    const int nit = it + gridDim.y;
    if (nit < n_items) stage(nit, sm + (cur ^ 1) * buf_floats);
    cp_async_commit();
    cp_async_wait<1>();  // this item's copies landed (the next item's may still be in flight)
    __syncthreads();
    const float* slab = sm + cur * buf_floats;
    const float* vec = slab + 32 * lda;
    const int u = a.t.item_u[it], pb = a.t.item_p[it];
    const int pr0 = a.s.rel_off[u], np = min(8, a.s.rel_off[u + 1] - pb);
    const int64_t ubase = a.t.pad_off[u];
    // warp w: outputs x = w + 8 xi (xi < 4) of the item's NV vectors (NV = 4 when it has <= 2 positions -- most items
    // -- else 16), lane = K part (kk = lane, lane + 32, ...): 4 slab and NV vector loads per 4 NV FMAs; then a
    // reduce-scatter butterfly over the 32 lanes (each level hands half of the values to the partner, the lane with
    // bit o set keeping the upper half) -- a fixed association, so the result is deterministic
    auto store = [&](int idx, float val) {  // idx = xi * NV + v
      const int nv = np <= 2 ? 4 : 16;
      const int xi = idx / nv, v = idx - xi * nv, xx = warp + 8 * xi;
      if (x0 + xx >= d || (v >> 1) >= np) return;
      const int p = pb + (v >> 1);
      if (BWD) {
        const int i = a.s.rel_occ[p];
        a.b.Gocc[((int64_t)((v & 1) ? dm.B + i : i)) * d + x0 + xx] = val;
      } else {
        a.t.U[(ubase + 2 * (p - pr0) + (v & 1)) * d + x0 + xx] = val;
      }
    };
    if (np <= 2) {
      float acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.f;
      for (int kk = lane; kk < d; kk += 32) {
        float m[4];
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) m[xi] = slab[(warp + 8 * xi) * lda + kk];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const float vv = vec[v * d + kk];
#pragma unroll
          for (int xi = 0; xi < 4; ++xi) acc[xi * 4 + v] = fmaf(m[xi], vv, acc[xi * 4 + v]);
        }
      }
#pragma unroll
      for (int lv = 0; lv < 4; ++lv) {  // 16 values -> 1 per lane pair (lane l: output l >> 1)
        const int o = 16 >> lv, half = 8 >> lv;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
          const float give = up ? acc[j] : acc[j + half];
          const float keep = up ? acc[j + half] : acc[j];
          acc[j] = keep + __shfl_xor_sync(0xffffffffu, give, o);
        }
      }
      acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
      if ((lane & 1) == 0) store(lane >> 1, acc[0]);
    } else {
      float acc[64];
#pragma unroll
      for (int j = 0; j < 64; ++j) acc[j] = 0.f;
      for (int kk = lane; kk < d; kk += 32) {
        float m[4];
#pragma unroll
        for (int xi = 0; xi < 4; ++xi) m[xi] = slab[(warp + 8 * xi) * lda + kk];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float vv = vec[v * d + kk];
#pragma unroll
          for (int xi = 0; xi < 4; ++xi) acc[xi * 16 + v] = fmaf(m[xi], vv, acc[xi * 16 + v]);
        }
      }
#pragma unroll
      for (int lv = 0; lv < 5; ++lv) {  // 64 values -> 2 per lane (lane l: outputs 2 l, 2 l + 1)
        const int o = 16 >> lv, half = 32 >> lv;
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int j = 0; j < half; ++j) {
          const float give = up ? acc[j] : acc[j + half];
          const float keep = up ? acc[j + half] : acc[j];
          acc[j] = keep + __shfl_xor_sync(0xffffffffu, give, o);
        }
      }
      store(2 * lane, acc[0]);
      store(2 * lane + 1, acc[1]);
    }
    __syncthreads();  // buffer cur is consumed before the copies of item it + 2 gridDim.y land in it
    cur ^= 1;
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------------
// positives: one CTA per relation-sorted position p, from Mh / Mt of k_tr_mv<0>
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tr_pos(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  __shared__ float red[8];
  const int p = blockIdx.x, i = a.s.rel_occ[p];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, d = dm.d;
  const int r = a.s.pr[i], mode = a.s.mode[i / dm.g];
  const int u = a.s.rel_inv[i];
  const float* smh = a.t.U + (a.t.pad_off[u] + 2 * (int64_t)(p - a.s.rel_off[u])) * d;  // Mh, then Mt
  const float* smt = smh + d;
  const float* rv = a.rel + (int64_t)r * d;
  float sq = 0.f;
  float* o = a.b.O + (int64_t)i * dm.dp;
  float* pv = a.t.Pv + (int64_t)i * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const float pe = smh[e] + rv[e] - smt[e];
    pv[e] = pe;
    sq += pe * pe;
    o[e] = mode == 0 ? smh[e] + rv[e] : smt[e] - rv[e];
  }
  sq = warp_sum(sq);
  if (lane == 0) red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w];
    const float f = dm.gamma - s;
    a.b.pstat[i] = s;
    if (dm.loss == KGE_LOSS_PAIRWISE) {  // reading c.9': the positive's terms come from its hinges
      a.b.wpos[i] = 0.f;
      a.b.lpos[i] = 0.f;
      a.b.pcnt[i] = 0;
    } else {
      a.b.wpos[i] = -sigmoid(-f) / (float)dm.B;
      a.b.lpos[i] = -log_sigmoid(f);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// grouped GEMMs (FFMA, 64x64 tiles, K-chunks of 16, 4x4 micro-tiles)
//   MODE 0: C[k x d]  = X'_c[k x d] * M_u^T                 group = pair group g       -> QX_g
//   MODE 1: C[k x d]  = dQ_g[k x d] * M_u                    group = pair group g       -> P_g (stored in QX_g)
//   MODE 2: C[d x d]  = sum_g dQ_g^T X'_c + U^T H            group = unique relation u  -> dM_u
// ------------------------------------------------------------------------------------------------
constexpr int GT = 64, GK = 16;

template <int MODE>
__global__ void __launch_bounds__(256) k_tr_gemm(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  const int grp = blockIdx.z;
  const int d = dm.d, k = dm.k;
  if (MODE < 2) {
    if (grp >= *T.n_groups) return;
  } else {
    if (grp >= *a.s.rel_n) return;
  }
  const int Mrows = MODE == 2 ? d : k, Ncols = d;
  const int m0 = blockIdx.y * GT, n0 = blockIdx.x * GT;
  if (m0 >= Mrows || n0 >= Ncols) return;
  __shared__ __align__(16) float As[GK][GT + 4];
  __shared__ __align__(16) float Bs[GK][GT + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};

  // A(m, kk) and B(kk, n) accessors for one term; a term is (A base, A pitch, A transposed?, B base, B pitch, B
  // transposed?, K)
  auto run_term = [&](const float* Ab, int lda, bool At, const float* Bb, int ldb, bool Bt, int K) {
    for (int k0 = 0; k0 < K; k0 += GK) {
      // coalesced: consecutive threads walk the operand's contiguous dimension (k for row-major A / transposed B,
      // m / n otherwise)
      for (int idx = threadIdx.x; idx < GK * GT; idx += blockDim.x) {
        const int kka = At ? idx / GT : idx % GK, mma = At ? idx % GT : idx / GK;
        const int kkb = Bt ? idx % GK : idx / GT, nnb = Bt ? idx / GK : idx % GT;
        float va = 0.f, vb = 0.f;
        const int gka = k0 + kka, gkb = k0 + kkb, gm = m0 + mma, gn = n0 + nnb;
        if (gka < K && gm < Mrows) va = At ? Ab[(int64_t)gka * lda + gm] : Ab[(int64_t)gm * lda + gka];
        if (gkb < K && gn < Ncols) vb = Bt ? Bb[(int64_t)gn * ldb + gkb] : Bb[(int64_t)gkb * ldb + gn];
        As[kka][mma] = va;
        Bs[kkb][nnb] = vb;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < GK; ++kk) {
        const float4 av = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
        const float4 bv = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
        const float ar[4] = {av.x, av.y, av.z, av.w}, br[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) acc[ii][jj] = fmaf(ar[ii], br[jj], acc[ii][jj]);
      }
      __syncthreads();
    }
  };

  float* out;
  if (MODE == 0) {
    const int u = T.grp_u[grp], c = T.grp_c[grp];
    const int r = a.s.rel_uniq[u];
    run_term(a.b.X + (int64_t)c * k * dm.dp, dm.dp, false, a.proj + (int64_t)r * d * d, d, true, d);
    out = T.QX + (int64_t)grp * k * d;
  } else if (MODE == 1) {
    const int u = T.grp_u[grp];
    const int r = a.s.rel_uniq[u];
    run_term(T.dQ + (int64_t)grp * k * d, d, false, a.proj + (int64_t)r * d * d, d, false, d);
    out = T.QX + (int64_t)grp * k * d;  // QX_g is dead after k_tr_score
  } else {
    const int u = grp;
    for (int g = T.rg_off[u]; g < T.rg_off[u + 1]; ++g) {
      const int c = T.grp_c[g];
      run_term(T.dQ + (int64_t)g * k * d, d, true, a.b.X + (int64_t)c * k * dm.dp, dm.dp, false, k);
    }
    const int q0 = T.pad_off[u], nq = 2 * (a.s.rel_off[u + 1] - a.s.rel_off[u]);
    run_term(T.U + (int64_t)q0 * d, d, true, T.H + (int64_t)q0 * d, d, false, nq);
    out = T.dM + (int64_t)u * d * d;
  }
#pragma unroll
  for (int ii = 0; ii < 4; ++ii) {
    const int m = m0 + ty * 4 + ii;
    if (m >= Mrows) continue;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int n = n0 + tx * 4 + jj;
      if (n < Ncols) out[(int64_t)m * Ncols + n] = acc[ii][jj];
    }
  }
}

// ------------------------------------------------------------------------------------------------
// k_tr_qx_tc: QX_g = X'_c M_u^T on tcgen05 (kind::tf32, TF32 negatives path): CTA = 128 negatives x N = d (<= 256)
// of one group, K = d streamed in 32-float k-blocks through a TMA -> mbarrier pipeline; two MMA-issuing threads own
// alternate K = 8 slices of every k-block (private TMEM accumulators at columns 0 / 256, added in a fixed order).
// Both operands are K-major: A = the chunk's X' rows, B = M_u's rows (M_u[a][b] is B[n = a][k = b]).
// ------------------------------------------------------------------------------------------------
struct TrTc {
  CUtensorMap mX;   // X' [C*k rows x d cols] (pitch dp), box {32, 128}
  CUtensorMap mM;   // proj [n_rel][d rows][d cols], box {32, N}: B of QX (K-major)
  CUtensorMap mMn;  // proj, box {32, 32}, SWIZZLE_128B_ATOM_32B: B of P = dQ M (MN-major, one box per 32-column block)
  CUtensorMap mdQ;  // dQ [B groups][k rows][d cols], box {32, 128}
  CUtensorMap mdQn;  // dQ, box {32, 32}, SWIZZLE_128B_ATOM_32B (A = dQ_g^T of dM, MN-major)
  CUtensorMap mXn;   // X' [C*k rows x d cols], box {32, 32}, SWIZZLE_128B_ATOM_32B (B of dM, MN-major)
  CUtensorMap mUn, mHn;  // padded U / H rows, box {32, 32}, SWIZZLE_128B_ATOM_32B (the U^T H term of dM)
  int N = 0;        // d rounded up to 16
};
constexpr int kTrStages = 2;  // two stages and one 256-column accumulator: two CTAs per SM (smem ~91 KB, TMEM 2 x 256)

__device__ __forceinline__ uint64_t sdesc_mn32(uint32_t saddr, uint32_t lbo) {
  // tf32 MN-major: SWIZZLE_128B_BASE32B (layout type 1), SBO = 512 B between 4-row K atoms (see tc.cu)
  uint64_t d = tc::sdesc(saddr, lbo, 512);
  d &= ~((uint64_t)7 << 61);
  d |= (uint64_t)1 << 61;
  return d;
}

// MODE 0: QX_g = X'_c M_u^T (k_tr_gemm<0>); MODE 1: P_g = dQ_g M_u (k_tr_gemm<1>), both into T.QX + g k d
template <int MODE>
__global__ void __launch_bounds__(128, 1)
    k_tr_tc(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, TrArgs a, int N, int chunk,
            int xmode) {  // xmode (timing experiments only, KGE_TR_XMODE): 1 = no epilogue stores
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kTrStages], empty[kTrStages], done;
  __shared__ uint32_t tbase;
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = dm.d, k = dm.k, m0 = blockIdx.x * 128;
  const int nkb = (d + 31) / 32, nnb = (N + 31) / 32;
  // MODE 0: blockIdx.y = group. MODE 1: blockIdx.y = chunk c, blockIdx.z = slice of the chunk's group list: the
  // slice's P_g = dQ_g M_u are accumulated in TMEM (one partial sum per slice, k_tr_reduce adds the slices in order)
  int grp = blockIdx.y, l0 = 0, nsteps = nkb;
  if (MODE == 0 && chunk < 0) {  // blockIdx.y = group, QX slot = group
    if (grp >= *T.n_groups) return;  // uniform per CTA, before any barrier / TMEM use
  } else if (MODE == 0) {  // one chunk: blockIdx.y = the chunk's y-th group, QX slot y
    const int gb = T.cg_off[chunk];
    if ((int)blockIdx.y >= T.cg_off[chunk + 1] - gb) return;
    grp = T.cg_list[gb + blockIdx.y];
  } else {
    const int c = blockIdx.y, S = gridDim.z, z = blockIdx.z;
    const int gb = T.cg_off[c], ng = T.cg_off[c + 1] - gb;
    l0 = gb + (int)(((int64_t)ng * z) / S);
    nsteps = (gb + (int)(((int64_t)ng * (z + 1)) / S) - l0) * nkb;
  }
  auto step_group = [&](int q) { return MODE == 0 ? grp : T.cg_list[l0 + q / nkb]; };
  const uint32_t A_BYTES = 128 * 128, STAGE = A_BYTES + (uint32_t)nnb * 4096;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTrStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], N > 128 ? 2 : 1);
    }
    tc::mbar_init(&done, N > 128 ? 2 : 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  pdl_wait();  // barriers / TMEM set up while the predecessor finished
  pdl_trigger();
  if (warp == 0 && lane == 0) {  // TMA producer
    for (int q = 0; q < nsteps; ++q) {
      const int s = q % kTrStages, kb = q % nkb, g = step_group(q);
      const int c = T.grp_c[g], r = a.s.rel_uniq[T.grp_u[g]];
      if (q >= kTrStages) tc::mbar_wait(&empty[s], ((q / kTrStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      if (MODE == 0) {
        tc::mbar_arrive_expect_tx(&full[s], A_BYTES + (uint32_t)N * 128);
        tc::tma_load_3d(sa, &mA, &full[s], kb * 32, c * k + m0, 0);
        tc::tma_load_3d(sa + A_BYTES, &mB, &full[s], kb * 32, 0, r);
      } else {
        tc::mbar_arrive_expect_tx(&full[s], STAGE);
        tc::tma_load_3d(sa, &mA, &full[s], kb * 32, m0, g);
        // rows a = kb*32.., every column block b = nb*32..: [nnb][32 K rows][32 N] in one 4D box
        tc::tma_load_4d(sa + A_BYTES, &mB, &full[s], 0, kb * 32, 0, r);
      }
    }
  } else if ((warp == 2 || warp == 3) && lane == 0 && (warp == 2 || N > 128)) {
    // MMA issuers split N: issuer 0 columns [0, 128), issuer 1 [128, N) -- two issue streams in parallel, one
    // complete accumulator per column, 256 TMEM columns in all (two CTAs per SM)
    const int qi = warp - 2;
    const int n0 = qi * 128, nn = qi ? N - 128 : (N < 128 ? N : 128);
    const uint32_t idesc = tc::idesc_tf32(128, nn, false, MODE == 1);
    const uint32_t acc = tmem + (uint32_t)n0;
    for (int q = 0; q < nsteps; ++q) {
      const int s = q % kTrStages;
      tc::mbar_wait(&full[s], (q / kTrStages) & 1);
      tc::tc_fence_after();
      const uint32_t sa = tc::smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int sl = 0; sl < 4; ++sl) {
        // N offset: K-major B = 128 rows of 128 B further; MN-major B = 4 blocks of 32 columns further
        const uint64_t bd = MODE == 0 ? tc::sdesc(sb + n0 * 128 + sl * 32, 16, 1024)
                                      : sdesc_mn32(sb + (n0 / 32) * 4096 + sl * 1024, 4096);
        tc::mma_tf32(acc, tc::sdesc(sa + sl * 32, 16, 1024), bd, idesc, (q | sl) ? 1u : 0u);
      }
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(&done);
  }
  __syncwarp();
  if (nsteps > 0) {
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
  }
  // epilogue: thread <-> row m0 + 32 warp + lane, stored to row pitch d (MODE 0: QX_g; MODE 1: the slice's partial
  // sum, slot (z C + c) of the same buffer)
  // Each warp's 32 x 32 chunk is transposed through shared memory (the pipeline stages are free once the MMAs
  // completed) so that every row segment is written by one coalesced 128-byte warp store.
  const int64_t slot = MODE == 0 ? (int64_t)blockIdx.y : (int64_t)blockIdx.z * dm.C + blockIdx.y;  // = grp if chunk < 0
  float* outw = T.QX + slot * k * d + (int64_t)(m0 + warp * 32) * d;  // this warp's first row
  const int nrow = min(32, k - (m0 + warp * 32));
  float* tw = reinterpret_cast<float*>(smem) + warp * (32 * 33);
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  for (int cb = 0; cb * 32 < d; ++cb) {
    uint32_t p0[32];
    if (nsteps > 0) {
      tc::tmem_ld32_nw(trow + cb * 32, p0);
      tc::tmem_wait_ld();
    } else {
#pragma unroll
      for (int x = 0; x < 32; ++x) p0[x] = 0u;
    }
#pragma unroll
    for (int x = 0; x < 32; ++x) tw[lane * 33 + x] = __uint_as_float(p0[x]);
    __syncwarp();
    const int col = cb * 32 + lane;
    if (col < d && xmode != 1)
      for (int rr = 0; rr < nrow; ++rr) outw[(int64_t)rr * d + col] = tw[rr * 33 + lane];
    __syncwarp();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

// dM_u = sum over the relation's groups g (in group order) of dQ_g^T X'_c  on tcgen05 (A = dQ_g^T and B = X'_c both
// MN-major, accumulated in TMEM), then + sum_q U_q^T H_q over its positives (K = 2 n_u, a few rows) in FFMA in the
// epilogue. CTA = 128 rows a of dM_u x N columns b; blockIdx.y = unique relation.
__global__ void __launch_bounds__(128, 1)
    k_tr_dm_tc(const __grid_constant__ CUtensorMap mdQn, const __grid_constant__ CUtensorMap mXn,
               const __grid_constant__ CUtensorMap mUn, const __grid_constant__ CUtensorMap mHn, TrArgs a, int N,
               int mode) {  // mode (timing experiments only, KGE_TR_DM_MODE): 1 = no M update, 2 = no epilogue
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[kTrStages], empty[kTrStages], done;
  __shared__ uint32_t tbase;
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  if ((int)blockIdx.y >= *a.s.rel_n) return;  // uniform per CTA
  const int u = T.rel_order[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int d = dm.d, k = dm.k, m0 = blockIdx.x * 128;
  {  // warm L2 with this CTA's rows of M_u for the fused Adagrad epilogue (HBM latency off its critical path)
    const float* Mu = a.proj + (int64_t)a.s.rel_uniq[u] * d * d;
    const int lines = (d + 31) / 32;
    for (int l = threadIdx.x; l < 128 * lines; l += blockDim.x) {
      const int rr = m0 + l / lines, cb = l - (l / lines) * lines;
      if (rr < d) asm volatile("prefetch.global.L2 [%0];" ::"l"(Mu + (int64_t)rr * d + 32 * cb));
    }
  }
  const int g0 = T.rg_off[u], g1 = T.rg_off[u + 1];
  const int nkg = (k + 31) / 32, nnb = (N + 31) / 32;
  const int nkq = (g1 - g0) * nkg;  // k-blocks over all groups of the relation, then over its padded U / H rows
  const int uq0 = T.pad_off[u], nku = (T.pad_off[u + 1] - uq0) / 32;
  const int nk = nkq + nku;
  const uint32_t A_BYTES = 128 * 128, STAGE = A_BYTES + (uint32_t)nnb * 4096;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTrStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], N > 128 ? 2 : 1);
    }
    tc::mbar_init(&done, N > 128 ? 2 : 1);
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&tbase, 256);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tbase;
  pdl_wait();  // barriers / TMEM set up while the predecessor finished
  pdl_trigger();
  if (warp == 0 && lane == 0) {  // TMA producer
    for (int q = 0; q < nk; ++q) {
      const int s = q % kTrStages;
      if (q >= kTrStages) tc::mbar_wait(&empty[s], ((q / kTrStages) - 1) & 1);
      uint8_t* sa = smem + s * STAGE;
      tc::mbar_arrive_expect_tx(&full[s], STAGE);
      if (q < nkq) {
        const int g = g0 + q / nkg, kb = q % nkg, c = T.grp_c[g];
        // A = dQ_g^T: [4 M-blocks of 32 a][32 K rows j][128 B]; B = X'_c: [N-blocks of 32 b][32 K rows j][128 B]
        tc::tma_load_4d(sa, &mdQn, &full[s], 0, kb * 32, m0 / 32, g);
        tc::tma_load_4d(sa + A_BYTES, &mXn, &full[s], 0, c * k + kb * 32, 0, 0);
      } else {  // + U^T H over the relation's positions: A = U^T (MN-major), B = H (MN-major), K = 32 rows
        const int row = uq0 + (q - nkq) * 32;
        tc::tma_load_4d(sa, &mUn, &full[s], 0, row, m0 / 32, 0);
        tc::tma_load_4d(sa + A_BYTES, &mHn, &full[s], 0, row, 0, 0);
      }
    }
  } else if ((warp == 2 || warp == 3) && lane == 0 && (warp == 2 || N > 128)) {  // issuers split N (see k_tr_tc)
    const int qi = warp - 2;
    const int n0 = qi * 128, nn = qi ? N - 128 : (N < 128 ? N : 128);
    const uint32_t idesc = tc::idesc_tf32(128, nn, true, true);
    const uint32_t acc = tmem + (uint32_t)n0;
    for (int q = 0; q < nk; ++q) {
      const int s = q % kTrStages;
      tc::mbar_wait(&full[s], (q / kTrStages) & 1);
      tc::tc_fence_after();
      const uint32_t sa = tc::smem_u32(smem + s * STAGE), sb = sa + A_BYTES;
#pragma unroll
      for (int sl = 0; sl < 4; ++sl)
        tc::mma_tf32(acc, sdesc_mn32(sa + sl * 1024, 4096), sdesc_mn32(sb + (n0 / 32) * 4096 + sl * 1024, 4096),
                     idesc, (q | sl) ? 1u : 0u);
      tc::mma_commit(&empty[s]);
    }
    tc::mma_commit(&done);
  }
  __syncwarp();
  if (nk > 0) {
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
  }
  // epilogue: row a = m0 + 32 warp + lane of dM_u straight from TMEM (the U^T H term was accumulated by the MMAs),
  // fused with the projection's Adagrad (reading c.11: one state per matrix, w = d*d). The CTAs of relation u -- one
  // cluster over the row blocks of dM_u -- add their sums of squares in cluster-rank order through distributed shared
  // memory; each then applies M_u -= lr dM_u / sqrt(state + eps) to its rows from TMEM (no dM round trip through HBM
  // and no separate pass over it). A split relation at P > 1 stores this rank's sum instead (dist.cu applies the
  // rank-ordered sum on every replica); a non-finite loss skips the update (KGE_ENONFINITE).
  __shared__ float s_sq[4];
  __shared__ float s_part;
  const int row = m0 + warp * 32 + lane;
  const int r = a.s.rel_uniq[u];
  const int sidx = a.split_index ? a.split_index[r] : -1;
  const bool skip = a.b.flags[2 + (a.s.info[0] & 1)] != 0;
  const int64_t w = (int64_t)d * d;
  const float st_old = a.proj_st[r];  // every CTA reads it before cluster rank 0 overwrites it (after the barrier)
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  auto chunk = [&](int cb, float* v) {
    uint32_t p0[32];
    tc::tmem_ld32_nw(trow + cb * 32, p0);
    tc::tmem_wait_ld();
#pragma unroll
    for (int x = 0; x < 32; ++x) v[x] = __uint_as_float(p0[x]);
  };
  // this warp's 32 rows of M_u into the freed pipeline shared memory (row pitch P4 float4, odd: the row-per-thread
  // float4 accesses below are conflict-free), in flight during the sums of squares and the cluster barriers
  const int d4 = d >> 2, P4 = d4 | 1, rw0 = m0 + warp * 32, nrw = min(32, d - rw0);
  float4* Ms = reinterpret_cast<float4*>(smem) + warp * 32 * P4;
  float4* Mg = reinterpret_cast<float4*>(a.proj + (int64_t)r * w) + (int64_t)rw0 * d4;
  const bool upd = !skip && sidx < 0 && mode == 0;
  if (upd)
    for (int rr = 0; rr < nrw; ++rr)
      for (int c = lane; c < d4; c += 32) cp_async16(Ms + rr * P4 + c, Mg + (int64_t)rr * d4 + c, true);
  cp_async_commit();
  float sq = 0.f;
  for (int cb = 0; cb * 32 < d && mode < 2; ++cb) {
    float v[32];
    chunk(cb, v);
    if (row < d && !skip) {
      if (sidx >= 0) {
        float* out = a.gproj_split + (int64_t)sidx * w + (int64_t)row * d;
#pragma unroll
        for (int x = 0; x < 32; x += 4)
          if (cb * 32 + x < d)
            *reinterpret_cast<float4*>(out + cb * 32 + x) = make_float4(v[x], v[x + 1], v[x + 2], v[x + 3]);
      } else {
#pragma unroll
        for (int x = 0; x < 32; ++x)
          if (cb * 32 + x < d) sq = fmaf(v[x], v[x], sq);
      }
    }
  }
  sq = warp_sum(sq);
  if (lane == 0) s_sq[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) s_part = ((s_sq[0] + s_sq[1]) + s_sq[2]) + s_sq[3];
  tc::cluster_sync();
  float total = 0.f;
  for (unsigned q = 0; q < gridDim.x; ++q) total += tc::ld_cluster_f32(tc::mapa_shared(tc::smem_u32(&s_part), q));
  const float st_new = st_old + total / (float)w;
  const float step = dm.lr / sqrtf(st_new + dm.eps);
  tc::cluster_sync();  // the peers' reads of s_part are done before any CTA leaves
  if (!skip && sidx < 0 && mode == 0) {
    if (tc::cluster_ctarank() == 0 && threadIdx.x == 0) a.proj_st[r] = st_new;
    // The warp's 32 rows of M_u are copied into shared memory in one cp.async round trip (the pipeline stages are
    // free once the MMAs completed; row pitch P4 float4, odd, so the row-per-thread float4 accesses below are
    // conflict-free), updated there from TMEM (thread = row), and written back with coalesced row stores.
    cp_async_wait<0>();  // the M_u rows issued before the sums of squares
    __syncwarp();
    for (int cb = 0; cb * 32 < d; ++cb) {
      float v[32];
      chunk(cb, v);  // warp-collective
      if (lane < nrw) {
#pragma unroll
        for (int x4 = 0; x4 < 8; ++x4) {
          const int c4 = cb * 8 + x4;
          if (c4 < d4) {
            float4 m = Ms[lane * P4 + c4];
            m.x -= step * v[4 * x4];
            m.y -= step * v[4 * x4 + 1];
            m.z -= step * v[4 * x4 + 2];
            m.w -= step * v[4 * x4 + 3];
            Ms[lane * P4 + c4] = m;
          }
        }
      }
    }
    __syncwarp();
    for (int rr = 0; rr < nrw; ++rr)
      for (int c = lane; c < d4; c += 32) Mg[(int64_t)rr * d4 + c] = Ms[rr * P4 + c];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

static size_t tr_tc_smem(int N) { return (size_t)kTrStages * (128 * 128 + (size_t)((N + 31) / 32) * 4096) + 1024; }
// k_tr_dm_tc: the pipeline stages, reused after the main loop for the 128 rows of M_u (pitch (d/4 | 1) float4)
static size_t tr_dm_smem(int N, int d) { return std::max(tr_tc_smem(N), (size_t)128 * ((d / 4) | 1) * 16 + 1024); }

// ------------------------------------------------------------------------------------------------
// per-group scores. CTA (t, g) = 32 negatives j of group g (warp w: j = 32 t + w + 8 u, u < 4, held in registers as
// V float4 per lane) against every positive of the group, RB positives at a time: one warp reduction per (positive,
// negative) distance. dQ_g[j] is complete in the warp that holds row j (sum over the group's positives in order);
// the dO_i partial of the tile is added over the 8 warps in warp order (shared memory) and stored per tile (dOp),
// which k_tr_chain sums in tile order -- a fixed order throughout, and the work of a large group (a frequent relation
// holding most of a chunk) is spread over k / 32 CTAs instead of one.
// ------------------------------------------------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(256) k_tr_score(TrArgs a, int chunk, int xmode, int fast) {
  // xmode (timing experiments only, KGE_TR_XMODE): 2 = no pair loop, 3 = no dQ stores
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  constexpr int RB = 4 / V;  // positives per block (registers: (2 JU + 2 RB) V float4 per lane)
  constexpr int JU = kTrJt / 8;  // negatives per warp
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  // launched per chunk (after k_tr_tc<0> of the chunk): blockIdx.y = the chunk's y-th group, its QX in slot y
  const int jt = blockIdx.x, njt = gridDim.x;
  __shared__ float red[8];
  __shared__ float4 sdo4[8][RB][32 * V];  // per-warp dO partials of a block of positives
  // work item (k_tr_groups): a slice of <= kTrSlice positions of group grp. chunk < 0: blockIdx.y = item, QX slot =
  // group; chunk >= 0 (launched per chunk after that chunk's projections): item si_off[chunk] + blockIdx.y, QX slot =
  // the group's index within the chunk
  const int item = chunk < 0 ? (int)blockIdx.y : T.si_off[chunk] + (int)blockIdx.y;
  if (item >= (chunk < 0 ? *T.n_sitems : T.si_off[chunk + 1])) return;
  const int grp = T.sitem_g[item];
  const int qslot = chunk < 0 ? grp : T.grp_lc[grp];
  const int d = dm.d, d4 = d >> 2, k = dm.k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = T.sitem_p[item], p1 = min(p0 + kTrSlice, T.grp_p1[grp]);
  const float4* QX = reinterpret_cast<const float4*>(T.QX + (int64_t)qslot * k * d);
  float4* dQ = reinterpret_cast<float4*>(T.dQ + (int64_t)grp * k * d);
  const float inv_bk = 1.f / ((float)dm.B * (float)dm.k);
  const bool pairwise = dm.loss == KGE_LOSS_PAIRWISE;
  float4 q[JU][V], dq[JU][V];
#pragma unroll
  for (int u = 0; u < JU; ++u)
#pragma unroll
    for (int m = 0; m < V; ++m) {
      const int j = jt * kTrJt + warp + 8 * u, c = lane + 32 * m;
      q[u][m] = j < k && c < d4 ? __ldcs(QX + (int64_t)j * d4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      dq[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  // the slice's o rows (d <= 256) are staged in shared memory once, together with the q loads: the positive blocks
  // below then wait on no global load
  constexpr bool STAGE = V <= 2;
  __shared__ float4 o_s[STAGE ? kTrSlice : 1][32 * V];
  __shared__ int ip_s[kTrSlice];
  if (STAGE) {
    constexpr int PER = (kTrSlice * 32 * V) / 256;
    float4 t[PER];
#pragma unroll
    for (int l = 0; l < PER; ++l) {
      const int x = threadIdx.x + 256 * l, rr = x / (32 * V), c = x % (32 * V);
      t[l] = p0 + rr < p1 && c < d4
                 ? reinterpret_cast<const float4*>(a.b.O + (int64_t)a.s.rel_occ[p0 + rr] * dm.dp)[c]
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int l = 0; l < PER; ++l) {
      const int x = threadIdx.x + 256 * l;
      o_s[x / (32 * V)][x % (32 * V)] = t[l];
    }
  }
  if (threadIdx.x < kTrSlice) ip_s[threadIdx.x] = p0 + (int)threadIdx.x < p1 ? a.s.rel_occ[p0 + threadIdx.x] : 0;
  __syncthreads();
  float lsum = 0.f, lprod = 1.f;
  for (int rb = p0; rb < p1 && xmode != 2; rb += RB) {
    const int nr = min(RB, p1 - rb);
    float4 o[RB][V], g[RB][V];
    int ip[RB];
    float fpos[RB];
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      ip[rr] = rr < nr ? ip_s[rb - p0 + rr] : 0;
      fpos[rr] = rr < nr && pairwise ? dm.gamma - a.b.pstat[ip[rr]] : 0.f;
      const float4* orow = reinterpret_cast<const float4*>(a.b.O + (int64_t)ip[rr] * dm.dp);
#pragma unroll
      for (int m = 0; m < V; ++m) {
        const int c = lane + 32 * m;
        if (STAGE)
          o[rr][m] = o_s[STAGE ? rb - p0 + rr : 0][c];  // zero beyond the slice / d4
        else
          o[rr][m] = rr < nr && c < d4 ? orow[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        g[rr][m] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int rr = 0; rr < RB; ++rr) {
      if (rr >= nr) break;  // warp-uniform
#pragma unroll
      for (int u = 0; u < JU; ++u) {
        const int j = jt * kTrJt + warp + 8 * u;
        if (j >= k) break;  // warp-uniform
        float s2 = 0.f;
#pragma unroll
        for (int m = 0; m < V; ++m) {
          const float ux = o[rr][m].x - q[u][m].x, uy = o[rr][m].y - q[u][m].y, uz = o[rr][m].z - q[u][m].z,
                      uw = o[rr][m].w - q[u][m].w;
          s2 = fmaf(ux, ux, s2);
          s2 = fmaf(uy, uy, s2);
          s2 = fmaf(uz, uz, s2);
          s2 = fmaf(uw, uw, s2);
        }
        s2 = warp_sum(s2);  // xor butterfly: every lane holds the same bits
        const float f = dm.gamma - s2;
        float coef;
        if (pairwise) {  // reading c.9'
          float dldf;
          int act;
          const float l = hinge_term(f, fpos[rr], dm.gamma, inv_bk, dldf, act);
          if (lane == 0) {
            lsum += l;
            if (act) atomicAdd(&a.b.pcnt[ip[rr]], 1);  // integer: exact in any order
          }
          coef = -2.f * dldf;
        } else {
          // e = exp(-|f|): sigma(f) = f >= 0 ? 1/(1+e) : e/(1+e); -log sigma(-f) = max(f, 0) + log1p(e), the log1p
          // terms summed as one log of their product (each factor in (1, 2], <= 64 per lane: no overflow) -- the
          // three-MUFU form of the tcgen05 forward epilogue
          // (the FP32 path -- FFMA projections -- keeps the accurate expf / log1pf forms of its 1e-5 bars)
          if (fast) {
            const float e = __expf(-fabsf(f));
            float r1;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(1.f + e));
            coef = -2.f * (f >= 0.f ? r1 : e * r1) * inv_bk;  // dL/df * df/d(s2)
            if (lane == 0) {
              lsum += fmaxf(f, 0.f);
              lprod *= 1.f + e;
            }
          } else {
            coef = -2.f * sigmoid(f) * inv_bk;
            if (lane == 0) lsum += -log_sigmoid(-f);
          }
        }
        if (lane == 0 && a.b.fdbg) a.b.fdbg[(int64_t)ip[rr] * k + j] = f;  // KGE_OPT_CAPTURE_NEG
#pragma unroll
        for (int m = 0; m < V; ++m) {  // dO_i += coef (o - q);  dQ_j += coef (q - o)
          const float4 w = make_float4(o[rr][m].x - q[u][m].x, o[rr][m].y - q[u][m].y, o[rr][m].z - q[u][m].z,
                                       o[rr][m].w - q[u][m].w);
          g[rr][m].x = fmaf(coef, w.x, g[rr][m].x);
          g[rr][m].y = fmaf(coef, w.y, g[rr][m].y);
          g[rr][m].z = fmaf(coef, w.z, g[rr][m].z);
          g[rr][m].w = fmaf(coef, w.w, g[rr][m].w);
          dq[u][m].x = fmaf(coef, -w.x, dq[u][m].x);
          dq[u][m].y = fmaf(coef, -w.y, dq[u][m].y);
          dq[u][m].z = fmaf(coef, -w.z, dq[u][m].z);
          dq[u][m].w = fmaf(coef, -w.w, dq[u][m].w);
        }
      }
    }
    // this tile's dO partials of the block: the 8 warps added in warp order
#pragma unroll
    for (int rr = 0; rr < RB; ++rr)
#pragma unroll
      for (int m = 0; m < V; ++m) sdo4[warp][rr][lane + 32 * m] = g[rr][m];
    __syncthreads();
    for (int x = threadIdx.x; x < nr * 32 * V; x += blockDim.x) {
      const int rr = x / (32 * V), c = x - rr * 32 * V;
      if (c >= d4) continue;
      float4 acc = sdo4[0][rr][c];
      for (int w = 1; w < 8; ++w) {
        const float4 y = sdo4[w][rr][c];
        acc.x += y.x;
        acc.y += y.y;
        acc.z += y.z;
        acc.w += y.w;
      }
      reinterpret_cast<float4*>(T.dOp + ((int64_t)jt * dm.B + ip_s[rb - p0 + rr]) * d)[c] = acc;
    }
    __syncthreads();
  }
  // dQ_g rows of this tile: a group of one slice stores them; the slices of a larger group park their partials in
  // dQs, and the last to arrive (integer counter per (group, tile)) adds them in slice order and stores dQ_g
  const int ms = T.ms_off[grp];
  const int sl = (p0 - T.grp_p0[grp]) / kTrSlice;
  float4* dst = ms < 0 ? dQ : reinterpret_cast<float4*>(T.dQs + (int64_t)(ms + sl) * k * d);
#pragma unroll
  for (int u = 0; u < JU; ++u) {
    const int j = jt * kTrJt + warp + 8 * u;
    if (j < k && xmode != 3)
#pragma unroll
      for (int m = 0; m < V; ++m)
        if (lane + 32 * m < d4) dst[(int64_t)j * d4 + lane + 32 * m] = dq[u][m];
  }
  lsum += __logf(lprod);
  lsum = warp_sum(lsum);
  if (lane == 0) red[warp] = lsum;
  __shared__ int s_last;
  if (ms >= 0) __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    a.b.lneg[(int64_t)item * njt + jt] = t;
    if (ms >= 0) {
      const int ns = (T.grp_p1[grp] - T.grp_p0[grp] + kTrSlice - 1) / kTrSlice;
      int* cnt = T.scnt + (int64_t)grp * njt + jt;
      s_last = atomicAdd(cnt, 1) == ns - 1;
      if (s_last) *cnt = 0;  // ready for the next step
    }
  }
  __syncthreads();
  if (ms >= 0 && s_last) {
    __threadfence();
    const int ns = (T.grp_p1[grp] - T.grp_p0[grp] + kTrSlice - 1) / kTrSlice;
    // slice order; every (row, column) load of a slice in flight at once (one L2 round trip per slice)
#pragma unroll
    for (int u = 0; u < JU; ++u)
#pragma unroll
      for (int m = 0; m < V; ++m) dq[u][m] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < ns; ++q) {
      const float4* src = reinterpret_cast<const float4*>(T.dQs + (int64_t)(ms + q) * k * d);
      float4 y[JU][V];
#pragma unroll
      for (int u = 0; u < JU; ++u)
#pragma unroll
        for (int m = 0; m < V; ++m) {
          const int j = jt * kTrJt + warp + 8 * u, c = lane + 32 * m;
          y[u][m] = j < k && c < d4 ? __ldcg(src + (int64_t)j * d4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int u = 0; u < JU; ++u)
#pragma unroll
        for (int m = 0; m < V; ++m) {
          dq[u][m].x += y[u][m].x;
          dq[u][m].y += y[u][m].y;
          dq[u][m].z += y[u][m].z;
          dq[u][m].w += y[u][m].w;
        }
    }
#pragma unroll
    for (int u = 0; u < JU; ++u) {
      const int j = jt * kTrJt + warp + 8 * u;
      if (j >= k) continue;
#pragma unroll
      for (int m = 0; m < V; ++m)
        if (lane + 32 * m < d4) dQ[(int64_t)j * d4 + lane + 32 * m] = dq[u][m];
    }
  }
}

static int tr_score_v(int d) { return d <= 128 ? 1 : (d <= 256 ? 2 : 4); }

// dX'_c[j][e] = sum over the chunk's groups (ascending group id) of P_g[j][e]  -> occurrence rows 2B + c*k + j
// (nslice > 0: the tcgen05 path's per-slice partial sums, slot z C + c, added in slice order)
__global__ void k_tr_reduce(TrArgs a, int nslice) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  const TrBuffers& T = a.t;
  const int64_t total = (int64_t)dm.C * dm.k * dm.d;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(q / ((int64_t)dm.k * dm.d));
    const int64_t je = q - (int64_t)c * dm.k * dm.d;
    float acc = 0.f;
    if (nslice > 0)
      for (int z = 0; z < nslice; ++z) acc += T.QX[((int64_t)z * dm.C + c) * dm.k * dm.d + je];
    else
      for (int l = T.cg_off[c]; l < T.cg_off[c + 1]; ++l) acc += T.QX[(int64_t)T.cg_list[l] * dm.k * dm.d + je];
    a.b.Gocc[((int64_t)2 * dm.B + (int64_t)c * dm.k) * dm.d + je] = acc;
  }
}

// ------------------------------------------------------------------------------------------------
// chain: one CTA per relation-sorted position p (+ one CTA for the loss)
//   tail: o = Mh + r : gMh = dO - 2w p, gMt = 2w p, dr = gMh
//   head: o = Mt - r : gMh = -2w p,     gMt = dO + 2w p, dr = -gMt
//   dh = M^T gMh, dt = M^T gMt ; dM_u += gMh h^T + gMt t^T (rows U/H at 2p, 2p+1)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_tr_chain(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == gridDim.x - 1) {
    // the loss: every thread of the CTA sums a strided share (eight loads in flight), then the 8 warps' sums are
    // added in warp order -- a fixed association
    __shared__ float s_sp[8], s_sn[8];
    float sp = 0.f, sn = 0.f;
    for (int i = threadIdx.x; i < dm.B; i += blockDim.x) sp += a.b.lpos[i];
    const int nparts = *a.t.n_sitems * tr_jtiles(dm.k);  // per (score item, tile of 32 negatives), k_tr_score
    for (int q0 = threadIdx.x; q0 < nparts; q0 += 8 * blockDim.x) {
      float y[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) y[t] = q0 + t * (int)blockDim.x < nparts ? a.b.lneg[q0 + t * blockDim.x] : 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t) sn += y[t];
    }
    sp = warp_sum(sp);
    sn = warp_sum(sn);
    if (lane == 0) {
      s_sp[threadIdx.x >> 5] = sp;
      s_sn[threadIdx.x >> 5] = sn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      sp = 0.f;
      sn = 0.f;
      for (int w8 = 0; w8 < 8; ++w8) {
        sp += s_sp[w8];
        sn += s_sn[w8];
      }
      {
        const float L = sp / (float)dm.B + sn / ((float)dm.B * (float)dm.k);
        store_loss(a.b.loss, a.s.info, L);
        const bool bad = !isfinite(L);
        a.b.flags[2 + (a.s.info[0] & 1)] = bad ? 1 : 0;
        if (bad) a.b.flags[0] = 1;
      }
    }
    return;
  }
  const int d = dm.d;
  const int p = blockIdx.x, i = a.s.rel_occ[p];
  const int r = a.s.pr[i], mode = a.s.mode[i / dm.g];
  const float w = dm.loss == KGE_LOSS_PAIRWISE ? -(float)a.b.pcnt[i] * (1.f / ((float)dm.B * (float)dm.k))
                                               : a.b.wpos[i];  // dL/df+ (reading c.9 / c.9')
  const float* pv = a.t.Pv + (int64_t)i * d;
  const float* dOp = a.t.dOp + (int64_t)i * d;  // tile t's partial at + t B d (k_tr_score)
  const int njt = tr_jtiles(dm.k);
  const int64_t tstride = (int64_t)dm.B * d;
  float* gR = a.b.Grel + (int64_t)i * dm.drel;
  const int u = a.s.rel_inv[i], pr0 = a.s.rel_off[u], pr1 = a.s.rel_off[u + 1];
  const int64_t urow = a.t.pad_off[u] + 2 * (p - pr0);  // padded per-relation layout (k_tr_groups)
  float* U = a.t.U + urow * d;
  float* H = a.t.H + urow * d;
  if (p == pr1 - 1)  // the relation's last position clears the padding rows after its 2 n_u rows
    for (int64_t q = (a.t.pad_off[u] + 2 * (pr1 - pr0)) * d + threadIdx.x; q < (int64_t)a.t.pad_off[u + 1] * d;
         q += blockDim.x) {
      a.t.U[q] = 0.f;
      a.t.H[q] = 0.f;
    }
  const float* hrow = a.ent.row(a.s.ph[i]);
  const float* trow = a.ent.row(a.s.pt[i]);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    const float tp = 2.f * w * pv[e];
    float dO = dOp[e];
    for (int t0 = 1; t0 < njt; t0 += 8) {  // the negative tiles in order, eight loads in flight
      float y[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) y[t] = t0 + t < njt ? dOp[(t0 + t) * tstride + e] : 0.f;
#pragma unroll
      for (int t = 0; t < 8; ++t)
        if (t0 + t < njt) dO += y[t];
    }
    const float gh = mode == 0 ? dO - tp : -tp;
    const float gt = mode == 0 ? tp : dO + tp;
    gR[e] = mode == 0 ? gh : -gt;
    U[e] = gh;
    U[d + e] = gt;
    H[e] = hrow[e];
    H[d + e] = trow[e];
  }
  (void)r;  // dh = M^T gMh, dt = M^T gMt: k_tr_mv<1> over the U rows written here
}

// Adagrad on M_u, one state per matrix (w = d*d)
__global__ void __launch_bounds__(1024) k_tr_proj(TrArgs a) {
  pdl_wait();  // the predecessor's outputs are final (programmatic dependent launch)
  pdl_trigger();
  const Dims& dm = a.dm;
  if (a.b.flags[2 + (a.s.info[0] & 1)]) return;
  const int u = blockIdx.x;
  if (u >= *a.s.rel_n) return;
  __shared__ float red[32];
  __shared__ float s_step;
  const int r = a.s.rel_uniq[u];
  const int64_t w = (int64_t)dm.d * dm.d;
  const float* G = a.t.dM + (int64_t)u * w;
  const int sidx = a.split_index ? a.split_index[r] : -1;
  if (sidx >= 0) {  // P > 1, split relation: this rank's sum; every replica applies the rank-ordered sum (dist.cu)
    float* dst = a.gproj_split + (int64_t)sidx * w;
    for (int64_t q = threadIdx.x; q < w; q += blockDim.x) dst[q] = G[q];
    return;
  }
  float sq = 0.f;
  for (int64_t q = threadIdx.x; q < w; q += blockDim.x) sq = fmaf(G[q], G[q], sq);
  sq = warp_sum(sq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += red[ww];
    const float st = a.proj_st[r] + s / (float)w;
    a.proj_st[r] = st;
    s_step = dm.lr / sqrtf(st + dm.eps);
  }
  __syncthreads();
  float* Mr = a.proj + (int64_t)r * w;
  for (int64_t q = threadIdx.x; q < w; q += blockDim.x) Mr[q] -= s_step * G[q];
}

// ------------------------------------------------------------------------------------------------
cudaError_t launch_gather_neg(kge_handle* h, const Slot& s);                      // step.cu
cudaError_t launch_update(kge_handle* h, const Slot& s);                          // step.cu

static void dbg(kge_handle* h, const char* what) {
  static const bool on = getenv("KGE_DEBUG_SYNC") != nullptr;
  if (!on) return;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  fprintf(stderr, "[kge] %s -> %s\n", what, cudaGetErrorString(e));
}

// Adagrad on the projection matrices of the step's unique relations (TransR, RESCAL: one state per matrix)
cudaError_t launch_proj_update(kge_handle* h, const Slot& s) {
  const Dims& dm = h->dims;
  TrArgs a{dm, s, h->rows, h->rel, h->proj, h->proj_st, h->buf, h->tr_buf, h->n_neg_parts,
           h->P > 1 ? h->dist.split_index : nullptr, h->dist.gproj_split};
  launch_pdl(k_tr_proj, dm.B, 1024, 0, h->stream, a);  // one matrix of d*d per CTA: 1024 threads stream it
  ++h->launches;
  return cudaGetLastError();
}

cudaError_t launch_transr_step(kge_handle* h, const Slot& s, int64_t step) {
  const Dims& dm = h->dims;
  (void)step;
  TrArgs a{dm, s, h->rows, h->rel, h->proj, h->proj_st, h->buf, h->tr_buf, h->n_neg_parts,
           h->P > 1 ? h->dist.split_index : nullptr, h->dist.gproj_split};
  cudaError_t e;
  launch_begin(h, KGE_K_GATHER);
  launch_pdl(k_tr_groups, 1, 1024, 0, h->stream, a); dbg(h, "k_tr_groups");
  e = launch_gather_neg(h, s);
  dbg(h, "gather_neg");
  if (e != cudaSuccess) return e;
  // k_tr_mv: one wave (two CTAs per SM), each CTA walking its items with the next one's slab prefetched into L2
  const dim3 gmv((dm.d + 31) / 32, std::max(1, 2 * 148 / ((dm.d + 31) / 32)));
  launch_pdl(k_tr_mv<0>, gmv, 256, tr_mv_smem(dm.d), h->stream, a); dbg(h, "k_tr_mv<0>");
  launch_pdl(k_tr_pos, dm.B, 256, 0, h->stream, a); dbg(h, "k_tr_pos");
  launch_end(h, KGE_K_GATHER);
  const dim3 gk((dm.d + GT - 1) / GT, (dm.k + GT - 1) / GT, dm.B);
  launch_begin(h, KGE_K_NEG_FWD);
  static const int xmode = getenv("KGE_TR_XMODE") ? atoi(getenv("KGE_TR_XMODE")) : 0;  // timing experiments only
  const int fast = h->tr_tc ? 1 : 0;  // three-MUFU logistic form on the TF32 path only
  auto score = [&](dim3 gs, int chunk) {
    switch (tr_score_v(dm.d)) {
      case 1: launch_pdl(k_tr_score<1>, gs, 256, 0, h->stream, a, chunk, xmode, fast); break;
      case 2: launch_pdl(k_tr_score<2>, gs, 256, 0, h->stream, a, chunk, xmode, fast); break;
      default: launch_pdl(k_tr_score<4>, gs, 256, 0, h->stream, a, chunk, xmode, fast); break;
    }
  };
  // every group in one launch; KGE_TR_CHUNKED=1 (experiment) runs projections + scores chunk by chunk so a chunk's QX
  // stays in L2 -- measured slower (1.74 vs 2.02 M pos/s: each chunk's score launch pays the latency of its longest
  // items again)
  static const bool global_fwd = getenv("KGE_TR_CHUNKED") == nullptr;
  if (h->tr_tc && global_fwd) {
    const TrTc* tt = static_cast<const TrTc*>(h->tr_tc);
    launch_pdl(k_tr_tc<0>, dim3((dm.k + 127) / 128, dm.B), 128, tr_tc_smem(tt->N), h->stream, tt->mX, tt->mM, a,
               tt->N, -1, xmode);
    score(dim3(tr_jtiles(dm.k), dm.B + dm.B / kTrSlice + 1), -1);
  } else if (h->tr_tc) {  // chunk by chunk: the chunk's projected negatives go to the first QX slots
    const TrTc* tt = static_cast<const TrTc*>(h->tr_tc);
    for (int c = 0; c < dm.C; ++c) {
      launch_pdl(k_tr_tc<0>, dim3((dm.k + 127) / 128, dm.g), 128, tr_tc_smem(tt->N), h->stream, tt->mX, tt->mM, a,
                 tt->N, c, xmode);
      dbg(h, "k_tr_tc<0>");
      score(dim3(tr_jtiles(dm.k), dm.g + dm.g / kTrSlice + 1), c);
      dbg(h, "k_tr_score");
    }
  } else {
    launch_pdl(k_tr_gemm<0>, gk, 256, 0, h->stream, a); dbg(h, "k_tr_gemm<0>");
    score(dim3(tr_jtiles(dm.k), dm.B + dm.B / kTrSlice + 1), -1);  // every group at once, QX slot = group
    dbg(h, "k_tr_score");
  }
  launch_end(h, KGE_K_NEG_FWD);
  launch_begin(h, KGE_K_NEG_BWD);
  // k_tr_tc<1>: CTAs (tile of 128 negatives, chunk, slice of the chunk's groups), about two per SM; the slices' partial
  // sums take slots z C + c of the QX buffer (B slots of k x d)
  const int jt = (dm.k + 127) / 128;
  const int nslice = std::max(1, std::min(2 * 148 / (jt * dm.C), dm.B / dm.C));
  if (h->tr_tc) {
    const TrTc* tt = static_cast<const TrTc*>(h->tr_tc);
    launch_pdl(k_tr_tc<1>, dim3(jt, dm.C, nslice), 128, tr_tc_smem(tt->N), h->stream, tt->mdQ, tt->mMn, a, tt->N, 0, 0);
    dbg(h, "k_tr_tc<1>");
  } else {
    launch_pdl(k_tr_gemm<1>, gk, 256, 0, h->stream, a); dbg(h, "k_tr_gemm<1>");
  }
  const int64_t tot = (int64_t)dm.C * dm.k * dm.d;
  launch_pdl(k_tr_reduce, (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, h->stream, a,
             h->tr_tc ? nslice : 0);
  dbg(h, "k_tr_reduce");
  launch_end(h, KGE_K_NEG_BWD);
  launch_begin(h, KGE_K_CHAIN);
  launch_pdl(k_tr_chain, dm.B + 1, 256, 0, h->stream, a); dbg(h, "k_tr_chain");
  launch_pdl(k_tr_mv<1>, gmv, 256, tr_mv_smem(dm.d), h->stream, a); dbg(h, "k_tr_mv<1>");
  const dim3 gm((dm.d + GT - 1) / GT, (dm.d + GT - 1) / GT, dm.B);
  if (h->tr_tc) {
    const TrTc* tt = static_cast<const TrTc*>(h->tr_tc);
    // cluster = the row blocks of one relation's dM (the fused Adagrad adds their sums of squares through DSMEM)
    const unsigned cx = (unsigned)((dm.d + 127) / 128);
    static const int dm_mode = getenv("KGE_TR_DM_MODE") ? atoi(getenv("KGE_TR_DM_MODE")) : 0;
    e = launch_pdl_cluster(k_tr_dm_tc, dim3(cx, dm.B), 128, tr_dm_smem(tt->N, dm.d), h->stream, cx, tt->mdQn, tt->mXn, tt->mUn,
                           tt->mHn, a, tt->N, dm_mode);
    if (e != cudaSuccess) return e;
    dbg(h, "k_tr_dm_tc");
  } else {
    launch_pdl(k_tr_gemm<2>, gm, 256, 0, h->stream, a); dbg(h, "k_tr_gemm<2>");
  }
  launch_end(h, KGE_K_CHAIN);
  e = launch_update(h, s);
  dbg(h, "update");
  if (e != cudaSuccess) return e;
  if (!h->tr_tc) {  // the tcgen05 path applies it in k_tr_dm_tc's epilogue
    launch_pdl(k_tr_proj, dm.B, 1024, 0, h->stream, a);
    dbg(h, "k_tr_proj");
  }
  h->launches += h->tr_tc ? (global_fwd ? 7 : 5 + 2 * dm.C) : 8;  // kernels launched here beyond the four launch_begin brackets (k_update counts itself)
  return cudaGetLastError();
}

// kge_score for TransR: f = gamma - ||M_r h + r - M_r t||^2 per triple (CTA per triple)
__global__ void __launch_bounds__(256) k_tr_score_triples(Dims dm, EntRows ent, const float* rel, const float* proj,
                                                          const int32_t* hs, const int32_t* rs, const int32_t* ts,
                                                          float* out) {
  __shared__ float sh[512], st[512], red[8];
  const int i = blockIdx.x, d = dm.d, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float* M = proj + (int64_t)rs[i] * d * d;
  const float* rv = rel + (int64_t)rs[i] * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    sh[e] = ent.row(hs[i])[e];
    st[e] = ent.row(ts[i])[e];
  }
  __syncthreads();
  float sq = 0.f;
  for (int row = warp; row < d; row += 8) {
    const float* mr = M + (int64_t)row * d;
    float ah = 0.f, at = 0.f;
    for (int b = lane; b < d; b += 32) {
      ah = fmaf(mr[b], sh[b], ah);
      at = fmaf(mr[b], st[b], at);
    }
    ah = warp_sum(ah);
    at = warp_sum(at);
    const float pe = ah + rv[row] - at;
    sq += lane == 0 ? pe * pe : 0.f;
  }
  sq = warp_sum(sq);
  if (lane == 0) red[warp] = sq;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.f;
    for (int w = 0; w < 8; ++w) s += red[w];
    out[i] = dm.gamma - s;
  }
}

cudaError_t launch_transr_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n,
                                float* out) {
  for (int64_t b = 0; b < n; b += 65535) {
    const int64_t m = std::min<int64_t>(65535, n - b);
    k_tr_score_triples<<<(unsigned)m, 256, 0, h->stream>>>(h->dims, h->rows, h->rel, h->proj, hs + b, rs + b, ts + b,
                                                           out + b);
    ++h->launches;
  }
  return cudaGetLastError();
}


bool transr_init(kge_handle* h) {
  const int smem = (int)tr_mv_smem(h->dims.d);
  return cudaFuncSetAttribute(k_tr_mv<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess &&
         cudaFuncSetAttribute(k_tr_mv<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess;
}

// after the step buffers exist (the maps name X' and the projection table)
void transr_tc_init(kge_handle* h) {
  // TF32 negatives path: the projections QX_g = X'_c M_u^T on tcgen05 (d <= 256), else FFMA
  const Dims& dm = h->dims;
  if (h->cfg.neg_precision == KGE_PREC_TF32 && dm.d <= 256 && dm.d % 4 == 0) {
    TrTc* tt = new TrTc();
    tt->N = (dm.d + 15) / 16 * 16;
    bool ok = make_map(&tt->mX, h->buf.X, dm.d, dm.C * dm.k, 1, dm.dp, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    ok = ok && make_map(&tt->mM, h->proj, dm.d, dm.d, (int)dm.n_relations, dm.d, tt->N, CU_TENSOR_MAP_SWIZZLE_128B);
    const int nnb = (tt->N + 31) / 32;
    ok = ok && make_map4c(&tt->mMn, h->proj, dm.d, dm.d, (int)dm.n_relations, dm.d, 32, nnb,
                          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    ok = ok && make_map(&tt->mdQ, h->tr_buf.dQ, dm.d, dm.k, dm.B, dm.d, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    ok = ok && make_map4c(&tt->mdQn, h->tr_buf.dQ, dm.d, dm.k, dm.B, dm.d, 32, 4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    ok = ok && make_map4c(&tt->mXn, h->buf.X, dm.d, dm.C * dm.k, 1, dm.dp, 32, nnb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const int urows = 2 * dm.B + 32 * dm.B;  // the padded U / H layout (k_tr_groups)
    ok = ok && make_map4c(&tt->mUn, h->tr_buf.U, dm.d, urows, 1, dm.d, 32, 4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    ok = ok && make_map4c(&tt->mHn, h->tr_buf.H, dm.d, urows, 1, dm.d, 32, nnb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    const size_t smem = tr_tc_smem(tt->N);
    ok = ok && cudaFuncSetAttribute(k_tr_tc<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
    ok = ok && cudaFuncSetAttribute(k_tr_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) == cudaSuccess;
    ok = ok && cudaFuncSetAttribute(k_tr_dm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)tr_dm_smem(tt->N, dm.d)) == cudaSuccess;
    if (ok) {
      h->tr_tc = tt;
    } else {
      cudaGetLastError();
      delete tt;
    }
  }
}

void transr_destroy(kge_handle* h) {
  delete static_cast<TrTc*>(h->tr_tc);
  h->tr_tc = nullptr;
}

}  // namespace kge
