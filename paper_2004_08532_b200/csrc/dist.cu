// dist.cu -- P > 1 ranks (one process per GPU of one node, or P handles on one device for the single-GPU emulation).
//
// Partitioning (PAPER.md:306-313 [3.1], 476-495 [3.4]; reading c.13):
//   * triples by relation: relations with count > N_t/P are SPLIT and their triples dealt round-robin per relation;
//     the rest go, by (count desc, id asc), to the currently lightest rank ("we sort the relations based on their
//     frequency ... greedily assign a relation to the partition with the smallest number of triplets so far").
//   * entity rows strided over the ranks ("strides them across all KVStore servers"): owner(e) =
//     e mod P, local row = e div P.
//   * relation rows replicated; a non-split relation is touched by its owner rank only (its rows "stay local and need
//     no communication", north_star); split relations are touched by every rank and their gradients summed in rank order.
// Exchange, fused into the kernels over peer memory (NVLink P2P through CUDA IPC mappings) instead of NCCL all-to-all:
//   * forward: k_gather / k_chain read an entity row straight from its owner's shard (EntRows accessor);
//   * gradient return: each rank writes one segment-summed gradient per unique entity it touched (Gu); after a device
//     barrier the owner pulls the gradients of its rows from every rank (k_owner_collect), sums them in rank order and
//     applies one Adagrad step per row (k_owner_update) -- the union-batch semantics of reading c.13;
//   * split relations: per-rank sums in GrelSplit, pulled and summed in rank order by every replica (k_split_rel);
//     TransR's projections M_r follow their relation: a non-split relation's M_r lives and is updated on its owner only
//     ("store all relation embeddings on GPUs and update relation embeddings in GPUs locally ... the
//     communication overhead drops from O(bd^2) to O(bd)"), a split relation's M_r is replicated and its rank sums are
//     exchanged like its row (GprojSplit).
// Device barriers (k_barrier: release/acquire flags at system scope in every peer) order the phases; a missing peer
// raises an error flag after KGE_OPT_BARRIER_MS instead of hanging.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "device_common.cuh"
#include "kge_internal.h"

namespace kge {

// ------------------------------------------------------------------------------------------------
// host: relation partition (reading c.13)
// ------------------------------------------------------------------------------------------------
// Philox4x32-10 on the host (the partition is computed by the host): the device helper's bijection
static uint32_t philox_host_x(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
  for (int round = 0; round < 10; ++round) {
    if (round) {
      k0 += kPhiloxW0;
      k1 += kPhiloxW1;
    }
    const uint64_t p0 = (uint64_t)kPhiloxM0 * c0, p1 = (uint64_t)kPhiloxM1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
    c0 = n0;
    c2 = n2;
  }
  return c0;
}

// randomise (reading c.13'): the non-split relations are ordered by (count desc, Philox(ctr = (r,
// epoch, 0, REPART), seed).x asc, id asc) -- a different greedy assignment every epoch, the SPLIT set unchanged
int32_t relation_partition(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, std::vector<int32_t>& owner,
                           bool randomise, uint64_t seed, uint32_t epoch) {
  std::vector<int64_t> cnt((size_t)nr, 0);
  for (int64_t i = 0; i < nt; ++i) cnt[(size_t)rels[i]]++;
  owner.assign((size_t)nr, 0);
  std::vector<int64_t> load((size_t)P, 0);
  std::vector<int64_t> rest;
  int32_t n_split = 0;
  for (int64_t r = 0; r < nr; ++r) {
    if (P > 1 && cnt[(size_t)r] * P > nt) {  // count > N_t / P, exact in integers
      owner[(size_t)r] = -1;
      ++n_split;
      for (int32_t w = 0; w < P; ++w) load[(size_t)w] += cnt[(size_t)r] / P + (w < cnt[(size_t)r] % P ? 1 : 0);
    } else {
      rest.push_back(r);
    }
  }
  std::vector<uint32_t> key(randomise ? (size_t)nr : 0);
  if (randomise)
    for (int64_t r : rest) key[(size_t)r] = philox_host_x((uint32_t)r, epoch, 0u, kTagRepart, (uint32_t)seed,
                                                          (uint32_t)(seed >> 32));
  std::stable_sort(rest.begin(), rest.end(), [&](int64_t a, int64_t b) {
    if (cnt[(size_t)a] != cnt[(size_t)b]) return cnt[(size_t)a] > cnt[(size_t)b];
    if (randomise && key[(size_t)a] != key[(size_t)b]) return key[(size_t)a] < key[(size_t)b];
    return a < b;
  });
  for (int64_t r : rest) {
    int32_t best = 0;
    for (int32_t w = 1; w < P; ++w)
      if (load[(size_t)w] < load[(size_t)best]) best = w;
    owner[(size_t)r] = best;
    load[(size_t)best] += cnt[(size_t)r];
  }
  return n_split;
}

int64_t rank_list(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, int32_t rank, const std::vector<int32_t>& owner,
                  std::vector<int32_t>* out) {
  std::vector<int64_t> dealt((size_t)nr, 0);
  int64_t n = 0;
  for (int64_t i = 0; i < nt; ++i) {
    const int64_t r = rels[i];
    int32_t o = owner[(size_t)r];
    if (o < 0) o = (int32_t)(dealt[(size_t)r]++ % P);
    if (o == rank) {
      if (out) out->push_back((int32_t)i);
      ++n;
    }
  }
  return n;
}

// ------------------------------------------------------------------------------------------------
// device: barrier, owner-side gradient collection and update, split relations
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

struct PeerFlags {
  uint64_t* f[kMaxRanks];  // rank q's flag array (P entries, one per writer)
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Device barrier of the P ranks. A rank that waits longer than timeout_ns (KGE_OPT_BARRIER_MS, default 2 min: a
// peer's host may be checkpointing or evaluating) leaves the spin and raises flags[1]; the next synchronising call
// reports it (KGE_ECUDA) -- a missing peer is an error, never a trapped context or an endless hang.
__global__ void k_barrier(PeerFlags pf, int P, int rank, uint64_t epoch, uint64_t timeout_ns, int32_t* flags) {
  const int q = threadIdx.x;
  if (q < P) {
    __threadfence_system();
    st_release_sys(pf.f[q] + rank, epoch);
  }
  __syncthreads();
  if (q < P) {
    const uint64_t t0 = globaltimer_ns();
    while (ld_acquire_sys(pf.f[rank] + q) < epoch) {
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicExch(flags + 1, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

struct OwnerArgs {
  Slot peer[kMaxRanks];         // every rank's sample slot of this step (peer pointers)
  const float* gu[kMaxRanks];   // every rank's per-unique gradient rows [n_occ x d]
  const int32_t* lossflag[kMaxRanks];  // every rank's flags array ([2 + step parity] = this step non-finite)
  int32_t P, rank, n_occ, d, par;  // par: this step's parity
  float lr, eps;
  int32_t* mark;     // [rows_local] slot of a touched local row, -1 otherwise
  int32_t* contrib;  // [P*n_occ x P] index of the row in rank w's unique list, -1 if absent
  int32_t* slot_row; // [P*n_occ] local row of a slot
  int32_t* n_slots;  // [1]
  float* ent;        // local shard
  float* ent_st;
};

// E1: every (rank w, unique index u) whose entity this rank owns claims a slot for its local row
__global__ void k_owner_collect(OwnerArgs a) {
  const int w = blockIdx.y;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.n_occ || u >= *a.peer[w].ent_n) return;
  const int32_t e = a.peer[w].ent_uniq[u];
  if (e % a.P != a.rank) return;
  const int32_t l = e / a.P;
  int32_t s = atomicCAS(a.mark + l, -1, -2);
  if (s == -1) {  // first claimant allocates the slot and publishes it
    s = atomicAdd(a.n_slots, 1);
    a.slot_row[s] = l;
    __threadfence();
    atomicExch(a.mark + l, s);
  } else {
    const long long t0 = clock64();
    while ((s = *(volatile int32_t*)(a.mark + l)) == -2) {
      if (clock64() - t0 > 4000000000ll) __trap();
    }
  }
  a.contrib[(int64_t)s * a.P + w] = u;
}

// E2: per claimed slot (warp): G = sum over ranks in rank order of their segment sums; one Adagrad step (c.11, c.13)
__global__ void __launch_bounds__(256) k_owner_update(OwnerArgs a) {
  const int lane = threadIdx.x & 31;
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= *a.n_slots) return;
  bool skip = false;  // a non-finite loss on any rank skips the step's update everywhere
  for (int w = 0; w < a.P; ++w) skip |= a.lossflag[w][2 + a.par] != 0;
  const int32_t l = a.slot_row[s];
  const int d = a.d, d4 = d >> 2;
  float* row = a.ent + (int64_t)l * d;
  if (!skip) {
    float4 g[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) g[m] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int w = 0; w < a.P; ++w) {
      const int32_t u = a.contrib[(int64_t)s * a.P + w];
      if (u < 0) continue;
      const float4* src = reinterpret_cast<const float4*>(a.gu[w] + (int64_t)u * d);
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        const int v = lane + 32 * m;
        if (v < d4) {
          const float4 x = src[v];
          g[m].x += x.x; g[m].y += x.y; g[m].z += x.z; g[m].w += x.w;
        }
      }
    }
    float sq = 0.f;
#pragma unroll
    for (int m = 0; m < 8; ++m)
      if (lane + 32 * m < d4) sq += g[m].x * g[m].x + g[m].y * g[m].y + g[m].z * g[m].z + g[m].w * g[m].w;
    sq = warp_sum(sq);
    const float st = a.ent_st[l] + sq / (float)d;
    if (lane == 0) a.ent_st[l] = st;
    const float step = a.lr / sqrtf(st + a.eps);
    float4* r4 = reinterpret_cast<float4*>(row);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int v = lane + 32 * m;
      if (v < d4) {
        float4 x = r4[v];
        x.x -= step * g[m].x; x.y -= step * g[m].y; x.z -= step * g[m].z; x.w -= step * g[m].w;
        r4[v] = x;
      }
    }
  }
  __syncwarp();
  if (lane < a.P) a.contrib[(int64_t)s * a.P + lane] = -1;
  if (lane == 0) a.mark[l] = -1;
}

struct SplitArgs {
  const float* gs[kMaxRanks];          // every rank's GrelSplit [n_split x drel]
  const int32_t* lossflag[kMaxRanks];
  const int32_t* split_list;           // [n_split] relation ids
  int32_t P, n_split, w, par;
  float lr, eps;
  float* rel;
  float* rel_st;
};

// split relations: every replica applies the same update from the rank-ordered sum (warp per relation)
__global__ void __launch_bounds__(256) k_split_rel(SplitArgs a) {
  const int lane = threadIdx.x & 31;
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (s >= a.n_split) return;
  for (int w = 0; w < a.P; ++w)
    if (a.lossflag[w][2 + a.par]) return;
  const int wd = a.w;
  float sq = 0.f;
  float* row = a.rel + (int64_t)a.split_list[s] * wd;
  // pass 1: squared norm of the summed gradient; pass 2: update (w <= 1024 floats; recompute the sums)
  for (int e = lane; e < wd; e += 32) {
    float g = 0.f;
    for (int q = 0; q < a.P; ++q) g += a.gs[q][(int64_t)s * wd + e];
    sq += g * g;
  }
  sq = warp_sum(sq);
  if (sq == 0.f) return;  // untouched this step on every rank: no update (exactly as the union step)
  const float st = a.rel_st[a.split_list[s]] + sq / (float)wd;
  const float step = a.lr / sqrtf(st + a.eps);
  for (int e = lane; e < wd; e += 32) {
    float g = 0.f;
    for (int q = 0; q < a.P; ++q) g += a.gs[q][(int64_t)s * wd + e];
    row[e] -= step * g;
  }
  if (lane == 0) a.rel_st[a.split_list[s]] = st;
}

struct PullArgs {
  const float* rel[kMaxRanks];
  const float* rel_st[kMaxRanks];
  const float* proj[kMaxRanks];
  const float* proj_st[kMaxRanks];
  const int32_t* owner_prev;  // [n_relations] owner in the epoch being left, -1 = split (replicas agree)
  int64_t nr;
  int32_t rank, drel, wproj;  // wproj: d*d (TransR) or 0
  float* rel_mine;
  float* rel_st_mine;
  float* proj_mine;
  float* proj_st_mine;
};

// epoch switch (repartition): copy every relation this rank did not own in the previous epoch from its owner (warp per
// relation: row, Adagrad state, TransR projection and its state)
__global__ void __launch_bounds__(256) k_pull_rel(PullArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= a.nr) return;
  const int o = a.owner_prev[r];
  if (o < 0 || o == a.rank) return;
  for (int e = lane; e < a.drel; e += 32) a.rel_mine[r * a.drel + e] = a.rel[o][r * a.drel + e];
  if (a.wproj)
    for (int64_t e = lane; e < a.wproj; e += 32) a.proj_mine[r * a.wproj + e] = a.proj[o][r * a.wproj + e];
  if (lane == 0) {
    a.rel_st_mine[r] = a.rel_st[o][r];
    if (a.wproj) a.proj_st_mine[r] = a.proj_st[o][r];
  }
}

cudaError_t dist_pull_relations(kge_handle* h, const int32_t* owner_prev) {
  PullArgs a{};
  for (int q = 0; q < h->P; ++q) {
    a.rel[q] = h->dist.peer_rel[q];
    a.rel_st[q] = h->dist.peer_rel_st[q];
    a.proj[q] = h->dist.peer_proj[q];
    a.proj_st[q] = h->dist.peer_proj_st[q];
  }
  a.owner_prev = owner_prev;
  a.nr = h->dims.n_relations;
  a.rank = h->rank;
  a.drel = h->dims.drel;
  a.wproj = h->proj ? h->dims.d * h->dims.d : 0;
  a.rel_mine = h->rel;
  a.rel_st_mine = h->rel_st;
  a.proj_mine = h->proj;
  a.proj_st_mine = h->proj_st;
  k_pull_rel<<<(unsigned)((a.nr + 7) / 8), 256, 0, h->stream>>>(a);
  ++h->launches;
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------
// host orchestration
// ------------------------------------------------------------------------------------------------
static PeerFlags peer_flags(const kge_handle* h) {
  PeerFlags pf{};
  for (int q = 0; q < h->P; ++q) pf.f[q] = h->dist.peer_flags[q];
  return pf;
}

cudaError_t dist_preload() {  // see step_preload (lazy loading vs spinning barriers)
  cudaFuncAttributes at;
  cudaError_t e = cudaFuncGetAttributes(&at, (const void*)k_barrier);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void*)k_owner_collect);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void*)k_owner_update);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void*)k_split_rel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&at, (const void*)k_pull_rel);
  return e;
}

// Barrier sequence `seq` (0: the step's main-stream barriers; 1: the lag = 1 update stream's) on stream st: each
// sequence has its own per-writer epoch slots in every rank's flag block and its own epoch counter.
static cudaError_t barrier_on(kge_handle* h, cudaStream_t st, int seq) {
  uint64_t& ep = seq == 0 ? h->dist.epoch : h->dist.epoch_u;
  ++ep;
  PeerFlags pf = peer_flags(h);
  for (int q = 0; q < h->P; ++q) pf.f[q] += seq * kMaxRanks;
  k_barrier<<<1, 32, 0, st>>>(pf, h->P, h->rank, ep, (uint64_t)h->barrier_ns, h->buf.flags);
  ++h->launches;
  return cudaGetLastError();
}

cudaError_t dist_barrier(kge_handle* h) { return barrier_on(h, h->stream, 0); }

// Slot with every pointer moved from my shared block to rank q's mapping of the same layout
static Slot peer_slot(const kge_handle* h, const Slot& mine, int q) {
  const char* base = (const char*)h->dist.shared;
  const char* pb = (const char*)h->dist.peer_shared[q];
  Slot s = mine;
  int32_t** f = reinterpret_cast<int32_t**>(&s);
  for (size_t i = 0; i < sizeof(Slot) / sizeof(int32_t*); ++i) f[i] = (int32_t*)(pb + ((const char*)f[i] - base));
  return s;
}

template <typename T>
static T* peer_ptr(const kge_handle* h, T* mine, int q) {  // the same object in rank q's shared block
  return (T*)((const char*)h->dist.peer_shared[q] + ((const char*)mine - (const char*)h->dist.shared));
}

cudaError_t dist_clear_split(kge_handle* h) {
  const Dist& D = h->dist;
  if (D.n_split == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(D.grel_split, 0, (size_t)D.n_split * h->dims.drel * 4, h->stream);
  if (e == cudaSuccess && D.gproj_split)
    e = cudaMemsetAsync(D.gproj_split, 0, (size_t)D.n_split * h->dims.d * h->dims.d * 4, h->stream);
  return e;
}

// Owner side of the entity exchange for step `step` on stream st: pull every rank's per-unique gradient sums of the
// rows this rank owns (gu: this rank's buffer of that step; peers' at the same offset), sum in rank order, one Adagrad
// step per row (reading c.13).
static cudaError_t owner_update(kge_handle* h, const Slot& s, int64_t step, float* gu, cudaStream_t st) {
  const Dims& dm = h->dims;
  Dist& D = h->dist;
  OwnerArgs oa{};
  for (int q = 0; q < h->P; ++q) {
    oa.peer[q] = peer_slot(h, s, q);
    oa.gu[q] = peer_ptr(h, gu, q);
    oa.lossflag[q] = peer_ptr(h, h->buf.flags, q);
  }
  oa.P = h->P;
  oa.rank = h->rank;
  oa.n_occ = dm.n_occ;
  oa.d = dm.d;
  oa.par = (int32_t)(step & 1);
  oa.lr = dm.lr;
  oa.eps = dm.eps;
  oa.mark = D.mark;
  oa.contrib = D.contrib;
  oa.slot_row = D.slot_row;
  oa.n_slots = D.n_slots;
  oa.ent = h->ent;
  oa.ent_st = h->ent_st;
  cudaError_t e = cudaMemsetAsync(D.n_slots, 0, 4, st);
  if (e != cudaSuccess) return e;
  k_owner_collect<<<dim3((dm.n_occ + 255) / 256, h->P), 256, 0, st>>>(oa);
  const int max_slots = h->P * dm.n_occ;
  k_owner_update<<<(max_slots + 7) / 8, 256, 0, st>>>(oa);
  h->launches += 2;
  return cudaGetLastError();
}

// split relations (and TransR's split projections): every replica applies the rank-ordered sum
static cudaError_t split_update(kge_handle* h, int64_t step) {
  const Dims& dm = h->dims;
  Dist& D = h->dist;
  if (D.n_split == 0) return cudaSuccess;
  SplitArgs sa{};
  for (int q = 0; q < h->P; ++q) {
    sa.gs[q] = peer_ptr(h, D.grel_split, q);
    sa.lossflag[q] = peer_ptr(h, h->buf.flags, q);
  }
  sa.split_list = D.split_list;
  sa.P = h->P;
  sa.n_split = D.n_split;
  sa.w = dm.drel;
  sa.par = (int32_t)(step & 1);
  sa.lr = dm.lr;
  sa.eps = dm.eps;
  sa.rel = h->rel;
  sa.rel_st = h->rel_st;
  k_split_rel<<<(D.n_split + 7) / 8, 256, 0, h->stream>>>(sa);
  ++h->launches;
  if (D.gproj_split) {  // TransR: the split relations' projections M_r, replicated like their rows (w = d*d)
    for (int q = 0; q < h->P; ++q) sa.gs[q] = peer_ptr(h, D.gproj_split, q);
    sa.w = dm.d * dm.d;
    sa.rel = h->proj;
    sa.rel_st = h->proj_st;
    k_split_rel<<<(D.n_split + 7) / 8, 256, 0, h->stream>>>(sa);
    ++h->launches;
  }
  return cudaGetLastError();
}

// After this rank's step kernels (lag = 0): B2, then the owner update of this step and the split relations.
// lag = 1 (reading c.12 at P > 1): B2 and the split relations now (relations stay synchronous); the owner update of
// this step's entity rows is held back -- dist_owner_update_lagged runs it during the next step.
cudaError_t dist_exchange_update(kge_handle* h, const Slot& s, int64_t step) {
  cudaError_t e = dist_barrier(h);  // B2: every rank's Gu / GrelSplit / sample slot is complete
  if (e != cudaSuccess) return e;
  launch_begin(h, KGE_K_UPDATE);
  if (h->cfg.lag == 0) e = owner_update(h, s, step, h->dist.gu_buf[0], h->stream);
  if (e == cudaSuccess) e = split_update(h, step);
  launch_end(h, KGE_K_UPDATE);
  return e;
}

// lag = 1, P > 1: the held-back owner update of step `step` on the update stream, once every rank has finished
// reading entity rows for the step after it (barrier sequence 1 behind this rank's ev_eread): it overlaps the rest
// of that step's forward / backward, and the next step's B1 waits for it (ev_eupd).
cudaError_t dist_owner_update_lagged(kge_handle* h, const Slot& s, int64_t step, cudaStream_t st) {
  cudaError_t e = barrier_on(h, st, 1);
  if (e == cudaSuccess) e = owner_update(h, s, step, h->dist.gu_buf[step & 1], st);
  return e;
}

// kge_flush at P > 1 (collective): the held-back owner update on the main stream after a barrier
cudaError_t dist_owner_flush(kge_handle* h, const Slot& s, int64_t step) {
  cudaError_t e = dist_barrier(h);
  if (e == cudaSuccess) e = owner_update(h, s, step, h->dist.gu_buf[step & 1], h->stream);
  return e;
}

}  // namespace kge

using namespace kge;

extern "C" {

int kge_partition(const int64_t* rels, int64_t n_triples, int64_t n_relations, int32_t world_size, int32_t rank,
                  int32_t* owner_out, int64_t* list_out, int64_t* n_list) {
  if (!rels || n_triples <= 0 || n_relations <= 0 || world_size < 1 || rank < 0 || rank >= world_size) {
    set_error("bad partition arguments");
    return KGE_EINVAL;
  }
  for (int64_t i = 0; i < n_triples; ++i)
    if (rels[i] < 0 || rels[i] >= n_relations) {
      set_error("relation id out of range");
      return KGE_ERANGE;
    }
  std::vector<int32_t> owner;
  relation_partition(rels, n_triples, n_relations, world_size, owner);
  if (owner_out) std::copy(owner.begin(), owner.end(), owner_out);
  std::vector<int32_t> lst;
  const int64_t n = rank_list(rels, n_triples, n_relations, world_size, rank, owner, list_out ? &lst : nullptr);
  if (list_out) for (int64_t i = 0; i < n; ++i) list_out[i] = lst[(size_t)i];
  if (n_list) *n_list = n;
  return KGE_OK;
}

int kge_locality_order(const int64_t* heads, const int64_t* tails, int64_t n_triples, int64_t n_entities,
                       int32_t world_size, int64_t* new_id_out, int64_t* edge_cut_out) {
  if (!heads || !tails || !new_id_out || n_triples < 0 || n_entities <= 0 || world_size < 1 ||
      world_size > n_entities) {
    set_error("bad locality-order arguments");
    return KGE_EINVAL;
  }
  // CSR of the undirected entity graph, neighbours ascending and distinct (self-loops dropped)
  std::vector<int64_t> deg((size_t)n_entities + 1, 0);
  for (int64_t i = 0; i < n_triples; ++i) {
    if (heads[i] < 0 || heads[i] >= n_entities || tails[i] < 0 || tails[i] >= n_entities) {
      set_error("entity id out of range");
      return KGE_ERANGE;
    }
    if (heads[i] != tails[i]) {
      ++deg[(size_t)heads[i] + 1];
      ++deg[(size_t)tails[i] + 1];
    }
  }
  for (int64_t e = 0; e < n_entities; ++e) deg[(size_t)e + 1] += deg[(size_t)e];
  std::vector<int64_t> nb((size_t)deg[(size_t)n_entities]), fill(deg.begin(), deg.end() - 1);
  for (int64_t i = 0; i < n_triples; ++i)
    if (heads[i] != tails[i]) {
      nb[(size_t)fill[(size_t)heads[i]]++] = tails[i];
      nb[(size_t)fill[(size_t)tails[i]]++] = heads[i];
    }
  std::vector<int64_t> start((size_t)n_entities), stop((size_t)n_entities);
  for (int64_t e = 0; e < n_entities; ++e) {
    auto b = nb.begin() + deg[(size_t)e], en = nb.begin() + deg[(size_t)e + 1];
    std::sort(b, en);
    start[(size_t)e] = deg[(size_t)e];
    stop[(size_t)e] = deg[(size_t)e] + (std::unique(b, en) - b);
  }
  // grow part w to exactly its shard size ceil((N_e - w) / P) breadth-first
  const int32_t P = world_size;
  std::vector<int32_t> part((size_t)n_entities, -1);
  std::vector<int64_t> frontier;
  int64_t seed = 0;
  for (int32_t w = 0; w < P; ++w) {
    const int64_t want = (n_entities - w + P - 1) / P;
    int64_t got = 0;
    frontier.clear();
    size_t at = 0;
    while (got < want) {
      if (at == frontier.size()) {
        while (part[(size_t)seed] >= 0) ++seed;
        part[(size_t)seed] = w;
        ++got;
        frontier.push_back(seed);
        continue;
      }
      const int64_t v = frontier[at++];
      for (int64_t q = start[(size_t)v]; q < stop[(size_t)v] && got < want; ++q) {
        const int64_t u = nb[(size_t)q];
        if (part[(size_t)u] < 0) {
          part[(size_t)u] = w;
          ++got;
          frontier.push_back(u);
        }
      }
    }
  }
  std::vector<int64_t> next((size_t)P, 0);
  for (int64_t e = 0; e < n_entities; ++e) new_id_out[e] = (int64_t)P * next[(size_t)part[(size_t)e]]++ + part[(size_t)e];
  if (edge_cut_out) {
    int64_t cut = 0;
    for (int64_t i = 0; i < n_triples; ++i) cut += part[(size_t)heads[i]] != part[(size_t)tails[i]];
    *edge_cut_out = cut;
  }
  return KGE_OK;
}

int kge_export(kge_handle* h, void* blob, size_t* blob_bytes) {
  if (!h || !blob_bytes) { set_error("NULL argument"); return KGE_EINVAL; }
  if (h->P < 2) { set_error("kge_export needs world_size > 1"); return KGE_ESTATE; }
  // entity shard, shared block, relation table and states, TransR projections and states (non-TransR: the relation
  // table's handle again in slots 4 and 5, ignored by kge_connect)
  const size_t need = 6 * sizeof(cudaIpcMemHandle_t);
  if (!blob) { *blob_bytes = need; return KGE_OK; }
  if (*blob_bytes < need) { set_error("blob too small"); return KGE_EINVAL; }
  cudaIpcMemHandle_t hs[6];
  cudaError_t e = cudaIpcGetMemHandle(&hs[0], h->ent);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs[1], h->dist.shared);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs[2], h->rel);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs[3], h->rel_st);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs[4], h->proj ? h->proj : h->rel);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hs[5], h->proj_st ? h->proj_st : h->rel);
  if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
  std::memcpy(blob, hs, need);
  *blob_bytes = need;
  return KGE_OK;
}

static int finish_connect(kge_handle* h) {
  Dist& D = h->dist;
  for (int q = 0; q < h->P; ++q) {
    h->rows.base[q] = D.peer_ent[q];
    D.peer_flags[q] = (uint64_t*)D.peer_shared[q];  // flags live at offset 0 of the shared block
  }
  h->rows.P = h->P;
  D.connected = true;
  return KGE_OK;
}

int kge_connect(kge_handle* h, const void* blobs, int32_t world_size) {
  if (!h || !blobs) { set_error("NULL argument"); return KGE_EINVAL; }
  if (world_size != h->P) { set_error("world_size mismatch"); return KGE_EINVAL; }
  const cudaIpcMemHandle_t* hs = (const cudaIpcMemHandle_t*)blobs;
  Dist& D = h->dist;
  for (int q = 0; q < h->P; ++q) {
    if (q == h->rank) {
      D.peer_ent[q] = h->ent;
      D.peer_shared[q] = D.shared;
      D.peer_rel[q] = h->rel;
      D.peer_rel_st[q] = h->rel_st;
      D.peer_proj[q] = h->proj;
      D.peer_proj_st[q] = h->proj_st;
      continue;
    }
    void* p[6] = {};
    const int nh = h->proj ? 6 : 4;
    for (int k = 0; k < nh; ++k) {
      cudaError_t e = cudaIpcOpenMemHandle(&p[k], hs[6 * q + k], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
      D.ipc_opened.push_back(p[k]);
    }
    D.peer_ent[q] = (float*)p[0];
    D.peer_shared[q] = p[1];
    D.peer_rel[q] = (float*)p[2];
    D.peer_rel_st[q] = (float*)p[3];
    D.peer_proj[q] = (float*)p[4];
    D.peer_proj_st[q] = (float*)p[5];
  }
  return finish_connect(h);
}

int kge_connect_local(kge_handle** hs, int32_t P) {
  if (!hs || P < 2 || P > kMaxRanks) { set_error("bad arguments"); return KGE_EINVAL; }
  for (int w = 0; w < P; ++w) {
    if (!hs[w] || hs[w]->P != P || hs[w]->rank != w) { set_error("handles must be ranks 0..P-1 of one world"); return KGE_EINVAL; }
    if (hs[w]->device != hs[0]->device) { set_error("kge_connect_local needs all handles on one device"); return KGE_EINVAL; }
  }
  for (int w = 0; w < P; ++w) {
    for (int q = 0; q < P; ++q) {
      hs[w]->dist.peer_ent[q] = hs[q]->ent;
      hs[w]->dist.peer_shared[q] = hs[q]->dist.shared;
      hs[w]->dist.peer_rel[q] = hs[q]->rel;
      hs[w]->dist.peer_rel_st[q] = hs[q]->rel_st;
      hs[w]->dist.peer_proj[q] = hs[q]->proj;
      hs[w]->dist.peer_proj_st[q] = hs[q]->proj_st;
    }
    finish_connect(hs[w]);
  }
  return KGE_OK;
}

int kge_relation_owner(const kge_handle* h, int64_t relation) {
  if (!h || relation < 0 || relation >= h->dims.n_relations) return -2;
  if (h->P == 1) return 0;
  return h->dist.rel_owner[(size_t)relation];
}

}  // extern "C"
