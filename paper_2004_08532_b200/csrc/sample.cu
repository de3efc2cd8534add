// sample.cu -- step (1) of the mini-batch loop (Sec. 3.1) on the device:
//   positives by a keyed Feistel permutation per epoch (reading c.2), joint negatives (reading
//   c.3), head/tail schedule (reading c.4), and the dedup of the rows the step touches (sort + segment, reading c.5)
//   -- all integer work, bit-exact with the oracle. Plus the table-init (reading c.6) and id-conversion kernels.
//
// Design (B200): sampling depends only on (seed, step), so one launch samples a whole window of steps ahead of the
// compute (grid.x = steps, grid.y = {entity, relation} dedup). Each CTA sorts its step's (id<<32 | occurrence) keys
// with an in-shared-memory bitonic network (n <= 16384 keys, one CTA, no global atomics), then a block scan turns
// the sorted run boundaries into unique ids, inverse map and segment offsets.
#include <cstdio>

#include "device_common.cuh"
#include "kge_internal.h"

namespace kge {

constexpr int kSampleThreads = 1024;  // block size limit of k_sample (registers capped at 64 per thread)
// Block size of a launch: a step sampled alone (caller batches; it runs next to the step kernels of the main stream)
// uses 256 threads, so it fits on an SM beside them -- a 1024-thread block needs an SM's whole register file and
// waited for a completely idle SM; the ring launches (32 steps ahead on the side stream) keep 1024.
static int sample_block(int n_steps) { return n_steps == 1 ? 256 : kSampleThreads; }

struct SampleArgs {
  SampleParams p;
  uint32_t fe_half;
  const Slot* slots;  // device array [ring]
  int32_t ring;
  int32_t loss_ring;  // the handle's loss ring (Slot::info[1] = step % loss_ring)
  int64_t step0;
  uint64_t* trace;    // KGE_TRACE diagnostics or nullptr
  uint64_t loss_dst;  // device-visible host address for the loss of step0 (n_steps == 1), or 0
  uint32_t* ready;    // n_steps == 1: counter each of the two CTAs bumps (release) once its half of the slot is
                      // written (k_wait_ready on the main stream acquires it), or nullptr
};

__device__ __forceinline__ int block_exclusive_scan(int v, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int nw = blockDim.x >> 5;
    int t = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) warp_tot[lane] = t;  // inclusive
    if (lane == 31) *total = t;
  }
  __syncthreads();
  const int base = wid ? warp_tot[wid - 1] : 0;
  return base + x - v;
}

__global__ void __launch_bounds__(kSampleThreads) k_sample(SampleArgs a) {
  extern __shared__ unsigned long long keys[];
  __shared__ int warp_tot[32];
  __shared__ int total;
  trace_stamp(a.trace, KGE_K_SAMPLE, 0);
  pdl_wait();  // the ring slots it overwrites may still be read by the previous step's kernels
  pdl_trigger();
  const SampleParams& p = a.p;
  const int64_t s = a.step0 + blockIdx.x;
  const Slot slot = a.slots[s % a.ring];
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    slot.info[0] = (int32_t)(uint32_t)s;
    slot.info[1] = (int32_t)(s % a.loss_ring);
    slot.info[2] = (int32_t)(uint32_t)a.loss_dst;
    slot.info[3] = (int32_t)(uint32_t)(a.loss_dst >> 32);
  }
  const bool ent_side = blockIdx.y == 0;
  const int tid = threadIdx.x;
  const int n = ent_side ? p.n_occ : p.B;
  const FeistelDomain dom{a.fe_half, (uint64_t)p.n_list};

  for (int i = tid; i < p.B; i += blockDim.x) {
    int32_t trip = -1, hv, rv, tv;
    if (p.given_h) {
      hv = p.given_h[i];
      rv = p.given_r[i];
      tv = p.given_t[i];
    } else {
      uint64_t q = (uint64_t)s * (uint64_t)p.B + (uint64_t)i;
      uint32_t epoch = (uint32_t)(q / (uint64_t)p.n_list);
      if (p.epoch_steps > 0) {  // repartition (reading c.13'): epoch e = s / S_E, the position within it
        const int64_t e = s / p.epoch_steps;
        epoch = (uint32_t)e;
        q = (uint64_t)(s - e * p.epoch_steps) * (uint64_t)p.B + (uint64_t)i;
      }
      const uint64_t pp = q % (uint64_t)p.n_list;
      const uint64_t idx = feistel_index(dom, p.k0, p.k1, epoch, pp);
      trip = p.list ? p.list[idx] : (int32_t)idx;
      hv = p.th[trip];
      rv = p.tr[trip];
      tv = p.tt[trip];
    }
    if (ent_side) {
      slot.pos[i] = trip;
      slot.ph[i] = hv;
      slot.pr[i] = rv;
      slot.pt[i] = tv;
      keys[i] = ((unsigned long long)(uint32_t)hv << 32) | (uint32_t)i;
      keys[p.B + i] = ((unsigned long long)(uint32_t)tv << 32) | (uint32_t)(p.B + i);
    } else {
      keys[i] = ((unsigned long long)(uint32_t)rv << 32) | (uint32_t)i;
    }
  }
  __syncthreads();  // the batch's heads / tails (slot.ph / pt) are complete for the in-batch negatives
  if (ent_side) {
    const int nneg = p.C * p.k;
    for (int q = tid; q < nneg; q += blockDim.x) {
      const int c = q / p.k, j = q - c * p.k;
      uint32_t id;
      if (j < p.kd) {  // degree-based in-batch slot: the drawn triplet's tail (tail mode) / head (head mode)
        const uint32_t t = deg_position(p.k0, p.k1, (uint32_t)p.B, (uint32_t)s, p.cg_base + c, (uint32_t)j);
        id = (uint32_t)(corrupt_mode(p.corrupt, (uint32_t)s, p.cg_base + c) == 0 ? slot.pt[t] : slot.ph[t]);
      } else if (p.local_P > 1) {  // local-shard negatives: rank w's shard {w + P m}
        const uint64_t n_w = (uint64_t)((p.n_entities - p.local_rank + p.local_P - 1) / p.local_P);
        id = (uint32_t)p.local_rank +
             (uint32_t)p.local_P * neg_entity(p.k0, p.k1, n_w, (uint32_t)s, p.cg_base + c, (uint32_t)j);
      } else {
        id = neg_entity(p.k0, p.k1, (uint64_t)p.n_entities, (uint32_t)s, p.cg_base + c, (uint32_t)j);
      }
      slot.neg[q] = (int32_t)id;
      keys[2 * p.B + q] = ((unsigned long long)id << 32) | (uint32_t)(2 * p.B + q);
    }
    for (int c = tid; c < p.C; c += blockDim.x) slot.mode[c] = corrupt_mode(p.corrupt, (uint32_t)s, p.cg_base + c);
  }
  // pad to a power of two
  int np2 = 64;  // >= one 64-key block of the warp-level stages (n_pad >= 64 on the host)
  while (np2 < n) np2 <<= 1;
  for (int q = n + tid; q < np2; q += blockDim.x) keys[q] = ~0ull;
  __syncthreads();
  trace_stamp(a.trace, KGE_K_SAMPLE, 1);

  // bitonic sort, ascending. Stages with distance j >= 32 exchange through shared memory (one barrier each); the
  // j < 32 stages of each merge run warp-synchronously on 64-key blocks held 2 per lane (no block barrier).
  const int lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int kk = 2; kk <= np2; kk <<= 1) {
    int j = kk >> 1;
    for (; j >= 32; j >>= 1) {
      const int lj = __ffs(j) - 1;
      for (int t = tid; t < (np2 >> 1); t += blockDim.x) {
        const int lo = ((t >> lj) << (lj + 1)) | (t & (j - 1));
        const int hi = lo + j;
        const bool up = (lo & kk) == 0;
        const unsigned long long x = keys[lo], y = keys[hi];
        if ((x > y) == up) {
          keys[lo] = y;
          keys[hi] = x;
        }
      }
      __syncthreads();
    }
    // remaining stages j = min(kk/2, 16) .. 1 stay inside aligned 64-key blocks: lane holds keys b+lane, b+lane+32
    for (int b = wid * 64; b < np2; b += nw * 64) {
      unsigned long long k0 = keys[b + lane], k1 = keys[b + lane + 32];
      const bool up = ((b + lane) & kk) == 0;  // direction of this kk-block (kk >= 64: same for the whole 64-block)
      for (int jj = j; jj > 0; jj >>= 1) {
        // element index e = b + lane (+32); partner e ^ jj lies in the same 32-half for jj <= 16
        const unsigned long long p0 = __shfl_xor_sync(0xffffffffu, k0, jj);
        const unsigned long long p1 = __shfl_xor_sync(0xffffffffu, k1, jj);
        const bool low = (lane & jj) == 0;
        const bool up0 = kk >= 64 ? up : (((b + lane) & kk) == 0);
        const bool up1 = kk >= 64 ? up : (((b + lane + 32) & kk) == 0);
        // keep min if (low == up) else max
        k0 = (low == up0) ? (p0 < k0 ? p0 : k0) : (p0 > k0 ? p0 : k0);
        k1 = (low == up1) ? (p1 < k1 ? p1 : k1) : (p1 > k1 ? p1 : k1);
      }
      keys[b + lane] = k0;
      keys[b + lane + 32] = k1;
    }
    __syncthreads();
  }

  trace_stamp(a.trace, KGE_K_SAMPLE, 2);
  // run boundaries -> unique ids, inverse map, segments (reading c.5)
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
  int cnt = 0;
  for (int q = b0; q < b1; ++q)
    if (q == 0 || (keys[q] >> 32) != (keys[q - 1] >> 32)) ++cnt;
  int uid = block_exclusive_scan(cnt, warp_tot, &total) - 1;
  int32_t* uniq = ent_side ? slot.ent_uniq : slot.rel_uniq;
  int32_t* inv = ent_side ? slot.ent_inv : slot.rel_inv;
  int32_t* off = ent_side ? slot.ent_off : slot.rel_off;
  int32_t* occ = ent_side ? slot.ent_occ : slot.rel_occ;
  for (int q = b0; q < b1; ++q) {
    const unsigned long long kv = keys[q];
    if (q == 0 || (kv >> 32) != (keys[q - 1] >> 32)) {
      ++uid;
      uniq[uid] = (int32_t)(kv >> 32);
      off[uid] = q;
    }
    const int32_t o = (int32_t)(kv & 0xffffffffu);
    occ[q] = o;
    inv[o] = uid;
  }
  if (tid == 0) {
    off[total] = n;
    if (ent_side)
      *slot.ent_n = total;
    else
      *slot.rel_n = total;
  }
  if (a.ready) {  // publish: every thread's slot writes, then one fenced increment per CTA
    __syncthreads();
    if (tid == 0) flow_release(a.ready, 1u);
  }
  trace_stamp(a.trace, KGE_K_SAMPLE, 7);
}

// Main-stream gate of a caller batch whose sample runs on a side stream (kge_train_batch): spins until the slot's
// counter reaches `want` (both k_sample CTAs published), then waits for its own stream predecessor, so the step's
// kernels that follow by PDL see the sample and the previous step complete. One CTA: the side-stream sampler always
// finds an SM. Times out after timeout_ns (flags[1] = 2: reported by the next flag check) instead of hanging.
__global__ void k_wait_ready(const uint32_t* ready, uint32_t want, uint64_t timeout_ns, int32_t* flags) {
  pdl_trigger();
  if (threadIdx.x == 0) {
    uint64_t t0 = 0;
    for (int it = 0;; ++it) {
      uint32_t v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready) : "memory");
      if ((int32_t)(v - want) >= 0) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (it == 0) t0 = t;
      else if (t - t0 > timeout_ns) { atomicExch(flags + 1, 2); break; }
      __nanosleep(32);
    }
  }
  __syncthreads();
  pdl_wait();
}

cudaError_t launch_wait_ready(kge_handle* h, const uint32_t* ready, uint32_t want) {
  return launch_pdl(k_wait_ready, dim3(1), dim3(32), 0, h->stream, ready, want, (uint64_t)5000000000ull, h->buf.flags);
}

size_t sample_smem_bytes(int n_pad) { return (size_t)n_pad * sizeof(unsigned long long); }

cudaError_t sample_init() {
  return cudaFuncSetAttribute(k_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

cudaError_t launch_sample(kge_handle* h, const SampleParams& p, const Slot* slots_dev, int ring, int64_t step0, int n_steps,
                          cudaStream_t stream, uint64_t loss_dst, uint32_t* ready) {
  SampleArgs a;
  a.p = p;
  a.fe_half = make_feistel_domain((uint64_t)p.n_list).half;
  a.slots = slots_dev;
  a.ring = ring;
  a.loss_ring = h->ring;
  a.step0 = step0;
  a.trace = h->dims.trace;
  a.loss_dst = loss_dst;
  a.ready = ready;
  size_t smem = sample_smem_bytes(p.n_pad);  // opt-in raised once by sample_init (never in the step path: the call
                                              // may synchronise, which would stall the multi-rank emulation)
  cudaStream_t main = h->stream;
  if (stream) h->stream = stream;  // the profiler brackets the launch on the stream it runs on
  launch_begin(h, KGE_K_SAMPLE);
  k_sample<<<dim3(n_steps, 2), sample_block(n_steps), smem, h->stream>>>(a);
  launch_end(h, KGE_K_SAMPLE);
  h->stream = main;
  return cudaGetLastError();
}

cudaError_t sample_graph_set(kge_handle* h, cudaGraphExec_t exec, cudaGraphNode_t node, const SampleParams& p,
                             const Slot* slots_dev, int ring, int64_t step0, int n_steps, uint64_t loss_dst,
                             uint32_t* ready) {
  SampleArgs a;
  a.p = p;
  a.fe_half = make_feistel_domain((uint64_t)p.n_list).half;
  a.slots = slots_dev;
  a.ring = ring;
  a.loss_ring = h->ring;
  a.step0 = step0;
  a.trace = h->dims.trace;
  a.loss_dst = loss_dst;
  a.ready = ready;
  void* args[] = {&a};
  cudaKernelNodeParams kp = {};
  kp.func = (void*)k_sample;
  kp.gridDim = dim3(n_steps, 2);
  kp.blockDim = dim3(sample_block(n_steps));
  kp.sharedMemBytes = (unsigned)sample_smem_bytes(p.n_pad);
  kp.kernelParams = args;
  return cudaGraphExecKernelNodeSetParams(exec, node, &kp);
}

// ---- table init (reading c.6) ----
// local row l holds global row l * row_stride + row_offset (entity shards: stride P, offset rank)
__global__ void k_init_table(float* __restrict__ tab, int64_t n_elem, int32_t w, uint32_t k0, uint32_t k1,
                             uint32_t table_id, float bound, int64_t row_stride, int64_t row_offset) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_elem; i += stride) {
    const int64_t lrow = i / w;
    const uint32_t col = (uint32_t)(i - lrow * w);
    tab[i] = init_value(k0, k1, table_id, (uint64_t)(lrow * row_stride + row_offset), col, bound);
  }
}

cudaError_t launch_init_table(kge_handle* h, float* tab, int64_t rows, int32_t w, uint32_t table_id, float bound,
                              int64_t row_stride, int64_t row_offset) {
  const int64_t n = rows * (int64_t)w;
  if (n == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 64);
  k_init_table<<<blocks, 256, 0, h->stream>>>(tab, n, w, h->k0, h->k1, table_id, bound, row_stride, row_offset);
  ++h->launches;
  return cudaGetLastError();
}

__global__ void k_convert_ids(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t n, int64_t limit,
                              int32_t* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t v = src[i];
    if (v < 0 || v >= limit) {
      atomicOr(bad, 1);
      dst[i] = 0;
    } else {
      dst[i] = (int32_t)v;
    }
  }
}

cudaError_t launch_convert_ids(kge_handle* h, const int64_t* src, int32_t* dst, int64_t n, int64_t limit, int32_t* bad) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 32);
  k_convert_ids<<<blocks, 256, 0, h->stream>>>(src, dst, n, limit, bad);
  ++h->launches;
  return cudaGetLastError();
}

}  // namespace kge
