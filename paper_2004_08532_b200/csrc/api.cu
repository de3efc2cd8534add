// api.cu -- the C-ABI of include/kge.h: validation, device memory, table init, the step loop and diagnostics.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <functional>
#include <vector>

#include "device_common.cuh"
#include "kge_internal.h"

namespace kge {

static thread_local std::string g_err;
bool g_pdl = true;

void set_error(const std::string& msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return KGE_ECUDA;
}

void launch_begin(kge_handle* h, int kid) {
  ++h->launches;
  if (!h->prof.on) return;
  if (h->prof.used + 2 > h->prof.ev.size()) {
    h->prof.ev.push_back(nullptr);
    h->prof.ev.push_back(nullptr);
    cudaEventCreate(&h->prof.ev[h->prof.ev.size() - 2]);
    cudaEventCreate(&h->prof.ev[h->prof.ev.size() - 1]);
  }
  cudaEventRecord(h->prof.ev[h->prof.used], h->stream);
  h->prof.kid.push_back(kid);
}

void launch_end(kge_handle* h, int kid) {
  static const bool dbg = getenv("KGE_DEBUG_SYNC") != nullptr;
  if (dbg) {
    cudaError_t e = cudaStreamSynchronize(h->stream);
    fprintf(stderr, "[kge] %s -> %s\n", kge_kernel_name(kid), cudaGetErrorString(e));
  }
  if (!h->prof.on) return;
  cudaEventRecord(h->prof.ev[h->prof.used + 1], h->stream);
  h->prof.used += 2;
}

static void* dalloc(kge_handle* h, size_t bytes) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);
  void* p = nullptr;
  if (h->cfg.dev_alloc) {
    p = h->cfg.dev_alloc(bytes, h->cfg.alloc_ctx);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    p = nullptr;
  }
  if (p) h->allocs.push_back(p);
  return p;
}

static void free_all(kge_handle* h) {
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) {
    if (h->cfg.dev_free)
      h->cfg.dev_free(p, h->cfg.alloc_ctx);
    else
      cudaFree(p);
  }
  h->allocs.clear();
}

#define CK(expr)                                         \
  do {                                                   \
    cudaError_t e_ = (expr);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #expr); \
  } while (0)

static float default_bound(float gamma, int dim) {
  if (gamma > 0.f) {
    volatile float num = gamma + 2.0f;
    volatile float v = num / (float)dim;
    return v;
  }
  volatile float sd = std::sqrt((float)dim);
  volatile float v = 1.0f / sd;
  return v;
}

static int validate(const kge_config* c) {
  if (!c) { set_error("cfg is NULL"); return KGE_EINVAL; }
  if (c->abi_version != KGE_ABI_VERSION) { set_error("abi_version mismatch"); return KGE_EINVAL; }
  if (c->model < 0 || c->model > KGE_RESCAL) { set_error("unknown model"); return KGE_EINVAL; }
  if (c->model == KGE_RESCAL && (c->neg_precision == KGE_PREC_BF16 || c->neg_precision == KGE_PREC_3XTF32 ||
                                  c->lag == 1)) {
    set_error("RESCAL: BF16 / 3xTF32 negatives and lag = 1 are not implemented");
    return KGE_EUNSUPPORTED;
  }
  if (c->dim <= 0 || c->dim % 4 != 0) { set_error("dim must be a positive multiple of 4"); return KGE_EINVAL; }
  if ((c->model == KGE_COMPLEX || c->model == KGE_ROTATE) && c->dim % 8 != 0) {
    set_error("ComplEx/RotatE need dim % 8 == 0 (d/2 complex coordinates, float4 halves)");
    return KGE_EINVAL;
  }
  if (c->dim > 1024) { set_error("dim > 1024 not supported"); return KGE_EINVAL; }
  if (c->batch_size <= 0 || c->chunk_size <= 0 || c->batch_size % c->chunk_size != 0) {
    set_error("chunk_size must divide batch_size (SPEC.md:209)");
    return KGE_EINVAL;
  }
  if (c->neg_k <= 0) { set_error("neg_k must be > 0"); return KGE_EINVAL; }
  const int64_t n_occ = 2 * (int64_t)c->batch_size + (int64_t)(c->batch_size / c->chunk_size) * c->neg_k;
  if (n_occ > 16384) { set_error("2B + (B/g)k must be <= 16384 (single-CTA dedup)"); return KGE_EINVAL; }
  if (c->n_entities <= 0 || c->n_relations <= 0) { set_error("empty vocabulary"); return KGE_EINVAL; }
  if (c->n_entities >= (1ll << 31) || c->n_relations >= (1ll << 31)) {
    set_error("n_entities / n_relations must be < 2^31");
    return KGE_ERANGE;
  }
  if (c->corrupt < 0 || c->corrupt > 2) { set_error("bad corrupt"); return KGE_EINVAL; }
  if (c->neg_precision < 0 || c->neg_precision > 3) { set_error("bad neg_precision"); return KGE_EINVAL; }
  if ((c->neg_precision == KGE_PREC_BF16 || c->neg_precision == KGE_PREC_3XTF32) && c->model == KGE_TRANSR) {
    set_error("BF16 / 3xTF32 negatives are not implemented for TransR (use TF32)");
    return KGE_EUNSUPPORTED;
  }
  if (c->lag != 0 && c->lag != 1) { set_error("lag must be 0 or 1"); return KGE_EINVAL; }
  if (c->neg_deg_k < 0 || c->neg_deg_k > c->neg_k) { set_error("neg_deg_k must be in [0, neg_k]"); return KGE_EINVAL; }
  if (c->neg_local != 0 && c->neg_local != 1) { set_error("neg_local must be 0 or 1"); return KGE_EINVAL; }
  if (c->loss != KGE_LOSS_LOGISTIC && c->loss != KGE_LOSS_PAIRWISE) { set_error("bad loss"); return KGE_EINVAL; }
  if (c->repartition != 0 && c->repartition != 1) { set_error("repartition must be 0 or 1"); return KGE_EINVAL; }
  if (c->placement != 0 && c->placement != 1) { set_error("placement must be 0 or 1"); return KGE_EINVAL; }
  if (c->placement == 1 && c->repartition) { set_error("placement = 1 replaces the relation partition (repartition = 0)"); return KGE_EINVAL; }
  if (c->neg_local && c->world_size > 1 && c->n_entities < c->world_size) {
    set_error("neg_local needs n_entities >= world_size (every shard non-empty)");
    return KGE_EINVAL;
  }
  if (c->lag == 1 && c->model == KGE_TRANSR) {
    set_error("lag = 1 is implemented for the non-TransR models");
    return KGE_EUNSUPPORTED;
  }
  if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size) { set_error("bad world_size/rank"); return KGE_EINVAL; }
  if (c->world_size > kMaxRanks) { set_error("world_size > 8 (one node) not supported"); return KGE_EINVAL; }
  if ((c->model == KGE_TRANSR || c->model == KGE_RESCAL) && c->dim > 512) {
    set_error("TransR / RESCAL support dim <= 512");
    return KGE_EINVAL;
  }
  return KGE_OK;
}

static size_t slot_ints(const Dims& d) {
  const size_t n_occ = d.n_occ, B = d.B;
  size_t n = B * 4 + (size_t)d.C * d.k + d.C + 1 + n_occ * 3 + (n_occ + 1) + 1 + B * 3 + (B + 1) + 4;
  return (n + 63) & ~size_t(63);  // 256-byte aligned slots
}

static void* rawalloc(kge_handle* h, size_t bytes) {  // plain cudaMalloc: IPC-exportable (P > 1)
  void* p = nullptr;
  if (cudaMalloc(&p, (bytes + 255) & ~size_t(255)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  h->dist.raw_allocs.push_back(p);
  return p;
}

static int carve_slot(kge_handle* h, int32_t* p, Slot& s) {
  const Dims& d = h->dims;
  const int n_occ = d.n_occ, B = d.B;
  s.pos = p; p += B;
  s.ph = p; p += B;
  s.pr = p; p += B;
  s.pt = p; p += B;
  s.neg = p; p += (size_t)d.C * d.k;
  s.mode = p; p += d.C;
  s.ent_n = p; p += 1;
  s.ent_uniq = p; p += n_occ;
  s.ent_inv = p; p += n_occ;
  s.ent_off = p; p += n_occ + 1;
  s.ent_occ = p; p += n_occ;
  s.rel_n = p; p += 1;
  s.rel_uniq = p; p += B;
  s.rel_inv = p; p += B;
  s.rel_off = p; p += B + 1;
  s.rel_occ = p; p += B;
  s.info = p; p += 4;
  return KGE_OK;
}

static SampleParams sample_params(const kge_handle* h, bool given, int gi = 0) {
  SampleParams p{};
  p.th = h->th;
  p.tr = h->tr;
  p.tt = h->tt;
  p.list = h->list;
  p.n_list = h->n_list;
  if (given) {
    const int32_t* gb = h->given + (size_t)gi * 3 * h->dims.B;
    p.given_h = gb;
    p.given_r = gb + h->dims.B;
    p.given_t = gb + 2 * h->dims.B;
  }
  p.n_entities = h->dims.n_entities;
  p.B = h->dims.B;
  p.g = h->dims.g;
  p.C = h->dims.C;
  p.k = h->dims.k;
  p.n_occ = h->dims.n_occ;
  p.n_pad = h->n_pad;
  p.k0 = h->k0;
  p.k1 = h->k1;
  p.corrupt = h->cfg.corrupt;
  p.cg_base = (uint32_t)(h->cfg.rank * h->dims.C);
  p.kd = h->cfg.neg_deg_k;
  p.local_P = h->cfg.neg_local && h->P > 1 ? h->P : 0;
  p.local_rank = h->rank;
  p.epoch_steps = h->epoch_steps;  // repartition: epochs of a fixed step count, the list is this epoch's
  return p;
}

// device copy of the slot table: stored right after flags[4] in the same allocation (see kge_init)
static Slot* d_slots(kge_handle* h) { return reinterpret_cast<Slot*>(h->buf.flags + 4); }

}  // namespace kge

using namespace kge;

extern "C" {

void kge_config_default(kge_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->abi_version = KGE_ABI_VERSION;
  c->model = KGE_TRANSE_L2;
  c->n_entities = 0;
  c->n_relations = 0;
  c->dim = 400;
  c->batch_size = 1024;
  c->chunk_size = 256;
  c->neg_k = 256;
  c->gamma = 12.0f;
  c->lr = 0.1f;
  c->adagrad_eps = 1e-10f;
  c->init_bound = 0.0f;
  c->seed = 1;
  c->corrupt = KGE_CORRUPT_ALTERNATE;
  c->neg_precision = KGE_PREC_TF32;
  c->rotate_variant = 0;
  c->lag = 0;
  c->neg_deg_k = 0;
  c->neg_local = 0;
  c->loss = KGE_LOSS_LOGISTIC;
  c->repartition = 0;
  c->placement = 0;
  c->world_size = 1;
  c->rank = 0;
}

const char* kge_last_error(void) { return g_err.c_str(); }

const char* kge_kernel_name(int32_t id) {
  static const char* names[] = {"k_sample", "k_gather", "k_neg_fwd", "k_neg_bwd", "k_chain", "k_update"};
  return (id >= 0 && id < KGE_K_COUNT) ? names[id] : "?";
}

int kge_init(kge_handle** out, const kge_config* cfg, const int64_t* heads, const int64_t* rels, const int64_t* tails,
             int64_t n_triples) {
  if (!out) { set_error("out is NULL"); return KGE_EINVAL; }
  *out = nullptr;
  int rc = validate(cfg);
  if (rc != KGE_OK) return rc;
  if (!heads || !rels || !tails || n_triples <= 0) { set_error("no triples"); return KGE_EINVAL; }
  if (n_triples >= (1ll << 31)) { set_error("n_triples must be < 2^31"); return KGE_ERANGE; }
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error("no CUDA device (this library has no CPU fallback)");
    return KGE_ECUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, dev);
  if (prop.major != 10) {
    set_error("libkge.so is built for sm_100a (B200); device is sm_" + std::to_string(prop.major * 10 + prop.minor));
    return KGE_ECUDA;
  }

  kge_handle* h = new kge_handle();
  h->cfg = *cfg;
  if (h->cfg.adagrad_eps <= 0.f) h->cfg.adagrad_eps = 1e-10f;
  h->device = dev;
  Dims& dm = h->dims;
  dm.model = cfg->model;
  dm.variant = cfg->rotate_variant;
  dm.family = family_of(cfg->model, cfg->rotate_variant);
  dm.d = cfg->dim;
  dm.drel = cfg->model == KGE_ROTATE ? cfg->dim / 2 : cfg->dim;
  dm.B = cfg->batch_size;
  dm.g = cfg->chunk_size;
  dm.C = dm.B / dm.g;
  dm.k = cfg->neg_k;
  dm.n_occ = 2 * dm.B + dm.C * dm.k;
  dm.gamma = cfg->gamma;
  dm.loss = cfg->loss;
  dm.lr = cfg->lr;
  dm.eps = h->cfg.adagrad_eps;
  dm.n_entities = cfg->n_entities;
  dm.n_relations = cfg->n_relations;
  dm.trace = nullptr;
  h->k0 = (uint32_t)cfg->seed;
  h->k1 = (uint32_t)(cfg->seed >> 32);
  dm.dp = ((dm.d + 2 + 31) / 32) * 32;  // O / X' pitch: room for the ones columns at d, d+1 (tc.cu)
  dm.kp = ((dm.k + 31) / 32) * 32;     // W pitch: whole 32-float k-blocks (tc.cu 4D maps; the pad stays zero)
  dm.dp16 = ((dm.d + 63) / 64) * 64;   // BF16 copies: whole 64-element (128-byte) k-blocks
  dm.kp16 = ((dm.k + 63) / 64) * 64;
  dm.bf16 = cfg->neg_precision == KGE_PREC_BF16 ? 1 : 0;
  dm.x3 = cfg->neg_precision == KGE_PREC_3XTF32 ? 1 : 0;
  h->dp = dm.dp;
  h->kp = dm.kp;
  h->n_pad = 64;  // the sampler's warp-level sort stages work on 64-key blocks
  while (h->n_pad < dm.n_occ) h->n_pad <<= 1;
  h->ring = 64;
  h->n_triples = n_triples;

  auto fail = [&](int code) {
    free_all(h);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return code;
  };

  if (cfg->cuda_stream) {
    h->stream = (cudaStream_t)cfg->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) return fail(cuda_fail(cudaGetLastError(), "stream"));
    h->own_stream = true;
  }

  // ---- triples -> device int32 (checked) ----
  h->th = (int32_t*)dalloc(h, n_triples * 4);
  h->tr = (int32_t*)dalloc(h, n_triples * 4);
  h->tt = (int32_t*)dalloc(h, n_triples * 4);
  int32_t* d_bad = (int32_t*)dalloc(h, 16);
  if (!h->th || !h->tr || !h->tt || !d_bad) { set_error("out of device memory (triples)"); return fail(KGE_ENOMEM); }
  {
    const int64_t chunk = 1 << 24;  // 16M ids (128 MB) staging
    int64_t* stage = nullptr;
    int64_t* d_stage = (int64_t*)dalloc(h, (size_t)std::min(chunk, n_triples) * 8);
    if (!d_stage || cudaMallocHost(&stage, (size_t)std::min(chunk, n_triples) * 8) != cudaSuccess) {
      cudaGetLastError();
      set_error("staging allocation failed");
      return fail(KGE_ENOMEM);
    }
    if (cudaMemsetAsync(d_bad, 0, 16, h->stream) != cudaSuccess) { cudaFreeHost(stage); return fail(cuda_fail(cudaGetLastError(), "memset")); }
    const int64_t* srcs[3] = {heads, rels, tails};
    int32_t* dsts[3] = {h->th, h->tr, h->tt};
    const int64_t lim[3] = {cfg->n_entities, cfg->n_relations, cfg->n_entities};
    for (int a = 0; a < 3; ++a) {
      for (int64_t b = 0; b < n_triples; b += chunk) {
        const int64_t m = std::min(chunk, n_triples - b);
        cudaStreamSynchronize(h->stream);  // staging buffer reuse
        std::memcpy(stage, srcs[a] + b, (size_t)m * 8);
        e = cudaMemcpyAsync(d_stage, stage, (size_t)m * 8, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess) e = launch_convert_ids(h, d_stage, dsts[a] + b, m, lim[a], d_bad);
        if (e != cudaSuccess) { cudaFreeHost(stage); return fail(cuda_fail(e, "triple upload")); }
      }
    }
    int32_t bad = 0;
    e = cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFreeHost(stage);
    if (e != cudaSuccess) return fail(cuda_fail(e, "triple upload"));
    if (bad) { set_error("triple id out of range"); return fail(KGE_ERANGE); }
  }
  h->P = cfg->world_size;
  h->rank = cfg->rank;
  h->list = nullptr;  // P = 1: identity list
  h->n_list = n_triples;
  if (h->P > 1) {  // relation partition (reading c.13) -> this rank's triple list
    std::vector<int32_t> owner, lst;
    const bool rp = cfg->repartition != 0;
    if (cfg->placement == 1) {  // head-owner placement (reading c.13''): every relation replicated (SPLIT)
      owner.assign((size_t)cfg->n_relations, -1);
      for (int64_t i = 0; i < n_triples; ++i)
        if (heads[i] % h->P == h->rank) lst.push_back((int32_t)i);
    } else {
      relation_partition(rels, n_triples, cfg->n_relations, h->P, owner, rp, cfg->seed, 0);
      rank_list(rels, n_triples, cfg->n_relations, h->P, h->rank, owner, &lst);
    }
    if (lst.empty()) { set_error("this rank received no triples"); return fail(KGE_EINVAL); }
    // repartition: room for any epoch's list, the relation column kept on the host for the per-epoch partitions
    h->list = (int32_t*)dalloc(h, (rp ? (size_t)n_triples : lst.size()) * 4);
    if (rp) {
      h->host_rels.assign(rels, rels + n_triples);
      h->epoch_steps = (n_triples + (int64_t)h->P * dm.B - 1) / ((int64_t)h->P * dm.B);
      h->cur_epoch = 0;
      h->d_owner_prev = (int32_t*)dalloc(h, (size_t)cfg->n_relations * 4);
      if (!h->d_owner_prev) return fail(KGE_ENOMEM);
    }
    std::vector<int32_t> split_list, split_index((size_t)cfg->n_relations, -1);
    for (int64_t r = 0; r < cfg->n_relations; ++r)
      if (owner[(size_t)r] < 0) {
        split_index[(size_t)r] = (int32_t)split_list.size();
        split_list.push_back((int32_t)r);
      }
    h->dist.n_split = (int32_t)split_list.size();
    h->dist.split_list = (int32_t*)dalloc(h, std::max<size_t>(1, split_list.size()) * 4);
    h->dist.split_index = (int32_t*)dalloc(h, (size_t)cfg->n_relations * 4);
    if (!h->list || !h->dist.split_list || !h->dist.split_index) return fail(KGE_ENOMEM);
    e = cudaMemcpy(h->list, lst.data(), lst.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !split_list.empty())
      e = cudaMemcpy(h->dist.split_list, split_list.data(), split_list.size() * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(h->dist.split_index, split_index.data(), split_index.size() * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return fail(cuda_fail(e, "partition upload"));
    h->n_list = (int64_t)lst.size();
    h->dist.rel_owner = owner;
  }

  // ---- tables ----
  const int64_t Ne = cfg->n_entities, Nr = cfg->n_relations;
  h->ent_rows = h->P > 1 ? (Ne - h->rank + h->P - 1) / h->P : Ne;  // shard: owner e mod P, local row e div P
  h->ent = (float*)(h->P > 1 ? rawalloc(h, (size_t)h->ent_rows * dm.d * 4) : dalloc(h, (size_t)Ne * dm.d * 4));
  h->ent_st = (float*)dalloc(h, (size_t)h->ent_rows * 4);
  // P > 1: relation tables IPC-exportable too (per-epoch repartition pulls rows from their previous owner)
  h->rel = (float*)(h->P > 1 ? rawalloc(h, (size_t)Nr * dm.drel * 4) : dalloc(h, (size_t)Nr * dm.drel * 4));
  h->rel_st = (float*)(h->P > 1 ? rawalloc(h, (size_t)Nr * 4) : dalloc(h, (size_t)Nr * 4));
  if (!h->ent || !h->ent_st || !h->rel || !h->rel_st) { set_error("out of device memory (tables)"); return fail(KGE_ENOMEM); }
  const float bound = cfg->init_bound > 0.f ? cfg->init_bound : default_bound(cfg->gamma, cfg->dim);
  const float rbound = cfg->model == KGE_ROTATE ? (float)M_PI : bound;
  e = launch_init_table(h, h->ent, h->ent_rows, dm.d, 0, bound, h->P, h->rank);
  if (e == cudaSuccess) e = launch_init_table(h, h->rel, Nr, dm.drel, 1, rbound);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->ent_st, 0, (size_t)h->ent_rows * 4, h->stream);
  h->rows = EntRows{};
  h->rows.base[0] = h->ent;
  h->rows.P = 1;
  h->rows.d = dm.d;
  if (e == cudaSuccess) e = cudaMemsetAsync(h->rel_st, 0, (size_t)Nr * 4, h->stream);
  if (e != cudaSuccess) return fail(cuda_fail(e, "table init"));
  if (cfg->model == KGE_TRANSR || cfg->model == KGE_RESCAL) {  // M_r, d x d row-major, same uniform law (c.6 / Q12)
    // + 256 B: the 4D TMA views of TransR read a ragged last column block past the last row (make_map4c)
    h->proj = (float*)(h->P > 1 ? rawalloc(h, (size_t)Nr * dm.d * dm.d * 4 + 256) : dalloc(h, (size_t)Nr * dm.d * dm.d * 4 + 256));
    h->proj_st = (float*)(h->P > 1 ? rawalloc(h, (size_t)Nr * 4) : dalloc(h, (size_t)Nr * 4));
    if (!h->proj || !h->proj_st) { set_error("out of device memory (TransR projections)"); return fail(KGE_ENOMEM); }
    e = launch_init_table(h, h->proj, Nr, dm.d * dm.d, 2, bound);
    if (e == cudaSuccess) e = cudaMemsetAsync(h->proj_st, 0, (size_t)Nr * 4, h->stream);
    if (e != cudaSuccess) return fail(cuda_fail(e, "projection init"));
    TrBuffers& T = h->tr_buf;
    const size_t B = dm.B;
    const size_t njt = (size_t)tr_jtiles(dm.k), nsi = B + B / kTrSlice + 1;
    int32_t* ib = (int32_t*)dalloc(h, (1 + 4 * B + (B + 1) + (dm.C + 1) + B + (B + 1) + 1 + 2 * (B + B / 8 + 1) + 1 +
                                       2 * nsi + B + B * njt + B + B + dm.C + 1) * 4);
    const bool tr = cfg->model == KGE_TRANSR;  // RESCAL needs only dM and the U / V (H) factor rows
    T.QX = (float*)dalloc(h, tr ? B * dm.k * dm.d * 4 : 4);
    T.dQ = (float*)dalloc(h, tr ? B * dm.k * dm.d * 4 + 256 : 4);
    T.dM = (float*)dalloc(h, B * dm.d * dm.d * 4);
    T.Pv = (float*)dalloc(h, B * dm.d * 4);
    const size_t urows = tr ? 2 * B + 32 * B : B;  // TransR: padded per-relation blocks (k_tr_dm_tc); RESCAL: B rows
    T.U = (float*)dalloc(h, urows * dm.d * 4 + 256);
    T.H = (float*)dalloc(h, urows * dm.d * 4 + 256);
    T.dOp = (float*)dalloc(h, tr ? (size_t)tr_jtiles(dm.k) * B * dm.d * 4 : 4);
    if (!ib || !T.QX || !T.dQ || !T.dM || !T.Pv || !T.U || !T.H || !T.dOp) { set_error("out of device memory (TransR)"); return fail(KGE_ENOMEM); }
    T.n_groups = ib; ib += 1;
    T.grp_u = ib; ib += B;
    T.grp_c = ib; ib += B;
    T.grp_p0 = ib; ib += B;
    T.grp_p1 = ib; ib += B;
    T.rg_off = ib; ib += B + 1;
    T.cg_off = ib; ib += dm.C + 1;
    T.cg_list = ib; ib += B;
    T.pad_off = ib; ib += B + 1;
    T.n_items = ib; ib += 1;
    T.item_u = ib; ib += B + B / 8 + 1;
    T.item_p = ib; ib += B + B / 8 + 1;
    T.n_sitems = ib; ib += 1;
    T.sitem_g = ib; ib += nsi;
    T.sitem_p = ib; ib += nsi;
    T.ms_off = ib; ib += B;
    T.scnt = ib; ib += B * njt;
    T.rel_order = ib; ib += B;
    T.grp_lc = ib; ib += B;
    T.si_off = ib; ib += dm.C + 1;
    T.dQs = (float*)dalloc(h, tr ? (2 * B / kTrSlice + 2) * dm.k * dm.d * 4 : 4);
    if (!T.dQs || cudaMemsetAsync(T.scnt, 0, B * njt * 4, h->stream) != cudaSuccess) {
      set_error("out of device memory (TransR)");
      return fail(KGE_ENOMEM);
    }
    if (cudaMemsetAsync(T.U, 0, urows * dm.d * 4, h->stream) != cudaSuccess ||
        cudaMemsetAsync(T.H, 0, urows * dm.d * 4, h->stream) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "TransR scratch"));
    if (!(tr ? transr_init(h) : rescal_init(h))) { set_error("TransR / RESCAL kernel setup failed"); return fail(KGE_ECUDA); }
  }

  // ---- sample ring + debug slot ----
  // sample ring (+ the debug slot) and the flags/slot-table block; for P > 1 they live in the exported shared block
  // together with the barrier flags and the per-unique gradient sums that peers read
  const size_t sl = slot_ints(dm);
  const int nslot = h->ring + 1 + kge_handle::kGiven;  // ring, debug slot, given-batch slots
  const size_t flags_bytes = ((16 + sizeof(Slot) * nslot) + 255) & ~size_t(255);
  const size_t ring_bytes = sl * 4 * nslot;
  int32_t* ring_base = nullptr;
  if (h->P > 1) {
    Dist& D = h->dist;
    const size_t gu_one = ((size_t)dm.n_occ * dm.d * 4 + 255) & ~size_t(255);
    const size_t gu_bytes = gu_one * (cfg->lag == 1 ? 2 : 1);
    const size_t gs_bytes = ((size_t)std::max(1, D.n_split) * dm.drel * 4 + 255) & ~size_t(255);
    const size_t gp_bytes = cfg->model == KGE_TRANSR || cfg->model == KGE_RESCAL
                                ? (size_t)std::max(1, D.n_split) * dm.d * dm.d * 4 : 0;
    D.shared_bytes = 256 + flags_bytes + ring_bytes + gu_bytes + gs_bytes + gp_bytes;
    char* sb = (char*)rawalloc(h, D.shared_bytes);
    if (!sb) { set_error("out of device memory (shared block)"); return fail(KGE_ENOMEM); }
    D.shared = sb;
    D.flags = (uint64_t*)sb;
    h->buf.flags = (int32_t*)(sb + 256);
    ring_base = (int32_t*)(sb + 256 + flags_bytes);
    D.gu = (float*)(sb + 256 + flags_bytes + ring_bytes);
    D.gu_buf[0] = D.gu;
    D.gu_buf[1] = cfg->lag == 1 ? (float*)(sb + 256 + flags_bytes + ring_bytes + gu_one) : D.gu;
    D.grel_split = (float*)(sb + 256 + flags_bytes + ring_bytes + gu_bytes);
    if (gp_bytes) D.gproj_split = (float*)(sb + 256 + flags_bytes + ring_bytes + gu_bytes + gs_bytes);
    e = cudaMemset(sb, 0, D.shared_bytes);
    const size_t max_slots = (size_t)h->P * dm.n_occ;
    D.mark = (int32_t*)dalloc(h, (size_t)h->ent_rows * 4);
    D.contrib = (int32_t*)dalloc(h, max_slots * h->P * 4);
    D.slot_row = (int32_t*)dalloc(h, max_slots * 4);
    D.n_slots = (int32_t*)dalloc(h, 16);
    if (!D.mark || !D.contrib || !D.slot_row || !D.n_slots) return fail(KGE_ENOMEM);
    if (e == cudaSuccess) e = cudaMemset(D.mark, 0xFF, (size_t)h->ent_rows * 4);
    if (e == cudaSuccess) e = cudaMemset(D.contrib, 0xFF, max_slots * h->P * 4);
    if (e != cudaSuccess) return fail(cuda_fail(e, "shared block init"));
  } else {
    ring_base = (int32_t*)dalloc(h, ring_bytes);
    h->buf.flags = (int32_t*)dalloc(h, flags_bytes);  // flags[4] then the device slot table
    if (!ring_base || !h->buf.flags) { set_error("out of device memory (ring)"); return fail(KGE_ENOMEM); }
  }
  h->slots.resize(h->ring);
  for (int i = 0; i < h->ring; ++i) carve_slot(h, ring_base + sl * i, h->slots[i]);
  carve_slot(h, ring_base + sl * h->ring, h->debug_slot);
  for (int i = 0; i < kge_handle::kGiven; ++i) carve_slot(h, ring_base + sl * (h->ring + 1 + i), h->given_slots[i]);
  {  // the side stream gets the highest priority: its sampler CTAs take the next free SM slot ahead of the step
     // kernels' (PDL-launched, waiting) CTAs, so the sample of step s+1 really overlaps step s
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "side stream"));
    for (int i = 0; i < kge_handle::kGiven; ++i)
      if (cudaStreamCreateWithPriority(&h->gside[i], cudaStreamNonBlocking, hi) != cudaSuccess)
        return fail(cuda_fail(cudaGetLastError(), "side stream"));
    if (cudaStreamCreateWithFlags(&h->ustream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_eread, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_eupd, cudaEventDisableTiming) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "update stream"));
  }
  for (int i = 0; i < 2; ++i)
    if (cudaEventCreateWithFlags(&h->ev_samp[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_free[i], cudaEventDisableTiming) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "events"));
  for (int i = 0; i < kge_handle::kGiven; ++i)
    if (cudaEventCreateWithFlags(&h->ev_gsamp[i], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&h->ev_gfree[i], cudaEventDisableTiming) != cudaSuccess)
      return fail(cuda_fail(cudaGetLastError(), "events"));
  h->given = (int32_t*)dalloc(h, (size_t)kge_handle::kGiven * 3 * dm.B * 4);
  h->gready = (uint32_t*)dalloc(h, kge_handle::kGiven * 4);
  if (!h->given || !h->gready || cudaMemsetAsync(h->gready, 0, kge_handle::kGiven * 4, h->stream) != cudaSuccess) {
    cudaGetLastError();
    set_error("out of device memory (caller-batch slots)");
    return fail(KGE_ENOMEM);
  }
  for (int i = 0; i < kge_handle::kStage; ++i)
    if (cudaEventCreateWithFlags(&h->stage_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return fail(KGE_ECUDA);
    }
  if (cudaMallocHost(&h->pinned_given, (size_t)kge_handle::kStage * 3 * dm.B * 4) != cudaSuccess ||
      cudaMallocHost(&h->pinned_loss, (size_t)h->ring * 4) != cudaSuccess ||
      cudaMallocHost(&h->pinned_sink, 16) != cudaSuccess) {
    cudaGetLastError();
    return fail(KGE_ENOMEM);
  }

  // ---- step buffers ----
  StepBuffers& b = h->buf;
  const int64_t nneg = (int64_t)dm.C * dm.k;
  h->n_neg_parts = dm.C * ((dm.g + 63) / 64) * ((dm.k + 63) / 64);
  const int64_t tc_parts = (int64_t)dm.C * ((dm.g + 127) / 128) * ((dm.k + 31) / 32) * 2;  // >= TC epilogue partials
  b.O = (float*)dalloc(h, (size_t)dm.B * dm.dp * 4);
  b.onorm = (float*)dalloc(h, (size_t)dm.B * 4);
  b.X = (float*)dalloc(h, (size_t)nneg * dm.dp * 4);
  b.xnorm = (float*)dalloc(h, (size_t)nneg * 4);
  b.W = (float*)dalloc(h, (size_t)dm.B * dm.kp * 4);
  if (dm.bf16) {  // BF16 operand copies of the tcgen05 kind::f16 path (pads stay zero)
    b.O16 = (uint16_t*)dalloc(h, (size_t)dm.B * dm.dp16 * 2);
    b.X16 = (uint16_t*)dalloc(h, (size_t)nneg * dm.dp16 * 2);
    b.W16 = (uint16_t*)dalloc(h, (size_t)dm.B * dm.kp16 * 2);
    if (!b.O16 || !b.X16 || !b.W16) { set_error("out of device memory (BF16 operands)"); return fail(KGE_ENOMEM); }
  }
  if (dm.x3) {  // 3xTF32 hi / lo splits (pads stay zero)
    b.O_hi = (float*)dalloc(h, (size_t)dm.B * dm.dp * 4);
    b.O_lo = (float*)dalloc(h, (size_t)dm.B * dm.dp * 4);
    b.X_hi = (float*)dalloc(h, (size_t)nneg * dm.dp * 4);
    b.X_lo = (float*)dalloc(h, (size_t)nneg * dm.dp * 4);
    b.W_hi = (float*)dalloc(h, (size_t)dm.B * dm.kp * 4);
    b.W_lo = (float*)dalloc(h, (size_t)dm.B * dm.kp * 4);
    if (!b.O_hi || !b.O_lo || !b.X_hi || !b.X_lo || !b.W_hi || !b.W_lo) {
      set_error("out of device memory (3xTF32 operands)");
      return fail(KGE_ENOMEM);
    }
  }
  b.wpos = (float*)dalloc(h, (size_t)dm.B * 4);
  b.lpos = (float*)dalloc(h, (size_t)dm.B * 4);
  b.pstat = (float*)dalloc(h, (size_t)dm.B * 4);
  b.pcnt = (int32_t*)dalloc(h, (size_t)dm.B * 4);
  const int64_t tr_parts = cfg->model == KGE_TRANSR ? (int64_t)(dm.B + dm.B / kTrSlice + 1) * tr_jtiles(dm.k) : 0;
  b.lneg = (float*)dalloc(h, (size_t)std::max<int64_t>(std::max<int64_t>(std::max<int64_t>(h->n_neg_parts, tc_parts),
                                                                         tr_parts), dm.B) * 4);
  b.flow = (uint32_t*)dalloc(h, (size_t)2 * dm.C * 4);
  {  // FFMA split-K scratch: tiles of the larger (backward) grid x up to 8 splits x 256 threads x 16 floats
    const int64_t tiles = (int64_t)((dm.d + 63) / 64) * ((std::max(dm.g, dm.k) + 63) / 64) * 2 * dm.C;
    h->ffma_ks_max = 8;
    h->ffma_part = (float4*)dalloc(h, (size_t)tiles * h->ffma_ks_max * 4 * 256 * sizeof(float4));
    h->ffma_cnt = (int32_t*)dalloc(h, (size_t)tiles * 4);
    if (!h->ffma_part || !h->ffma_cnt) { set_error("out of device memory (FFMA scratch)"); return fail(KGE_ENOMEM); }
  }
  b.rowsumW = (float*)dalloc(h, (size_t)dm.B * 2 * ((dm.k + 31) / 32) * 4);   // tc.cu partial row sums of W
  b.colsumW = (float*)dalloc(h, (size_t)nneg * ((dm.g + 127) / 128) * 4);     // tc.cu partial column sums of W
  b.dO = (float*)dalloc(h, (size_t)dm.B * dm.d * 4);
  b.Gocc = (float*)dalloc(h, (size_t)(cfg->lag == 1 ? 2 : 1) * dm.n_occ * dm.d * 4);
  h->gocc2[0] = b.Gocc;
  h->gocc2[1] = cfg->lag == 1 && b.Gocc ? b.Gocc + (size_t)dm.n_occ * dm.d : b.Gocc;
  b.Grel = (float*)dalloc(h, (size_t)dm.B * dm.drel * 4);
  b.loss = (float*)dalloc(h, (size_t)h->ring * 4);
  h->seg_cnt = (int32_t*)dalloc(h, (size_t)(dm.B + dm.n_occ) * 4);
  if (!b.O || !b.onorm || !b.X || !b.xnorm || !b.W || !b.wpos || !b.lpos || !b.pstat || !b.lneg || !b.rowsumW || !b.colsumW ||
      !b.dO || !b.Gocc || !b.Grel || !b.loss || !b.flags || !h->seg_cnt) {
    set_error("out of device memory (workspace)");
    return fail(KGE_ENOMEM);
  }
  e = cudaMemsetAsync(b.flags, 0, 16, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(b.flow, 0, (size_t)2 * dm.C * 4, h->stream);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(h->ffma_cnt, 0, (size_t)((dm.d + 63) / 64) * ((std::max(dm.g, dm.k) + 63) / 64) * 2 * dm.C * 4,
                        h->stream);
  // padding of O / X' (see tc.cu): zeros, plus O[:, d] = 1 and X'[:, d+1] = 1 -- written once, never overwritten
  if (e == cudaSuccess) e = cudaMemsetAsync(b.O, 0, (size_t)dm.B * dm.dp * 4, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(b.X, 0, (size_t)nneg * dm.dp * 4, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(b.W, 0, (size_t)dm.B * dm.kp * 4, h->stream);
  if (e == cudaSuccess && dm.bf16) e = cudaMemsetAsync(b.O16, 0, (size_t)dm.B * dm.dp16 * 2, h->stream);
  if (e == cudaSuccess && dm.bf16) e = cudaMemsetAsync(b.X16, 0, (size_t)nneg * dm.dp16 * 2, h->stream);
  if (e == cudaSuccess && dm.bf16) e = cudaMemsetAsync(b.W16, 0, (size_t)dm.B * dm.kp16 * 2, h->stream);
  for (float* p : {b.O_hi, b.O_lo})
    if (e == cudaSuccess && p) e = cudaMemsetAsync(p, 0, (size_t)dm.B * dm.dp * 4, h->stream);
  for (float* p : {b.X_hi, b.X_lo})
    if (e == cudaSuccess && p) e = cudaMemsetAsync(p, 0, (size_t)nneg * dm.dp * 4, h->stream);
  for (float* p : {b.W_hi, b.W_lo})
    if (e == cudaSuccess && p) e = cudaMemsetAsync(p, 0, (size_t)dm.B * dm.kp * 4, h->stream);
  if (e == cudaSuccess) {
    std::vector<float> ones((size_t)std::max<int64_t>(dm.B, nneg), 1.0f);
    e = cudaMemcpy2DAsync(b.O + dm.d, (size_t)dm.dp * 4, ones.data(), 4, 4, dm.B, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(b.X + dm.d + 1, (size_t)dm.dp * 4, ones.data(), 4, 4, nneg, cudaMemcpyHostToDevice, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  }
  if (e == cudaSuccess)
    e = cudaMemsetAsync(b.Gocc, 0, (size_t)(cfg->lag == 1 ? 2 : 1) * dm.n_occ * dm.d * 4, h->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(h->seg_cnt, 0, (size_t)(dm.B + dm.n_occ) * 4, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_slots(h), h->slots.data(), sizeof(Slot) * h->ring, cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_slots(h) + h->ring, &h->debug_slot, sizeof(Slot), cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_slots(h) + h->ring + 1, h->given_slots, sizeof(Slot) * kge_handle::kGiven, cudaMemcpyHostToDevice,
                        h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return fail(cuda_fail(e, "workspace init"));
  if (getenv("KGE_TRACE")) {  // diagnostics: per-CTA stamps, read with kge_debug_trace
    const size_t tb = (size_t)KGE_K_COUNT * kTraceCtas * kTraceSlots * 8;
    dm.trace = (uint64_t*)dalloc(h, tb);
    if (!dm.trace || cudaMemset(dm.trace, 0, tb) != cudaSuccess) return fail(KGE_ENOMEM);
  }
  if (sample_init() != cudaSuccess || step_preload() != cudaSuccess || dist_preload() != cudaSuccess)
    return fail(cuda_fail(cudaGetLastError(), "kernel preload"));
  if (cfg->model == KGE_TRANSR)  // per (score item, tile of 32 negatives)
    h->n_neg_parts = (dm.B + dm.B / kTrSlice + 1) * tr_jtiles(dm.k);
  if (cfg->neg_precision != KGE_PREC_FP32 && cfg->model != KGE_TRANSR) tc_init(h);
  if (cfg->model == KGE_TRANSR) transr_tc_init(h);  // DistMult / ComplEx / TransE-L2 on tcgen05
  if (tc_supported(h)) h->n_neg_parts = tc_neg_parts(h);
  *out = h;
  return KGE_OK;
}

static int ensure_sampled(kge_handle* h, int64_t s) {
  if (h->epoch_steps > 0) {  // repartition: the list changes at epoch boundaries, so every step is sampled on its own
    cudaError_t e = launch_sample(h, sample_params(h, false), d_slots(h), h->ring, s, 1);
    if (e != cudaSuccess) return cuda_fail(e, "sample");
    h->half_first[0] = h->half_first[1] = -1;
    return KGE_OK;
  }
  const int H = h->ring / 2;
  const int64_t hs = s - s % H;  // first step of s's ring half
  const int q = (int)((hs / H) % 2);
  SampleParams p = sample_params(h, false);
  cudaError_t e = cudaSuccess;
  if (h->half_first[q] != hs) {  // not sampled ahead (first call, kge_set_step, a caller batch): sample it in order
    e = launch_sample(h, p, d_slots(h), h->ring, hs, H);
    if (e != cudaSuccess) return cuda_fail(e, "sample");
    h->half_first[q] = hs;
    h->half_waited[q] = true;
  } else if (!h->half_waited[q]) {
    e = cudaStreamWaitEvent(h->stream, h->ev_samp[q], 0);
    if (e != cudaSuccess) return cuda_fail(e, "sample wait");
    h->half_waited[q] = true;
  }
  return KGE_OK;
}

static int join_updates(kge_handle* h);
static int check_flags(kge_handle* h) {
  const int rj = join_updates(h);
  if (rj != KGE_OK) return rj;
  int32_t f[4];
  cudaError_t e = cudaMemcpyAsync(f, h->buf.flags, 16, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sync");
  if (f[1] == 2) {
    set_error("caller-batch sample gate timed out (the side-stream sample of a step never completed)");
    return KGE_ECUDA;
  }
  if (f[1]) {
    set_error("device barrier timed out: a peer rank did not reach the step (KGE_OPT_BARRIER_MS)");
    return KGE_ECUDA;
  }
  if (f[0]) {
    cudaMemsetAsync(h->buf.flags, 0, 4, h->stream);
    set_error("a step produced a non-finite loss; its update was skipped");
    return KGE_ENONFINITE;
  }
  return KGE_OK;
}

// Fill the other ring half with steps [hs + H, hs + 2H) on the side stream. Its slots were last read by steps < hs,
// all enqueued before this point on the main stream (and, lag = 1, by the held-back entity update enqueued with
// step s on the update stream). (P > 1 samples in order on the main stream: with several ranks sharing one device,
// as the emulated-rank tests do, side-stream samplers could hold the SMs the ranks' device barriers need.)
static int prefetch_half(kge_handle* h, int64_t s) {
  const int H = h->ring / 2;
  const int64_t hs = s - s % H;
  const int q = (int)((hs / H) % 2);
  if (h->P != 1 || h->half_first[1 - q] == hs + H) return KGE_OK;
  SampleParams p = sample_params(h, false);
  cudaError_t e = cudaEventRecord(h->ev_free[1 - q], h->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h->side, h->ev_free[1 - q], 0);
  if (e == cudaSuccess && h->eupd_enqueued) e = cudaStreamWaitEvent(h->side, h->ev_eupd, 0);
  if (e == cudaSuccess) e = launch_sample(h, p, d_slots(h), h->ring, hs + H, H, h->side);
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_samp[1 - q], h->side);
  if (e != cudaSuccess) return cuda_fail(e, "sample ahead");
  h->half_first[1 - q] = hs + H;
  h->half_waited[1 - q] = false;
  return KGE_OK;
}

// One step on the main stream. lag = 1 (reading c.12): the step's gather waits for the entity update of step s-2;
// the entity update of step s-1 is enqueued on the update stream behind this step's last entity-table read
// (ev_eread) and the current step's is held back.
static int enqueue_step(kge_handle* h, const Slot& slot, int64_t s, int gi) {
  cudaError_t e = cudaSuccess;
  if (h->cfg.lag == 1) {
    if (h->eupd_enqueued) e = cudaStreamWaitEvent(h->stream, h->ev_eupd, 0);
    h->buf.Gocc = h->gocc2[s & 1];
  }
  h->next_slot = gi >= 0 ? d_slots(h) + h->ring + 1 + (gi + 1) % kge_handle::kGiven : d_slots(h) + (s + 1) % h->ring;
  if (h->P > 1) h->dist.gu = h->dist.gu_buf[h->cfg.lag == 1 ? (s & 1) : 0];
  if (e == cudaSuccess) e = launch_step(h, slot, s);
  if (e == cudaSuccess && h->P > 1) e = dist_exchange_update(h, slot, s);
  if (e != cudaSuccess) return cuda_fail(e, "step");
  if (h->cfg.lag == 1 && h->P > 1) {
    // the owner update of step s-1 (its per-unique sums were exchanged in step s-1) on the update stream, behind this
    // step's last entity-table read and a barrier of every rank's (sequence 1); the next step's B1 waits for it
    if (h->pend_step >= 0) {
      e = cudaStreamWaitEvent(h->ustream, h->ev_eread, 0);
      if (e == cudaSuccess) e = dist_owner_update_lagged(h, h->pend_slot, h->pend_step, h->ustream);
      if (e == cudaSuccess) e = cudaEventRecord(h->ev_eupd, h->ustream);
      if (e != cudaSuccess) return cuda_fail(e, "lagged owner update");
      h->eupd_enqueued = true;
    }
    h->pend_step = s;
    h->pend_slot = slot;
    h->pend_gi = gi;
  } else if (h->cfg.lag == 1) {
    if (h->pend_step >= 0) {
      const Dims& dm = h->dims;
      e = cudaStreamWaitEvent(h->ustream, h->ev_eread, 0);
      if (e == cudaSuccess)
        e = launch_update_range(h, h->pend_slot, dm.B, dm.B + dm.n_occ, h->ustream, h->gocc2[h->pend_step & 1]);
      if (e == cudaSuccess) e = cudaEventRecord(h->ev_eupd, h->ustream);
      if (e == cudaSuccess && h->pend_gi >= 0) e = cudaEventRecord(h->ev_gfree[h->pend_gi], h->ustream);
      if (e != cudaSuccess) return cuda_fail(e, "entity update");
      h->eupd_enqueued = true;
    }
    h->pend_step = s;
    h->pend_slot = slot;
    h->pend_gi = gi;
  }
  return KGE_OK;
}

// the main stream waits for the update stream (table reads / writes from the host API see every enqueued update)
static int join_updates(kge_handle* h) {
  if (h->eupd_enqueued) {
    cudaError_t e = cudaStreamWaitEvent(h->stream, h->ev_eupd, 0);
    if (e != cudaSuccess) return cuda_fail(e, "join");
  }
  return KGE_OK;
}

int kge_flush(kge_handle* h) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  int rc = join_updates(h);
  if (rc != KGE_OK || h->pend_step < 0) return rc;
  const Dims& dm = h->dims;
  cudaError_t e = h->P > 1 ? dist_owner_flush(h, h->pend_slot, h->pend_step)  // collective (every rank calls it)
                           : launch_update_range(h, h->pend_slot, dm.B, dm.B + dm.n_occ, h->stream,
                                                 h->gocc2[h->pend_step & 1]);
  if (e == cudaSuccess && h->pend_gi >= 0) e = cudaEventRecord(h->ev_gfree[h->pend_gi], h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "flush");
  h->pend_step = -1;
  h->pend_gi = -1;
  return KGE_OK;
}

// repartition (reading c.13'): the partition of epoch e; every rank pulls the relation rows (states, TransR M_r) it did
// not own in the previous epoch from their owner, between two barriers, then samples from its epoch-e list
static int switch_epoch(kge_handle* h, int64_t e) {
  const int64_t Nr = h->dims.n_relations;
  std::vector<int32_t> owner, lst;
  relation_partition(h->host_rels.data(), (int64_t)h->host_rels.size(), Nr, h->P, owner, true, h->cfg.seed,
                     (uint32_t)e);
  rank_list(h->host_rels.data(), (int64_t)h->host_rels.size(), Nr, h->P, h->rank, owner, &lst);
  if (lst.empty()) { set_error("this rank received no triples in an epoch's partition"); return KGE_EINVAL; }
  h->owner_prev = h->dist.rel_owner;  // kept alive for the asynchronous copy
  cudaError_t err = cudaMemcpyAsync(h->d_owner_prev, h->owner_prev.data(), (size_t)Nr * 4, cudaMemcpyHostToDevice,
                                    h->stream);
  if (err == cudaSuccess) err = dist_barrier(h);  // every rank finished the previous epoch's updates
  if (err == cudaSuccess) err = dist_pull_relations(h, h->d_owner_prev);
  if (err == cudaSuccess) err = dist_barrier(h);  // nobody updates a row a peer is still pulling
  // the new list through one of two pinned staging buffers (no stream synchronisation: with several ranks driven by one
  // host thread a synchronising copy would wait on a barrier the other ranks have not enqueued yet); a buffer is
  // reused two switches later, after its copy's event
  const int b = h->list_flip;
  h->list_flip ^= 1;
  if (err == cudaSuccess && !h->pin_list[b]) {
    err = cudaMallocHost((void**)&h->pin_list[b], h->host_rels.size() * 4);
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&h->ev_list[b], cudaEventDisableTiming);
  } else if (err == cudaSuccess) {
    err = cudaEventSynchronize(h->ev_list[b]);
  }
  if (err == cudaSuccess) {
    std::copy(lst.begin(), lst.end(), h->pin_list[b]);
    err = cudaMemcpyAsync(h->list, h->pin_list[b], lst.size() * 4, cudaMemcpyHostToDevice, h->stream);
  }
  if (err == cudaSuccess) err = cudaEventRecord(h->ev_list[b], h->stream);
  if (err != cudaSuccess) return cuda_fail(err, "epoch repartition");
  h->n_list = (int64_t)lst.size();
  h->dist.rel_owner = owner;
  h->cur_epoch = e;
  return KGE_OK;
}

int kge_train_step(kge_handle* h, int64_t n_steps, float* loss_out) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  if (n_steps < 0) { set_error("n_steps < 0"); return KGE_EINVAL; }
  if (h->P > 1 && !h->dist.connected) { set_error("world_size > 1: call kge_connect first"); return KGE_ESTATE; }
  for (int64_t it = 0; it < n_steps; ++it) {
    const int64_t s = h->step;
    if (s >= (1ll << 32)) { set_error("step index exceeds 2^32 (one Philox counter word)"); return KGE_ERANGE; }
    if (h->P > 1) {
      // B1: every owner has applied step s-1 (lag = 1: step s-2, joined from the update stream first) before anyone
      // gathers rows or overwrites a slot peers read
      int rj = join_updates(h);
      if (rj == KGE_OK && h->epoch_steps > 0 && s / h->epoch_steps != h->cur_epoch) rj = switch_epoch(h, s / h->epoch_steps);
      if (rj != KGE_OK) return rj;
      cudaError_t e = dist_barrier(h);
      if (e == cudaSuccess) e = dist_clear_split(h);
      if (e != cudaSuccess) return cuda_fail(e, "barrier");
    }
    int rc = ensure_sampled(h, s);
    if (rc != KGE_OK) return rc;
    rc = enqueue_step(h, h->slots[s % h->ring], s, -1);
    if (rc != KGE_OK) return rc;
    rc = prefetch_half(h, s);
    if (rc != KGE_OK) return rc;
    cudaError_t e = cudaSuccess;
    if (loss_out) {
      e = cudaMemcpyAsync(h->pinned_loss + (it % h->ring), h->buf.loss + (s % h->ring), 4, cudaMemcpyDeviceToHost, h->stream);
      if (e != cudaSuccess) return cuda_fail(e, "loss readback");
    }
    h->step = s + 1;
    if (loss_out && ((it + 1) % h->ring == 0 || it + 1 == n_steps)) {
      e = cudaStreamSynchronize(h->stream);
      if (e != cudaSuccess) return cuda_fail(e, "sync");
      const int64_t first = it - (it % h->ring);
      for (int64_t q = first; q <= it; ++q) loss_out[q] = h->pinned_loss[q % h->ring];
    }
  }
  if (loss_out) return check_flags(h);
  return KGE_OK;
}

// Enqueue one step on a caller-supplied batch; loss_dev_to: host destination of an async loss copy (or NULL).
static bool use_graphs(const kge_handle* h) {
  static const bool off = getenv("KGE_NO_GRAPHS") != nullptr || getenv("KGE_DEBUG_SYNC") != nullptr;
  return h->P == 1 && h->cfg.lag == 0 && !off && !h->prof.on && h->dims.trace == nullptr;
}

// capture `body` (launches on stream st) into an instantiated graph; the first node of the given type is returned
static cudaError_t capture_graph(kge_handle* h, cudaStream_t st, const std::function<cudaError_t()>& body,
                                 cudaGraphExec_t* exec, cudaGraphNodeType want, cudaGraphNode_t* node) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return e;
  const int64_t l0 = h->launches;
  cudaError_t eb = body();
  cudaError_t ee = cudaStreamEndCapture(st, &g);
  h->g_launches = (int32_t)(h->launches - l0);
  h->launches = l0;
  if (eb != cudaSuccess || ee != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    return eb != cudaSuccess ? eb : ee;
  }
  size_t n = 0;
  e = cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (e == cudaSuccess) e = cudaGraphGetNodes(g, nodes.data(), &n);
  *node = nullptr;
  for (size_t i = 0; e == cudaSuccess && i < n && !*node; ++i) {
    cudaGraphNodeType t;
    e = cudaGraphNodeGetType(nodes[i], &t);
    if (e == cudaSuccess && t == want) *node = nodes[i];
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(exec, g, 0);
  if (e == cudaSuccess)
    h->graphs.push_back(g);  // kept alive: node parameter updates name nodes of the source graph
  else
    cudaGraphDestroy(g);
  return e;
}

// graph path of train_batch_enqueue (P == 1): see kge_handle::g_samp / g_step
#define KGE_GCHK(call, what)                        \
  do {                                              \
    cudaError_t _e = (call);                        \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)
// device-visible address of a caller's pinned loss float (0: pageable, the loss is copied back instead)
static uint64_t loss_device_address(float* loss_host) {
  if (!loss_host) return 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, loss_host) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
    return (uint64_t)(uintptr_t)at.devicePointer;
  cudaGetLastError();
  return 0;
}

// Caller batch behind a device gate (P == 1, lag 0, the gather-first step of every model but TransR / RESCAL): the
// upload + sample run as one graph on the slot's side stream as in batch_graphs, but the main stream does not wait
// for it with a stream event. The step kernels are launched directly, each with PDL, behind k_wait_ready -- one CTA
// that spins on the slot's ready counter (bumped by both k_sample CTAs) and then waits for the previous step's last
// kernel. A cross-stream event wait or a graph boundary ends the PDL chain (the next step's kernels could only launch
// once the previous step had fully drained, ~3.7 us per step measured end to end); with the gate the chain runs from
// one step's update into the next step's gather as in kge_train_step.
static bool use_gate(const kge_handle* h) {
  static const bool off = getenv("KGE_NO_GATE") != nullptr;
  return !off && use_graphs(h) && h->dims.model != KGE_TRANSR && h->dims.model != KGE_RESCAL;
}

static int batch_gated(kge_handle* h, int gi, int64_t s, float* loss_host) {
  const int B = h->dims.B;
  SampleParams p = sample_params(h, true, gi);
  const Slot* gslot = d_slots(h) + h->ring + 1 + gi;
  cudaStream_t ss = h->gside[gi];
  uint32_t* rd = h->gready + gi;
  if (!h->g_samp[gi]) {
    int32_t* st = h->pinned_given + (size_t)gi * 3 * B;
    int32_t* gb = h->given + (size_t)gi * 3 * B;
    KGE_GCHK(capture_graph(h, ss, [&]() {
               cudaError_t x = cudaMemcpyAsync(gb, st, (size_t)3 * B * 4, cudaMemcpyHostToDevice, ss);
               return x == cudaSuccess ? launch_sample(h, p, gslot, 1, s, 1, ss, 0, rd) : x;
             }, &h->g_samp[gi], cudaGraphNodeTypeKernel, &h->g_samp_node[gi]), "capture sample graph");
  }
  const uint64_t dst = loss_device_address(loss_host);
  KGE_GCHK(cudaStreamWaitEvent(ss, h->ev_gfree[gi], 0), "wait slot");
  KGE_GCHK(sample_graph_set(h, h->g_samp[gi], h->g_samp_node[gi], p, gslot, 1, s, 1, dst, rd), "sample node params");
  KGE_GCHK(cudaGraphLaunch(h->g_samp[gi], ss), "sample graph launch");
  KGE_GCHK(cudaEventRecord(h->stage_ev[gi], ss), "event");
  ++h->launches;
  h->gcount[gi] += 1;
  KGE_GCHK(launch_wait_ready(h, rd, 2u * h->gcount[gi]), "sample gate");
  ++h->launches;
  const int rc = enqueue_step(h, h->given_slots[gi], s, gi);
  if (rc != KGE_OK) return rc;
  KGE_GCHK(cudaEventRecord(h->ev_gfree[gi], h->stream), "event");
  if (loss_host && !dst)
    KGE_GCHK(cudaMemcpyAsync(loss_host, h->buf.loss + (s % h->ring), 4, cudaMemcpyDeviceToHost, h->stream),
             "loss readback");
  return KGE_OK;
}

static int batch_graphs(kge_handle* h, int gi, int64_t s, float* loss_host) {
  const int B = h->dims.B;
  SampleParams p = sample_params(h, true, gi);
  const Slot* gslot = d_slots(h) + h->ring + 1 + gi;
  cudaStream_t ss = h->gside[gi];
  if (!h->g_samp[gi]) {
    int32_t* st = h->pinned_given + (size_t)gi * 3 * B;
    int32_t* gb = h->given + (size_t)gi * 3 * B;
    KGE_GCHK(capture_graph(h, ss, [&]() {
               cudaError_t x = cudaMemcpyAsync(gb, st, (size_t)3 * B * 4, cudaMemcpyHostToDevice, ss);
               return x == cudaSuccess ? launch_sample(h, p, gslot, 1, s, 1, ss) : x;
             }, &h->g_samp[gi], cudaGraphNodeTypeKernel, &h->g_samp_node[gi]), "capture sample graph");
  }
  if (!h->g_step[gi]) {
    h->next_slot = d_slots(h) + h->ring + 1 + (gi + 1) % kge_handle::kGiven;
    KGE_GCHK(capture_graph(h, h->stream, [&]() {
               cudaError_t x = launch_step(h, h->given_slots[gi], s);
               return x == cudaSuccess ? cudaMemcpyAsync(h->pinned_sink, h->buf.loss, 4, cudaMemcpyDeviceToHost, h->stream)
                                       : x;
             }, &h->g_step[gi], cudaGraphNodeTypeMemcpy, &h->g_loss_node[gi]), "capture step graph");
  }
  const int32_t kernels = h->g_launches;
  // the loss goes straight from the kernel that reduces it to the caller's pinned (device-visible) float: a 4-byte
  // D2H copy node costs ~10 us on the step's critical path. Pageable targets keep the copy.
  const uint64_t dst = loss_device_address(loss_host);
  KGE_GCHK(cudaStreamWaitEvent(ss, h->ev_gfree[gi], 0), "wait slot");
  KGE_GCHK(sample_graph_set(h, h->g_samp[gi], h->g_samp_node[gi], p, gslot, 1, s, 1, dst), "sample node params");
  KGE_GCHK(cudaGraphLaunch(h->g_samp[gi], ss), "sample graph launch");
  KGE_GCHK(cudaEventRecord(h->stage_ev[gi], ss), "event");
  KGE_GCHK(cudaEventRecord(h->ev_gsamp[gi], ss), "event");
  KGE_GCHK(cudaStreamWaitEvent(h->stream, h->ev_gsamp[gi], 0), "wait sample");
  const bool copy = loss_host && !dst;
  if (copy)
    KGE_GCHK(cudaGraphExecMemcpyNodeSetParams1D(h->g_step[gi], h->g_loss_node[gi], loss_host, h->buf.loss + (s % h->ring),
                                                4, cudaMemcpyDeviceToHost),
             "loss node params");
  if (copy != h->g_loss_on[gi]) {
    KGE_GCHK(cudaGraphNodeSetEnabled(h->g_step[gi], h->g_loss_node[gi], copy ? 1 : 0), "loss node");
    h->g_loss_on[gi] = copy;
  }
  KGE_GCHK(cudaGraphLaunch(h->g_step[gi], h->stream), "step graph launch");
  KGE_GCHK(cudaEventRecord(h->ev_gfree[gi], h->stream), "event");
  h->launches += 1 + kernels;
  return KGE_OK;
}
#undef KGE_GCHK

static int train_batch_enqueue(kge_handle* h, const int64_t* heads, const int64_t* rels, const int64_t* tails,
                               float* loss_host) {
  if (!h || !heads || !rels || !tails) { set_error("NULL argument"); return KGE_EINVAL; }
  if (h->P > 1 && !h->dist.connected) { set_error("world_size > 1: call kge_connect first"); return KGE_ESTATE; }
  const int B = h->dims.B;
  const int64_t s = h->step;
  // host-side range check + int32 narrowing into a pinned staging buffer (ring of kStage; a buffer is reused only
  // after its previous H2D copy completed), then one H2D copy
  const int si = (int)(s % kge_handle::kGiven);  // staging buffer = given slot (kStage == kGiven)
  int32_t* st = h->pinned_given + (size_t)si * 3 * B;
  static const bool hprof = getenv("KGE_HOST_PROF") != nullptr;  // diagnostics: host time per phase
  static double hp[4] = {0, 0, 0, 0};
  static int64_t hn = 0;
  auto now = []() { timespec t; clock_gettime(CLOCK_MONOTONIC, &t); return t.tv_sec * 1e6 + t.tv_nsec * 1e-3; };
  const double t0 = hprof ? now() : 0.0;
  cudaError_t e = cudaEventSynchronize(h->stage_ev[si]);
  if (e != cudaSuccess) return cuda_fail(e, "staging reuse");
  const double t1 = hprof ? now() : 0.0;
  struct HostProf {
    bool on; double t0, t1; double* hp; int64_t* hn; double (*now)();
    double t2 = 0;
    ~HostProf() {
      if (!on) return;
      const double t3 = now();
      hp[0] += t1 - t0; hp[1] += t2 - t1; hp[2] += t3 - t2; ++*hn;
      if (*hn % 1000 == 0)
        fprintf(stderr, "[kge host] per call: event sync %.2f us, narrowing %.2f us, enqueue %.2f us (%lld calls)\n",
                hp[0] / *hn, hp[1] / *hn, hp[2] / *hn, (long long)*hn);
    }
  } hpr{hprof, t0, t1, hp, &hn, +now};
  {  // branch-free (vectorisable) narrowing and range check; the error is reported after the loop
    const uint64_t ne = (uint64_t)h->dims.n_entities, nr = (uint64_t)h->dims.n_relations;
    uint64_t bad = 0;
    int32_t* sh = st;
    int32_t* sr = st + B;
    int32_t* stt = st + 2 * B;
    for (int i = 0; i < B; ++i) {  // unsigned compares: negative ids wrap to huge values
      bad |= (uint64_t)((uint64_t)heads[i] >= ne) | (uint64_t)((uint64_t)tails[i] >= ne) |
             (uint64_t)((uint64_t)rels[i] >= nr);
      sh[i] = (int32_t)heads[i];
      sr[i] = (int32_t)rels[i];
      stt[i] = (int32_t)tails[i];
    }
    if (bad) {
      set_error("batch id out of range");
      return KGE_ERANGE;
    }
  }
  if (hprof) hpr.t2 = now();
  if (h->epoch_steps > 0) {
    set_error("kge_train_batch: caller batches with repartition = 1 are not supported (the partition is the sampler's)");
    return KGE_EUNSUPPORTED;
  }
  if (h->P > 1) {  // B1 (see kge_train_step); every rank must call kge_train_batch for this step
    const int rj = join_updates(h);
    if (rj != KGE_OK) return rj;
    e = dist_barrier(h);
    if (e == cudaSuccess) e = dist_clear_split(h);
    if (e != cudaSuccess) return cuda_fail(e, "barrier");
  }
  if (use_gate(h) || use_graphs(h)) {
    const int rc = use_gate(h) ? batch_gated(h, si, s, loss_host) : batch_graphs(h, si, s, loss_host);
    if (rc != KGE_OK) return rc;
    h->step = s + 1;
    return KGE_OK;
  }
  // given slot gi of this step: upload + sample on the side stream (overlapping the previous step's kernels), after
  // the step that last used the slot released it
  // (P > 1: everything on the main stream, see ensure_sampled)
  const int gi = (int)(s % kge_handle::kGiven);
  cudaStream_t ss = h->P == 1 ? h->gside[gi] : h->stream;
  e = h->P == 1 ? cudaStreamWaitEvent(ss, h->ev_gfree[gi], 0) : cudaSuccess;
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->given + (size_t)gi * 3 * B, st, (size_t)3 * B * 4, cudaMemcpyHostToDevice, ss);
  if (e == cudaSuccess) e = cudaEventRecord(h->stage_ev[si], ss);
  if (e != cudaSuccess) return cuda_fail(e, "batch upload");
  // sample negatives + dedup for this step from the given positives
  SampleParams p = sample_params(h, true, gi);
  e = launch_sample(h, p, d_slots(h) + h->ring + 1 + gi, 1, s, 1, ss);
  if (e == cudaSuccess && h->P == 1) e = cudaEventRecord(h->ev_gsamp[gi], ss);
  if (e == cudaSuccess && h->P == 1) e = cudaStreamWaitEvent(h->stream, h->ev_gsamp[gi], 0);
  if (e != cudaSuccess) return cuda_fail(e, "sample");
  const int rcs = enqueue_step(h, h->given_slots[gi], s, gi);
  if (rcs != KGE_OK) return rcs;
  if (h->P == 1 && h->cfg.lag == 0) e = cudaEventRecord(h->ev_gfree[gi], h->stream);  // lag 1: after its entity update
  if (e != cudaSuccess) return cuda_fail(e, "step");
  h->step = s + 1;
  if (loss_host) {
    e = cudaMemcpyAsync(loss_host, h->buf.loss + (s % h->ring), 4, cudaMemcpyDeviceToHost, h->stream);
    if (e != cudaSuccess) return cuda_fail(e, "loss readback");
  }
  return KGE_OK;
}

int kge_train_batch(kge_handle* h, const int64_t* heads, const int64_t* rels, const int64_t* tails, float* loss_out) {
  const int rc = train_batch_enqueue(h, heads, rels, tails, loss_out ? h->pinned_loss : nullptr);
  if (rc != KGE_OK || !loss_out) return rc;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "loss readback");
  *loss_out = h->pinned_loss[0];
  return check_flags(h);
}

int kge_train_batch_async(kge_handle* h, const int64_t* heads, const int64_t* rels, const int64_t* tails,
                          float* loss_host) {
  return train_batch_enqueue(h, heads, rels, tails, loss_host);
}

int kge_sample(kge_handle* h, int64_t step, int64_t* pos_idx, int64_t* neg, int8_t* mode, int64_t* uniq_ent,
               int64_t* n_uniq_ent, int32_t* inv_ent, int64_t* uniq_rel, int64_t* n_uniq_rel, int32_t* inv_rel) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  if (step < 0 || step >= (1ll << 32)) { set_error("step out of range"); return KGE_ERANGE; }
  SampleParams p = sample_params(h, false);
  cudaError_t e = launch_sample(h, p, d_slots(h) + h->ring, 1, step, 1);
  if (e != cudaSuccess) return cuda_fail(e, "sample");
  const Dims& d = h->dims;
  const Slot& s = h->debug_slot;
  std::vector<int32_t> pos(d.B), ng((size_t)d.C * d.k), md(d.C), ue(d.n_occ), ie(d.n_occ), ur(d.B), ir(d.B);
  int32_t ne = 0, nr = 0;
  e = cudaMemcpyAsync(pos.data(), s.pos, d.B * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ng.data(), s.neg, ng.size() * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(md.data(), s.mode, d.C * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ue.data(), s.ent_uniq, d.n_occ * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ie.data(), s.ent_inv, d.n_occ * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ur.data(), s.rel_uniq, d.B * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(ir.data(), s.rel_inv, d.B * 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&ne, s.ent_n, 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nr, s.rel_n, 4, cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sample readback");
  if (pos_idx) for (int i = 0; i < d.B; ++i) pos_idx[i] = pos[i];
  if (neg) for (size_t i = 0; i < ng.size(); ++i) neg[i] = ng[i];
  if (mode) for (int i = 0; i < d.C; ++i) mode[i] = (int8_t)md[i];
  if (uniq_ent) for (int i = 0; i < ne; ++i) uniq_ent[i] = ue[i];
  if (n_uniq_ent) *n_uniq_ent = ne;
  if (inv_ent) std::memcpy(inv_ent, ie.data(), ie.size() * 4);
  if (uniq_rel) for (int i = 0; i < nr; ++i) uniq_rel[i] = ur[i];
  if (n_uniq_rel) *n_uniq_rel = nr;
  if (inv_rel) std::memcpy(inv_rel, ir.data(), ir.size() * 4);
  return KGE_OK;
}

static float* table_ptr(kge_handle* h, int32_t table, int32_t* w, int64_t* rows) {
  const Dims& d = h->dims;
  switch (table) {
    case 0: *w = d.d; *rows = d.n_entities; return h->ent;
    case 1: *w = d.drel; *rows = d.n_relations; return h->rel;
    case 2: *w = d.d * d.d; *rows = d.n_relations; return h->proj;
    case 3: *w = 1; *rows = d.n_entities; return h->ent_st;
    case 4: *w = 1; *rows = d.n_relations; return h->rel_st;
    case 5: *w = 1; *rows = d.n_relations; return h->proj_st;
  }
  return nullptr;
}

int32_t kge_table_width(const kge_handle* h, int32_t table) {
  if (!h) return 0;
  int32_t w = 0;
  int64_t rows = 0;
  float* p = table_ptr(const_cast<kge_handle*>(h), table, &w, &rows);
  return p ? w : 0;
}

// Readers / writers of the tables (rows, scores, ranks, set_step) see every update: one rank applies a held-back
// entity update itself; with P > 1 that update is collective, so the caller flushes on every rank first (KGE_ESTATE).
static int flush_for_io(kge_handle* h, bool entity_tables) {
  if (h->P == 1) return kge_flush(h);
  const int rj = join_updates(h);
  if (rj != KGE_OK) return rj;
  if (entity_tables && h->pend_step >= 0) {
    set_error("lag = 1 with world_size > 1: call kge_flush on every rank before reading or writing entity rows");
    return KGE_ESTATE;
  }
  return KGE_OK;
}

static int rows_io(kge_handle* h, int32_t table, const int64_t* ids, int64_t n, float* host, bool write) {
  if (!h || (n > 0 && (!ids || !host))) { set_error("NULL argument"); return KGE_EINVAL; }
  int32_t w;
  int64_t rows;
  float* tab = table_ptr(h, table, &w, &rows);
  if (!tab) { set_error("table not present for this model"); return KGE_EINVAL; }
  if (n == 0) return KGE_OK;
  // lag = 1: the held-back entity update belongs to the table the caller reads / overwrites
  const int rj = flush_for_io(h, table == 0 || table == 3);
  if (rj != KGE_OK) return rj;
  std::vector<int32_t> ids32(n);
  const bool sharded = h->P > 1 && (table == 0 || table == 3);
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= rows) { set_error("row id out of range"); return KGE_ERANGE; }
    if (sharded && ids[i] % h->P != h->rank) { set_error("entity row not owned by this rank (owner = id mod P)"); return KGE_ERANGE; }
    ids32[i] = (int32_t)(sharded ? ids[i] / h->P : ids[i]);
  }
  int32_t* d_ids = nullptr;
  float* d_buf = nullptr;
  CK(cudaMallocAsync((void**)&d_ids, n * 4, h->stream));
  CK(cudaMallocAsync((void**)&d_buf, (size_t)n * w * 4, h->stream));
  CK(cudaMemcpyAsync(d_ids, ids32.data(), n * 4, cudaMemcpyHostToDevice, h->stream));
  if (write) CK(cudaMemcpyAsync(d_buf, host, (size_t)n * w * 4, cudaMemcpyHostToDevice, h->stream));
  CK(launch_rows(h, tab, w, d_ids, n, d_buf, write));
  if (!write) CK(cudaMemcpyAsync(host, d_buf, (size_t)n * w * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaFreeAsync(d_ids, h->stream));
  CK(cudaFreeAsync(d_buf, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KGE_OK;
}

int kge_get_rows(kge_handle* h, int32_t table, const int64_t* ids, int64_t n, float* out) {
  return rows_io(h, table, ids, n, out, false);
}
int kge_set_rows(kge_handle* h, int32_t table, const int64_t* ids, int64_t n, const float* in) {
  return rows_io(h, table, ids, n, const_cast<float*>(in), true);
}

int kge_score(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, float* out) {
  if (!h || (n > 0 && (!hs || !rs || !ts || !out))) { set_error("NULL argument"); return KGE_EINVAL; }
  if (h->P > 1 && !h->dist.connected) { set_error("world_size > 1: call kge_connect first"); return KGE_ESTATE; }
  if (n == 0) return KGE_OK;
  std::vector<int32_t> ids((size_t)3 * n);
  for (int64_t i = 0; i < n; ++i) {
    if (hs[i] < 0 || hs[i] >= h->dims.n_entities || ts[i] < 0 || ts[i] >= h->dims.n_entities || rs[i] < 0 ||
        rs[i] >= h->dims.n_relations) {
      set_error("triple id out of range");
      return KGE_ERANGE;
    }
    ids[i] = (int32_t)hs[i];
    ids[n + i] = (int32_t)rs[i];
    ids[2 * n + i] = (int32_t)ts[i];
  }
  const int rj = flush_for_io(h, true);  // lag = 1: score the tables with every enqueued update applied
  if (rj != KGE_OK) return rj;
  int32_t* d_ids = nullptr;
  float* d_out = nullptr;
  CK(cudaMallocAsync((void**)&d_ids, (size_t)3 * n * 4, h->stream));
  CK(cudaMallocAsync((void**)&d_out, (size_t)n * 4, h->stream));
  CK(cudaMemcpyAsync(d_ids, ids.data(), (size_t)3 * n * 4, cudaMemcpyHostToDevice, h->stream));
  CK(launch_score(h, d_ids, d_ids + n, d_ids + 2 * n, n, d_out));
  CK(cudaMemcpyAsync(out, d_out, (size_t)n * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaFreeAsync(d_ids, h->stream));
  CK(cudaFreeAsync(d_out, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KGE_OK;
}

// checks a CSR list (off[n+1] from 0, non-decreasing; ids in [0, n_entities)) and packs its ids as int32
static int pack_list(const int64_t* off, const int64_t* ids, int64_t n, int64_t n_ent, bool dedup,
                     std::vector<int64_t>& o, std::vector<int32_t>& v) {
  if (off[0] != 0) { set_error("list offsets must start at 0"); return KGE_EINVAL; }
  o.assign(1, 0);
  for (int64_t i = 0; i < n; ++i) {
    if (off[i + 1] < off[i]) { set_error("list offsets must be non-decreasing"); return KGE_EINVAL; }
    if (off[i + 1] > off[i] && !ids) { set_error("NULL list ids"); return KGE_EINVAL; }
    const size_t b = v.size();
    for (int64_t j = off[i]; j < off[i + 1]; ++j) {
      if (ids[j] < 0 || ids[j] >= n_ent) { set_error("list entity id out of range"); return KGE_ERANGE; }
      v.push_back((int32_t)ids[j]);
    }
    if (dedup) {
      std::sort(v.begin() + b, v.end());
      v.erase(std::unique(v.begin() + b, v.end()), v.end());
    }
    o.push_back((int64_t)v.size());
  }
  return KGE_OK;
}

// validates and narrows the query triples; common to kge_rank / kge_rank_sampled
static int rank_queries(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n,
                        int32_t corrupt, std::vector<int32_t>& ids) {
  if (!h || (n > 0 && (!hs || !rs || !ts))) { set_error("NULL argument"); return KGE_EINVAL; }
  if (h->dims.model == KGE_TRANSR || h->dims.model == KGE_RESCAL || h->P > 1) {
    set_error("kge_rank: TransR, RESCAL and world_size > 1 are not supported");
    return KGE_EUNSUPPORTED;
  }
  if (corrupt < 0 || corrupt > 2) { set_error("corrupt_head must be 0 (tail), 1 (head) or 2 (both)"); return KGE_EINVAL; }
  ids.resize((size_t)3 * n);
  for (int64_t i = 0; i < n; ++i) {
    if (hs[i] < 0 || hs[i] >= h->dims.n_entities || ts[i] < 0 || ts[i] >= h->dims.n_entities || rs[i] < 0 ||
        rs[i] >= h->dims.n_relations) {
      set_error("triple id out of range");
      return KGE_ERANGE;
    }
    ids[i] = (int32_t)hs[i];
    ids[n + i] = (int32_t)rs[i];
    ids[2 * n + i] = (int32_t)ts[i];
  }
  return flush_for_io(h, true);  // lag = 1: rank against the tables with every enqueued update applied
}

// both sides pooled in one S_i (reading c.15'): rank = 1 + #{tail side >=} + #{head side >=} = r_tail + r_head - 1
static void pool_sides(const std::vector<int64_t>& r, int64_t n, int32_t corrupt, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = corrupt == 2 ? r[(size_t)i] + r[(size_t)(n + i)] - 1 : r[(size_t)i];
}

int kge_rank(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, int32_t corrupt_head,
             const int64_t* cand_off, const int64_t* cand_ids, const int64_t* filt_off, const int64_t* filt_ids,
             int64_t* ranks_out) {
  std::vector<int32_t> ids;
  if (n > 0 && !ranks_out) { set_error("NULL argument"); return KGE_EINVAL; }
  if (cand_off && filt_off) {
    set_error("kge_rank: the filter applies to the all-entity protocol only (cand_off must be NULL)");
    return KGE_EINVAL;
  }
  if (cand_off && corrupt_head == 2) {
    set_error("kge_rank: pooled sides with candidate lists is kge_rank_sampled (the lists carry one side each)");
    return KGE_EINVAL;
  }
  int rc = rank_queries(h, hs, rs, ts, n, corrupt_head, ids);
  if (rc != KGE_OK || n == 0) return rc;
  const int nside = corrupt_head == 2 ? 2 : 1;
  std::vector<int64_t> co, fo;
  std::vector<int32_t> cv, fv;
  if (cand_off) {
    rc = pack_list(cand_off, cand_ids, n, h->dims.n_entities, false, co, cv);
    if (rc != KGE_OK) return rc;
  }
  if (filt_off) {  // pooled sides: 2n lists, the tail side's first
    rc = pack_list(filt_off, filt_ids, nside * n, h->dims.n_entities, true, fo, fv);
    if (rc != KGE_OK) return rc;
  }
  // one device block: ids | offsets (8-byte aligned) | list ids | ranks
  const size_t b_ids = (size_t)3 * n * 4, b_co = co.size() * 8, b_fo = fo.size() * 8;
  const size_t o_co = (b_ids + 7) & ~(size_t)7, o_fo = o_co + b_co, o_cv = o_fo + b_fo;
  const size_t o_fv = o_cv + cv.size() * 4, o_out = (o_fv + fv.size() * 4 + 7) & ~(size_t)7;
  char* d = nullptr;
  CK(cudaMallocAsync((void**)&d, o_out + (size_t)nside * n * 8, h->stream));
  CK(cudaMemcpyAsync(d, ids.data(), b_ids, cudaMemcpyHostToDevice, h->stream));
  if (b_co) CK(cudaMemcpyAsync(d + o_co, co.data(), b_co, cudaMemcpyHostToDevice, h->stream));
  if (b_fo) CK(cudaMemcpyAsync(d + o_fo, fo.data(), b_fo, cudaMemcpyHostToDevice, h->stream));
  if (!cv.empty()) CK(cudaMemcpyAsync(d + o_cv, cv.data(), cv.size() * 4, cudaMemcpyHostToDevice, h->stream));
  if (!fv.empty()) CK(cudaMemcpyAsync(d + o_fv, fv.data(), fv.size() * 4, cudaMemcpyHostToDevice, h->stream));
  const int32_t* di = reinterpret_cast<const int32_t*>(d);
  int64_t* d_out = reinterpret_cast<int64_t*>(d + o_out);
  // every entity a candidate on a TF32 handle of a contraction family: the tcgen05 ranking kernel (rank_tc.cu) -- it
  // returns the counts, the rank is 1 + count; otherwise the FFMA streaming kernel
  const bool tcr = !cand_off && rank_tc_supported(h) && getenv("KGE_RANK_FFMA") == nullptr;
  for (int sd = 0; sd < nside; ++sd) {
    const int side = nside == 2 ? sd : (corrupt_head ? 1 : 0);
    const int64_t* fo_d = filt_off ? reinterpret_cast<const int64_t*>(d + o_fo) + (size_t)sd * n : nullptr;
    if (tcr)
      CK(launch_rank_tc(h, di, di + n, di + 2 * n, n, side, fo_d, reinterpret_cast<const int32_t*>(d + o_fv),
                        d_out + (size_t)sd * n));
    else
      CK(launch_rank(h, di, di + n, di + 2 * n, n, side, cand_off ? reinterpret_cast<const int64_t*>(d + o_co) : nullptr,
                     reinterpret_cast<const int32_t*>(d + o_cv), fo_d, reinterpret_cast<const int32_t*>(d + o_fv),
                     d_out + (size_t)sd * n));
  }
  std::vector<int64_t> r((size_t)nside * n);
  CK(cudaMemcpyAsync(r.data(), d_out, (size_t)nside * n * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaFreeAsync(d, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (tcr)
    for (auto& x : r) x += 1;
  pool_sides(r, n, corrupt_head, ranks_out);
  return KGE_OK;
}

int kge_rank_sampled(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n,
                     int32_t corrupt, int32_t n_uniform, int32_t n_degree, uint64_t eval_seed, int64_t* ranks_out) {
  std::vector<int32_t> ids;
  if (n > 0 && !ranks_out) { set_error("NULL argument"); return KGE_EINVAL; }
  if (n_uniform < 0 || n_degree < 0 || (int64_t)n_uniform + n_degree > (1 << 24)) {
    set_error("n_uniform, n_degree must be >= 0 with a sum <= 2^24");
    return KGE_EINVAL;
  }
  int rc = rank_queries(h, hs, rs, ts, n, corrupt, ids);
  if (rc != KGE_OK || n == 0) return rc;
  const int nside = corrupt == 2 ? 2 : 1;
  const int64_t m = (int64_t)n_uniform + n_degree;
  std::vector<int64_t> co((size_t)n + 1);
  for (int64_t i = 0; i <= n; ++i) co[(size_t)i] = i * m;
  // one device block: ids | offsets | candidates of side 0 | of side 1 | ranks
  const size_t b_ids = ((size_t)3 * n * 4 + 7) & ~(size_t)7, b_co = co.size() * 8, b_c = (size_t)n * m * 4;
  const size_t o_co = b_ids, o_c0 = o_co + b_co, o_c1 = o_c0 + b_c, o_out = (o_c1 + (nside - 1) * b_c + 7) & ~(size_t)7;
  char* d = nullptr;
  CK(cudaMallocAsync((void**)&d, o_out + (size_t)nside * n * 8, h->stream));
  CK(cudaMemcpyAsync(d, ids.data(), (size_t)3 * n * 4, cudaMemcpyHostToDevice, h->stream));
  CK(cudaMemcpyAsync(d + o_co, co.data(), b_co, cudaMemcpyHostToDevice, h->stream));
  int32_t* c0 = reinterpret_cast<int32_t*>(d + o_c0);
  int32_t* c1 = nside == 2 ? reinterpret_cast<int32_t*>(d + o_c1) : nullptr;
  CK(launch_eval_cand(h, n, n_uniform, n_degree, corrupt == 2 ? 1 : 0, eval_seed, c0, c1));
  const int32_t* di = reinterpret_cast<const int32_t*>(d);
  int64_t* d_out = reinterpret_cast<int64_t*>(d + o_out);
  for (int sd = 0; sd < nside; ++sd)
    CK(launch_rank(h, di, di + n, di + 2 * n, n, nside == 2 ? sd : (corrupt ? 1 : 0),
                   reinterpret_cast<const int64_t*>(d + o_co), sd ? c1 : c0, nullptr, nullptr, d_out + (size_t)sd * n));
  std::vector<int64_t> r((size_t)nside * n);
  CK(cudaMemcpyAsync(r.data(), d_out, (size_t)nside * n * 8, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaFreeAsync(d, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  pool_sides(r, n, corrupt, ranks_out);
  return KGE_OK;
}

int kge_link_metrics(const int64_t* ranks, int64_t n, double* out) {
  if (!ranks || !out || n <= 0) { set_error("kge_link_metrics: empty rank list or NULL argument"); return KGE_EINVAL; }
  double h1 = 0, h3 = 0, h10 = 0, mr = 0, mrr = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (ranks[i] < 1) { set_error("ranks must be >= 1"); return KGE_EINVAL; }
    h1 += ranks[i] <= 1;
    h3 += ranks[i] <= 3;
    h10 += ranks[i] <= 10;
    mr += (double)ranks[i];
    mrr += 1.0 / (double)ranks[i];
  }
  out[0] = h1 / n;
  out[1] = h3 / n;
  out[2] = h10 / n;
  out[3] = mr / n;
  out[4] = mrr / n;
  return KGE_OK;
}

int64_t kge_step(const kge_handle* h) { return h ? h->step : -1; }

int32_t kge_neg_path(const kge_handle* h) {
  if (!h) return -1;
  if (h->dims.model == KGE_TRANSR) return h->tr_tc ? KGE_PATH_TF32 : KGE_PATH_FFMA;
  if (!tc_supported(h)) return KGE_PATH_FFMA;
  return h->dims.bf16 ? KGE_PATH_BF16 : (h->dims.x3 ? KGE_PATH_3XTF32 : KGE_PATH_TF32);
}

int kge_read_losses(kge_handle* h, int64_t first_step, int64_t n, float* out) {
  if (!h || (n > 0 && !out)) { set_error("NULL argument"); return KGE_EINVAL; }
  if (first_step < 0 || first_step + n > h->step || first_step < h->step - h->ring) {
    set_error("losses are kept for the last 64 steps only");
    return KGE_ERANGE;
  }
  std::vector<float> ring(h->ring);
  CK(cudaMemcpyAsync(ring.data(), h->buf.loss, (size_t)h->ring * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  for (int64_t i = 0; i < n; ++i) out[i] = ring[(first_step + i) % h->ring];
  return check_flags(h);
}

int kge_set_step(kge_handle* h, int64_t step) {
  if (!h || step < 0) { set_error("bad argument"); return KGE_EINVAL; }
  const int rf = kge_flush(h);  // lag = 1: a held-back entity update belongs to the step sequence being left
  if (rf != KGE_OK) return rf;
  h->step = step;
  return KGE_OK;
}

int kge_sync(kge_handle* h) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  return check_flags(h);
}

// Profiling gate: the main stream is held by a spinning kernel until kge_profile_end, so every bracketed launch is
// already queued when the GPU reaches it -- the event pairs then time the kernel alone, not the host's submission
// latency (measured: without the gate each bracket also held ~8 us of host API time). The spin gives up after 2 s
// (a caller that enqueues more work than the queue holds is delayed, never hung).
__global__ void k_profile_gate(const volatile int32_t* flag) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (*flag) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 2000000000ull) return;
    __nanosleep(1000);
  }
}

int kge_profile_begin(kge_handle* h) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  if (!h->prof_gate) {
    if (cudaHostAlloc((void**)&h->prof_gate, 64, cudaHostAllocMapped) != cudaSuccess) {
      cudaGetLastError();
      h->prof_gate = nullptr;
    }
  }
  h->prof.on = true;
  h->prof.used = 0;
  h->prof.kid.clear();
  g_pdl = false;  // isolated per-kernel times (see g_pdl)
  if (h->prof_gate) {
    *(volatile int32_t*)h->prof_gate = 0;
    int32_t* dflag = nullptr;
    if (cudaHostGetDevicePointer((void**)&dflag, h->prof_gate, 0) == cudaSuccess) {
      k_profile_gate<<<1, 1, 0, h->stream>>>(dflag);
      h->prof_gated = true;
    } else {
      cudaGetLastError();
    }
  }
  return KGE_OK;
}

int kge_profile_end(kge_handle* h, int32_t n_kernels, double* avg_ms, int64_t* launches) {
  if (!h || !h->prof.on) { set_error("profiling not active"); return KGE_ESTATE; }
  h->prof.on = false;
  g_pdl = true;
  if (h->prof_gated) {  // release the queued launches
    __atomic_store_n(h->prof_gate, 1, __ATOMIC_SEQ_CST);
    h->prof_gated = false;
  }
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaStreamSynchronize(h->side));
  for (int i = 0; i < kge_handle::kGiven; ++i) CK(cudaStreamSynchronize(h->gside[i]));
  std::vector<double> sum(KGE_K_COUNT, 0.0);
  std::vector<int64_t> cnt(KGE_K_COUNT, 0);
  for (size_t p = 0; p < h->prof.kid.size(); ++p) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->prof.ev[2 * p], h->prof.ev[2 * p + 1]));
    sum[h->prof.kid[p]] += ms;
    cnt[h->prof.kid[p]] += 1;
  }
  for (int k = 0; k < n_kernels && k < KGE_K_COUNT; ++k) {
    if (avg_ms) avg_ms[k] = cnt[k] ? sum[k] / cnt[k] : 0.0;
    if (launches) launches[k] = cnt[k];
  }
  return KGE_OK;
}

int64_t kge_launch_count(const kge_handle* h) { return h ? h->launches : 0; }

int kge_set_option(kge_handle* h, int32_t option, int64_t value) {
  if (!h) { set_error("NULL handle"); return KGE_EINVAL; }
  switch (option) {
    case KGE_OPT_FFMA_SPLITK:
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8) {
        set_error("KGE_OPT_FFMA_SPLITK must be 0 (automatic), 1, 2, 4 or 8");
        return KGE_EINVAL;
      }
      h->ffma_ks_force = (int32_t)value;
      return KGE_OK;
    case KGE_OPT_CAPTURE_NEG:
      if (value != 0 && value != 1) { set_error("KGE_OPT_CAPTURE_NEG must be 0 or 1"); return KGE_EINVAL; }
      if (value && !h->fdbg_buf) {
        h->fdbg_buf = (float*)dalloc(h, (size_t)h->dims.B * h->dims.k * 4);
        if (!h->fdbg_buf) { set_error("out of device memory (capture buffer)"); return KGE_ENOMEM; }
        CK(cudaMemsetAsync(h->fdbg_buf, 0xFF, (size_t)h->dims.B * h->dims.k * 4, h->stream));  // NaN until written
      }
      h->buf.fdbg = value ? h->fdbg_buf : nullptr;
      return KGE_OK;
    case KGE_OPT_BARRIER_MS:
      if (value <= 0) { set_error("KGE_OPT_BARRIER_MS must be > 0"); return KGE_EINVAL; }
      h->barrier_ns = value * 1000000ll;
      return KGE_OK;
  }
  set_error("unknown option");
  return KGE_EINVAL;
}

int kge_debug_neg_scores(kge_handle* h, float* out) {
  if (!h || !out) { set_error("NULL argument"); return KGE_EINVAL; }
  if (!h->buf.fdbg) { set_error("negative-score capture is off (KGE_OPT_CAPTURE_NEG)"); return KGE_ESTATE; }
  CK(cudaMemcpyAsync(out, h->buf.fdbg, (size_t)h->dims.B * h->dims.k * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return KGE_OK;
}

int kge_debug_trace(kge_handle* h, uint64_t* out, int64_t n) {
  if (!h || !out) { set_error("NULL argument"); return KGE_EINVAL; }
  if (!h->dims.trace) { set_error("start with KGE_TRACE=1 in the environment"); return KGE_ESTATE; }
  const int64_t total = (int64_t)KGE_K_COUNT * kTraceCtas * kTraceSlots;
  CK(cudaStreamSynchronize(h->stream));
  CK(cudaMemcpy(out, h->dims.trace, (size_t)std::min(n, total) * 8, cudaMemcpyDeviceToHost));
  return KGE_OK;
}

void kge_destroy(kge_handle* h) {
  if (!h) return;
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->dist.ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : h->dist.raw_allocs) cudaFree(p);
  h->dist.raw_allocs.clear();
  free_all(h);
  for (cudaEvent_t ev : h->prof.ev)
    if (ev) cudaEventDestroy(ev);
  if (h->pinned_given) cudaFreeHost(h->pinned_given);
  for (int i = 0; i < kge_handle::kStage; ++i)
    if (h->stage_ev[i]) cudaEventDestroy(h->stage_ev[i]);
  if (h->pinned_loss) cudaFreeHost(h->pinned_loss);
  if (h->prof_gate) cudaFreeHost(h->prof_gate);
  for (int b = 0; b < 2; ++b) {
    if (h->pin_list[b]) cudaFreeHost(h->pin_list[b]);
    if (h->ev_list[b]) cudaEventDestroy(h->ev_list[b]);
  }
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->ustream) {
    cudaStreamSynchronize(h->ustream);
    cudaStreamDestroy(h->ustream);
  }
  if (h->ev_eread) cudaEventDestroy(h->ev_eread);
  if (h->ev_eupd) cudaEventDestroy(h->ev_eupd);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_samp[i]) cudaEventDestroy(h->ev_samp[i]);
    if (h->ev_free[i]) cudaEventDestroy(h->ev_free[i]);
  }
  for (int i = 0; i < kge_handle::kGiven; ++i) {
    if (h->ev_gsamp[i]) cudaEventDestroy(h->ev_gsamp[i]);
    if (h->ev_gfree[i]) cudaEventDestroy(h->ev_gfree[i]);
  }
  if (h->side) cudaStreamDestroy(h->side);
  for (int i = 0; i < kge_handle::kGiven; ++i)
    if (h->gside[i]) {
      cudaStreamSynchronize(h->gside[i]);
      cudaStreamDestroy(h->gside[i]);
    }
  for (int i = 0; i < kge_handle::kGiven; ++i) {
    if (h->g_samp[i]) cudaGraphExecDestroy(h->g_samp[i]);
    if (h->g_step[i]) cudaGraphExecDestroy(h->g_step[i]);
  }
  for (cudaGraph_t g : h->graphs) cudaGraphDestroy(g);
  if (h->pinned_sink) cudaFreeHost(h->pinned_sink);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  tc_destroy(h);
  transr_destroy(h);
  delete h;
}

}  // extern "C"
