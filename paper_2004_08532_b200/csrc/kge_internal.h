// kge_internal.h -- host-side state of a kge_handle and the launchers each .cu file exports.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/kge.h"

namespace kge {

enum Family : int32_t {  // pair-score family of the chunked negative contraction
  FAM_DOT = 0,   // DistMult, ComplEx: f = o . x
  FAM_L2 = 1,    // TransE-L2: f = gamma - sqrt(sum (o-x)^2)
  FAM_L2SQ = 2,  // RotatE (Table 1, squared), TransR: f = gamma - sum (o-x)^2
  FAM_L1 = 3,    // TransE-L1: f = gamma - sum |o-x|
  FAM_CMOD = 4   // RotatE modulus variant: f = gamma - sum_c |z_c|
};

inline Family family_of(int model, int rotate_variant) {
  switch (model) {
    case KGE_TRANSE_L1: return FAM_L1;
    case KGE_TRANSE_L2: return FAM_L2;
    case KGE_DISTMULT:
    case KGE_COMPLEX: return FAM_DOT;
    case KGE_ROTATE: return rotate_variant ? FAM_CMOD : FAM_L2SQ;
    case KGE_RESCAL: return FAM_DOT;  // o = M^T h | M t, then o . x' (rescal.cu)
    default: return FAM_L2SQ;
  }
}

constexpr int kMaxRanks = 8;

// Entity-row accessor: P == 1 -> the local table; P > 1 -> owner (e mod P) shard, local row e div P (possibly a peer
// mapping over NVLink).
struct EntRows {
  const float* base[kMaxRanks];
  int32_t P;
  int32_t d;
  __host__ __device__ __forceinline__ const float* row(int64_t e) const {
    return P == 1 ? base[0] + e * d : base[e % P] + (e / P) * (int64_t)d;
  }
};

// Per-step sample slot (device pointers into one ring allocation).
struct Slot {
  int32_t* pos;      // [B] triple index
  int32_t* ph;       // [B]
  int32_t* pr;       // [B]
  int32_t* pt;       // [B]
  int32_t* neg;      // [C*k]
  int32_t* mode;     // [C]
  int32_t* ent_n;    // [1] number of unique entities
  int32_t* ent_uniq; // [n_occ]
  int32_t* ent_inv;  // [n_occ]
  int32_t* ent_off;  // [n_occ + 1]
  int32_t* ent_occ;  // [n_occ] occurrences sorted by (id, occ)
  int32_t* rel_n;    // [1]
  int32_t* rel_uniq; // [B]
  int32_t* rel_inv;  // [B]
  int32_t* rel_off;  // [B + 1]
  int32_t* rel_occ;  // [B]
  int32_t* info;     // [4]: the step (mod 2^32), its loss slot (step % loss ring) and the 64-bit device-visible host
                     // address its loss is also stored to (0: none), written by k_sample -- so the step kernels'
                     // parameters depend on the slot only and one captured graph serves every step
};

struct SampleParams {
  const int32_t* th;
  const int32_t* tr;
  const int32_t* tt;
  const int32_t* list;   // rank's triple list, or nullptr for identity
  int64_t n_list;
  const int32_t* given_h;  // caller-supplied positives (kge_train_batch), or nullptr
  const int32_t* given_r;
  const int32_t* given_t;
  int64_t n_entities;
  int32_t B, g, C, k, n_occ, n_pad;  // n_pad: power of two >= n_occ
  uint32_t k0, k1;
  int32_t corrupt;
  uint32_t cg_base;  // rank * C
  int32_t kd;        // degree-based in-batch slots per chunk (kge_config::neg_deg_k)
  int32_t local_P, local_rank;  // local-shard negatives (kge_config::neg_local): P > 1 and this rank, else local_P = 0
  int64_t epoch_steps;  // repartition (reading c.13'): steps per epoch (epoch e = s / epoch_steps, position within it),
                        // 0 = the classic per-rank epochs of reading c.2
};

struct StepBuffers {
  float* O;        // [B x d] combined o_i
  float* onorm;    // [B] ||o_i||^2 (TC L2 path)
  float* X;        // [C*k x d] gathered negative rows
  float* xnorm;    // [C*k]
  float* W;        // [B x k] dL/dS coefficient (C chunks of g x k)
  uint16_t* O16;   // BF16 path: bf16 copies of O [B x dp16], X' [C*k x dp16] (written by the gather) and W [B x kp16]
  uint16_t* X16;   // (written by the forward epilogue), or nullptr
  uint16_t* W16;
  float* O_hi;     // 3xTF32 path: tf32 hi / lo splits of O, X' (gather) and W (forward epilogue), pitch dp / kp
  float* O_lo;
  float* X_hi;
  float* X_lo;
  float* W_hi;
  float* W_lo;
  float* wpos;     // [B] dL/df+
  float* lpos;     // [B] per-positive loss term
  float* pstat;    // [B] pair statistic of each positive (L2: squared distance)
  int32_t* pcnt;   // [B] pairwise ranking loss: active hinges of positive i (integer atomics of the forward epilogues;
                   // zeroed by the gather): dL/df+_i = -pcnt_i / (B k)
  float* lneg;     // [n_neg_parts] per-tile negative loss partials
  float* rowsumW;  // [B]
  float* colsumW;  // [C*k]
  float* dO;       // [B x d]
  float* Gocc;     // [n_occ x d] per-occurrence entity gradients
  float* Grel;     // [B x d_r]
  float* Gproj;    // [B x d*d] (TransR)
  float* loss;     // [ring] per-step loss
  uint32_t* flow;  // [2 C] dataflow counters of the tcgen05 path: [c] rows of chunk c gathered, [C + c] forward CTAs of
                   // chunk c done -- k_tc_fwd / k_tc_bwd start a chunk on these instead of waiting for the whole
                   // predecessor grid; k_update resets them for the next step
  int32_t* flags;  // [4]: [0] non-finite seen, [1] device barrier timed out (P > 1), [2 + step parity] this step's
                   // loss is non-finite (its update is skipped)
  float* fdbg;     // [B x k] captured negative pair scores (KGE_OPT_CAPTURE_NEG), or nullptr
};

// TransR scratch (transr.cu)
struct TrBuffers {
  int32_t* n_groups;  // [1]
  int32_t* grp_u;     // [B] unique-relation index of group
  int32_t* grp_c;     // [B] chunk of group
  int32_t* grp_p0;    // [B] first position in rel_occ
  int32_t* grp_p1;    // [B]
  int32_t* rg_off;    // [B + 1] groups of unique relation u: [rg_off[u], rg_off[u+1])
  int32_t* cg_off;    // [C + 1]
  int32_t* cg_list;   // [B] groups of each chunk, ascending id
  float* QX;          // [B x k x d] projected negatives per group (then P_g)
  float* dQ;          // [B x k x d]
  float* dM;          // [B x d x d] per unique relation
  float* Pv;          // [B x d]  p = Mh + r - Mt
  float* U;           // [(2B + 32 B) x d] gMh, gMt rows (relation-sorted; relation u's 2 n_u rows start at pad_off[u],
  float* H;           // padded to whole 32-row k-blocks with zero rows) / h, t rows, the same layout
  int32_t* pad_off;   // [B + 1] first U / H row of each unique relation (multiples of 32)
  int32_t* n_items;   // [1] k_tr_mv work items: runs of <= 8 positions of one relation
  int32_t* item_u;    // [B + B/8 + 1] unique relation of item
  int32_t* item_p;    // [B + B/8 + 1] first relation-sorted position of item
  int32_t* n_sitems;  // [1] k_tr_score work items: slices of <= kTrSlice positions of one group
  int32_t* sitem_g;   // [B + B/kTrSlice + 1] group of item
  int32_t* sitem_p;   // [B + B/kTrSlice + 1] first relation-sorted position of item
  int32_t* ms_off;    // [B] groups with several slices: first slot of their dQ partials in dQs, else -1
  int32_t* scnt;      // [B x k/32] arrival counters per (group, tile) of the multi-slice groups (reset by the last)
  float* dQs;         // [(2 B / kTrSlice + 2) x k x d] per-slice dQ partials of the multi-slice groups
  int32_t* rel_order;  // [B] unique relations by descending group count (k_tr_dm_tc: the longest CTAs start first)
  int32_t* grp_lc;     // [B] index of a group within its chunk's list
  int32_t* si_off;     // [C + 1] score items of chunk c: [si_off[c], si_off[c + 1])
  float* dOp;         // [kTrJt-tiles x B x d] dO partials of k_tr_score, one per tile of 32 negatives (summed in tile
                      // order by k_tr_chain)
};
constexpr int kTrJt = 32;     // negatives per k_tr_score CTA
constexpr int kTrSlice = 16;  // positives per k_tr_score CTA (a group with more is cut into slices)
__host__ __device__ inline int tr_jtiles(int k) { return (k + kTrJt - 1) / kTrJt; }

// multi-rank state (dist.cu)
struct Dist {
  void* shared = nullptr;       // cudaMalloc'd block exported to peers: flags | ring | Gu | GrelSplit
  size_t shared_bytes = 0;
  uint64_t* flags = nullptr;    // [kMaxRanks] barrier epochs written by each rank
  float* gu = nullptr;          // [n_occ x d] per-unique entity gradient sums of the step being enqueued (= gu_buf[0],
                                // or gu_buf[step & 1] with lag = 1: the owner update of step s-1 reads the other one)
  float* gu_buf[2] = {};
  float* grel_split = nullptr;  // [n_split x drel]
  float* gproj_split = nullptr; // TransR: [n_split x d*d] per-rank sums of the split relations' projection gradients
  int32_t n_split = 0;
  int32_t* split_list = nullptr;   // [n_split] device
  int32_t* split_index = nullptr;  // [n_relations] device, -1 if not split
  std::vector<int32_t> rel_owner;  // host copy of the relation partition
  int32_t* mark = nullptr;      // [rows_local]
  int32_t* contrib = nullptr;   // [P*n_occ x P]
  int32_t* slot_row = nullptr;  // [P*n_occ]
  int32_t* n_slots = nullptr;   // [1]
  float* peer_ent[kMaxRanks] = {};
  void* peer_shared[kMaxRanks] = {};
  float* peer_rel[kMaxRanks] = {};     // every rank's relation table, states and (TransR) projections: the per-epoch
  float* peer_rel_st[kMaxRanks] = {};  // repartition pulls a relation from its previous owner
  float* peer_proj[kMaxRanks] = {};
  float* peer_proj_st[kMaxRanks] = {};
  uint64_t* peer_flags[kMaxRanks] = {};
  std::vector<void*> ipc_opened;
  std::vector<void*> raw_allocs;  // cudaMalloc'd (IPC-exportable) allocations
  uint64_t epoch = 0;            // barrier sequence 0 (main stream)
  uint64_t epoch_u = 0;          // barrier sequence 1 (lag = 1 update stream)
  bool connected = false;
};

struct Dims {
  uint64_t* trace;  // diagnostics (KGE_TRACE=1 at init): per-kernel, per-CTA globaltimer stamps, else nullptr
  int32_t model, family, variant;
  int32_t loss;  // kge_loss
  int32_t d, drel, B, g, C, k, n_occ;
  int32_t dp, kp;  // padded row pitch of O / X' (d + 2 rounded up to 32) and of W (k rounded up to 32)
  int32_t dp16, kp16;  // BF16 copies: pitch of O16 / X16 (d rounded up to 64) and of W16 (k rounded up to 64)
  int32_t bf16;        // 1: the tcgen05 path contracts BF16 operand copies (KGE_PREC_BF16)
  int32_t x3;          // 1: 3xTF32 split precision (KGE_PREC_3XTF32)
  float gamma, lr, eps;
  int64_t n_entities, n_relations;
};

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // pairs
  std::vector<int32_t> kid;
  size_t used = 0;
};

}  // namespace kge

struct kge_handle {
  kge_config cfg{};
  kge::Dims dims{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // tables
  float* ent = nullptr;
  float* rel = nullptr;
  float* proj = nullptr;
  float* ent_st = nullptr;
  float* rel_st = nullptr;
  float* proj_st = nullptr;
  // graph
  int32_t* th = nullptr;
  int32_t* tr = nullptr;
  int32_t* tt = nullptr;
  int32_t* list = nullptr;
  int64_t n_triples = 0, n_list = 0;
  // per-epoch repartition (kge_config::repartition, P > 1)
  std::vector<int64_t> host_rels;
  int64_t epoch_steps = 0, cur_epoch = -1;
  int32_t* d_owner_prev = nullptr;  // [n_relations] owner map of the epoch being left (device, for the pull)
  std::vector<int32_t> owner_prev;  // its host source
  int32_t* pin_list[2] = {};        // pinned staging of the epoch lists
  cudaEvent_t ev_list[2] = {};
  int list_flip = 0;
  // sampling ring
  int32_t ring = 0;
  std::vector<kge::Slot> slots;
  kge::Slot debug_slot{};
  // sampling runs on a side stream ahead of the steps (k_sample is a pure function of (seed, step)): the ring is two
  // halves of ring/2 steps; while the main stream works through one half the side stream fills the other
  cudaStream_t side = nullptr;
  // lag = 1 (reading c.12): the entity update of step s runs on ustream after step s+1 stops reading the entity table
  // (ev_eread) and before step s+2's gather (ev_eupd); Gocc is double-buffered by step parity
  cudaStream_t ustream = nullptr;
  cudaEvent_t ev_eread = nullptr, ev_eupd = nullptr;
  int64_t pend_step = -1;   // step whose entity update is held back (-1: none)
  kge::Slot pend_slot{};
  int32_t pend_gi = -1;     // its caller-batch slot, or -1 (ring slot)
  bool eupd_enqueued = false;
  float* gocc2[2] = {};     // the two Gocc buffers (lag = 1), else both = buf.Gocc
  // FFMA negative kernels: deterministic split-K scratch (partial tiles + arrival counters)
  float4* ffma_part = nullptr;
  int32_t* ffma_cnt = nullptr;
  int32_t ffma_ks_max = 1;  // the split factor the scratch was sized for
  int32_t ffma_ks_force = 0;  // KGE_OPT_FFMA_SPLITK (0 = automatic)
  float* fdbg_buf = nullptr;  // KGE_OPT_CAPTURE_NEG target, allocated on first use; buf.fdbg points here when on
  int64_t barrier_ns = 120000000000ll;  // KGE_OPT_BARRIER_MS
  const kge::Slot* next_slot = nullptr;  // device slot of the step after the one being enqueued (row prefetch)
  cudaEvent_t ev_samp[2] = {}, ev_free[2] = {};
  int64_t half_first[2] = {-1, -1};  // first step held by each ring half (-1: none)
  bool half_waited[2] = {false, false};
  // caller-supplied batches (kge_train_batch): kGiven slots sampled on the side stream, so the sample of batch s+1
  // overlaps step s
  static constexpr int kGiven = 8;
  kge::Slot given_slots[kGiven] = {};
  cudaStream_t gside[kGiven] = {};  // one high-priority stream per given slot: the single-step samples of consecutive
                                    // batches (~50 us each) run concurrently instead of queueing on one stream
  cudaEvent_t ev_gsamp[kGiven] = {}, ev_gfree[kGiven] = {};
  // CUDA graphs of the caller-batch path (P == 1, no profiler / trace / debug sync), one pair per given slot: the
  // upload + sample (side stream) and the step kernels + loss readback (main stream); per launch only the sampler's
  // step and the readback addresses change (node parameter updates), which keeps the host cost per step far below
  // the device time
  cudaGraphExec_t g_samp[kGiven] = {}, g_step[kGiven] = {};
  cudaGraphNode_t g_samp_node[kGiven] = {}, g_loss_node[kGiven] = {};
  bool g_loss_on[kGiven] = {true, true, true, true, true, true, true, true};  // state of each D2H loss node
  std::vector<cudaGraph_t> graphs;  // source graphs of the instantiated ones
  int32_t g_launches = 0;       // kernels per captured step (launch counter)
  float* pinned_sink = nullptr;  // readback target when the caller passes no loss pointer
  int32_t* given = nullptr;  // [kGiven][3 x B] device copies of caller positives (one per given slot)
  // device-side sample gate (P == 1, lag 0, step kernels launched directly with PDL): k_sample of given slot i bumps
  // gready[i] once per CTA, the step's k_wait_ready waits for 2 x (samples enqueued into slot i) = 2 x gcount[i]
  uint32_t* gready = nullptr;
  uint32_t gcount[kGiven] = {};
  static constexpr int kStage = kGiven;  // staging buffer i feeds given slot i (the captured upload reads it)
  int32_t* pinned_given = nullptr;  // host pinned staging: kStage buffers of 3B int32 (caller-supplied batches)
  cudaEvent_t stage_ev[kStage] = {};  // recorded after each staging buffer's H2D copy
  float* pinned_loss = nullptr;
  // step
  kge::StepBuffers buf{};
  int32_t n_neg_parts = 0;
  int64_t step = 0;
  int64_t launches = 0;
  kge::Profiler prof;
  int32_t* prof_gate = nullptr;  // mapped pinned flag of the profiling gate (kge_profile_begin / end)
  bool prof_gated = false;
  std::vector<void*> allocs;
  // sizes
  uint32_t k0 = 0, k1 = 0;
  int32_t n_pad = 0;
  int32_t dp = 0, kp = 0;
  void* tc = nullptr;  // TcState (tc.cu)
  kge::TrBuffers tr_buf{};
  void* tr_tc = nullptr;  // TransR tcgen05 projection state (transr.cu), or nullptr (FFMA)
  // ranks
  int32_t P = 1, rank = 0;
  int64_t ent_rows = 0;  // rows of the local entity table (shard when P > 1)
  int32_t* seg_cnt = nullptr;  // [B + n_occ] k_update segment arrival counters
  kge::EntRows rows{};
  kge::Dist dist;
};

namespace kge {

// Programmatic dependent launch on/off (off while the profiler brackets each launch with events, so the per-kernel
// times are those of each kernel alone rather than including the wait for its predecessor)
extern bool g_pdl;

// Launch with programmatic stream serialization (PDL); see pdl_wait / pdl_trigger in device_common.cuh.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// PDL launch with a thread-block cluster of (cx, 1, 1)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_cluster(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                      unsigned cx, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cx;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// launch bracketing for the profiler / launch counter
void launch_begin(kge_handle* h, int kid);
void launch_end(kge_handle* h, int kid);

// sample.cu
size_t sample_smem_bytes(int n_pad);
cudaError_t sample_init();
cudaError_t launch_sample(kge_handle* h, const SampleParams& p, const Slot* slots_dev_array, int ring, int64_t step0, int n_steps,
                          cudaStream_t stream = nullptr, uint64_t loss_dst = 0,
                          uint32_t* ready = nullptr);  // nullptr stream: h->stream
// main-stream gate for a side-stream sample (see k_wait_ready)
cudaError_t launch_wait_ready(kge_handle* h, const uint32_t* ready, uint32_t want);
// re-point a captured k_sample node at another first step
cudaError_t sample_graph_set(kge_handle* h, cudaGraphExec_t exec, cudaGraphNode_t node, const SampleParams& p,
                             const Slot* slots_dev_array, int ring, int64_t step0, int n_steps, uint64_t loss_dst,
                             uint32_t* ready = nullptr);
cudaError_t launch_init_table(kge_handle* h, float* tab, int64_t rows, int32_t w, uint32_t table_id, float bound,
                              int64_t row_stride = 1, int64_t row_offset = 0);
cudaError_t launch_convert_ids(kge_handle* h, const int64_t* src, int32_t* dst, int64_t n, int64_t limit, int32_t* bad);

// step.cu
cudaError_t launch_step(kge_handle* h, const Slot& s, int64_t step);
cudaError_t launch_score(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, float* out);
cudaError_t launch_rank(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, int head,
                        const int64_t* cand_off, const int32_t* cand, const int64_t* filt_off, const int32_t* filt,
                        int64_t* ranks);
cudaError_t launch_rows(kge_handle* h, float* tab, int32_t w, const int32_t* ids, int64_t n, float* buf, bool write);
bool rank_tc_supported(const kge_handle* h);  // rank_tc.cu: tcgen05 all-entity ranking for this handle
cudaError_t launch_rank_tc(kge_handle* h, const int32_t* hs, const int32_t* rs, const int32_t* ts, int64_t n, int head,
                           const int64_t* filt_off, const int32_t* filt, int64_t* ranks);  // ranks - 1 (counts)
cudaError_t launch_eval_cand(kge_handle* h, int64_t n, int32_t n_uniform, int32_t n_degree, int32_t both,
                             uint64_t seed, int32_t* cand_t, int32_t* cand_h);

cudaError_t launch_gather_neg(kge_handle* h, const Slot& s);
cudaError_t launch_update(kge_handle* h, const Slot& s);
cudaError_t launch_update_range(kge_handle* h, const Slot& s, int lo, int hi, cudaStream_t st, float* gocc);

// transr.cu
cudaError_t launch_transr_step(kge_handle* h, const Slot& s, int64_t step);
cudaError_t launch_proj_update(kge_handle* h, const Slot& s);
// rescal.cu
cudaError_t launch_rescal_step(kge_handle* h, const Slot& s, int64_t step);
bool rescal_init(kge_handle* h);
bool transr_init(kge_handle* h);
void transr_destroy(kge_handle* h);
void transr_tc_init(kge_handle* h);  // tcgen05 projections (TF32 negatives path)

// dist.cu
int32_t relation_partition(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, std::vector<int32_t>& owner,
                           bool randomise = false, uint64_t seed = 0, uint32_t epoch = 0);
int64_t rank_list(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, int32_t rank,
                  const std::vector<int32_t>& owner, std::vector<int32_t>* out);
cudaError_t dist_barrier(kge_handle* h);
cudaError_t dist_preload();
cudaError_t step_preload();
cudaError_t dist_exchange_update(kge_handle* h, const Slot& s, int64_t step);
cudaError_t dist_clear_split(kge_handle* h);  // zero this rank's split-relation gradient sums before a step
cudaError_t dist_pull_relations(kge_handle* h, const int32_t* owner_prev);  // epoch switch (repartition)
cudaError_t dist_owner_update_lagged(kge_handle* h, const Slot& s, int64_t step, cudaStream_t st);
cudaError_t dist_owner_flush(kge_handle* h, const Slot& s, int64_t step);

// tc.cu
bool tc_init(kge_handle* h);
void tc_destroy(kge_handle* h);
bool tc_supported(const kge_handle* h);
int32_t tc_neg_parts(const kge_handle* h);
// the step's loss goes to the ring slot named by the sample slot (Slot::info); when tc_fuses_chain(h) the backward
// kernel also applies the positive chain
// rule and reduces the loss (k_chain is not launched)
cudaError_t launch_tc_neg(kge_handle* h, const Slot& s);
bool tc_fuses_chain(const kge_handle* h);
bool tc_flow();  // chunk-level dataflow counters on (KGE_FLOW=1)
// 3D TMA map over a [chunks x rows x cols] fp32 buffer (row pitch in floats), box {32, box_rows, 1}; out-of-range
// columns / rows read as zeros
bool make_map(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows,
              CUtensorMapSwizzle sw);
bool make_map4c(CUtensorMap* m, const float* base, int cols, int rows, int chunks, int pitch, int box_rows, int box_kb,
                CUtensorMapSwizzle sw);  // tc.cu

}  // namespace kge
