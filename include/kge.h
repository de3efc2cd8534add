/* kge.h -- C-ABI of libkge.so, the B200-native (sm_100a) DGL-KE mini-batch KGE training step.
 *
 * The operation is the four-step mini-batch loop of PAPER.md:314-344 (Sec. 3.1):
 *   (1) sample b positive triplets of the local partition and their negatives (joint negative
 *       sampling PAPER.md:417-428, Sec. 3.3: chunks of g positives share k uniformly drawn corrupting entities),
 *   (2) fetch the entity and relation rows the batch touches,
 *   (3) forward + backward of the Table-1 score (Sec. 2) under the logistic loss,
 *       negatives scored as a generalised matrix product o x t'^T,
 *   (4) apply sparse row-wise Adagrad to the touched rows (sparse updates PAPER.md:262-266,
 *       472-474), duplicate-row gradients summed by sort + segmented reduce first.
 * Readings of the paper where it is silent (RNG, positive order, head/tail schedule, margin placement, loss
 * normalisation, init, optimizer) are DESIGN.md "Readings" = SURVEY.md 8(c) c.1-c.14; the CPU oracle in oracle/
 * implements the same readings independently.
 *
 * Conventions for every entry point:
 *  - Return value is a kge_status; nothing throws across the ABI. On a non-OK return kge_last_error() gives a
 *    thread-local message. A failed call leaves the handle usable unless it returns KGE_ECUDA / KGE_ENCCL.
 *  - Host pointers are caller-owned and only read / written during the call. Device memory (tables, triples,
 *    workspaces) is owned by the handle, allocated through cfg.dev_alloc / dev_free when given (PyTorch's caching
 *    allocator in the Python binding) else cudaMalloc, and freed by kge_destroy.
 *  - Work is enqueued on cfg.cuda_stream (NULL -> a stream the handle creates). Calls that only enqueue return
 *    before the GPU finishes; calls with host outputs synchronise that stream before returning.
 *  - Ids are int64 at the ABI; the device stores int32, so n_entities, n_relations, n_triples must be < 2^31.
 *  - Not thread-safe per handle. With world_size > 1, kge_init and kge_train_step are collective (every rank calls
 *    them in the same order, NCCL semantics).
 *  - There is no CPU fallback: without a usable sm_100 device kge_init returns KGE_ECUDA.
 */
#ifndef KGE_H
#define KGE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KGE_ABI_VERSION 4  /* 2: kge_config::neg_deg_k; 3: kge_config::neg_local (validated: 0 or 1); 4: loss */

typedef struct kge_handle kge_handle; /* opaque, library-owned */

/* Table 1 models. */
typedef enum {
  KGE_TRANSE_L1 = 0, /* gamma - ||h + r - t||_1 */
  KGE_TRANSE_L2 = 1, /* gamma - ||h + r - t||_2 (not squared) */
  KGE_DISTMULT = 2,  /* h^T diag(r) t */
  KGE_COMPLEX = 3,   /* Re(h^T diag(r) conj(t)); rows [re(d/2) | im(d/2)] */
  KGE_ROTATE = 4,    /* gamma - ||h o e^{i theta} - t||^2 (variant 1: gamma - sum_j |.|); relation = d/2 phases */
  KGE_TRANSR = 5,    /* gamma - ||M_r h + r - M_r t||_2^2, M_r d x d row-major */
  KGE_RESCAL = 6     /* h^T M_r t, M_r d x d row-major in table 2; the relation table (1, 4) is unused
                        (never updated); TF32 / FP32 negatives only (BF16, lag = 1: KGE_EUNSUPPORTED) */
} kge_model;

typedef enum {
  KGE_OK = 0,
  KGE_EINVAL = -1,       /* bad configuration / argument (g does not divide B, odd d for ComplEx/RotatE, k<=0, ...) */
  KGE_ERANGE = -2,       /* an id out of range, or a size >= 2^31 */
  KGE_ENOMEM = -3,       /* device allocation failed */
  KGE_ECUDA = -4,        /* CUDA error (incl. no sm_100 device); handle should be destroyed */
  KGE_ENCCL = -5,        /* NCCL error */
  KGE_ENONFINITE = -6,   /* a step produced a non-finite loss; that step's update was skipped on the device */
  KGE_ESTATE = -7,       /* call not valid in the handle's state */
  KGE_EUNSUPPORTED = -8  /* valid request this build does not implement */
} kge_status;

/* Corruption schedule (reading c.4; "corrupt the head entities in a similar fashion"). */
typedef enum { KGE_CORRUPT_TAIL = 0, KGE_CORRUPT_HEAD = 1, KGE_CORRUPT_ALTERNATE = 2 } kge_corrupt;

/* Arithmetic of the chunked negative contraction. FP32 = FFMA (all models; the parity path);
 * TF32 = tcgen05 tensor cores with TMEM accumulators (DistMult, ComplEx, and TransE-L2 / Table-1 RotatE via
 * ||o - x||^2 = ||o||^2 - 2 o.x + ||x||^2; TransR projections); BF16 = the same contractions (forward S = O X'^T and
 * both backward GEMMs) on BF16 copies of O, X' and W with fp32 TMEM accumulators (kind::f16; not for TransR:
 * KGE_EUNSUPPORTED). 3XTF32 = the same contractions in split precision: every operand x =
 * hi + lo (hi a tf32 value, lo = x - hi exact), S = hi.hi + hi.lo + lo.hi on the tensor cores -- FP32-level
 * accuracy at three MMAs per K slice (not for TransR / RESCAL: KGE_EUNSUPPORTED). TransE-L1 and the RotatE modulus
 * variant are not contractions and run FFMA at any setting (kge_neg_path reports which path a handle took). */
typedef enum { KGE_PREC_FP32 = 0, KGE_PREC_TF32 = 1, KGE_PREC_BF16 = 2, KGE_PREC_3XTF32 = 3 } kge_precision;

/* Loss (PAPER.md:239-249 [2], "two loss functions are commonly used"): LOGISTIC = sum log(1 + exp(-y f)) (L243;
 * normalisation reading c.9: mean over positives + mean over negatives); PAIRWISE = the pairwise ranking loss
 * sum max(0, gamma - f+ + f-) (L247-249; reading c.9': each positive paired with its chunk's k negatives, mean over
 * the B*k pairs, hinge subgradient 0 at 0). */
typedef enum { KGE_LOSS_LOGISTIC = 0, KGE_LOSS_PAIRWISE = 1 } kge_loss;

typedef struct {
  int32_t abi_version;     /* = KGE_ABI_VERSION */
  int32_t model;           /* kge_model */
  int64_t n_entities;      /* |V| */
  int64_t n_relations;     /* number of relation types */
  int32_t dim;             /* d: floats per entity row; multiple of 4 (of 8 for ComplEx/RotatE) */
  int32_t batch_size;      /* b positives per step per rank */
  int32_t chunk_size;      /* g positives sharing one negative set; must divide batch_size */
  int32_t neg_k;           /* k negatives per chunk */
  float gamma;             /* margin gamma; enters f = gamma + f_T1 for distance models (reading Q7) */
  float lr;                /* Adagrad learning rate */
  float adagrad_eps;       /* epsilon inside sqrt(state + eps); <= 0 -> 1e-10 */
  float init_bound;        /* <= 0 -> (gamma+2)/d if gamma > 0 else 1/sqrt(d) (reading c.6) */
  uint64_t seed;           /* Philox key for sampling and init (reading c.1) */
  int32_t corrupt;         /* kge_corrupt */
  int32_t neg_precision;   /* kge_precision */
  int32_t rotate_variant;  /* RotatE: 0 = Table-1 squared (default), 1 = modulus sum */
  int32_t lag;             /* 0 = synchronous (reading c.12). 1 = the paper's overlap of the entity update with the next
                              mini-batch (PAPER.md:515-534 [3.5]) made deterministic: step s reads entity rows updated
                              by steps <= s-2 and relation rows by steps <= s-1; the entity update of the last step
                              is held back until the next step or kge_flush. With world_size > 1 the held-back part
                              is the owner's Adagrad step of the exchanged entity gradients, run on an update stream
                              while the next step computes (after every rank's entity reads of that step). TransR ->
                              KGE_EUNSUPPORTED. */
  int32_t world_size;      /* P ranks (one process per GPU) */
  int32_t rank;            /* this rank */
  void* nccl_comm;         /* reserved, ignored: the P > 1 exchange runs over CUDA-IPC peer memory inside the step
                              kernels (handles from kge_export / kge_connect, rendezvous by the caller's process group;
                              DESIGN.md §6 gives the bytes / latency argument against an NCCL all-to-all) */
  const void* nccl_unique_id; /* reserved, ignored (as nccl_comm) */
  void* cuda_stream;       /* cudaStream_t to enqueue on, or NULL */
  void* (*dev_alloc)(size_t bytes, void* ctx); /* optional device allocator */
  void (*dev_free)(void* ptr, void* ctx);
  void* alloc_ctx;
  int32_t neg_deg_k;       /* slots j < neg_deg_k of every chunk are degree-based in-batch negatives (PAPER.md:437-448
                              [3.3]: the tail (tail corruption) / head (head corruption) of a uniformly drawn triplet
                              of the mini-batch, Philox stream DEG = 4); the rest uniform. 0 (default) = all uniform;
                              must be <= neg_k */
  int32_t neg_local;       /* 1: with world_size > 1 the uniform negatives of rank w come from its own entity shard
                              {e : e mod P == w} (PAPER.md:451-456 [3.3] local negatives: no remote rows for them);
                              the draw of reading c.3 mapped to e = w + P * floor(u * n_w / 2^64). Default 0 */
  int32_t loss;            /* a kge_loss value; default LOGISTIC */
  int32_t repartition;     /* 1 with world_size > 1: a different, randomised relation partition every epoch (PAPER.md:
                              497-501 [3.4]; reading c.13': epochs of ceil(N_t / (P B)) steps on every rank, the
                              non-split relations ordered by (count desc, Philox(r, epoch, REPART = 6) asc); the SPLIT
                              set is unchanged). At an epoch boundary kge_train_step re-partitions (host) and every rank
                              pulls the relations it did not own from their previous owner. Default 0; sampled steps
                              only (kge_train_batch with repartition: KGE_EUNSUPPORTED) */
  int32_t placement;       /* world_size > 1: 0 = relation partition (reading c.13); 1 = head-owner
                              placement (PAPER.md:395-406 [3.2], reading c.13''): triple i trains on the rank owning its
                              head (h mod P), so every head row is local; all relations are then replicated and their
                              gradients exchanged (the SPLIT path). With kge_locality_order's renumbering and
                              neg_local = 1 most rows of a step are local. Default 0; not with repartition */
} kge_config;

/* Fill *cfg with defaults (ABI version, TransE-L2, d=400, B=1024, g=256, k=256, gamma=12, lr=0.1, eps=1e-10,
 * seed=1, ALTERNATE, TF32, P=1). Never fails. */
void kge_config_default(kge_config* cfg);

/* Create a handle: validate cfg, copy the triples (h, r, t) of the whole graph to the device,
 * compute this rank's triple list (relation partitioning PAPER.md:476-495 when world_size > 1), allocate and
 * Philox-initialise the tables (reading c.6) and zero the Adagrad states.
 * heads/rels/tails: host int64[n_triples], caller-owned, read during the call only.
 * Errors: KGE_EINVAL (config), KGE_ERANGE (id out of range / sizes >= 2^31), KGE_ENOMEM, KGE_ECUDA, KGE_ENCCL. */
int kge_init(kge_handle** out, const kge_config* cfg, const int64_t* heads, const int64_t* rels, const int64_t* tails,
             int64_t n_triples);

/* Run the sampler of step `step` (steps (1) of Sec. 3.1 and the dedup of the touched rows) and copy its results to
 * host buffers; any pointer may be NULL. Sizes: pos_idx[B] (triple indices), neg[C*k] (C = B/g, chunk-major),
 * mode[C] (0 tail, 1 head), uniq_ent[2B+C*k] (ascending distinct entity ids over occurrences
 * [h_0..h_{B-1}, t_0..t_{B-1}, neg...]), inv_ent[2B+C*k] (position of each occurrence's id in uniq_ent),
 * uniq_rel[B], inv_rel[B] likewise for [r_0..r_{B-1}]. Synchronous. Does not advance the step counter. */
int kge_sample(kge_handle* h, int64_t step, int64_t* pos_idx, int64_t* neg, int8_t* mode, int64_t* uniq_ent,
               int64_t* n_uniq_ent, int32_t* inv_ent, int64_t* uniq_rel, int64_t* n_uniq_rel, int32_t* inv_rel);

/* Enqueue n_steps training steps (sample -> gather -> score fwd/bwd -> dedup-sum -> Adagrad), advancing the step
 * counter. loss_out: host float[n_steps] receiving each step's loss (then the call synchronises), or NULL (the call
 * returns after enqueueing). KGE_ENONFINITE is reported by the first synchronising call after the offending step. */
int kge_train_step(kge_handle* h, int64_t n_steps, float* loss_out);

/* One step on a caller-supplied batch of B positive triples (host int64 heads/rels/tails[B]); negatives are still
 * drawn on the device for the current step counter. Copies the batch host->device, runs the step, and (if loss_out
 * is not NULL) reads the loss back. This is the end-to-end entry for a host-side sampler. */
int kge_train_batch(kge_handle* h, const int64_t* heads, const int64_t* rels, const int64_t* tails, float* loss_out);

/* Asynchronous kge_train_batch for a pipelined host loop: the batch is range-checked and staged synchronously (the
 * caller's arrays may be reused on return), the H2D copy, the step and -- if loss_host is not NULL -- the D2H copy of
 * the step's loss into loss_host are enqueued and the call returns. loss_host should be pinned (cudaMallocHost /
 * torch pin_memory) and is valid after the next kge_sync; KGE_ENONFINITE is reported by that kge_sync.
 * The upload and sample run on a side stream; the step's first kernel waits for them on the device (a ready counter,
 * 5 s limit: KGE_ECUDA "sample gate timed out" from the next synchronising call, which should never happen). */
int kge_train_batch_async(kge_handle* h, const int64_t* heads, const int64_t* rels, const int64_t* tails,
                          float* loss_host);

/* Scores f(h, r, t) of n triples with the current tables (Table 1 with the margin of reading Q7). out: host
 * float[n]. Synchronous. KGE_ERANGE on an out-of-range id. */
int kge_score(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, float* out);

/* Link-prediction ranks (PAPER.md:652-665 [5.3] evaluation methodology). For each test triple i
 * the true entity is scored against its corruptions with the current tables -- candidates and the true triple through
 * the same arithmetic (o = combine(h, r) or combine'(r, t), then the pair score of Table 1). corrupt_head: 0 = the
 * tail is replaced, 1 = the head, 2 = both: one list S_i holding the corruptions (h', r, t) AND (h, r, t') (the
 * paper's first protocol, reading c.15'). rank_i = 1 + #{corruptions c != the positive, not filtered : f(c) >=
 * f(true)} -- ties rank the positive last (reading c.15).
 *   cand_off == NULL: every entity corrupts the side(s) (first protocol; raw if filt_off == NULL).
 *   cand_off/cand_ids: the side's candidates cand_ids[cand_off[i] .. cand_off[i+1]) (duplicates count once per
 *     occurrence, the true entity is skipped); not with corrupt_head = 2 (KGE_EINVAL: see kge_rank_sampled).
 *   filt_off/filt_ids: filtered first protocol -- the corrupted entities that form a known triple are removed
 *     (never scored); per query list i = filt_ids[filt_off[i] .. filt_off[i+1]) (duplicates removed here). With
 *     corrupt_head = 2 there are 2n lists (offsets [2n+1]): lists 0..n-1 hold the tail side, n..2n-1 the head side.
 *     Only with cand_off == NULL, else KGE_EINVAL.
 * Offsets: host int64, from 0, non-decreasing (KGE_EINVAL otherwise); ids: host int64, each in [0, N_e)
 * (KGE_ERANGE otherwise). hs/rs/ts: host int64[n]; ranks_out: host int64[n], owned by the caller. Synchronous.
 * KGE_EUNSUPPORTED for TransR or world_size > 1. */
int kge_rank(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, int32_t corrupt_head,
             const int64_t* cand_off, const int64_t* cand_ids, const int64_t* filt_off, const int64_t* filt_ids,
             int64_t* ranks_out);

/* Second protocol (PAPER.md:656-658 [5.3]: "2000 negative triplets; 1000 sampled uniformly from the entire set of
 * negative samples and 1000 sampled proportionally to the degree of the corrupted entities", unfiltered), candidates
 * drawn on the device (reading c.15'): slot j < n_uniform + n_degree of query i draws u from Philox(ctr = (j/2,
 * lo32(i), hi32(i), EVAL = 5), key = eval_seed); uniform slots take an entity uniform over N_e (corrupt = 2: a
 * (side, entity) pair uniform over the 2 N_e corruptions), degree slots a uniform endpoint of the graph's triples (an
 * entity drawn proportionally to its degree; corrupt = 2: plus a uniform side bit). Ranks as kge_rank over these
 * candidates (corrupt 0 / 1 / 2 as there). Synchronous; errors as kge_rank, KGE_EINVAL for negative counts. */
int kge_rank_sampled(kge_handle* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n,
                     int32_t corrupt, int32_t n_uniform, int32_t n_degree, uint64_t eval_seed, int64_t* ranks_out);

/* Hit@1, Hit@3, Hit@10, MR and MRR of n ranks (PAPER.md:660-664 [5.3] formulas) into out[5] (host). KGE_EINVAL for
 * n <= 0 or a rank < 1. */
int kge_link_metrics(const int64_t* ranks, int64_t n, double* out);

/* Read / overwrite rows of a table: 0 entity [N_e x d], 1 relation [N_r x d_r] (d_r = d, or d/2 for RotatE),
 * 2 TransR projection [N_r x d*d], 3 entity Adagrad state [N_e x 1], 4 relation state, 5 projection state.
 * ids: host int64[n]; out/in: host float[n x width]. Synchronous. KGE_EINVAL for a table the model lacks. */
int kge_get_rows(kge_handle* h, int32_t table, const int64_t* ids, int64_t n, float* out);
int kge_set_rows(kge_handle* h, int32_t table, const int64_t* ids, int64_t n, const float* in);
int32_t kge_table_width(const kge_handle* h, int32_t table);

/* Arithmetic the chunked negative contraction of this handle runs in: KGE_PATH_FFMA (FP32 FFMA
 * tiles: the FP32 precision, and TransE-L1 / the RotatE modulus variant at any precision), KGE_PATH_TF32 (tcgen05
 * kind::tf32 with TMEM accumulators: DistMult, ComplEx, TransE-L2, Table-1 RotatE, TransR projections), KGE_PATH_BF16
 * (tcgen05 kind::f16 on BF16 operands, the same models but TransR). -1 for NULL. */
enum { KGE_PATH_FFMA = 0, KGE_PATH_TF32 = 1, KGE_PATH_BF16 = 2, KGE_PATH_3XTF32 = 3 };
int32_t kge_neg_path(const kge_handle* h);

/* Next step index (steps are counter-based: (seed, step) fixes every sample, so resume is exact). */
int64_t kge_step(const kge_handle* h);
int kge_set_step(kge_handle* h, int64_t step);
/* lag = 1: apply the held-back entity update of the last step now (no-op when none / lag = 0). kge_set_step flushes.
 * One rank: kge_get_rows / kge_set_rows / kge_score / kge_rank flush implicitly. world_size > 1: collective (every rank
 * calls it, like kge_train_step); reading or writing entity rows (tables 0, 3) or scoring while an update is held back
 * returns KGE_ESTATE. */
int kge_flush(kge_handle* h);

/* Wait for all enqueued work; reports KGE_ENONFINITE if any step since the last check had a non-finite loss. */
int kge_sync(kge_handle* h);

/* Losses of recent steps (the last 64) from the device ring; synchronises. For the single-process multi-rank emulation,
 * where a per-call loss readback would block the other ranks' progress. */
int kge_read_losses(kge_handle* h, int64_t first_step, int64_t n, float* out);

/* ---- P > 1 ranks (one process per GPU of one node) ----
 * Partition (reading c.13; PAPER.md:476-495 [3.4]): relations with count > N_t/P are split and their triples dealt
 * round-robin; the others go, by frequency, to the lightest rank. Entity rows are sharded owner = e mod P, local row =
 * e div P. After kge_init, every rank exports the IPC handles of its shard and exchange block
 * (kge_export), the caller gathers the P blobs (e.g. torch.distributed.all_gather_object) and passes them, in rank
 * order, to kge_connect. kge_train_step is then collective: gather reads rows from their owners over NVLink, owners pull
 * the per-rank gradient sums of their rows and apply one Adagrad step per row (the union-batch semantics of c.13).
 * For table 0 / 3, kge_get_rows / kge_set_rows take global ids owned by this rank. */
/* METIS-style locality ordering (PAPER.md:395-406 [3.2] deploys METIS; reading c.13'', SPEC's BFS-grown balanced
 * partitioner): part w of the entity graph (the undirected edges (h_i, t_i)) takes exactly ceil((N_e - w) / P)
 * entities -- from the lowest-id unassigned entity, breadth-first with neighbours in ascending id, an entity joining
 * when discovered, a new seed when the frontier empties -- and new_id[e] = P j + w (j = e's position in part w by
 * ascending old id) puts part w on rank w's shard (owner = id mod P). The caller renumbers its triples (and evaluation
 * data) with new_id before kge_init; with placement = 1 a triple's head and tail then share a rank unless the edge is
 * cut. new_id_out: host int64[n_entities]; edge_cut_out: triples whose endpoints fall in different parts (or NULL).
 * Host only; KGE_EINVAL / KGE_ERANGE for bad sizes or ids. */
int kge_locality_order(const int64_t* heads, const int64_t* tails, int64_t n_triples, int64_t n_entities,
                       int32_t world_size, int64_t* new_id_out, int64_t* edge_cut_out);
int kge_partition(const int64_t* rels, int64_t n_triples, int64_t n_relations, int32_t world_size, int32_t rank,
                  int32_t* owner_out /* [n_relations] rank or -1 = split, or NULL */,
                  int64_t* list_out /* this rank's triple indices (ascending), or NULL */, int64_t* n_list);
int kge_export(kge_handle* h, void* blob, size_t* blob_bytes); /* blob == NULL: *blob_bytes <- size needed */
int kge_connect(kge_handle* h, const void* blobs /* world_size blobs, rank order */, int32_t world_size);
/* Single-process emulation: ranks 0..P-1 as P handles on one device, connected directly (tests / one-GPU parity). */
int kge_connect_local(kge_handle** hs, int32_t world_size);
int kge_relation_owner(const kge_handle* h, int64_t relation); /* rank, -1 = split (replicated), -2 = bad id */

/* Run-time options (diagnostics and robustness knobs; none changes the result of a step):
 *   KGE_OPT_FFMA_SPLITK   : split-K factor of the FFMA negative kernels, 0 = automatic (default), else 1, 2, 4 or 8
 *                           (forces the deterministic parked-partial reduction at any shape; KGE_EINVAL otherwise).
 *   KGE_OPT_CAPTURE_NEG   : 1 = the following training steps (kge_train_step) also store every negative pair score
 *                           f-_{i,j} (the g x k chunk products) into a library buffer read by
 *                           kge_debug_neg_scores; 0 = off (default). Not captured into the caller-batch CUDA graphs.
 *   KGE_OPT_BARRIER_MS    : P > 1 device-barrier timeout in milliseconds (default 120000). A rank that waits longer
 *                           for a peer leaves the barrier, and the next synchronising call returns KGE_ECUDA
 *                           ("device barrier timed out") instead of hanging or trapping the context. */
enum { KGE_OPT_FFMA_SPLITK = 0, KGE_OPT_CAPTURE_NEG = 1, KGE_OPT_BARRIER_MS = 2 };
int kge_set_option(kge_handle* h, int32_t option, int64_t value);
/* Negative pair scores f-_{i,j} of the last step run with KGE_OPT_CAPTURE_NEG on: out = host float[B * k], row i =
 * positive i of the batch (chunk i / g), column j = negative slot j of that chunk -- the scores the negative kernels
 * fed into the loss (FP32 FFMA, TF32/BF16 tcgen05 or TransR path). Synchronous. KGE_ESTATE if capture is off. */
int kge_debug_neg_scores(kge_handle* h, float* out);

/* Diagnostics. Kernel ids for kge_profile_end. Between begin and end every kernel launch of the step is bracketed by
 * CUDA events on the stream it runs on, and programmatic dependent launch is off (each kernel starts after its
 * predecessor completed), so the durations are those of each kernel alone; begin also holds the main stream behind a
 * gate kernel that end releases, so the bracketed launches are all queued when the GPU reaches them and the event
 * pairs exclude the host's submission latency (keep a profiled region to a few dozen steps: the gate gives up after
 * 2 s); end synchronises and returns the average device duration (ms) and the number of launches per kernel id. kge_launch_count: total kernel launches the handle
 * has issued. */
enum { KGE_K_SAMPLE = 0, KGE_K_GATHER = 1, KGE_K_NEG_FWD = 2, KGE_K_NEG_BWD = 3, KGE_K_CHAIN = 4, KGE_K_UPDATE = 5,
       KGE_K_COUNT = 6 };
int kge_profile_begin(kge_handle* h);
int kge_profile_end(kge_handle* h, int32_t n_kernels, double* avg_ms, int64_t* launches);
int64_t kge_launch_count(const kge_handle* h);
/* Diagnostics (handle created with KGE_TRACE=1 in the environment): per kernel id, per CTA (2048), 8 globaltimer stamps
 * of the latest launch (slot 0 = CTA start, 7 = end, 1-2 = setup / main-loop done for the tensor-core kernels). */
int kge_debug_trace(kge_handle* h, uint64_t* out, int64_t n);

void kge_destroy(kge_handle* h);
const char* kge_last_error(void);
const char* kge_kernel_name(int32_t kernel_id);

#ifdef __cplusplus
}
#endif
#endif
