/* oracle.h -- plain, slow, obviously-correct CPU oracle of the DGL-KE mini-batch training step.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call this library. The product path (libkge.so and the
 * paper_2004_08532_b200 package) never links, imports or executes it, and shares no code with it.
 *
 * What it computes (citations: PAPER.md = /root/reference/PAPER.md, section in brackets;
 * SURVEY = /root/repo/SURVEY.md 8(c) readings c.1 .. c.14, restated in DESIGN.md "Readings"):
 *   - Philox4x32-10 counter RNG (c.1; constants of the standard Random123 / curand bijection)
 *   - positive selection by a keyed Feistel permutation per epoch (c.2; PAPER.md:260-261 [2], 317-318 [3.1])
 *   - joint negative sampling: k uniform entity ids per chunk of g positives (c.3; PAPER.md:417-422 [3.3])
 *   - head/tail corruption schedule (c.4; PAPER.md:251-255 [2], 420-422 [3.3])
 *   - dedup of touched rows (c.5; sparse updates PAPER.md:262-266 [2], 472-474 [3.4])
 *   - table init (c.6; not in the paper)
 *   - Table-1 score functions (PAPER.md:216-237 [2], Table 1) and their hand-derived gradients (c.10)
 *   - chunk decomposition o = combine(h, r) (PAPER.md:429-435 [3.3]) -- used only to pin that it
 *     equals the naive per-triple definition, which is what the step uses (c.8)
 *   - logistic loss (PAPER.md:239-246 [2], eq. at; normalisation c.9) and pairwise ranking loss
 *     (PAPER.md:247-249 [2]; reading c.9': mean over the B*k (positive, its chunk's negative) pairs)
 *   - sparse row-wise Adagrad after dedup-sum (c.11; PAPER.md:336-338 [3.1] "apply an optimization
 *     algorithm")
 *   - greedy relation partitioning with heavy-relation split (c.13; PAPER.md:484-495 [3.4])
 *   - P-rank step = one step over the union of the P rank batches, losses summed (c.13)
 * Precision: double (reference) or float (to quantify fp32 spread); built -O2 -ffp-contract=off.
 */
#ifndef KGE_ORACLE_H
#define KGE_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_TRANSE_L1 = 0, ORC_TRANSE_L2 = 1, ORC_DISTMULT = 2, ORC_COMPLEX = 3, ORC_ROTATE = 4, ORC_TRANSR = 5,
       ORC_RESCAL = 6 /* h^T M_r t (Table 1); M_r d x d row-major in table 2, no relation vector */ };
enum { ORC_TAIL = 0, ORC_HEAD = 1, ORC_ALTERNATE = 2 };

typedef struct {
  int32_t model;
  int32_t precision;        /* 0 = double, 1 = float */
  int64_t n_entities, n_relations;
  int32_t dim;              /* d */
  int32_t batch, chunk, neg_k; /* B, g, k */
  float gamma, lr, eps, init_bound; /* init_bound <= 0 -> (gamma+2)/d if gamma>0 else 1/sqrt(d) */
  uint64_t seed;
  int32_t corrupt;          /* ORC_TAIL / ORC_HEAD / ORC_ALTERNATE */
  int32_t rotate_variant;   /* 0 = Table-1 squared, 1 = modulus sum */
  int32_t world_size;       /* P simulated ranks */
  int32_t lazy_rows;        /* 1: rows materialised on first touch (Freebase-sized N_e) */
  int32_t lag;              /* 0: synchronous; 1: the entity-table update of step s is applied after step s+1 computed
                               its gradients (deterministic form of PAPER.md:515-534; relations stay synchronous) */
  int32_t neg_deg_k;        /* slots j < neg_deg_k of each chunk are degree-based in-batch negatives,
                               the rest uniform; 0 = all uniform */
  int32_t neg_local;        /* 1: uniform negatives of rank w are drawn from its own entity shard {e : e mod P == w}
                               ("local" negatives; no remote rows for them) */
  int32_t loss;             /* ORC_LOSS_LOGISTIC (c.9) or ORC_LOSS_PAIRWISE (c.9') */
  int32_t repartition;      /* 1 with world_size > 1: a randomised relation partition per epoch of ceil(N_t/(P B))
                               steps (reading c.13') */
  int32_t placement;        /* 0: relation partition (c.13); 1: head-owner placement (c.13'') */
} orc_config;
enum { ORC_LOSS_LOGISTIC = 0, ORC_LOSS_PAIRWISE = 1 };

typedef void (*orc_triple_fn)(void* ctx, int64_t i, int64_t* h, int64_t* r, int64_t* t);

/* ---- primitives ---- */
void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t orc_feistel_index(uint64_t n, uint64_t seed, uint32_t epoch, uint64_t p);
int64_t orc_neg_id(uint64_t seed, int64_t n_entities, uint32_t step, uint32_t cg, uint32_t j);
int32_t orc_mode(int32_t corrupt, uint32_t step, uint32_t cg);
float orc_init_value(uint64_t seed, int32_t table, int64_t row, int64_t col, float bound);
float orc_default_bound(float gamma, int32_t dim);

/* relation partition; owner_out[n_rel] = rank or -1 (SPLIT). Returns #split relations. */
int32_t orc_relation_partition(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P,
                               int32_t* owner_out);
/* triple indices of `rank` (ascending). Returns count; idx_out may be NULL (count only). */
/* c.13' the randomised partition of epoch `epoch` */
/* c.13'' BFS-grown balanced partition of the entity graph and the renumbering that puts part w on rank w's shard
 * (new_id_out [n_entities], part_out [n_entities] or NULL); returns the edge cut */
int64_t orc_locality_order(const int64_t* heads, const int64_t* tails, int64_t n_triples, int64_t n_entities, int32_t P,
                           int64_t* new_id_out, int32_t* part_out);
int32_t orc_relation_partition_epoch(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P, uint64_t seed,
                                     uint32_t epoch, int32_t* owner_out);
int64_t orc_rank_triples(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P, int32_t rank,
                         int64_t* idx_out);

/* ---- scores / grads / loss / optimizer (double) ---- */
/* rel width: d (TransE, DistMult, ComplEx, TransR), d/2 (RotatE); M: d*d row-major (TransR) or NULL */
double orc_score(int32_t model, int32_t variant, double gamma, int32_t d, const double* h, const double* r,
                 const double* t, const double* M);
float orc_score_f(int32_t model, int32_t variant, float gamma, int32_t d, const float* h, const float* r,
                  const float* t, const float* M);
void orc_score_grad(int32_t model, int32_t variant, double gamma, int32_t d, const double* h, const double* r,
                    const double* t, const double* M, double upstream, double* dh, double* dr, double* dt,
                    double* dM);
/* decomposed chunk scorer (c.8): mode 0 tail (x replaces t), 1 head (x replaces h). out[g*k] */
void orc_score_group(int32_t model, int32_t variant, double gamma, int32_t d, int32_t mode, int32_t g, int32_t k,
                     const double* H, const double* R, const double* T, const double* M, const double* X,
                     double* out);
/* c.15' second-protocol candidates of n_queries queries: ent/side [n_queries x (n_uniform +
 * n_degree)], side 0 = tail replaced, 1 = head replaced (both = 0: all 0). th/tt: the graph's heads and tails. */
void orc_eval_candidates(uint64_t seed, int64_t n_ent, int64_t n_trip, const int64_t* th, const int64_t* tt,
                         int64_t n_queries, int64_t n_uniform, int64_t n_degree, int32_t both, int64_t* ent,
                         int32_t* side);
/* c.9' pairwise ranking loss: L = (1/(B k)) sum_i sum_j max(0, gamma - f+_i + f-_ij) over
 * pos[B] and neg[B*k] (row i = the negatives paired with positive i); dpos[B], dneg[B*k] = dL/df (hinge at 0:
 * subgradient 0). Returns L. */
double orc_ranking_loss(const double* pos, const double* neg, int64_t B, int64_t k, double gamma, double* dpos,
                        double* dneg);
double orc_logistic_loss(const double* pos, int64_t n_pos, const double* neg, int64_t n_neg, int64_t B, int64_t k,
                         double* dpos, double* dneg);
void orc_adagrad(double* row, double* state, const double* g, int32_t w, double lr, double eps);

/* dedup: uniq ascending distinct ids; inv[o]; seg_off[n_uniq+1]; seg_occ = occurrences in (id, occ) order */
int64_t orc_dedup(const int64_t* ids, int64_t n, int64_t* uniq, int32_t* inv, int64_t* seg_off, int64_t* seg_occ);

/* ---- the training step ---- */
void* orc_create(const orc_config* cfg, const int64_t* heads, const int64_t* rels, const int64_t* tails,
                 int64_t n_triples, orc_triple_fn fn, void* ctx);
void orc_destroy(void* h);
int orc_sample(void* h, int64_t step, int32_t rank, int64_t* pos_idx, int64_t* neg, int8_t* mode);
/* entity occurrence ids of one rank-step [h..., t..., neg...] and relation occurrence ids [r...] */
int orc_occurrences(void* h, int64_t step, int32_t rank, int64_t* ent_occ, int64_t* rel_occ);
int orc_train(void* h, int64_t n_steps, double* losses);
/* lag = 1: apply the pending entity update of the last step (no-op otherwise). */
int orc_flush(void* h);
int orc_get_rows(void* h, int32_t table, const int64_t* ids, int64_t n, double* out);
int orc_set_rows(void* h, int32_t table, const int64_t* ids, int64_t n, const double* in);
int orc_score_triples(void* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, double* out);
int64_t orc_next_step(void* h);
void orc_set_step(void* h, int64_t s);
int32_t orc_table_width(void* h, int32_t table);

#ifdef __cplusplus
}
#endif
#endif
