/* synth.h -- seeded synthetic knowledge-graph generator (INPUT GENERATION ONLY).
 *
 * This module is shared by the CPU oracle (oracle/) and the CUDA path's tests / bench as the
 * single source of synthetic triples. It holds none of the method's arithmetic: no Philox, no
 * sampling, no scores. Its RNG is SplitMix64 (deliberately a different generator from the
 * method's Philox4x32-10, so nothing the method computes can leak in through here).
 *
 * Recipe (SURVEY.md 8(d) "Synthetic inputs"):
 *   triple i:  r = pi_R(Zipf_{alpha_r}(N_r)),  h = pi_E(Zipf_{alpha_e}(N_e)),  t = pi_E(Zipf_{alpha_e}(N_e))
 *   Zipf draws by inverse-CDF of the continuous power law on [1, N+1); pi_* are keyed affine
 *   bijections (a*x+b mod N, gcd(a,N)=1) that scatter hub ids across the id space.
 *   Every triple is a pure function of (graph_seed, i): any range can be regenerated lazily.
 *   Self-loops and duplicate triples are allowed (SPEC.md:56 keeps duplicates).
 */
#ifndef KGE_SYNTH_H
#define KGE_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t n_entities;   /* N_e */
  int64_t n_relations;  /* N_r */
  int64_t n_triples;    /* N_t */
  double alpha_e;       /* Zipf exponent for entities (0 = uniform) */
  double alpha_r;       /* Zipf exponent for relations (0 = uniform) */
  uint64_t graph_seed;
} synth_graph;

/* Triple i (0 <= i < n_triples) -> (h, r, t). */
void synth_triple(const synth_graph* g, int64_t i, int64_t* h, int64_t* r, int64_t* t);

/* Triples [begin, begin+n) into caller arrays (any may be NULL). OpenMP-parallel. */
void synth_triples(const synth_graph* g, int64_t begin, int64_t n, int64_t* h, int64_t* r, int64_t* t);

/* Same, writing int32 ids (ids must be < 2^31). */
void synth_triples_i32(const synth_graph* g, int64_t begin, int64_t n, int32_t* h, int32_t* r, int32_t* t);

#ifdef __cplusplus
}
#endif
#endif
