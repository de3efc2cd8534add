/* synth.c -- see synth.h. Input generation only; no method arithmetic. */
#include "synth.h"
#include <math.h>

static inline uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static inline double unit(uint64_t seed, uint64_t i, uint64_t slot) {
  uint64_t u = mix64(seed ^ mix64(i * 4u + slot));
  return (double)(u >> 11) * (1.0 / 9007199254740992.0); /* [0,1) */
}

static inline int64_t zipf_rank(double u, int64_t n, double alpha) {
  double x;
  int64_t k;
  if (n <= 1) return 0;
  if (alpha == 0.0) {
    k = (int64_t)(u * (double)n);
  } else if (fabs(alpha - 1.0) < 1e-12) {
    x = exp(u * log((double)n + 1.0));
    k = (int64_t)floor(x) - 1;
  } else {
    double a = 1.0 - alpha;
    x = pow(1.0 + u * (pow((double)n + 1.0, a) - 1.0), 1.0 / a);
    k = (int64_t)floor(x) - 1;
  }
  if (k < 0) k = 0;
  if (k >= n) k = n - 1;
  return k;
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) { uint64_t t = a % b; a = b; b = t; }
  return a;
}

/* keyed affine bijection on [0, n): x -> (a*x + b) mod n */
static void affine_key(uint64_t seed, uint64_t tag, int64_t n, uint64_t* a, uint64_t* b) {
  uint64_t nn = (uint64_t)(n > 0 ? n : 1);
  uint64_t aa = 0;
  if (nn > 1) {
    aa = mix64(seed ^ (tag * 0x632BE59BD9B4E019ull)) % nn;
    if (aa == 0) aa = 1;
    while (gcd_u64(aa, nn) != 1) {
      aa += 1;
      if (aa >= nn) aa = 1;
    }
  }
  *a = aa;
  *b = nn > 1 ? mix64(seed ^ (tag * 0x9E3779B97F4A7C15ull + 7)) % nn : 0;
}

static inline int64_t affine(uint64_t a, uint64_t b, int64_t n, int64_t x) {
  if (n <= 1) return 0;
  unsigned __int128 v = (unsigned __int128)a * (uint64_t)x + b;
  return (int64_t)(v % (uint64_t)n);
}

typedef struct { uint64_t ae, be, ar, br; } keys_t;

static keys_t make_keys(const synth_graph* g) {
  keys_t k;
  affine_key(g->graph_seed, 1, g->n_entities, &k.ae, &k.be);
  affine_key(g->graph_seed, 2, g->n_relations, &k.ar, &k.br);
  return k;
}

static inline void one(const synth_graph* g, const keys_t* k, int64_t i, int64_t* h, int64_t* r, int64_t* t) {
  uint64_t s = g->graph_seed;
  int64_t rr = zipf_rank(unit(s, (uint64_t)i, 0), g->n_relations, g->alpha_r);
  int64_t hh = zipf_rank(unit(s, (uint64_t)i, 1), g->n_entities, g->alpha_e);
  int64_t tt = zipf_rank(unit(s, (uint64_t)i, 2), g->n_entities, g->alpha_e);
  *r = affine(k->ar, k->br, g->n_relations, rr);
  *h = affine(k->ae, k->be, g->n_entities, hh);
  *t = affine(k->ae, k->be, g->n_entities, tt);
}

void synth_triple(const synth_graph* g, int64_t i, int64_t* h, int64_t* r, int64_t* t) {
  keys_t k = make_keys(g);
  one(g, &k, i, h, r, t);
}

void synth_triples(const synth_graph* g, int64_t begin, int64_t n, int64_t* h, int64_t* r, int64_t* t) {
  keys_t k = make_keys(g);
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    int64_t a, b, c;
    one(g, &k, begin + i, &a, &b, &c);
    if (h) h[i] = a;
    if (r) r[i] = b;
    if (t) t[i] = c;
  }
}

void synth_triples_i32(const synth_graph* g, int64_t begin, int64_t n, int32_t* h, int32_t* r, int32_t* t) {
  keys_t k = make_keys(g);
  int64_t i;
#pragma omp parallel for schedule(static)
  for (i = 0; i < n; ++i) {
    int64_t a, b, c;
    one(g, &k, begin + i, &a, &b, &c);
    if (h) h[i] = (int32_t)a;
    if (r) r[i] = (int32_t)b;
    if (t) t[i] = (int32_t)c;
  }
}
