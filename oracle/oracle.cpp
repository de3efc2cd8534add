// oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h). Plain, slow, single-threaded (ORC_THREADS > 1: the
// independent per-row loops of the step in parallel, bit-identical results) CPU oracle of the
// DGL-KE mini-batch KGE training step. Every function cites the passage it follows; readings of the paper
// where it is silent are SURVEY.md 8(c) c.1..c.14, restated in DESIGN.md "Readings of the paper".
// Build: g++ -O2 -ffp-contract=off -fPIC -shared (no fast-math). Shares no code with the CUDA path.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <unordered_map>
#include <vector>

namespace {

// Threads of the optional parallel loops of the training step (ORC_THREADS, default 1 = the single-threaded oracle).
// The loops run over independent output rows (positive i, negative slot (c, j)); every value is computed by the same
// operations in the same order as with one thread, and the loss is still summed serially -- results are identical.
int threads() {
  const char* v = std::getenv("ORC_THREADS");
  const int n = v ? std::atoi(v) : 1;
  return n > 1 ? n : 1;
}

// ------------------------------------------------------------------------------------------------
// c.1 Philox4x32-10 (Salmon et al., Random123; the bijection CUDA's curand uses). Not in the paper:
// the north_star names "Philox counter-based" sampling.
// ------------------------------------------------------------------------------------------------
const uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
const uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;
const uint32_t TAG_NEG = 1, TAG_PERM = 2, TAG_INIT = 3, TAG_DEG = 4, TAG_EVAL = 5, TAG_REPART = 6;

void philox(const uint32_t in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t x0 = in[0], x1 = in[1], x2 = in[2], x3 = in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t p0 = (uint64_t)PHILOX_M0 * x0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * x2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

void seed_key(uint64_t seed, uint32_t key[2]) {
  key[0] = (uint32_t)seed;
  key[1] = (uint32_t)(seed >> 32);
}

// c.2 positive selection: pi_e is a 4-round balanced Feistel network on 2^m >= N with cycle walking.
// m = max(2, 2*ceil(ceil(log2 N)/2)); round function F_i(R) = Philox(ctr=(R, i, e, PERM), key)[0] & mask.
uint64_t ceil_log2(uint64_t n) {
  uint64_t b = 0;
  while ((1ull << b) < n) ++b;
  return b;
}

uint64_t feistel_once(uint64_t x, uint32_t half, uint64_t seed, uint32_t epoch) {
  uint32_t key[2];
  seed_key(seed, key);
  uint64_t mask = (1ull << half) - 1;
  uint64_t L = x >> half, R = x & mask;
  for (uint32_t i = 0; i < 4; ++i) {
    uint32_t ctr[4] = {(uint32_t)R, i, epoch, TAG_PERM}, o[4];
    philox(ctr, key, o);
    uint64_t F = (uint64_t)o[0] & mask;
    uint64_t nl = R, nr = L ^ F;
    L = nl;
    R = nr;
  }
  return (L << half) | R;
}

uint64_t feistel_index(uint64_t n, uint64_t seed, uint32_t epoch, uint64_t p) {
  uint64_t lg = ceil_log2(n);
  uint64_t m = 2 * ((lg + 1) / 2);
  if (m < 2) m = 2;
  uint32_t half = (uint32_t)(m / 2);
  uint64_t x = feistel_once(p, half, seed, epoch);
  while (x >= n) x = feistel_once(x, half, seed, epoch);
  return x;
}

// c.3 joint negatives (PAPER.md:417-422 [3.3] "uniformly sample k entities"): for chunk cg, slot j,
// x = Philox(ctr=(j/2, cg, s, NEG), key); even j uses (w0,w1), odd j (w2,w3); u = w_b<<32 | w_a;
// id = floor(u * N / 2^64) (multiply-high; no rejection).
int64_t neg_id(uint64_t seed, int64_t n_ent, uint32_t step, uint32_t cg, uint32_t j) {
  uint32_t key[2];
  seed_key(seed, key);
  uint32_t ctr[4] = {j / 2u, cg, step, TAG_NEG}, o[4];
  philox(ctr, key, o);
  uint64_t u = (j & 1u) ? (((uint64_t)o[3] << 32) | o[2]) : (((uint64_t)o[1] << 32) | o[0]);
  unsigned __int128 prod = (unsigned __int128)u * (uint64_t)n_ent;
  return (int64_t)(uint64_t)(prod >> 64);
}

// Degree-based in-batch negatives (PAPER.md:437-448 [3.3]: "uniformly sampling some of the mini-batch's triplets and
// connecting the sampled head (tail) entities with the tail (head) entities of the mini-batch's triplets"; reading
// c.3'): slot j < k_deg of chunk cg draws a batch position t = floor(u * B / 2^64) from Philox(ctr=(j/2, cg, s, DEG))
// (words as in c.3); the negative is that triplet's tail (tail corruption) or head (head corruption), so an entity is
// drawn with probability proportional to its degree in the mini-batch.
int64_t deg_pos(uint64_t seed, int64_t B, uint32_t step, uint32_t cg, uint32_t j) {
  uint32_t key[2];
  seed_key(seed, key);
  uint32_t ctr[4] = {j / 2u, cg, step, TAG_DEG}, o[4];
  philox(ctr, key, o);
  uint64_t u = (j & 1u) ? (((uint64_t)o[3] << 32) | o[2]) : (((uint64_t)o[1] << 32) | o[0]);
  unsigned __int128 prod = (unsigned __int128)u * (uint64_t)B;
  return (int64_t)(uint64_t)(prod >> 64);
}

// c.15' second-protocol candidates (PAPER.md:656-658 [5.3]: "we use only 2000 negative triplets; 1000 sampled
// uniformly from the entire set of negative samples and 1000 sampled proportionally to the degree of the corrupted
// entities"): slot j of query i draws u from Philox(ctr=(j/2, lo32(i), hi32(i), EVAL), key = eval seed), words as in
// c.3. Uniform slots (j < n_uniform): an entity uniform over the N_e entities -- with both sides pooled (mode 2) a
// corruption uniform over the 2 N_e (side, entity) pairs: p = floor(u * 2 N_e / 2^64), side = p & 1, e = p >> 1.
// Degree slots: an endpoint uniform over the 2 N_t triple endpoints (entity drawn proportionally to its degree in the
// graph): p = floor(u * 2 N_t / 2^64) (mode 2: * 4 N_t, side = p & 1, p >>= 1), e = (p & 1) ? t[p >> 1] : h[p >> 1].
// side 0 = the tail is replaced, 1 = the head.
void eval_candidate(uint64_t seed, int64_t n_ent, int64_t n_trip, const int64_t* th, const int64_t* tt, int64_t i,
                    int64_t j, int64_t n_uniform, int32_t both, int64_t* ent, int32_t* side) {
  uint32_t key[2];
  seed_key(seed, key);
  uint32_t ctr[4] = {(uint32_t)(j / 2), (uint32_t)i, (uint32_t)((uint64_t)i >> 32), TAG_EVAL}, o[4];
  philox(ctr, key, o);
  uint64_t u = (j & 1) ? (((uint64_t)o[3] << 32) | o[2]) : (((uint64_t)o[1] << 32) | o[0]);
  const uint64_t range = j < n_uniform ? (uint64_t)n_ent * (both ? 2u : 1u) : (uint64_t)n_trip * (both ? 4u : 2u);
  uint64_t p = (uint64_t)(((unsigned __int128)u * range) >> 64);
  *side = 0;
  if (both) {
    *side = (int32_t)(p & 1u);
    p >>= 1;
  }
  if (j < n_uniform) {
    *ent = (int64_t)p;
  } else {
    const int64_t q = (int64_t)(p >> 1);
    *ent = (p & 1u) ? tt[q] : th[q];
  }
}

// c.4 corruption schedule; "corrupt the head entities in a similar fashion".
int32_t mode_of(int32_t corrupt, uint32_t step, uint32_t cg) {
  if (corrupt == ORC_TAIL) return ORC_TAIL;
  if (corrupt == ORC_HEAD) return ORC_HEAD;
  return ((uint64_t)step + cg) % 2 == 0 ? ORC_TAIL : ORC_HEAD;
}

// c.6 init: u = Philox(ctr=(col, row_lo, row_hi ^ (table<<24), INIT))[0]; v = bound * ((float)(int32)u * 2^-31)
float init_value(uint64_t seed, int32_t table, int64_t row, int64_t col, float bound) {
  uint32_t key[2];
  seed_key(seed, key);
  uint32_t ctr[4] = {(uint32_t)col, (uint32_t)(uint64_t)row,
                     (uint32_t)((uint64_t)row >> 32) ^ ((uint32_t)table << 24), TAG_INIT};
  uint32_t o[4];
  philox(ctr, key, o);
  volatile float f = (float)(int32_t)o[0];  // RN int -> float
  volatile float s = f * 0x1p-31f;          // exact power-of-two scale
  volatile float v = bound * s;             // one RN multiply
  return v;
}

float default_bound(float gamma, int32_t dim) {
  if (gamma > 0.0f) {
    volatile float num = gamma + 2.0f;
    volatile float v = num / (float)dim;
    return v;
  }
  volatile float sd = std::sqrt((float)dim);
  volatile float v = 1.0f / sd;
  return v;
}

// ------------------------------------------------------------------------------------------------
// Table 1 score functions (PAPER.md:216-237 [2]). Distance models carry the margin: f = gamma + f_T1
// (reading Q7). DistMult / ComplEx use f = f_T1. Layouts: ComplEx and RotatE entities [re(d/2)|im(d/2)]
// (SPEC.md:106); RotatE relation = d/2 phases theta; TransR M_r is d x d row-major.
// ------------------------------------------------------------------------------------------------
template <typename T>
T score_t(int32_t model, int32_t variant, T gamma, int32_t d, const T* h, const T* r, const T* t, const T* M) {
  switch (model) {
    case ORC_TRANSE_L1: {  // -||h + r - t||_1
      T s = 0;
      for (int32_t e = 0; e < d; ++e) s += std::fabs(h[e] + r[e] - t[e]);
      return gamma - s;
    }
    case ORC_TRANSE_L2: {  // -||h + r - t||_2 (not squared)
      T s = 0;
      for (int32_t e = 0; e < d; ++e) {
        T x = h[e] + r[e] - t[e];
        s += x * x;
      }
      return gamma - std::sqrt(s);
    }
    case ORC_DISTMULT: {  // h^T diag(r) t, evaluated as sum r_j*(h_j*t_j) so f(h,r,t)=f(t,r,h) exactly
      T s = 0;
      for (int32_t e = 0; e < d; ++e) s += r[e] * (h[e] * t[e]);
      return s;
    }
    case ORC_COMPLEX: {  // Re(h^T diag(r) conj(t))
      int32_t n = d / 2;
      T s = 0;
      for (int32_t e = 0; e < n; ++e) {
        T hr = h[e], hi = h[e + n], rr = r[e], ri = r[e + n], tr = t[e], ti = t[e + n];
        s += hr * rr * tr + hi * rr * ti + hr * ri * ti - hi * ri * tr;
      }
      return s;
    }
    case ORC_ROTATE: {  // -||h o r - t||^2 (Table 1 as printed) or -sum_j |h_j r_j - t_j| (variant 1)
      int32_t n = d / 2;
      T s = 0;
      for (int32_t e = 0; e < n; ++e) {
        T a = h[e], b = h[e + n], c = std::cos(r[e]), sn = std::sin(r[e]);
        T u = a * c - b * sn - t[e];
        T v = a * sn + b * c - t[e + n];
        if (variant == 0)
          s += u * u + v * v;
        else
          s += std::sqrt(u * u + v * v);
      }
      return gamma - s;
    }
    case ORC_RESCAL: {  // h^T M_r t = sum_a sum_b h_a M_ab t_b (Table 1)
      T s = 0;
      for (int32_t a = 0; a < d; ++a) {
        T mt = 0;
        for (int32_t b = 0; b < d; ++b) mt += M[(int64_t)a * d + b] * t[b];
        s += h[a] * mt;
      }
      return s;
    }
    case ORC_TRANSR: {  // -||M_r h + r - M_r t||_2^2
      T s = 0;
      for (int32_t a = 0; a < d; ++a) {
        T mh = 0, mt = 0;
        for (int32_t b = 0; b < d; ++b) {
          mh += M[(int64_t)a * d + b] * h[b];
          mt += M[(int64_t)a * d + b] * t[b];
        }
        T p = mh + r[a] - mt;
        s += p * p;
      }
      return gamma - s;
    }
  }
  return 0;
}

// Gradients (c.10; not in the paper, derived). Adds upstream * df/d(param) into dh, dr, dt, dM.
template <typename T>
void grad_t(int32_t model, int32_t variant, int32_t d, const T* h, const T* r, const T* t, const T* M, T up, T* dh,
            T* dr, T* dt, T* dM) {
  switch (model) {
    case ORC_TRANSE_L1: {
      for (int32_t e = 0; e < d; ++e) {
        T x = h[e] + r[e] - t[e];
        T sg = x > 0 ? T(1) : (x < 0 ? T(-1) : T(0));  // sgn(0) = 0
        dh[e] += -up * sg;
        dr[e] += -up * sg;
        dt[e] += up * sg;
      }
      return;
    }
    case ORC_TRANSE_L2: {
      T s = 0;
      for (int32_t e = 0; e < d; ++e) {
        T x = h[e] + r[e] - t[e];
        s += x * x;
      }
      T nrm = std::sqrt(s);
      T den = nrm > T(1e-12) ? nrm : T(1e-12);
      for (int32_t e = 0; e < d; ++e) {
        T x = h[e] + r[e] - t[e];
        T gx = -up * (x / den);
        dh[e] += gx;
        dr[e] += gx;
        dt[e] -= gx;
      }
      return;
    }
    case ORC_DISTMULT: {
      for (int32_t e = 0; e < d; ++e) {
        dh[e] += up * (r[e] * t[e]);
        dr[e] += up * (h[e] * t[e]);
        dt[e] += up * (h[e] * r[e]);
      }
      return;
    }
    case ORC_COMPLEX: {
      int32_t n = d / 2;
      for (int32_t e = 0; e < n; ++e) {
        T hr = h[e], hi = h[e + n], rr = r[e], ri = r[e + n], tr = t[e], ti = t[e + n];
        dh[e] += up * (rr * tr + ri * ti);
        dh[e + n] += up * (rr * ti - ri * tr);
        dr[e] += up * (hr * tr + hi * ti);
        dr[e + n] += up * (hr * ti - hi * tr);
        dt[e] += up * (hr * rr - hi * ri);
        dt[e + n] += up * (hi * rr + hr * ri);
      }
      return;
    }
    case ORC_ROTATE: {
      int32_t n = d / 2;
      for (int32_t e = 0; e < n; ++e) {
        T a = h[e], b = h[e + n], c = std::cos(r[e]), sn = std::sin(r[e]);
        T u = a * c - b * sn - t[e];
        T v = a * sn + b * c - t[e + n];
        T fac;
        if (variant == 0) {
          fac = T(2);
        } else {
          T m = std::sqrt(u * u + v * v);
          fac = T(1) / (m > T(1e-12) ? m : T(1e-12));
        }
        // f = gamma - sum phi(u,v); d phi/du = fac*u, d phi/dv = fac*v
        dh[e] += up * (-fac * (u * c + v * sn));
        dh[e + n] += up * (-fac * (-u * sn + v * c));
        dt[e] += up * (fac * u);
        dt[e + n] += up * (fac * v);
        dr[e] += up * (-fac * (u * (-a * sn - b * c) + v * (a * c - b * sn)));
      }
      return;
    }
    case ORC_RESCAL: {  // dh_a = sum_b M_ab t_b, dt_b = sum_a h_a M_ab, dM_ab = h_a t_b; no relation vector
      for (int32_t a = 0; a < d; ++a) {
        T mt = 0;
        for (int32_t b = 0; b < d; ++b) mt += M[(int64_t)a * d + b] * t[b];
        dh[a] += up * mt;
      }
      for (int32_t b = 0; b < d; ++b) {
        T hm = 0;
        for (int32_t a = 0; a < d; ++a) hm += h[a] * M[(int64_t)a * d + b];
        dt[b] += up * hm;
      }
      if (dM)
        for (int32_t a = 0; a < d; ++a)
          for (int32_t b = 0; b < d; ++b) dM[(int64_t)a * d + b] += up * (h[a] * t[b]);
      (void)dr;
      return;
    }
    case ORC_TRANSR: {
      std::vector<T> p(d);
      for (int32_t a = 0; a < d; ++a) {
        T mh = 0, mt = 0;
        for (int32_t b = 0; b < d; ++b) {
          mh += M[(int64_t)a * d + b] * h[b];
          mt += M[(int64_t)a * d + b] * t[b];
        }
        p[a] = mh + r[a] - mt;
      }
      for (int32_t a = 0; a < d; ++a) dr[a] += up * (T(-2) * p[a]);
      for (int32_t b = 0; b < d; ++b) {
        T mtp = 0;  // (M^T p)_b
        for (int32_t a = 0; a < d; ++a) mtp += M[(int64_t)a * d + b] * p[a];
        dh[b] += up * (T(-2) * mtp);
        dt[b] += up * (T(2) * mtp);
      }
      if (dM)
        for (int32_t a = 0; a < d; ++a)
          for (int32_t b = 0; b < d; ++b) dM[(int64_t)a * d + b] += up * (T(-2) * p[a] * (h[b] - t[b]));
      return;
    }
  }
}

// c.9: log sigma(x) = min(x,0) - log1p(exp(-|x|)); sigma stable.
template <typename T>
T log_sigmoid(T x) {
  return std::min(x, T(0)) - std::log1p(std::exp(-std::fabs(x)));
}
template <typename T>
T sigmoid(T x) {
  if (x >= 0) return T(1) / (T(1) + std::exp(-x));
  T e = std::exp(x);
  return e / (T(1) + e);
}

// c.9' pairwise ranking loss (PAPER.md:247-249 [2]): minimize sum over positives and their negatives of
// max(0, gamma - f(h,r,t) + f(h',r',t')). The negatives of positive i are its chunk's k joint negatives (PAPER.md:
// 417-422); the sum is normalised by the B*k pairs like the negative term of c.9 (the scale is irrelevant under
// Adagrad up to eps). A hinge exactly at 0 contributes subgradient 0. fneg: [B x k], row i = positive i.
template <typename T>
T ranking_loss(const T* fpos, const T* fneg, int64_t B, int64_t k, T gamma, T* dpos, T* dneg) {
  T ln = 0;
  const T inv = T(1) / ((T)B * (T)k);
  for (int64_t i = 0; i < B; ++i) {
    int64_t active = 0;
    for (int64_t j = 0; j < k; ++j) {
      const T m = gamma - fpos[i] + fneg[i * k + j];
      const bool on = m > T(0);
      if (on) {
        ln += m;
        ++active;
      }
      if (dneg) dneg[i * k + j] = on ? inv : T(0);
    }
    if (dpos) dpos[i] = -(T)active * inv;
  }
  return ln * inv;
}

// ------------------------------------------------------------------------------------------------
// Row stores. Dense, or lazily materialised from the init law (c.6) on first touch.
// ------------------------------------------------------------------------------------------------
template <typename T>
struct RowStore {
  int64_t n = 0;
  int32_t w = 0;
  int32_t table = 0;
  float bound = 0;
  uint64_t seed = 0;
  bool lazy = false;
  bool is_state = false;
  std::vector<T> dense;
  std::unordered_map<int64_t, std::vector<T>> sparse;

  void init(int64_t n_, int32_t w_, int32_t table_, float bound_, uint64_t seed_, bool lazy_, bool state_) {
    n = n_; w = w_; table = table_; bound = bound_; seed = seed_; lazy = lazy_; is_state = state_;
    if (!lazy) {
      dense.assign((size_t)n * w, T(0));
      if (!is_state)
        for (int64_t i = 0; i < n; ++i)
          for (int32_t c = 0; c < w; ++c) dense[(size_t)i * w + c] = (T)init_value(seed, table, i, c, bound);
    }
  }
  T* row(int64_t i) {
    if (!lazy) return &dense[(size_t)i * w];
    auto it = sparse.find(i);
    if (it != sparse.end()) return it->second.data();
    std::vector<T> v((size_t)w, T(0));
    if (!is_state)
      for (int32_t c = 0; c < w; ++c) v[c] = (T)init_value(seed, table, i, c, bound);
    auto res = sparse.emplace(i, std::move(v));
    return res.first->second.data();
  }
};

// c.13' per-epoch randomisation (PAPER.md:497-501 [3.4]: "we introduce randomization in the partitioning algorithm
// and at the start of each epoch we compute a somewhat different relation partitioning"; SPEC.md reshuffle_partition:
// ties broken by a seed- and epoch-dependent permutation, SPLIT set unchanged): the sort key of relation r in epoch e.
uint32_t repart_key(uint64_t seed, uint32_t epoch, int64_t r) {
  uint32_t key[2];
  seed_key(seed, key);
  uint32_t ctr[4] = {(uint32_t)r, epoch, 0u, TAG_REPART}, o[4];
  philox(ctr, key, o);
  return o[0];
}

// c.13 relation partition (PAPER.md:484-492 [3.4]): relations with count > N_t/P are SPLIT and their
// triples dealt round-robin (per relation, ascending triple index); the rest sorted by (count desc, id asc)
// and each given to the currently lightest rank (ties -> lowest rank). Loads start from the dealt split triples.
// With `randomise` the non-split order is (count desc, repart_key(seed, epoch, r) asc, id asc) (c.13').
int32_t relation_partition(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, std::vector<int32_t>& owner,
                           std::vector<int64_t>& counts, bool randomise = false, uint64_t seed = 0,
                           uint32_t epoch = 0) {
  counts.assign((size_t)nr, 0);
  for (int64_t i = 0; i < nt; ++i) counts[(size_t)rels[i]]++;
  owner.assign((size_t)nr, 0);
  std::vector<int64_t> load((size_t)P, 0);
  int32_t n_split = 0;
  std::vector<int64_t> order;
  for (int64_t r = 0; r < nr; ++r) {
    // count > N_t / P  <=>  count * P > N_t (exact integer comparison)
    if (P > 1 && counts[(size_t)r] * P > nt) {
      owner[(size_t)r] = -1;
      ++n_split;
      for (int32_t w = 0; w < P; ++w) load[(size_t)w] += counts[(size_t)r] / P + (w < counts[(size_t)r] % P ? 1 : 0);
    } else {
      order.push_back(r);
    }
  }
  std::vector<uint32_t> key((size_t)nr, 0u);
  if (randomise)
    for (int64_t r : order) key[(size_t)r] = repart_key(seed, epoch, r);
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
    if (counts[(size_t)a] != counts[(size_t)b]) return counts[(size_t)a] > counts[(size_t)b];
    if (key[(size_t)a] != key[(size_t)b]) return key[(size_t)a] < key[(size_t)b];
    return a < b;
  });
  for (int64_t r : order) {
    int32_t best = 0;
    for (int32_t w = 1; w < P; ++w)
      if (load[(size_t)w] < load[(size_t)best]) best = w;
    owner[(size_t)r] = best;
    load[(size_t)best] += counts[(size_t)r];
  }
  return n_split;
}

// c.13'' head-owner placement (PAPER.md:395-406 [3.2]: a machine holds "all entities and triplets incident to the
// entities" of its partition; SPEC: single ownership by the head's part): triple i belongs to the rank owning its
// head, h_i mod P; every relation may then appear on every rank (all replicated, their gradients summed in rank
// order -- the union-step semantics of c.13 do not change).
void head_owner_lists(const std::vector<int64_t>& heads, int32_t P, std::vector<std::vector<int64_t>>& lists) {
  lists.assign((size_t)P, {});
  for (size_t i = 0; i < heads.size(); ++i) lists[(size_t)(heads[i] % P)].push_back((int64_t)i);
}

// c.13'' METIS-style locality ordering (PAPER.md:395-406 deploys METIS; SPEC's built-in substitute
// partition_graph_greedy: BFS-grown balanced parts). Part w takes exactly n_w = ceil((N_e - w) / P) entities (the
// size of rank w's shard under owner = e mod P): starting from the lowest-id unassigned entity, breadth-first over the
// undirected entity graph of the triples (neighbours in ascending id, an entity joins the part when discovered) until
// the part is full (a new seed = the lowest unassigned id when the frontier empties). The renumbering new(e) = P j + w
// (j = position of e among part w's entities in ascending old id) puts part w on rank w's shard. Returns the edge cut
// (triples whose head and tail fall in different parts).
int64_t locality_order(const int64_t* heads, const int64_t* tails, int64_t nt, int64_t ne, int32_t P,
                       std::vector<int64_t>& new_id, std::vector<int32_t>& part) {
  std::vector<std::vector<int64_t>> adj((size_t)ne);
  for (int64_t i = 0; i < nt; ++i) {
    if (heads[i] == tails[i]) continue;
    adj[(size_t)heads[i]].push_back(tails[i]);
    adj[(size_t)tails[i]].push_back(heads[i]);
  }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  part.assign((size_t)ne, -1);
  int64_t next_seed = 0;
  for (int32_t w = 0; w < P; ++w) {
    const int64_t target = (ne - w + P - 1) / P;
    int64_t size = 0;
    std::vector<int64_t> queue;
    size_t head = 0;
    while (size < target) {
      if (head == queue.size()) {  // frontier empty: seed with the lowest unassigned entity
        while (part[(size_t)next_seed] >= 0) ++next_seed;
        part[(size_t)next_seed] = w;
        ++size;
        queue.push_back(next_seed);
        continue;
      }
      const int64_t v = queue[head++];
      for (int64_t u : adj[(size_t)v]) {
        if (size >= target) break;
        if (part[(size_t)u] < 0) {
          part[(size_t)u] = w;
          ++size;
          queue.push_back(u);
        }
      }
    }
  }
  new_id.assign((size_t)ne, -1);
  std::vector<int64_t> cnt((size_t)P, 0);
  for (int64_t e = 0; e < ne; ++e) {
    const int32_t w = part[(size_t)e];
    new_id[(size_t)e] = (int64_t)P * cnt[(size_t)w]++ + w;
  }
  int64_t cut = 0;
  for (int64_t i = 0; i < nt; ++i) cut += part[(size_t)heads[i]] != part[(size_t)tails[i]];
  return cut;
}

void rank_lists(const int64_t* rels, int64_t nt, int64_t nr, int32_t P, std::vector<std::vector<int64_t>>& lists,
                bool randomise = false, uint64_t seed = 0, uint32_t epoch = 0) {
  lists.assign((size_t)P, {});
  if (P == 1) {
    lists[0].resize((size_t)nt);
    for (int64_t i = 0; i < nt; ++i) lists[0][(size_t)i] = i;
    return;
  }
  std::vector<int32_t> owner;
  std::vector<int64_t> counts;
  relation_partition(rels, nt, nr, P, owner, counts, randomise, seed, epoch);
  std::vector<int64_t> dealt((size_t)nr, 0);
  for (int64_t i = 0; i < nt; ++i) {
    int64_t r = rels[i];
    int32_t o = owner[(size_t)r];
    if (o < 0) o = (int32_t)(dealt[(size_t)r]++ % P);
    lists[(size_t)o].push_back(i);
  }
}

int64_t dedup(const int64_t* ids, int64_t n, int64_t* uniq, int32_t* inv, int64_t* seg_off, int64_t* seg_occ) {
  // c.5: uniq = sorted distinct ids; segments list occurrences in increasing occurrence index (stable sort).
  std::vector<int64_t> occ((size_t)n);
  std::iota(occ.begin(), occ.end(), 0);
  std::stable_sort(occ.begin(), occ.end(), [&](int64_t a, int64_t b) { return ids[a] < ids[b]; });
  int64_t nu = 0;
  for (int64_t p = 0; p < n; ++p) {
    int64_t o = occ[(size_t)p];
    if (p == 0 || ids[o] != ids[occ[(size_t)p - 1]]) {
      if (uniq) uniq[nu] = ids[o];
      if (seg_off) seg_off[nu] = p;
      ++nu;
    }
    if (inv) inv[o] = (int32_t)(nu - 1);
    if (seg_occ) seg_occ[p] = o;
  }
  if (seg_off) seg_off[nu] = n;
  return nu;
}

// ------------------------------------------------------------------------------------------------
// The trainer: PAPER.md:314-344 [3.1] four steps (sample, fetch, forward/backward, apply) at lag 0 (c.12),
// P ranks simulated as one step over the union of their batches with summed losses (c.13).
// ------------------------------------------------------------------------------------------------
struct Base {
  orc_config cfg{};
  std::vector<int64_t> H, R, Tt;  // triples (empty when generated through fn)
  orc_triple_fn fn = nullptr;
  void* ctx = nullptr;
  int64_t nt = 0;
  std::vector<std::vector<int64_t>> lists;  // per-rank triple index lists (empty lists[0] -> identity)
  bool identity_list = false;
  // c.13' (cfg.repartition, P > 1): epochs of S_E = ceil(N_t / (P B)) steps on every rank, the partition of epoch e
  // recomputed with the epoch's keys; lists cached for epoch cur_epoch
  std::vector<int64_t> RR;  // relation of every triple
  mutable std::vector<std::vector<int64_t>> ep_lists;
  mutable int64_t cur_epoch = -1;
  bool repart() const { return cfg.repartition && cfg.world_size > 1; }
  int64_t epoch_steps() const {
    const int64_t pb = (int64_t)cfg.world_size * cfg.batch;
    return (nt + pb - 1) / pb;
  }
  const std::vector<int64_t>& epoch_list(int64_t e, int32_t rank) const {
    if (e != cur_epoch) {
      rank_lists(RR.data(), nt, cfg.n_relations, cfg.world_size, ep_lists, true, cfg.seed, (uint32_t)e);
      cur_epoch = e;
    }
    return ep_lists[(size_t)rank];
  }
  int64_t step = 0;
  virtual ~Base() {}
  virtual int train(int64_t n, double* losses) = 0;
  virtual int get_rows(int32_t table, const int64_t* ids, int64_t n, double* out) = 0;
  virtual int set_rows(int32_t table, const int64_t* ids, int64_t n, const double* in) = 0;
  virtual int score_triples(const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, double* out) = 0;
  virtual int32_t width(int32_t table) = 0;
  virtual int flush() = 0;

  void triple(int64_t i, int64_t& h, int64_t& r, int64_t& t) const {
    if (fn) {
      fn(ctx, i, &h, &r, &t);
    } else {
      h = H[(size_t)i]; r = R[(size_t)i]; t = Tt[(size_t)i];
    }
  }
  int64_t list_size(int32_t rank) const { return identity_list ? nt : (int64_t)lists[(size_t)rank].size(); }
  int64_t list_at(int32_t rank, int64_t p) const { return identity_list ? p : lists[(size_t)rank][(size_t)p]; }

  int32_t C() const { return cfg.batch / cfg.chunk; }

  // c.2 + c.3 + c.4
  void sample(int64_t s, int32_t rank, int64_t* pos, int64_t* neg, int8_t* mode) const {
    const int64_t B = cfg.batch, k = cfg.neg_k;
    if (repart()) {  // c.13': epoch e = s / S_E on every rank, position within the epoch wraps on this epoch's list
      const int64_t SE = epoch_steps(), e = s / SE;
      const std::vector<int64_t>& l = epoch_list(e, rank);
      const uint64_t nl = l.size();
      for (int64_t i = 0; i < B; ++i) {
        const uint64_t q = (uint64_t)(s - e * SE) * (uint64_t)B + (uint64_t)i;
        pos[i] = l[(size_t)feistel_index(nl, cfg.seed, (uint32_t)e, q % nl)];
      }
    } else {
      int64_t nl = list_size(rank);
      for (int64_t i = 0; i < B; ++i) {
        uint64_t q = (uint64_t)s * (uint64_t)B + (uint64_t)i;
        uint32_t e = (uint32_t)(q / (uint64_t)nl);
        uint64_t p = q % (uint64_t)nl;
        pos[i] = list_at(rank, (int64_t)feistel_index((uint64_t)nl, cfg.seed, e, p));
      }
    }
    for (int32_t c = 0; c < C(); ++c) {
      uint32_t cg = (uint32_t)(rank * C() + c);
      const int32_t md = mode_of(cfg.corrupt, (uint32_t)s, cg);
      if (mode) mode[c] = (int8_t)md;
      if (neg)
        for (int64_t j = 0; j < k; ++j) {
          if (j < cfg.neg_deg_k) {  // in-batch: the sampled triplet's tail (tail mode) / head (head mode)
            int64_t hh, rr, tt;
            triple(pos[deg_pos(cfg.seed, B, (uint32_t)s, cg, (uint32_t)j)], hh, rr, tt);
            neg[c * k + j] = md == ORC_TAIL ? tt : hh;
          } else if (cfg.neg_local && cfg.world_size > 1) {
            // local-shard negatives (PAPER.md:451-456 [3.3]: "sample entities from the local partition"; reading
            // c.3''): the c.3 draw mapped onto rank w's shard e = w + P * m, m uniform in [0, n_w)
            const int64_t P = cfg.world_size, n_w = (cfg.n_entities - rank + P - 1) / P;
            neg[c * k + j] = rank + P * neg_id(cfg.seed, n_w, (uint32_t)s, cg, (uint32_t)j);
          } else {
            neg[c * k + j] = neg_id(cfg.seed, cfg.n_entities, (uint32_t)s, cg, (uint32_t)j);
          }
        }
    }
  }
};

template <typename T>
struct Trainer : Base {
  RowStore<T> ent, rel, proj, ent_st, rel_st, proj_st;
  int32_t d = 0, drel = 0;
  bool has_proj = false;

  void setup() {
    d = cfg.dim;
    drel = cfg.model == ORC_ROTATE ? d / 2 : d;
    has_proj = cfg.model == ORC_TRANSR || cfg.model == ORC_RESCAL;
    float bound = cfg.init_bound > 0 ? cfg.init_bound : default_bound(cfg.gamma, d);
    float rbound = cfg.model == ORC_ROTATE ? (float)M_PI : bound;  // RotatE phases in [-pi, pi)
    bool lazy = cfg.lazy_rows != 0;
    ent.init(cfg.n_entities, d, 0, bound, cfg.seed, lazy, false);
    rel.init(cfg.n_relations, drel, 1, rbound, cfg.seed, false, false);
    ent_st.init(cfg.n_entities, 1, 3, 0, cfg.seed, lazy, true);
    rel_st.init(cfg.n_relations, 1, 4, 0, cfg.seed, false, true);
    if (has_proj) {
      proj.init(cfg.n_relations, d * d, 2, bound, cfg.seed, true, false);  // materialised on first touch
      proj_st.init(cfg.n_relations, 1, 5, 0, cfg.seed, true, true);
    }
  }

  RowStore<T>* store(int32_t table) {
    switch (table) {
      case 0: return &ent;
      case 1: return &rel;
      case 2: return has_proj ? &proj : nullptr;
      case 3: return &ent_st;
      case 4: return &rel_st;
      case 5: return has_proj ? &proj_st : nullptr;
    }
    return nullptr;
  }
  int32_t width(int32_t table) override {
    RowStore<T>* s = store(table);
    return s ? s->w : 0;
  }

  T score_ids(int64_t h, int64_t r, int64_t t) {
    return score_t<T>(cfg.model, cfg.rotate_variant, (T)cfg.gamma, d, ent.row(h), rel.row(r), ent.row(t),
                      has_proj ? proj.row(r) : nullptr);
  }

  int train(int64_t n_steps, double* losses) override {
    const int32_t P = cfg.world_size, B = cfg.batch, k = cfg.neg_k, g = cfg.chunk, Cn = C();
    const int64_t n_occ = 2 * (int64_t)B + (int64_t)Cn * k;
    for (int64_t it = 0; it < n_steps; ++it, ++step) {
      const int64_t s = step;
      // (1) sample every rank's batch
      std::vector<int64_t> pos((size_t)B), neg((size_t)Cn * k);
      std::vector<int8_t> mode((size_t)Cn);
      std::vector<int64_t> ent_ids((size_t)P * n_occ), rel_ids((size_t)P * B);
      std::vector<T> Gent((size_t)P * n_occ * d, T(0)), Grel((size_t)P * B * drel, T(0));
      std::vector<T> Gproj;
      if (has_proj) Gproj.assign((size_t)P * B * d * d, T(0));
      T loss_total = 0;
      for (int32_t w = 0; w < P; ++w) {
        sample(s, w, pos.data(), neg.data(), mode.data());
        std::vector<int64_t> hh((size_t)B), rr((size_t)B), tt((size_t)B);
        for (int32_t i = 0; i < B; ++i) triple(pos[(size_t)i], hh[(size_t)i], rr[(size_t)i], tt[(size_t)i]);
        int64_t* eo = &ent_ids[(size_t)w * n_occ];
        for (int32_t i = 0; i < B; ++i) {
          eo[i] = hh[(size_t)i];
          eo[B + i] = tt[(size_t)i];
          rel_ids[(size_t)w * B + i] = rr[(size_t)i];
        }
        for (int64_t q = 0; q < (int64_t)Cn * k; ++q) eo[2 * B + q] = neg[(size_t)q];
        // (2)+(3) fetch rows and score: positives f+_i = f(h_i, r_i, t_i); negatives naive per triple (c.8)
        // (rows are materialised serially first: the optional parallel loops below only read the stores)
        for (int32_t i = 0; i < B; ++i) {
          ent.row(hh[(size_t)i]);
          ent.row(tt[(size_t)i]);
          rel.row(rr[(size_t)i]);
          if (has_proj) proj.row(rr[(size_t)i]);
        }
        for (int64_t q = 0; q < (int64_t)Cn * k; ++q) ent.row(neg[(size_t)q]);
        const int nth = threads();
        std::vector<T> fpos((size_t)B), fneg((size_t)B * k), dpos((size_t)B), dneg((size_t)B * k);
        for (int32_t i = 0; i < B; ++i) fpos[(size_t)i] = score_ids(hh[(size_t)i], rr[(size_t)i], tt[(size_t)i]);
#pragma omp parallel for num_threads(nth) schedule(dynamic, 8) if (nth > 1)
        for (int32_t i = 0; i < B; ++i) {
          int32_t c = i / g;
          for (int32_t j = 0; j < k; ++j) {
            int64_t x = neg[(size_t)c * k + j];
            fneg[(size_t)i * k + j] = mode[(size_t)c] == ORC_TAIL ? score_ids(hh[(size_t)i], rr[(size_t)i], x)
                                                                  : score_ids(x, rr[(size_t)i], tt[(size_t)i]);
          }
        }
        if (cfg.loss == ORC_LOSS_PAIRWISE) {  // pairwise ranking loss, reading c.9'
          loss_total += ranking_loss<T>(fpos.data(), fneg.data(), B, k, (T)cfg.gamma, dpos.data(), dneg.data());
        } else {  // logistic loss, c.9 normalisation
          T lp = 0, ln = 0;
          for (int32_t i = 0; i < B; ++i) {
            lp += log_sigmoid(fpos[(size_t)i]);
            dpos[(size_t)i] = -sigmoid(-fpos[(size_t)i]) / (T)B;
          }
          for (int64_t q = 0; q < (int64_t)B * k; ++q) {
            ln += log_sigmoid(-fneg[(size_t)q]);
            dneg[(size_t)q] = sigmoid(fneg[(size_t)q]) / ((T)B * (T)k);
          }
          loss_total += -lp / (T)B - ln / ((T)B * (T)k);
        }
        // backward: per-occurrence gradients (c.10); positive term first, then j = 0..k-1
        T* G = &Gent[(size_t)w * n_occ * d];
        T* GR = &Grel[(size_t)w * B * drel];
#pragma omp parallel for num_threads(nth) schedule(dynamic, 8) if (nth > 1)
        for (int32_t i = 0; i < B; ++i) {
          std::vector<T> sink((size_t)d, T(0));
          int32_t c = i / g;
          T* gh = G + (size_t)i * d;
          T* gt = G + (size_t)(B + i) * d;
          T* gr = GR + (size_t)i * drel;
          T* gm = has_proj ? &Gproj[((size_t)w * B + i) * d * d] : nullptr;
          const T* M = has_proj ? proj.row(rr[(size_t)i]) : nullptr;
          grad_t<T>(cfg.model, cfg.rotate_variant, d, ent.row(hh[(size_t)i]), rel.row(rr[(size_t)i]),
                    ent.row(tt[(size_t)i]), M, dpos[(size_t)i], gh, gr, gt, gm);
          for (int32_t j = 0; j < k; ++j) {
            int64_t x = neg[(size_t)c * k + j];
            T up = dneg[(size_t)i * k + j];
            std::fill(sink.begin(), sink.end(), T(0));
            if (mode[(size_t)c] == ORC_TAIL)
              grad_t<T>(cfg.model, cfg.rotate_variant, d, ent.row(hh[(size_t)i]), rel.row(rr[(size_t)i]), ent.row(x),
                        M, up, gh, gr, sink.data(), gm);
            else
              grad_t<T>(cfg.model, cfg.rotate_variant, d, ent.row(x), rel.row(rr[(size_t)i]), ent.row(tt[(size_t)i]),
                        M, up, sink.data(), gr, gt, gm);
          }
        }
        // negatives: sum over i in the chunk, ascending (c.10)
#pragma omp parallel for num_threads(nth) schedule(dynamic, 4) if (nth > 1)
        for (int64_t cj = 0; cj < (int64_t)Cn * k; ++cj) {
            const int32_t c = (int32_t)(cj / k), j = (int32_t)(cj % k);
            std::vector<T> junk_r((size_t)drel), junk_e((size_t)d), junk_m(has_proj ? (size_t)d * d : 0);
            int64_t x = neg[(size_t)c * k + j];
            T* gx = G + (size_t)(2 * B + c * k + j) * d;
            for (int32_t i = c * g; i < (c + 1) * g; ++i) {
              const T* M = has_proj ? proj.row(rr[(size_t)i]) : nullptr;
              T up = dneg[(size_t)i * k + j];
              if (mode[(size_t)c] == ORC_TAIL)
                grad_t<T>(cfg.model, cfg.rotate_variant, d, ent.row(hh[(size_t)i]), rel.row(rr[(size_t)i]), ent.row(x),
                          M, up, junk_e.data(), junk_r.data(), gx, has_proj ? junk_m.data() : nullptr);
              else
                grad_t<T>(cfg.model, cfg.rotate_variant, d, ent.row(x), rel.row(rr[(size_t)i]), ent.row(tt[(size_t)i]),
                          M, up, gx, junk_r.data(), junk_e.data(), has_proj ? junk_m.data() : nullptr);
            }
          }
      }
      if (losses) losses[it] = (double)loss_total;
      // (4) apply: dedup over the union (rank-major occurrence order), sum in segment order, Adagrad (c.11).
      // lag = 1 (reading c.12): relations (and TransR projections) are updated now; the entity
      // update of this step is held back and applied after the next step has computed its gradients, i.e. step s
      // reads entity rows updated by steps <= s-2 -- the previous step's entity update is applied here, after this
      // step's forward/backward
      apply(rel, rel_st, rel_ids, Grel, drel);
      if (has_proj) apply(proj, proj_st, rel_ids, Gproj, d * d);
      if (cfg.lag == 1) {
        flush();
        pend_ids.swap(ent_ids);
        pend_G.swap(Gent);
        pending = true;
      } else {
        apply(ent, ent_st, ent_ids, Gent, d);
      }
    }
    return 0;
  }

  // lag = 1: the held-back entity update of the last step
  std::vector<int64_t> pend_ids;
  std::vector<T> pend_G;
  bool pending = false;
  int flush() override {
    if (pending) apply(ent, ent_st, pend_ids, pend_G, d);
    pending = false;
    return 0;
  }

  void apply(RowStore<T>& tab, RowStore<T>& st, const std::vector<int64_t>& ids, const std::vector<T>& G, int32_t w) {
    int64_t n = (int64_t)ids.size();
    std::vector<int64_t> uniq((size_t)n), seg_off((size_t)n + 1), seg_occ((size_t)n);
    std::vector<int32_t> inv((size_t)n);
    int64_t nu = dedup(ids.data(), n, uniq.data(), inv.data(), seg_off.data(), seg_occ.data());
    // c.13: with P ranks the occurrences are rank-major; each rank's occurrences of a row are summed first (in
    // occurrence order) and the rank sums are added in rank order -- "entity gradients meet at the owner and are
    // summed", "split relations ... all-gathered and summed in rank order". P = 1: one plain sum.
    const int64_t per = n / cfg.world_size;
    std::vector<T> gsum((size_t)w), gpart((size_t)w);
    for (int64_t u = 0; u < nu; ++u) {
      std::fill(gsum.begin(), gsum.end(), T(0));
      std::fill(gpart.begin(), gpart.end(), T(0));
      int64_t cur = -1;
      for (int64_t p = seg_off[(size_t)u]; p < seg_off[(size_t)u + 1]; ++p) {
        const int64_t o = seg_occ[(size_t)p];
        if (o / per != cur) {
          if (cur >= 0)
            for (int32_t c = 0; c < w; ++c) gsum[(size_t)c] += gpart[(size_t)c];
          std::fill(gpart.begin(), gpart.end(), T(0));
          cur = o / per;
        }
        const T* go = &G[(size_t)o * w];
        for (int32_t c = 0; c < w; ++c) gpart[(size_t)c] += go[c];
      }
      for (int32_t c = 0; c < w; ++c) gsum[(size_t)c] += gpart[(size_t)c];
      T* row = tab.row(uniq[(size_t)u]);
      T* s = st.row(uniq[(size_t)u]);
      T sq = 0;
      for (int32_t c = 0; c < w; ++c) sq += gsum[(size_t)c] * gsum[(size_t)c];
      s[0] += sq / (T)w;
      T den = std::sqrt(s[0] + (T)cfg.eps);
      for (int32_t c = 0; c < w; ++c) row[c] -= (T)cfg.lr * gsum[(size_t)c] / den;
    }
  }

  int get_rows(int32_t table, const int64_t* ids, int64_t n, double* out) override {
    RowStore<T>* s = store(table);
    if (!s) return -1;
    for (int64_t i = 0; i < n; ++i) {
      if (ids[i] < 0 || ids[i] >= s->n) return -2;
      T* r = s->row(ids[i]);
      for (int32_t c = 0; c < s->w; ++c) out[(size_t)i * s->w + c] = (double)r[c];
    }
    return 0;
  }
  int set_rows(int32_t table, const int64_t* ids, int64_t n, const double* in) override {
    RowStore<T>* s = store(table);
    if (!s) return -1;
    for (int64_t i = 0; i < n; ++i) {
      if (ids[i] < 0 || ids[i] >= s->n) return -2;
      T* r = s->row(ids[i]);
      for (int32_t c = 0; c < s->w; ++c) r[c] = (T)in[(size_t)i * s->w + c];
    }
    return 0;
  }
  int score_triples(const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, double* out) override {
    const int nth = threads();
    if (nth > 1)  // materialise lazily stored rows serially; the parallel loop then only reads the stores
      for (int64_t i = 0; i < n; ++i) {
        ent.row(hs[i]);
        ent.row(ts[i]);
        rel.row(rs[i]);
        if (has_proj) proj.row(rs[i]);
      }
#pragma omp parallel for num_threads(nth) schedule(static) if (nth > 1)
    for (int64_t i = 0; i < n; ++i) out[i] = (double)score_ids(hs[i], rs[i], ts[i]);
    return 0;
  }
};

// c.8 decomposition: o = combine(h, r) for tail mode, combine'(r, t) for head mode,
// then a pair score of o against each sampled entity x. Used only to pin "joint == naive".
void combine(int32_t model, int32_t d, int32_t mode, const double* h, const double* r, const double* t,
             const double* M, double* o) {
  int32_t n = d / 2;
  switch (model) {
    case ORC_TRANSE_L1:
    case ORC_TRANSE_L2:
      for (int32_t e = 0; e < d; ++e) o[e] = mode == 0 ? h[e] + r[e] : t[e] - r[e];
      return;
    case ORC_DISTMULT:
      for (int32_t e = 0; e < d; ++e) o[e] = mode == 0 ? h[e] * r[e] : r[e] * t[e];
      return;
    case ORC_COMPLEX:
      for (int32_t e = 0; e < n; ++e) {
        double rr = r[e], ri = r[e + n];
        if (mode == 0) {
          o[e] = h[e] * rr - h[e + n] * ri;
          o[e + n] = h[e] * ri + h[e + n] * rr;
        } else {
          o[e] = rr * t[e] + ri * t[e + n];
          o[e + n] = rr * t[e + n] - ri * t[e];
        }
      }
      return;
    case ORC_ROTATE:
      for (int32_t e = 0; e < n; ++e) {
        double c = std::cos(r[e]), s = std::sin(r[e]);
        if (mode == 0) {  // h * e^{i theta}
          o[e] = h[e] * c - h[e + n] * s;
          o[e + n] = h[e] * s + h[e + n] * c;
        } else {  // t * e^{-i theta}
          o[e] = t[e] * c + t[e + n] * s;
          o[e + n] = -t[e] * s + t[e + n] * c;
        }
      }
      return;
    case ORC_RESCAL:  // tail: o = M^T h (f = o . t'); head: o = M t (f = h' . o)
      for (int32_t a = 0; a < d; ++a) {
        double acc = 0;
        for (int32_t b = 0; b < d; ++b) acc += mode == 0 ? h[b] * M[(int64_t)b * d + a] : M[(int64_t)a * d + b] * t[b];
        o[a] = acc;
      }
      return;
    case ORC_TRANSR:
      for (int32_t a = 0; a < d; ++a) {
        double acc = 0;
        const double* x = mode == 0 ? h : t;
        for (int32_t b = 0; b < d; ++b) acc += M[(int64_t)a * d + b] * x[b];
        o[a] = mode == 0 ? acc + r[a] : acc - r[a];
      }
      return;
  }
}

double pair_score(int32_t model, int32_t variant, double gamma, int32_t d, const double* o, const double* x,
                  const double* M) {
  int32_t n = d / 2;
  double s = 0;
  switch (model) {
    case ORC_TRANSE_L1:
      for (int32_t e = 0; e < d; ++e) s += std::fabs(o[e] - x[e]);
      return gamma - s;
    case ORC_TRANSE_L2:
      for (int32_t e = 0; e < d; ++e) s += (o[e] - x[e]) * (o[e] - x[e]);
      return gamma - std::sqrt(s);
    case ORC_DISTMULT:
    case ORC_COMPLEX:
    case ORC_RESCAL:
      for (int32_t e = 0; e < d; ++e) s += o[e] * x[e];
      return s;
    case ORC_ROTATE:
      for (int32_t e = 0; e < n; ++e) {
        double u = o[e] - x[e], v = o[e + n] - x[e + n];
        s += variant == 0 ? u * u + v * v : std::sqrt(u * u + v * v);
      }
      return gamma - s;
    case ORC_TRANSR:
      for (int32_t a = 0; a < d; ++a) {
        double q = 0;
        for (int32_t b = 0; b < d; ++b) q += M[(int64_t)a * d + b] * x[b];
        s += (o[a] - q) * (o[a] - q);
      }
      return gamma - s;
  }
  return 0;
}

}  // namespace

// ================================================================================================
// C API
// ================================================================================================
extern "C" {

void orc_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) { philox(ctr, key, out); }
uint64_t orc_feistel_index(uint64_t n, uint64_t seed, uint32_t epoch, uint64_t p) {
  return feistel_index(n, seed, epoch, p);
}
int64_t orc_neg_id(uint64_t seed, int64_t n_entities, uint32_t step, uint32_t cg, uint32_t j) {
  return neg_id(seed, n_entities, step, cg, j);
}
int32_t orc_mode(int32_t corrupt, uint32_t step, uint32_t cg) { return mode_of(corrupt, step, cg); }
float orc_init_value(uint64_t seed, int32_t table, int64_t row, int64_t col, float bound) {
  return init_value(seed, table, row, col, bound);
}
float orc_default_bound(float gamma, int32_t dim) { return default_bound(gamma, dim); }

int32_t orc_relation_partition(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P, int32_t* owner_out) {
  std::vector<int32_t> owner;
  std::vector<int64_t> counts;
  int32_t ns = relation_partition(rels, n_triples, n_rel, P, owner, counts);
  for (int64_t r = 0; r < n_rel; ++r) owner_out[r] = owner[(size_t)r];
  return ns;
}
int64_t orc_locality_order(const int64_t* heads, const int64_t* tails, int64_t n_triples, int64_t n_entities, int32_t P,
                           int64_t* new_id_out, int32_t* part_out) {
  std::vector<int64_t> nid;
  std::vector<int32_t> part;
  const int64_t cut = locality_order(heads, tails, n_triples, n_entities, P, nid, part);
  std::copy(nid.begin(), nid.end(), new_id_out);
  if (part_out) std::copy(part.begin(), part.end(), part_out);
  return cut;
}
int32_t orc_relation_partition_epoch(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P, uint64_t seed,
                                     uint32_t epoch, int32_t* owner_out) {
  std::vector<int32_t> owner;
  std::vector<int64_t> counts;
  int32_t ns = relation_partition(rels, n_triples, n_rel, P, owner, counts, true, seed, epoch);
  for (int64_t r = 0; r < n_rel; ++r) owner_out[r] = owner[(size_t)r];
  return ns;
}
int64_t orc_rank_triples(const int64_t* rels, int64_t n_triples, int64_t n_rel, int32_t P, int32_t rank,
                         int64_t* idx_out) {
  std::vector<std::vector<int64_t>> lists;
  rank_lists(rels, n_triples, n_rel, P, lists);
  const auto& l = lists[(size_t)rank];
  if (idx_out) std::copy(l.begin(), l.end(), idx_out);
  return (int64_t)l.size();
}

double orc_score(int32_t model, int32_t variant, double gamma, int32_t d, const double* h, const double* r,
                 const double* t, const double* M) {
  return score_t<double>(model, variant, gamma, d, h, r, t, M);
}
float orc_score_f(int32_t model, int32_t variant, float gamma, int32_t d, const float* h, const float* r,
                  const float* t, const float* M) {
  return score_t<float>(model, variant, gamma, d, h, r, t, M);
}
void orc_score_grad(int32_t model, int32_t variant, double gamma, int32_t d, const double* h, const double* r,
                    const double* t, const double* M, double upstream, double* dh, double* dr, double* dt,
                    double* dM) {
  (void)gamma;
  grad_t<double>(model, variant, d, h, r, t, M, upstream, dh, dr, dt, dM);
}
void orc_score_group(int32_t model, int32_t variant, double gamma, int32_t d, int32_t mode, int32_t g, int32_t k,
                     const double* H, const double* R, const double* T, const double* M, const double* X,
                     double* out) {
  int32_t drel = model == ORC_ROTATE ? d / 2 : d;
  std::vector<double> o((size_t)d);
  for (int32_t i = 0; i < g; ++i) {
    const double* Mi = M ? M + (size_t)i * d * d : nullptr;
    combine(model, d, mode, H + (size_t)i * d, R + (size_t)i * drel, T + (size_t)i * d, Mi, o.data());
    for (int32_t j = 0; j < k; ++j) out[(size_t)i * k + j] = pair_score(model, variant, gamma, d, o.data(), X + (size_t)j * d, Mi);
  }
}
void orc_eval_candidates(uint64_t seed, int64_t n_ent, int64_t n_trip, const int64_t* th, const int64_t* tt,
                         int64_t n_queries, int64_t n_uniform, int64_t n_degree, int32_t both, int64_t* ent,
                         int32_t* side) {
  const int64_t m = n_uniform + n_degree;
  for (int64_t i = 0; i < n_queries; ++i)
    for (int64_t j = 0; j < m; ++j) eval_candidate(seed, n_ent, n_trip, th, tt, i, j, n_uniform, both, ent + i * m + j,
                                                   side + i * m + j);
}
double orc_ranking_loss(const double* pos, const double* neg, int64_t B, int64_t k, double gamma, double* dpos,
                        double* dneg) {
  return ranking_loss<double>(pos, neg, B, k, gamma, dpos, dneg);
}
double orc_logistic_loss(const double* pos, int64_t n_pos, const double* neg, int64_t n_neg, int64_t B, int64_t k,
                         double* dpos, double* dneg) {
  double lp = 0, ln = 0;
  for (int64_t i = 0; i < n_pos; ++i) {
    lp += log_sigmoid(pos[i]);
    if (dpos) dpos[i] = -sigmoid(-pos[i]) / (double)B;
  }
  for (int64_t q = 0; q < n_neg; ++q) {
    ln += log_sigmoid(-neg[q]);
    if (dneg) dneg[q] = sigmoid(neg[q]) / ((double)B * (double)k);
  }
  return -lp / (double)B - ln / ((double)B * (double)k);
}
void orc_adagrad(double* row, double* state, const double* g, int32_t w, double lr, double eps) {
  double sq = 0;
  for (int32_t c = 0; c < w; ++c) sq += g[c] * g[c];
  state[0] += sq / (double)w;
  double den = std::sqrt(state[0] + eps);
  for (int32_t c = 0; c < w; ++c) row[c] -= lr * g[c] / den;
}
int64_t orc_dedup(const int64_t* ids, int64_t n, int64_t* uniq, int32_t* inv, int64_t* seg_off, int64_t* seg_occ) {
  return dedup(ids, n, uniq, inv, seg_off, seg_occ);
}

void* orc_create(const orc_config* cfg, const int64_t* heads, const int64_t* rels, const int64_t* tails,
                 int64_t n_triples, orc_triple_fn fn, void* ctx) {
  if (!cfg || cfg->batch <= 0 || cfg->chunk <= 0 || cfg->batch % cfg->chunk != 0 || cfg->neg_k <= 0) return nullptr;
  if ((cfg->model == ORC_COMPLEX || cfg->model == ORC_ROTATE) && cfg->dim % 2 != 0) return nullptr;
  if (cfg->world_size < 1 || n_triples <= 0) return nullptr;
  if (cfg->lag != 0 && cfg->lag != 1) return nullptr;
  if (cfg->neg_deg_k < 0 || cfg->neg_deg_k > cfg->neg_k) return nullptr;
  Base* b;
  if (cfg->precision == 1) {
    auto* t = new Trainer<float>();
    t->cfg = *cfg;
    t->setup();
    b = t;
  } else {
    auto* t = new Trainer<double>();
    t->cfg = *cfg;
    t->setup();
    b = t;
  }
  b->nt = n_triples;
  b->fn = fn;
  b->ctx = ctx;
  if (!fn) {
    b->H.assign(heads, heads + n_triples);
    b->R.assign(rels, rels + n_triples);
    b->Tt.assign(tails, tails + n_triples);
  }
  if (cfg->world_size == 1) {
    b->identity_list = true;
  } else {
    std::vector<int64_t> rr((size_t)n_triples);
    for (int64_t i = 0; i < n_triples; ++i) {
      int64_t h, r, t;
      b->triple(i, h, r, t);
      rr[(size_t)i] = r;
    }
    if (cfg->placement == 1) {  // c.13'' head-owner placement
      std::vector<int64_t> hh((size_t)n_triples);
      for (int64_t i = 0; i < n_triples; ++i) {
        int64_t h, r, t;
        b->triple(i, h, r, t);
        hh[(size_t)i] = h;
      }
      head_owner_lists(hh, cfg->world_size, b->lists);
    } else {
      rank_lists(rr.data(), n_triples, cfg->n_relations, cfg->world_size, b->lists);
    }
    for (const auto& l : b->lists)
      if (l.empty()) {
        delete b;
        return nullptr;
      }
    b->RR.swap(rr);
  }
  return b;
}
void orc_destroy(void* h) { delete static_cast<Base*>(h); }
int orc_sample(void* h, int64_t step, int32_t rank, int64_t* pos_idx, int64_t* neg, int8_t* mode) {
  static_cast<Base*>(h)->sample(step, rank, pos_idx, neg, mode);
  return 0;
}
int orc_occurrences(void* hp, int64_t step, int32_t rank, int64_t* ent_occ, int64_t* rel_occ) {
  Base* b = static_cast<Base*>(hp);
  const int32_t B = b->cfg.batch, k = b->cfg.neg_k, Cn = b->C();
  std::vector<int64_t> pos((size_t)B), neg((size_t)Cn * k);
  b->sample(step, rank, pos.data(), neg.data(), nullptr);
  for (int32_t i = 0; i < B; ++i) {
    int64_t hh, rr, tt;
    b->triple(pos[(size_t)i], hh, rr, tt);
    if (ent_occ) {
      ent_occ[i] = hh;
      ent_occ[B + i] = tt;
    }
    if (rel_occ) rel_occ[i] = rr;
  }
  if (ent_occ)
    for (int64_t q = 0; q < (int64_t)Cn * k; ++q) ent_occ[2 * B + q] = neg[(size_t)q];
  return 0;
}
int orc_train(void* h, int64_t n_steps, double* losses) { return static_cast<Base*>(h)->train(n_steps, losses); }
int orc_flush(void* h) { return static_cast<Base*>(h)->flush(); }
int orc_get_rows(void* h, int32_t table, const int64_t* ids, int64_t n, double* out) {
  return static_cast<Base*>(h)->get_rows(table, ids, n, out);
}
int orc_set_rows(void* h, int32_t table, const int64_t* ids, int64_t n, const double* in) {
  return static_cast<Base*>(h)->set_rows(table, ids, n, in);
}
int orc_score_triples(void* h, const int64_t* hs, const int64_t* rs, const int64_t* ts, int64_t n, double* out) {
  return static_cast<Base*>(h)->score_triples(hs, rs, ts, n, out);
}
int64_t orc_next_step(void* h) { return static_cast<Base*>(h)->step; }
// continue from step s (counter-based sampling: (seed, s) fixes the sample; teacher-forced spot checks)
void orc_set_step(void* h, int64_t s) { static_cast<Base*>(h)->step = s; }
int32_t orc_table_width(void* h, int32_t table) { return static_cast<Base*>(h)->width(table); }

}  // extern "C"
