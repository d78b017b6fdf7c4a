/*
 * kron_gen.h -- the seeded synthetic INPUT generator (Graph500-style Kronecker / R-MAT).
 *
 * This header is the single definition of the benchmark input.  It is shared by the
 * host generator (inputs/kron_host.c, used by tests and the CPU oracle leg) and the
 * device generator (inputs/kron_dev.cu, used by bench.py), so both produce bit-identical
 * tuple lists.  It holds NONE of the BFS method's arithmetic: no partitioning, no CSC,
 * no traversal.  (The oracle never includes it; it receives plain edge arrays.)
 *
 * What it generates ("make_graph" R-MAT, edge factor 16;
 * parameters A,B,C,D = 0.57,0.19,0.19,0.05 from BASELINE.json / SPEC.md S:71):
 *   M = edgefactor * 2^scale directed tuples (s_k, d_k), k = 0..M-1, ids < 2^scale.
 *   For bit b < scale of tuple k draw one 64-bit word h = H(key, 64k + b):
 *       U1 = low 32 bits, U2 = high 32 bits
 *       ii_b = U1 > T_AB                       (P(ii=1) = C+D = 0.24)
 *       jj_b = U2 > (ii_b ? T_CN : T_AN)       (P(jj=1|ii=0) = B/(A+B), P(jj=1|ii=1) = D/(C+D))
 *   s_raw = sum ii_b 2^b, d_raw = sum jj_b 2^b  (the Graph500 kronecker_generator recursion)
 *   s = pi(s_raw), d = pi(d_raw) with pi a seeded bijection of [0, 2^scale) (Graph500
 *   scrambles vertex ids; SURVEY.md §8(c) reading 13).
 *   Duplicates and self-loops are kept.
 * H is the splitmix64 output function evaluated at counter x (a counter-based generator,
 * so any rank / the host can regenerate any tuple range independently).
 */
#ifndef KRON_GEN_H
#define KRON_GEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define KRON_FN __host__ __device__ __forceinline__
#else
#define KRON_FN static inline
#endif

#define KRON_GOLDEN 0x9E3779B97F4A7C15ULL

/* splitmix64 finaliser */
KRON_FN uint64_t kron_fmix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

/* key derived from a user seed */
KRON_FN uint64_t kron_key(uint64_t seed) { return kron_fmix(seed ^ 0x5DEECE66DULL); }

/* counter-based 64-bit draw number x of stream `key` (splitmix64's x-th output) */
KRON_FN uint64_t kron_hash(uint64_t key, uint64_t x) { return kron_fmix(key + (x + 1ULL) * KRON_GOLDEN); }

/* R-MAT thresholds as u32 comparands: floor(p * 2^32). */
typedef struct {
  uint32_t t_ab; /* A+B            */
  uint32_t t_an; /* A/(A+B)        */
  uint32_t t_cn; /* C/(C+D)        */
  int scale;
  uint64_t key;
  uint64_t mask;      /* 2^scale - 1 */
  uint64_t mul1, add1, mul2, add2; /* scramble constants */
} kron_params;

KRON_FN uint32_t kron_thr(double p) {
  double t = p * 4294967296.0;
  if (t >= 4294967295.0) return 0xFFFFFFFFu;
  if (t <= 0.0) return 0u;
  return (uint32_t)t;
}

/* Graph500 defaults A,B,C = 0.57,0.19,0.19 (D = 0.05). */
KRON_FN kron_params kron_make_params(int scale, uint64_t seed) {
  kron_params p;
  const double A = 0.57, B = 0.19, C = 0.19, D = 1.0 - A - B - C;
  p.t_ab = kron_thr(A + B);
  p.t_an = kron_thr(A / (A + B));
  p.t_cn = kron_thr(C / (C + D));
  p.scale = scale;
  p.key = kron_key(seed);
  p.mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1ULL);
  /* scramble constants come from a counter range disjoint from tuple draws (x < 2^43) */
  p.mul1 = kron_hash(p.key, (1ULL << 60) + 1) | 1ULL;
  p.add1 = kron_hash(p.key, (1ULL << 60) + 2);
  p.mul2 = kron_hash(p.key, (1ULL << 60) + 3) | 1ULL;
  p.add2 = kron_hash(p.key, (1ULL << 60) + 4);
  return p;
}

/* pi: bijection of [0, 2^scale): odd multiply, xorshift, add (each invertible mod 2^scale) */
KRON_FN uint64_t kron_scramble(const kron_params* p, uint64_t x) {
  const int sh = (p->scale + 1) / 2;
  x = (x * p->mul1) & p->mask;
  if (sh > 0) x ^= x >> sh;
  x = (x + p->add1) & p->mask;
  x = (x * p->mul2) & p->mask;
  if (sh > 0) x ^= x >> sh;
  x = (x + p->add2) & p->mask;
  return x;
}

/* tuple k -> (s, d) */
KRON_FN void kron_tuple(const kron_params* p, uint64_t k, uint64_t* s, uint64_t* d) {
  uint64_t si = 0, di = 0;
  for (int b = 0; b < p->scale; ++b) {
    uint64_t h = kron_hash(p->key, k * 64ULL + (uint64_t)b);
    uint32_t u1 = (uint32_t)h, u2 = (uint32_t)(h >> 32);
    uint64_t ii = u1 > p->t_ab;
    uint64_t jj = u2 > (ii ? p->t_cn : p->t_an);
    si |= ii << b;
    di |= jj << b;
  }
  *s = kron_scramble(p, si);
  *d = kron_scramble(p, di);
}

/* Root candidates: candidate t of root stream `root_seed`, uniform over [0, nverts). The caller
 * keeps candidates with degree >= 1 (self-loops excluded) that were not drawn before. */
KRON_FN uint64_t kron_root_candidate(uint64_t root_seed, uint64_t t, uint64_t nverts) {
  uint64_t h = kron_hash(kron_key(root_seed ^ 0xA5A5A5A5ULL), t);
  return nverts ? (h % nverts) : 0;
}

#endif /* KRON_GEN_H */
