/*
 * kron_host.c -- host twin of the seeded Kronecker input generator (definition in kron_gen.h).
 * Input generation only: no BFS arithmetic.  Built as libkron_host.so; used by the tests and
 * by the CPU-oracle leg of bench.py.  Bit-identical to the device generator (inputs/kron_dev.cu).
 */
#include "kron_gen.h"
#include <stddef.h>

/* Tuples [k0, k0+count) of the scale/seed graph into s[], d[] (u64 ids). */
void kron_host_generate(int scale, uint64_t seed, uint64_t k0, uint64_t count, uint64_t* s, uint64_t* d) {
  kron_params p = kron_make_params(scale, seed);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) {
    kron_tuple(&p, k0 + (uint64_t)i, &s[i], &d[i]);
  }
}

/* Same, narrowed to u32 ids (scale <= 32). */
void kron_host_generate_u32(int scale, uint64_t seed, uint64_t k0, uint64_t count, uint32_t* s, uint32_t* d) {
  kron_params p = kron_make_params(scale, seed);
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)count; ++i) {
    uint64_t a, b;
    kron_tuple(&p, k0 + (uint64_t)i, &a, &b);
    s[i] = (uint32_t)a;
    d[i] = (uint32_t)b;
  }
}

uint64_t kron_host_scramble(int scale, uint64_t seed, uint64_t x) {
  kron_params p = kron_make_params(scale, seed);
  return kron_scramble(&p, x);
}

uint64_t kron_host_root_candidate(uint64_t root_seed, uint64_t t, uint64_t nverts) {
  return kron_root_candidate(root_seed, t, nverts);
}

void kron_host_thresholds(uint32_t* out3) {
  kron_params p = kron_make_params(1, 0);
  out3[0] = p.t_ab;
  out3[1] = p.t_an;
  out3[2] = p.t_cn;
}
