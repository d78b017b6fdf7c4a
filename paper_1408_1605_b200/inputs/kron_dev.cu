// kron_dev.cu -- device twin of the seeded Kronecker input generator (definition: kron_gen.h).
// Input generation only (no BFS arithmetic); built as libkron_dev.so and used by bench.py to
// create the Graph500-style tuple list directly in HBM.  Bit-identical to kron_host.c.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kron_gen.h"

__global__ void k_kron_generate(kron_params p, uint64_t k0, uint64_t count, uint64_t* s, uint64_t* d) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t a, b;
    kron_tuple(&p, k0 + i, &a, &b);
    s[i] = a;
    d[i] = b;
  }
}

extern "C" {

// Tuples [k0, k0+count) of the (scale, seed) graph into device arrays s[], d[] on `stream`.
// Returns a cudaError_t value (0 = success). Asynchronous.
int kron_device_generate(int scale, uint64_t seed, uint64_t k0, uint64_t count, uint64_t* s, uint64_t* d,
                         void* stream) {
  if (scale < 0 || scale > 32) return (int)cudaErrorInvalidValue;
  if (!count) return 0;
  kron_params p = kron_make_params(scale, seed);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (count + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  k_kron_generate<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p, k0, count, s, d);
  return (int)cudaGetLastError();
}

}
