// engine.h -- internal helpers shared by engine.cu (ABI, level loop, transport) and build_graph.cu.
#pragma once
#include <vector>

#include "bfs_internal.h"

namespace bfs200 {

int set_err(int status, const char* fmt, ...);
int cuda_fail(Graph& G, cudaError_t e, const char* what, const char* file, int line);
int nccl_fail(Graph& G, ncclResult_t r, const char* what, const char* file, int line);
bool is_device_ptr(const void* p);

// graph-lifetime device allocation (tracked, freed by bfs_destroy)
int G_alloc(Graph& G, void** p, size_t bytes);

// call-lifetime device scratch: freed when the Scratch goes out of scope
struct Scratch {
  std::vector<void*> ptrs;
  template <typename T>
  cudaError_t alloc(T** p, size_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = (T*)q;
    return e;
  }
  void release(void* p) {
    for (auto& q : ptrs)
      if (q == p) {
        cudaFree(q);
        q = nullptr;
      }
  }
  ~Scratch() {
    for (void* q : ptrs)
      if (q) cudaFree(q);
  }
};

#define CKR(x)                                                                   \
  do {                                                                           \
    cudaError_t _e = (x);                                                        \
    if (_e != cudaSuccess) return ::bfs200::cuda_fail(G, _e, #x, __FILE__, __LINE__); \
  } while (0)
#define NKR(x)                                                                   \
  do {                                                                           \
    ncclResult_t _r = (x);                                                       \
    if (_r != ncclSuccess) return ::bfs200::nccl_fail(G, _r, #x, __FILE__, __LINE__); \
  } while (0)

// transport (NCCL, world_size > 1)
int comm_allreduce_int_max(Graph& G, int* v);
int comm_exchange_counts(Graph& G, const unsigned long long* d_send_counts, unsigned long long* d_recv_counts);
int comm_alltoallv_u64(Graph& G, const unsigned long long* send, const unsigned long long* soff,
                       const unsigned long long* scnt, unsigned long long* recv, const unsigned long long* roff,
                       const unsigned long long* rcnt);
int comm_allreduce_u32_sum(Graph& G, uint32_t* buf, uint64_t n);
int comm_reduce_scatter_u32(Graph& G, const uint32_t* full, uint32_t* mine, uint64_t block);

int build_graph(Graph& G, const uint64_t* src, const uint64_t* dst, uint64_t m);

}  // namespace bfs200
