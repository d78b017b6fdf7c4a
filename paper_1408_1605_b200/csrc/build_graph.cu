// build_graph.cu -- graph construction: tuples -> 2D partition -> per-rank CSC/CSR (not timed).
//
// PAPER.md P:300-303 ("the graph is partitioned as described in Section 2DPart")
// (symmetrise), P:275-291 (local (N/R) x (N/C) matrix stored as CSC: `col` offsets + `row`
// indices).  Each tuple (a, b), a != b, is inserted as edge a->b and b->a; edge u->v goes to
// P_ij with i = (v/block) mod R, j = u/(N/C) as column
// local_col(u) = u mod N/C and row local_row(v) = (v/block/R)*block + v mod block.
// Duplicates collapse and self-loops are dropped.  tdeg[v] counts every input
// tuple with source v (the m_comp numerator), duplicates and self-loops included.
//
// Internal relabeling (layout only): inside every vertex block the vertices are
// renumbered by descending degree; ownership (the block) never changes and all outputs are in the
// original ids.  The expansion keeps the visited bits of the hot (highest-degree) prefixes in
// shared memory.
// To keep the minimum-id parent rule in original ids, CSC rows are ordered by ORIGINAL row id
// and CSR rows by ORIGINAL column id (the stored indices are the relabeled ones).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <vector>

#include "engine.h"

namespace bfs200 {

typedef unsigned long long ull;

struct PartMap {
  uint64_t block, ncols, nverts;
  int R, C, rbits;
  __device__ __forceinline__ int dest(uint64_t u, uint64_t v) const {
    const int i = (int)((v / block) % (uint64_t)R);
    const int j = (int)(u / ncols);
    return j * R + i;
  }
  // CSC sort key: relabeled local column, then relabeled local row (so each column lists its
  // rows hot prefix first; the expansion skips warp groups that are all hot and visited)
  __device__ __forceinline__ ull key(uint64_t u, uint64_t v, const uint32_t* fwd) const {
    const uint64_t lc = (uint64_t)fwd[u] % ncols;
    const uint64_t vb = v / block;
    const uint64_t lr = (vb / (uint64_t)R) * block + (fwd[v] - vb * block);
    return ((ull)lc << rbits) | (ull)lr;
  }
};

constexpr int kBuildThreads = 256;
constexpr int kBuildPer = 8;  // tuples per thread per CTA chunk
constexpr int kMaxP = 64;

// count directed entries per destination rank; validate ids; tuple-source histogram (tdeg)
// and endpoint histogram (sdeg, non-self-loop, for the hot-prefix relabeling)
__global__ void __launch_bounds__(kBuildThreads) k_count(const uint64_t* src, const uint64_t* dst, uint64_t m,
                                                         PartMap pm, int P, ull* counts, uint32_t* tdeg_all,
                                                         uint32_t* sdeg_all, int* err) {
  __shared__ unsigned int sc[kMaxP];
  for (int q = threadIdx.x; q < P; q += blockDim.x) sc[q] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBuildThreads * kBuildPer;
  for (int q = 0; q < kBuildPer; ++q) {
    const uint64_t k = base + (uint64_t)q * kBuildThreads + threadIdx.x;
    if (k >= m) break;
    const uint64_t a = src[k], b = dst[k];
    if (a >= pm.nverts || b >= pm.nverts) {
      atomicOr(err, 1);
      continue;
    }
    atomicAdd(tdeg_all + a, 1u);
    if (a == b) continue;
    atomicAdd(sdeg_all + a, 1u);
    atomicAdd(sdeg_all + b, 1u);
    atomicAdd(&sc[pm.dest(a, b)], 1u);
    atomicAdd(&sc[pm.dest(b, a)], 1u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < P; q += blockDim.x)
    if (sc[q]) atomicAdd(counts + q, (ull)sc[q]);
}

// scatter keys into per-destination buckets; cursors[r] starts at the bucket offset
__global__ void __launch_bounds__(kBuildThreads) k_scatter(const uint64_t* src, const uint64_t* dst, uint64_t m,
                                                           PartMap pm, int P, ull* cursors, ull* keys,
                                                           const uint32_t* fwd) {
  __shared__ unsigned int sc[kMaxP];
  __shared__ ull sbase[kMaxP];
  for (int q = threadIdx.x; q < P; q += blockDim.x) sc[q] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kBuildThreads * kBuildPer;
  uint64_t a[kBuildPer], b[kBuildPer];
  unsigned int pos1[kBuildPer], pos2[kBuildPer];
  int d1[kBuildPer], d2[kBuildPer];
  for (int q = 0; q < kBuildPer; ++q) {
    const uint64_t k = base + (uint64_t)q * kBuildThreads + threadIdx.x;
    d1[q] = -1;
    if (k >= m) continue;
    a[q] = src[k];
    b[q] = dst[k];
    if (a[q] == b[q]) continue;
    d1[q] = pm.dest(a[q], b[q]);
    d2[q] = pm.dest(b[q], a[q]);
    pos1[q] = atomicAdd(&sc[d1[q]], 1u);
    pos2[q] = atomicAdd(&sc[d2[q]], 1u);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < P; q += blockDim.x) sbase[q] = sc[q] ? atomicAdd(cursors + q, (ull)sc[q]) : 0ull;
  __syncthreads();
  for (int q = 0; q < kBuildPer; ++q) {
    if (d1[q] < 0) continue;
    keys[sbase[d1[q]] + pos1[q]] = pm.key(a[q], b[q], fwd);
    keys[sbase[d2[q]] + pos2[q]] = pm.key(b[q], a[q], fwd);
  }
}

// ---- relabeling helpers
__global__ void k_degree_keys(const uint32_t* sdeg, uint64_t npad, uint64_t block, ull* keys, uint32_t* vals) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < npad; v += (uint64_t)gridDim.x * blockDim.x) {
    keys[v] = ((ull)(v / block) << 32) | (ull)(0xFFFFFFFFu - sdeg[v]);  // block, then degree descending
    vals[v] = (uint32_t)v;
  }
}

// full per-block degree sort: relabeled id k <- vertex sorted[k] (blocks stay in place: the sort
// key starts with the block)
__global__ void k_perm_from_sorted(const uint32_t* sorted, uint64_t n, uint32_t* fwd, uint32_t* inv) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = sorted[k];
    fwd[v] = (uint32_t)k;
    inv[k] = v;
  }
}

// saturated column degrees for the K3 count pass: min(col[u+1] - col[u], 255)
__global__ void k_deg8(const ull* col, uint64_t n, uint8_t* out) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = (uint8_t)min(col[t + 1] - col[t], 255ull);
}

__global__ void k_narrow(const ull* in, uint64_t n, uint32_t* out) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = (uint32_t)in[t];
}

// ---- CSC / CSR assembly
// row[t] = the key's relabeled local row
__global__ void k_keys_to_rows(const ull* keys, uint64_t n, int rbits, uint32_t* row) {
  const ull rmask = (1ull << rbits) - 1;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    row[t] = (uint32_t)(keys[t] & rmask);
}

// CSC key (col' << rbits | row') -> CSR key (row' << cbits | orig col)
__global__ void k_csr_keys(ull* keys, uint64_t n, int rbits, int cbits, uint64_t cbase, const uint32_t* inv) {
  const ull rmask = (1ull << rbits) - 1;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const ull k = keys[t];
    const uint64_t lr = k & rmask, lc = k >> rbits;
    const uint64_t lc_orig = inv[cbase + lc] - cbase;
    keys[t] = ((ull)lr << cbits) | (ull)lc_orig;
  }
}

// csr_col[t] = relabeled local column of the ORIGINAL local column in the key's low bits
__global__ void k_keys_to_cols(const ull* keys, uint64_t n, int cbits, uint64_t cbase, const uint32_t* fwd,
                               uint32_t* out) {
  const ull cmask = (1ull << cbits) - 1;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    out[t] = (uint32_t)(fwd[cbase + (keys[t] & cmask)] - cbase);
}

// off[c] = first position with key >= c << shift (lower bound), c in [0, nc]
__global__ void k_offsets(const ull* keys, uint64_t n, int shift, uint64_t nc, ull* off) {
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= nc; c += (uint64_t)gridDim.x * blockDim.x) {
    const ull target = (ull)c << shift;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    off[c] = lo;
  }
}

__global__ void k_slice(const uint32_t* src, uint64_t base, uint64_t n, uint32_t sub, uint32_t* dst) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
    dst[t] = src[base + t] - sub;
}

static int bits_for(uint64_t n) {  // bits to represent values < n
  int b = 0;
  while (b < 64 && (1ull << b) < n) ++b;
  return b;
}

// Degree relabeling: perm_fwd (original -> relabeled global id) and perm_inv on
// device.  Inside every vertex block the vertices are ordered by descending non-self-loop degree
// (ties by original id): one radix sort of (block, -degree) keys, then position k of the sorted
// order is relabeled offset k.
static int compute_relabel(Graph& G, const uint32_t* sdeg, uint32_t* fwd, uint32_t* inv) {
  cudaStream_t s = G.stream;
  const Geom& g = G.g;
  const uint64_t P = (uint64_t)g.R * g.C;
  Scratch sc;
  ull *keys = nullptr, *keys2 = nullptr;
  uint32_t *vals = nullptr, *vals2 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  const int kb = 32 + bits_for(P);
  CKR(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (uint64_t)g.npad, 0, kb, s));
  CKR(sc.alloc(&keys, g.npad * 8));
  CKR(sc.alloc(&keys2, g.npad * 8));
  CKR(sc.alloc(&vals, g.npad * 4));
  CKR(sc.alloc(&vals2, g.npad * 4));
  CKR(sc.alloc(&tmp, tmp_bytes));
  k_degree_keys<<<4096, 256, 0, s>>>(sdeg, g.npad, g.block, keys, vals);
  CKR(cudaGetLastError());
  CKR(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (uint64_t)g.npad, 0, kb, s));
  k_perm_from_sorted<<<4096, 256, 0, s>>>(vals2, g.npad, fwd, inv);
  CKR(cudaGetLastError());
  CKR(cudaStreamSynchronize(s));
  return BFS_OK;
}

// Sorted/deduplicated CSC (and, for 2D, CSR) of one rank from its bucket of keys (consumed).
static int csc_from_keys(Graph& G, Rank& rk, ull* keys, uint64_t n, int rbits, const uint32_t* fwd,
                         const uint32_t* inv) {
  cudaStream_t s = G.stream;
  const Geom& g = G.g;
  const int cbits = bits_for(g.ncols());
  const int kbits = rbits + cbits;
  Scratch sc;
  ull* sorted = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, tmp2 = 0;
  ull* nsel = nullptr;
  int rc = BFS_OK;
  if (n) {
    CKR(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys, (uint64_t)n, 0, kbits, s));
    CKR(cub::DeviceSelect::Unique(nullptr, tmp2, keys, keys, nsel, (uint64_t)n, s));
    tmp_bytes = tmp_bytes > tmp2 ? tmp_bytes : tmp2;
    CKR(sc.alloc(&sorted, n * sizeof(ull)));
    CKR(sc.alloc(&tmp, tmp_bytes));
    CKR(sc.alloc(&nsel, sizeof(ull)));
    CKR(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, (uint64_t)n, 0, kbits, s));
    CKR(cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, keys, nsel, (uint64_t)n, s));
    ull h_nsel = 0;
    CKR(cudaMemcpyAsync(&h_nsel, nsel, sizeof(ull), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
    sc.release(sorted);
    sc.release(tmp);
    sc.release(nsel);
    sorted = nullptr;
    rk.nnz = h_nsel;
  } else {
    rk.nnz = 0;
  }
  // + 4 entries: K1's bulk copies round a tile's byte range out to 16-B boundaries
  rc = G_alloc(G, (void**)&rk.row, (rk.nnz + 4) * sizeof(uint32_t));
  if (rc) return rc;
  rc = G_alloc(G, (void**)&rk.col, (g.ncols() + 1) * sizeof(ull));
  if (rc) return rc;
  if (rk.nnz) {
    k_keys_to_rows<<<4096, 256, 0, s>>>(keys, rk.nnz, rbits, rk.row);
    CKR(cudaGetLastError());
  }
  const uint64_t nc = g.ncols() + 1;
  k_offsets<<<(unsigned)((nc + 255) / 256), 256, 0, s>>>(keys, rk.nnz, rbits, g.ncols(), rk.col);
  CKR(cudaGetLastError());
  if (rk.nnz < (1ull << 32)) {  // 32-bit copy for the unpack / degree scan (K3 reads half the bytes)
    rc = G_alloc(G, (void**)&rk.col32, nc * sizeof(uint32_t));
    if (rc) return rc;
    k_narrow<<<1024, 256, 0, s>>>(rk.col, nc, rk.col32);
    CKR(cudaGetLastError());
  }
  rc = G_alloc(G, (void**)&rk.deg8, (g.ncols() + 32) * sizeof(uint8_t));  // ncols is a multiple of 32
  if (rc) return rc;
  k_deg8<<<1024, 256, 0, s>>>(rk.col, g.ncols(), rk.deg8);
  CKR(cudaGetLastError());
  CKR(cudaStreamSynchronize(s));
  // CSR of the same local matrix for the parent pass (rows scanned in ascending ORIGINAL
  // column order; the CSC lists rows in relabeled order, so even a 1x1 grid needs its own copy)
  const uint64_t cbase = (uint64_t)rk.j * g.ncols();
  rc = G_alloc(G, (void**)&rk.csr_col, (rk.nnz ? rk.nnz : 1) * sizeof(uint32_t));
  if (rc) return rc;
  rc = G_alloc(G, (void**)&rk.csr_ptr, (g.nrows() + 1) * sizeof(ull));
  if (rc) return rc;
  if (rk.nnz) {
    k_csr_keys<<<4096, 256, 0, s>>>(keys, rk.nnz, rbits, cbits, cbase, inv);
    CKR(cudaGetLastError());
    tmp_bytes = 0;
    CKR(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys, keys, (uint64_t)rk.nnz, 0, rbits + cbits, s));
    CKR(sc.alloc(&sorted, rk.nnz * sizeof(ull)));
    CKR(sc.alloc(&tmp, tmp_bytes));
    CKR(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, keys, sorted, (uint64_t)rk.nnz, 0, rbits + cbits, s));
    k_keys_to_cols<<<4096, 256, 0, s>>>(sorted, rk.nnz, cbits, cbase, fwd, rk.csr_col);
    CKR(cudaGetLastError());
  }
  const uint64_t nr = g.nrows() + 1;
  k_offsets<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(sorted, rk.nnz, cbits, g.nrows(), rk.csr_ptr);
  CKR(cudaGetLastError());
  if (rk.nnz < (1ull << 32)) {  // 32-bit copy for the parent pass
    rc = G_alloc(G, (void**)&rk.csr_ptr32, nr * sizeof(uint32_t));
    if (rc) return rc;
    k_narrow<<<1024, 256, 0, s>>>(rk.csr_ptr, nr, rk.csr_ptr32);
    CKR(cudaGetLastError());
  }
  CKR(cudaStreamSynchronize(s));
  return BFS_OK;
}

// rows with at least one entry (csr_ptr[r+1] > csr_ptr[r]) -> *out
__global__ void k_count_nz_rows(const ull* ptr, uint64_t nrows, ull* out) {
  unsigned c = 0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += (uint64_t)gridDim.x * blockDim.x)
    c += ptr[r + 1] > ptr[r] ? 1u : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (ull)c);
}

// per-rank slices of the permutation: fwd_own / inv_own (local offsets of the owned block) and
// inv_col (relabeled local column -> ORIGINAL global id, the value stored as parent)
static int rank_maps(Graph& G, Rank& rk, const uint32_t* fwd, const uint32_t* inv) {
  cudaStream_t s = G.stream;
  const Geom& g = G.g;
  int rc;
  if ((rc = G_alloc(G, (void**)&rk.fwd_own, g.block * 4))) return rc;
  if ((rc = G_alloc(G, (void**)&rk.inv_own, g.block * 4))) return rc;
  if ((rc = G_alloc(G, (void**)&rk.inv_col, g.ncols() * 4))) return rc;
  {
    Scratch sc;
    ull* cnt = nullptr;
    ull h = 0;
    CKR(sc.alloc(&cnt, sizeof(ull)));
    CKR(cudaMemsetAsync(cnt, 0, sizeof(ull), s));
    k_count_nz_rows<<<1024, 256, 0, s>>>(rk.csr_ptr, g.nrows(), cnt);
    CKR(cudaGetLastError());
    CKR(cudaMemcpyAsync(&h, cnt, sizeof(ull), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
    rk.nz_rows = h;
  }
  const uint64_t vb = (uint64_t)rk.r * g.block;
  k_slice<<<1024, 256, 0, s>>>(fwd, vb, g.block, (uint32_t)vb, rk.fwd_own);
  k_slice<<<1024, 256, 0, s>>>(inv, vb, g.block, (uint32_t)vb, rk.inv_own);
  k_slice<<<1024, 256, 0, s>>>(inv, (uint64_t)rk.j * g.ncols(), g.ncols(), 0u, rk.inv_col);
  CKR(cudaGetLastError());
  return BFS_OK;
}

// Build every local rank's CSC/CSR, maps and tdeg.  src/dst: host or device arrays of m tuples.
int build_graph(Graph& G, const uint64_t* src, const uint64_t* dst, uint64_t m) {
  cudaStream_t s = G.stream;
  const Geom& g = G.g;
  const int P = g.R * g.C;
  if (P > kMaxP) return set_err(BFS_EINVAL, "R*C must be <= 64");
  PartMap pm{g.block, g.ncols(), g.nverts, g.R, g.C, bits_for(g.nrows())};
  const bool src_dev = is_device_ptr(src), dst_dev = is_device_ptr(dst);
  if (src_dev != dst_dev) return set_err(BFS_EINVAL, "src and dst must both be host or both device pointers");

  // ---- histograms and per-destination counts
  Scratch sc;
  uint32_t *tdeg_all = nullptr, *sdeg_all = nullptr;
  ull* counts = nullptr;
  int* err = nullptr;
  CKR(sc.alloc(&tdeg_all, g.npad * sizeof(uint32_t)));
  CKR(sc.alloc(&sdeg_all, g.npad * sizeof(uint32_t)));
  CKR(sc.alloc(&counts, 2 * kMaxP * sizeof(ull)));
  CKR(sc.alloc(&err, sizeof(int)));
  CKR(cudaMemsetAsync(tdeg_all, 0, g.npad * sizeof(uint32_t), s));
  CKR(cudaMemsetAsync(sdeg_all, 0, g.npad * sizeof(uint32_t), s));
  CKR(cudaMemsetAsync(counts, 0, 2 * kMaxP * sizeof(ull), s));
  CKR(cudaMemsetAsync(err, 0, sizeof(int), s));
  const uint64_t chunk = src_dev ? (m ? m : 1) : (1ull << 26);
  uint64_t* stage_s = nullptr;
  uint64_t* stage_d = nullptr;
  if (!src_dev && m) {
    CKR(sc.alloc(&stage_s, chunk * sizeof(uint64_t)));
    CKR(sc.alloc(&stage_d, chunk * sizeof(uint64_t)));
  }
  auto for_chunks = [&](auto&& fn) -> int {
    for (uint64_t k0 = 0; k0 < m; k0 += chunk) {
      const uint64_t len = (m - k0 < chunk) ? (m - k0) : chunk;
      const uint64_t* ps = src + k0;
      const uint64_t* pd = dst + k0;
      if (!src_dev) {
        CKR(cudaMemcpyAsync(stage_s, ps, len * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        CKR(cudaMemcpyAsync(stage_d, pd, len * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
        ps = stage_s;
        pd = stage_d;
      }
      const uint64_t per = (uint64_t)kBuildThreads * kBuildPer;
      fn(ps, pd, len, (unsigned)((len + per - 1) / per));
      CKR(cudaGetLastError());
      if (!src_dev) CKR(cudaStreamSynchronize(s));
    }
    return BFS_OK;
  };
  int rc = for_chunks([&](const uint64_t* ps, const uint64_t* pd, uint64_t len, unsigned grid) {
    k_count<<<grid, kBuildThreads, 0, s>>>(ps, pd, len, pm, P, counts, tdeg_all, sdeg_all, err);
  });
  if (rc) return rc;
  ull h_counts[kMaxP];
  int h_err = 0;
  CKR(cudaMemcpyAsync(h_counts, counts, P * sizeof(ull), cudaMemcpyDeviceToHost, s));
  CKR(cudaMemcpyAsync(&h_err, err, sizeof(int), cudaMemcpyDeviceToHost, s));
  CKR(cudaStreamSynchronize(s));
  if (G.world_size > 1) {
    int any_err = h_err;
    rc = comm_allreduce_int_max(G, &any_err);
    if (rc) return rc;
    h_err = any_err;
  }
  if (h_err) return set_err(BFS_ERANGE, "an edge endpoint is >= nverts");
  if (G.world_size > 1) {
    rc = comm_allreduce_u32_sum(G, sdeg_all, g.npad);
    if (rc) return rc;
  }

  // ---- hot-prefix relabeling (perm_fwd kept for root / degree lookups)
  uint32_t* inv = nullptr;
  rc = G_alloc(G, (void**)&G.perm_fwd, g.npad * 4);
  if (rc) return rc;
  CKR(sc.alloc(&inv, g.npad * 4));
  rc = compute_relabel(G, sdeg_all, G.perm_fwd, inv);
  if (rc) return rc;
  sc.release(sdeg_all);

  // ---- bucket keys by destination rank
  ull offs[kMaxP + 1];
  offs[0] = 0;
  for (int q = 0; q < P; ++q) offs[q + 1] = offs[q] + h_counts[q];
  ull* keys = nullptr;
  CKR(sc.alloc(&keys, (offs[P] ? offs[P] : 1) * sizeof(ull)));
  ull* cursors = counts + kMaxP;
  CKR(cudaMemcpyAsync(cursors, offs, P * sizeof(ull), cudaMemcpyHostToDevice, s));
  rc = for_chunks([&](const uint64_t* ps, const uint64_t* pd, uint64_t len, unsigned grid) {
    k_scatter<<<grid, kBuildThreads, 0, s>>>(ps, pd, len, pm, P, cursors, keys, G.perm_fwd);
  });
  if (rc) return rc;
  CKR(cudaStreamSynchronize(s));
  if (stage_s) {
    sc.release(stage_s);
    sc.release(stage_d);
    stage_s = stage_d = nullptr;
  }

  if (G.world_size == 1) {
    // loopback (or 1x1): every bucket is local
    for (Rank& rk : G.ranks) {
      rc = csc_from_keys(G, rk, keys + offs[rk.r], h_counts[rk.r], pm.rbits, G.perm_fwd, inv);
      if (rc) return rc;
      rc = G_alloc(G, (void**)&rk.tdeg, g.block * sizeof(uint32_t));
      if (rc) return rc;
      CKR(cudaMemcpyAsync(rk.tdeg, tdeg_all + (uint64_t)rk.r * g.block, g.block * sizeof(uint32_t),
                          cudaMemcpyDeviceToDevice, s));
      rc = rank_maps(G, rk, G.perm_fwd, inv);
      if (rc) return rc;
    }
    CKR(cudaStreamSynchronize(s));
    sc.release(keys);
  } else {
    // NCCL: exchange bucket sizes, then the buckets (grouped send/recv over the world comm)
    Rank& rk = G.ranks[0];
    ull* recv_counts = nullptr;
    CKR(sc.alloc(&recv_counts, kMaxP * sizeof(ull)));
    rc = comm_exchange_counts(G, counts /*device counts[P]*/, recv_counts);
    if (rc) return rc;
    ull h_rc[kMaxP];
    CKR(cudaMemcpyAsync(h_rc, recv_counts, P * sizeof(ull), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
    ull roffs[kMaxP + 1];
    roffs[0] = 0;
    for (int q = 0; q < P; ++q) roffs[q + 1] = roffs[q] + h_rc[q];
    ull* rkeys = nullptr;
    CKR(sc.alloc(&rkeys, (roffs[P] ? roffs[P] : 1) * sizeof(ull)));
    rc = comm_alltoallv_u64(G, keys, offs, h_counts, rkeys, roffs, h_rc);
    if (rc) return rc;
    CKR(cudaStreamSynchronize(s));
    sc.release(keys);
    rc = csc_from_keys(G, rk, rkeys, roffs[P], pm.rbits, G.perm_fwd, inv);
    sc.release(rkeys);
    if (rc) return rc;
    rc = G_alloc(G, (void**)&rk.tdeg, g.block * sizeof(uint32_t));
    if (rc) return rc;
    rc = comm_reduce_scatter_u32(G, tdeg_all, rk.tdeg, g.block);
    if (rc) return rc;
    rc = rank_maps(G, rk, G.perm_fwd, inv);
    if (rc) return rc;
    CKR(cudaStreamSynchronize(s));
  }
  return BFS_OK;
}

}  // namespace bfs200
