// kernels.cu -- hot-path kernels of libbfs200 for sm_100a (B200).
//
// Per BFS level on rank P_ij (Alg.2):
//   K3 k_scan_count / k_scan_tiles / k_scan_emit : frontier bitmap -> ascending column list,
//        row offsets, exclusive degree scan `cumul` and the per-tile
//        first-vertex table used to map threads to edges (Fig. t2d_map).
//   K1 k_expand<E> : one thread per E consecutive frontier edges; the
//        visited-bitmap filter (Alg.3 lines 5-6); the parent claim by atomicMin of the global
//        id (deterministic minimum rule, R1) and the discovered-row bitmap by atomicOr
//        (Alg.3 line 7, bitmap pack fused: P:900-903).
//   K2 k_update : OR of the received fold segments, new = OR & ~visited, level, visited,
//        next frontier bitmap, lowest-column winner.
// All hot-path arithmetic is integer.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "kernels.cuh"

namespace bfs200 {

typedef unsigned long long ull;

// ------------------------------------------------------------------ small helpers
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void load8(const uint32_t* __restrict__ bm, uint64_t w0, uint64_t nwords, uint32_t (&x)[8]) {
  if (w0 + 8 <= nwords) {
    const uint4* p = reinterpret_cast<const uint4*>(bm + w0);
    uint4 a = __ldg(p), b = __ldg(p + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = (w0 + q < nwords) ? __ldg(bm + w0 + q) : 0u;
  }
}

// ------------------------------------------------------------------ init (Alg.2 lines 1-10)
__global__ void k_seed_root(uint32_t* visited, uint32_t* all_front, int32_t* level, uint32_t* pred, uint8_t* winner,
                            uint64_t t, uint64_t row_local, uint64_t col_local, uint32_t root, int j) {
  visited[row_local >> 5] |= 1u << (row_local & 31);  // bmap[LOCAL_ROW(r)] <- 1
  all_front[col_local >> 5] |= 1u << (col_local & 31);  // front[0] <- LOCAL_COL(r)
  level[t] = 0;                                          // level[LOCAL_ROW(r)] <- 0
  pred[row_local] = root;                                // pred[LOCAL_ROW(r)] <- r
  if (winner) winner[t] = (uint8_t)j;
}

cudaError_t launch_init(const Geom& g, Rank& rk, bool owner, uint64_t root, cudaStream_t s) {
  const uint64_t rw = g.nrows() / 32, cw = g.ncols() / 32;
  cudaMemsetAsync(rk.visited, 0, rw * 4, s);
  cudaMemsetAsync(rk.disc, 0, rw * 4, s);
  cudaMemsetAsync(rk.all_front, 0, cw * 4, s);
  cudaMemsetAsync(rk.pred, 0xFF, g.nrows() * 4, s);
  cudaMemsetAsync(rk.level, 0xFF, g.block * 4, s);
  if (owner) {
    const uint64_t t = root - (uint64_t)rk.r * g.block;
    k_seed_root<<<1, 1, 0, s>>>(rk.visited, rk.all_front, rk.level, rk.pred, rk.winner, t,
                                (uint64_t)rk.j * g.block + t, (uint64_t)rk.i * g.block + t, (uint32_t)root, rk.j);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3: unpack + degree scan
struct CS {
  unsigned int c;
  ull s;
};
struct CSAdd {
  __device__ __forceinline__ CS operator()(const CS& a, const CS& b) const { return CS{a.c + b.c, a.s + b.s}; }
};

// per tile of kScanTileWords words: number of frontier columns with degree > 0 and their degree sum
__global__ void __launch_bounds__(kScanThreads) k_scan_count(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                              const ull* __restrict__ col, uint32_t* tile_cnt,
                                                              ull* tile_sum) {
  typedef cub::BlockReduce<CS, kScanThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const uint64_t w0 = (uint64_t)blockIdx.x * kScanTileWords + threadIdx.x * 8;
  uint32_t x[8];
  load8(bm, w0, nwords, x);
  CS acc{0u, 0ull};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t b = x[q];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const uint64_t u = (w0 + q) * 32 + bit;
      const ull d = __ldg(col + u + 1) - __ldg(col + u);
      acc.c += d ? 1u : 0u;
      acc.s += d;
    }
  }
  CS tot = BR(tmp).Reduce(acc, CSAdd());
  if (threadIdx.x == 0) {
    tile_cnt[blockIdx.x] = tot.c;
    tile_sum[blockIdx.x] = tot.s;
  }
}

// exclusive scan over tiles (one CTA); writes n, edges, cumul[n]; resets the update counter
__global__ void __launch_bounds__(1024) k_scan_tiles(int ntiles, const uint32_t* tile_cnt, const ull* tile_sum,
                                                     uint32_t* cnt_off, ull* sum_off, LevelInfo* info, ull* cumul) {
  typedef cub::BlockScan<CS, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  __shared__ CS carry;
  if (threadIdx.x == 0) carry = CS{0u, 0ull};
  __syncthreads();
  for (int base = 0; base < ntiles; base += 1024) {
    const int t = base + threadIdx.x;
    CS v = (t < ntiles) ? CS{tile_cnt[t], tile_sum[t]} : CS{0u, 0ull};
    CS ex, agg;
    BS(tmp).ExclusiveScan(v, ex, CS{0u, 0ull}, CSAdd(), agg);
    const CS c0 = carry;
    if (t < ntiles) {
      cnt_off[t] = c0.c + ex.c;
      sum_off[t] = c0.s + ex.s;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry = CS{c0.c + agg.c, c0.s + agg.s};
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    info->n = carry.c;
    info->edges = carry.s;
    info->newv = 0;
    cumul[carry.c] = carry.s;
  }
}

// emit the list, row offsets, cumul and, for every expansion tile starting inside a column's
// edge range, the index of that column (tile_k): the thread->edge mapping table.
__global__ void __launch_bounds__(kScanThreads) k_scan_emit(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                             const ull* __restrict__ col, const uint32_t* cnt_off,
                                                             const ull* sum_off, uint32_t* flist, ull* rowoff,
                                                             ull* cumul, uint32_t* tile_k, uint32_t tile_edges) {
  typedef cub::BlockScan<CS, kScanThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t w0 = (uint64_t)blockIdx.x * kScanTileWords + threadIdx.x * 8;
  uint32_t x[8];
  load8(bm, w0, nwords, x);
  CS acc{0u, 0ull};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t b = x[q];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const uint64_t u = (w0 + q) * 32 + bit;
      const ull d = __ldg(col + u + 1) - __ldg(col + u);
      acc.c += d ? 1u : 0u;
      acc.s += d;
    }
  }
  CS ex;
  BS(tmp).ExclusiveScan(acc, ex, CS{0u, 0ull}, CSAdd());
  uint64_t k = cnt_off[blockIdx.x] + ex.c;
  ull e = sum_off[blockIdx.x] + ex.s;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t b = x[q];
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const uint64_t u = (w0 + q) * 32 + bit;
      const ull c0 = __ldg(col + u), d = __ldg(col + u + 1) - c0;
      if (!d) continue;
      flist[k] = (uint32_t)u;
      rowoff[k] = c0;
      cumul[k] = e;
      // tiles whose first edge lies in [e, e+d)
      for (ull t = (e + tile_edges - 1) / tile_edges; t * tile_edges < e + d; ++t) tile_k[t] = (uint32_t)k;
      ++k;
      e += d;
    }
  }
}

cudaError_t launch_scan(const Geom& g, Rank& rk, uint32_t tile_edges, cudaStream_t s) {
  const uint64_t nwords = g.ncols() / 32;
  const int ntiles = (int)((nwords + kScanTileWords - 1) / kScanTileWords);
  k_scan_count<<<ntiles, kScanThreads, 0, s>>>(rk.all_front, nwords, rk.col, rk.tile_cnt, rk.tile_sum);
  k_scan_tiles<<<1, 1024, 0, s>>>(ntiles, rk.tile_cnt, rk.tile_sum, rk.tile_cnt_off, rk.tile_sum_off, rk.info,
                                  rk.cumul);
  k_scan_emit<<<ntiles, kScanThreads, 0, s>>>(rk.all_front, nwords, rk.col, rk.tile_cnt_off, rk.tile_sum_off,
                                              rk.flist, rk.rowoff, rk.cumul, rk.tile_k, tile_edges);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1: frontier expansion
// Tile of TILE = 256*E consecutive frontier edges per CTA iteration (grid-stride over tiles,
// persistent grid sized from the SM count).  The tile's columns (<= TILE+1) are staged in
// shared memory (edge begin within the tile, row offset, column id); each thread maps its
// first edge by binary search in shared memory and the next E-1 by linear advance.
template <int E>
__global__ void __launch_bounds__(kExpandThreads) k_expand(const uint32_t* __restrict__ row,
                                                           const uint32_t* __restrict__ flist,
                                                           const ull* __restrict__ rowoff,
                                                           const ull* __restrict__ cumul,
                                                           const uint32_t* __restrict__ tile_k,
                                                           const LevelInfo* __restrict__ info,
                                                           const uint32_t* __restrict__ visited, uint32_t* pred,
                                                           uint32_t* disc, uint32_t col_base) {
  constexpr int TILE = kExpandThreads * E;
  extern __shared__ __align__(16) unsigned char smem[];
  ull* s_off = reinterpret_cast<ull*>(smem);               // [TILE+2]
  uint32_t* s_beg = reinterpret_cast<uint32_t*>(s_off + TILE + 2);  // [TILE+2]
  uint32_t* s_u = s_beg + TILE + 2;                         // [TILE+2]
  const ull n = info->n, total = info->edges;
  if (total == 0) return;
  const ull ntiles = (total + TILE - 1) / TILE;
  for (ull tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const ull t0 = tile * TILE;
    const uint32_t len = (uint32_t)min((ull)TILE, total - t0);
    const uint32_t klo = tile_k[tile];
    const uint32_t khi = (tile + 1 < ntiles) ? tile_k[tile + 1] : (uint32_t)(n - 1);
    const uint32_t cnt = khi - klo + 1;
    for (uint32_t idx = threadIdx.x; idx < cnt; idx += kExpandThreads) {
      const ull c = cumul[klo + idx];
      const uint32_t beg = c > t0 ? (uint32_t)(c - t0) : 0u;
      s_beg[idx] = beg;
      s_off[idx] = rowoff[klo + idx] + (t0 + beg - c);
      s_u[idx] = flist[klo + idx];
    }
    if (threadIdx.x == 0) s_beg[cnt] = 0xFFFFFFFFu;
    __syncthreads();
    const uint32_t le = threadIdx.x * E;
    if (le < len) {
      // greatest idx < cnt with s_beg[idx] <= le (binsearch_maxle, Alg.3 line 2)
      uint32_t lo = 0, hi = cnt - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_beg[mid] <= le) lo = mid; else hi = mid - 1;
      }
      uint32_t idx = lo;
      uint32_t v[E], u[E];
#pragma unroll
      for (int q = 0; q < E; ++q) {
        const uint32_t e = le + q;
        if (e < len) {
          while (s_beg[idx + 1] <= e) ++idx;  // linear advance
          v[q] = ld_stream_u32(row + s_off[idx] + (e - s_beg[idx]));  // Alg.3 line 4
          u[q] = s_u[idx];
        } else {
          v[q] = 0xFFFFFFFFu;
        }
      }
      uint32_t w[E];
#pragma unroll
      for (int q = 0; q < E; ++q) w[q] = (v[q] != 0xFFFFFFFFu) ? __ldg(visited + (v[q] >> 5)) : 0xFFFFFFFFu;
#pragma unroll
      for (int q = 0; q < E; ++q) {
        if (v[q] == 0xFFFFFFFFu) continue;
        const uint32_t m = 1u << (v[q] & 31);
        if (w[q] & m) continue;  // already visited (Alg.3 lines 5-6)
        const uint32_t ug = col_base + u[q];
        if (ug < *(volatile uint32_t*)(pred + v[q])) atomicMin(pred + v[q], ug);  // parent claim
        atomicOr(disc + (v[q] >> 5), m);                                          // discovered row
      }
    }
    __syncthreads();
  }
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

template <int E>
static cudaError_t launch_expand_t(const Geom& g, Rank& rk, cudaStream_t s) {
  constexpr int TILE = kExpandThreads * E;
  const size_t smem = (size_t)(TILE + 2) * (8 + 4 + 4);
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaFuncSetAttribute(k_expand<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_expand<E>, kExpandThreads, smem);
    if (blocks_per_sm <= 0) blocks_per_sm = 1;
  }
  const int grid = num_sms() * blocks_per_sm;
  k_expand<E><<<grid, kExpandThreads, smem, s>>>(rk.row, rk.flist, rk.rowoff, rk.cumul, rk.tile_k, rk.info,
                                                  rk.visited, rk.pred, rk.disc, (uint32_t)(rk.j * g.ncols()));
  return cudaGetLastError();
}

cudaError_t launch_expand(const Geom& g, Rank& rk, int E, cudaStream_t s) {
  switch (E) {
    case 1: return launch_expand_t<1>(g, rk, s);
    case 2: return launch_expand_t<2>(g, rk, s);
    case 4: return launch_expand_t<4>(g, rk, s);
    case 8: return launch_expand_t<8>(g, rk, s);
    case 16: return launch_expand_t<16>(g, rk, s);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ K2: frontier update
// Thread per (segment m, word w) of the local rows.  Owned segment m == j: new vertices are the
// rows received from any column (own discoveries included) that are not yet visited; the
// lowest sending column is recorded as the parent's column (winner).  Other segments: mark the
// rows this rank discovered as visited so they are sent at most once.
__global__ void __launch_bounds__(256) k_update(uint32_t* visited, uint32_t* disc, const uint32_t* recv,
                                                uint32_t* front_seg, int32_t* level, uint8_t* winner,
                                                LevelInfo* info, uint64_t W, int C, int j, int lvl) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t newbits = 0;
  if (gid < W * (uint64_t)C) {
    const int m = (int)(gid / W);
    const uint64_t w = gid - (uint64_t)m * W;
    if (m != j) {
      visited[gid] |= disc[gid];
      disc[gid] = 0;
    } else {
      const uint32_t vis = visited[gid];
      uint32_t claimed = 0;
      for (int c = 0; c < C; ++c) {
        const uint32_t x = ((c == j) ? disc[gid] : recv[(uint64_t)c * W + w]) & ~vis & ~claimed;
        if (x && winner) {
          uint32_t b = x;
          while (b) {
            const int bit = __ffs(b) - 1;
            b &= b - 1;
            winner[w * 32 + bit] = (uint8_t)c;
          }
        }
        claimed |= x;
      }
      newbits = claimed;
      visited[gid] = vis | newbits;
      disc[gid] = 0;
      front_seg[w] = newbits;
      uint32_t b = newbits;
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        level[w * 32 + bit] = lvl;
      }
    }
  }
  unsigned int cnt = __popc(newbits);
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&info->newv, (ull)cnt);
}

cudaError_t launch_update(const Geom& g, Rank& rk, int lvl, cudaStream_t s) {
  const uint64_t W = g.words_block();
  const uint64_t nthreads = W * (uint64_t)g.C;
  const unsigned grid = (unsigned)((nthreads + 255) / 256);
  k_update<<<grid, 256, 0, s>>>(rk.visited, rk.disc, rk.recv, rk.all_front + (uint64_t)rk.i * W, rk.level,
                                g.C > 1 ? rk.winner : nullptr, rk.info, W, g.C, rk.j, lvl);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ outputs
// parent for owned t: unreached -> -1; winner column == own column (always with C == 1) ->
// pred of the own row segment; otherwise left for the resolution exchange.
__global__ void k_finalize(const int32_t* level, const uint32_t* pred_own, const uint8_t* winner, int j,
                           uint64_t block, int64_t* parent_out, int32_t* level_out) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= block) return;
  const int32_t lv = level[t];
  if (parent_out) {
    int64_t p = -1;
    if (lv >= 0 && (!winner || winner[t] == (uint8_t)j)) p = (int64_t)pred_own[t];
    parent_out[t] = p;
  }
  if (level_out) level_out[t] = lv;
}

cudaError_t launch_finalize(const Geom& g, Rank& rk, int64_t* parent_out, int32_t* level_out, cudaStream_t s) {
  const unsigned grid = (unsigned)((g.block + 255) / 256);
  k_finalize<<<grid, 256, 0, s>>>(rk.level, rk.pred + (uint64_t)rk.j * g.block, g.C > 1 ? rk.winner : nullptr, rk.j,
                                  g.block, parent_out, level_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ parent resolution (C > 1)
// request bitmaps: req[c] has bit t for owned reached t whose winner column is c != j
__global__ void k_req_build(const uint32_t* vis_own, const uint8_t* winner, uint32_t* req, uint64_t W, int C, int j) {
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W) return;
  uint32_t b = vis_own[w];
  while (b) {
    const int bit = __ffs(b) - 1;
    b &= b - 1;
    const int c = winner[w * 32 + bit];
    if (c != j) req[(uint64_t)c * W + w] |= 1u << bit;
  }
}

cudaError_t launch_req_build(const Geom& g, Rank& rk, cudaStream_t s) {
  const uint64_t W = g.words_block();
  cudaMemsetAsync(rk.req, 0, W * g.C * 4, s);
  k_req_build<<<(unsigned)((W + 255) / 256), 256, 0, s>>>(rk.visited + (uint64_t)rk.j * W, rk.winner, rk.req, W, g.C,
                                                           rk.j);
  return cudaGetLastError();
}

struct PopcOp {
  __device__ __forceinline__ uint32_t operator()(const uint32_t x) const { return (uint32_t)__popc(x); }
};

size_t popc_scan_tmp_bytes(uint64_t nwords) {
  size_t bytes = 0;
  cub::TransformInputIterator<uint32_t, PopcOp, const uint32_t*> it((const uint32_t*)nullptr, PopcOp());
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (uint32_t*)nullptr, (uint64_t)nwords + 1);
  return bytes;
}

// off[w] = sum_{w' < w} popc(bits[w']), for w in [0, nwords]; bits must have nwords+1 readable
// words is NOT required: the transform reads bits[w] only for w < nwords+1 -> pass a padded array.
cudaError_t launch_popc_scan(const uint32_t* bits, uint32_t* off, uint64_t nwords, void* tmp, size_t tmp_bytes,
                             cudaStream_t s) {
  cub::TransformInputIterator<uint32_t, PopcOp, const uint32_t*> it(bits, PopcOp());
  return cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, it, off, (uint64_t)nwords + 1, s);
}

// responder: for every requesting column c != j, pack pred of the requested rows of segment c
// in ascending order into resp[c*block ...]
__global__ void k_resp_pack(const uint32_t* reqin, const uint32_t* off, const uint32_t* pred, uint32_t* resp,
                            uint64_t W, uint64_t block, int C, int j) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= W * (uint64_t)C) return;
  const int c = (int)(gid / W);
  if (c == j) return;
  const uint64_t w = gid - (uint64_t)c * W;
  uint32_t b = reqin[gid];
  uint64_t pos = off[gid] - off[(uint64_t)c * W];
  while (b) {
    const int bit = __ffs(b) - 1;
    b &= b - 1;
    resp[(uint64_t)c * block + pos++] = pred[(uint64_t)c * block + w * 32 + bit];
  }
}

cudaError_t launch_resp_pack(const Geom& g, Rank& rk, cudaStream_t s) {
  const uint64_t W = g.words_block();
  const uint64_t n = W * g.C;
  k_resp_pack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rk.reqin, rk.off_in, rk.pred, rk.resp, W, g.block, g.C,
                                                          rk.j);
  return cudaGetLastError();
}

// owner: scatter the answers for its requests (req_off holds the popc scan of req here)
__global__ void k_resp_scatter(const uint32_t* req, const uint32_t* off, const uint32_t* respin, int64_t* parent,
                               uint64_t W, uint64_t block, int C, int j) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= W * (uint64_t)C) return;
  const int c = (int)(gid / W);
  if (c == j) return;
  const uint64_t w = gid - (uint64_t)c * W;
  uint32_t b = req[gid];
  uint64_t pos = off[gid] - off[(uint64_t)c * W];
  while (b) {
    const int bit = __ffs(b) - 1;
    b &= b - 1;
    parent[w * 32 + bit] = (int64_t)respin[(uint64_t)c * block + pos++];
  }
}

cudaError_t launch_resp_scatter(const Geom& g, Rank& rk, int64_t* parent_out, cudaStream_t s) {
  const uint64_t W = g.words_block();
  const uint64_t n = W * g.C;
  k_resp_scatter<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rk.req, rk.off_req, rk.respin, parent_out, W, g.block,
                                                             g.C, rk.j);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ m_comp, degree
__global__ void __launch_bounds__(256) k_mcomp(const int32_t* level, const uint32_t* tdeg, uint64_t block, ull* out) {
  typedef cub::BlockReduce<ull, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  ull acc = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x; t < block; t += (uint64_t)gridDim.x * 256)
    if (level[t] >= 0) acc += tdeg[t];
  ull tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0 && tot) atomicAdd(out, tot);
}

cudaError_t launch_mcomp(const Geom& g, Rank& rk, ull* out, cudaStream_t s) {
  k_mcomp<<<num_sms() * 4, 256, 0, s>>>(rk.level, rk.tdeg, g.block, out);
  return cudaGetLastError();
}

__global__ void k_degree(const ull* col, uint64_t u, ull* out) { *out += col[u + 1] - col[u]; }

cudaError_t launch_degree(Rank& rk, uint64_t u, ull* out, cudaStream_t s) {
  k_degree<<<1, 1, 0, s>>>(rk.col, u, out);
  return cudaGetLastError();
}

}  // namespace bfs200

namespace bfs200 {
// totals[c] = popcount of segment c of a bitmap whose exclusive popcount scan is off
__global__ void k_seg_totals(const uint32_t* off, uint64_t W, int C, unsigned long long* totals) {
  const int c = threadIdx.x;
  if (c < C) totals[c] = off[(uint64_t)(c + 1) * W] - off[(uint64_t)c * W];
}
cudaError_t launch_seg_totals(const uint32_t* off, uint64_t W, int C, unsigned long long* totals, cudaStream_t s) {
  k_seg_totals<<<1, 64, 0, s>>>(off, W, C, totals);
  return cudaGetLastError();
}
}  // namespace bfs200
