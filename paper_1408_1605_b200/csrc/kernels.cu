// kernels.cu -- hot-path kernels of libbfs200 for sm_100a (B200).
//
// Per BFS level on rank P_ij (Alg.2):
//   K3 k_scan_count / k_scan_segs / k_scan_emit : frontier bitmap -> ascending list of frontier
//        columns with local degree > 0, their row offsets, the exclusive degree scan `cumul`
//         and the per-tile first-column table that maps threads to edges
//        (Fig. t2d_map).  Warp-cooperative bitmap unpack.
//   K1 k_expand<E> : one thread per E consecutive frontier edges; the
//        visited filter (Alg.3 lines 5-6) and the discovered-row bitmap by atomicOr (Alg.3 line
//        7; bitmap pack fused).
//   K4 k_parent : parent claim for every row discovered in this level: the minimum frontier
//        column adjacent to it (ascending CSR row scan, first frontier member) -- the
//        deterministic form of Alg.3 line 17 (R1), without per-edge atomics.
//   K2 k_update : OR of the received fold segments, new = OR & ~visited, level, visited,
//        next frontier bitmap, lowest-column winner.
// All hot-path arithmetic is integer.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include <stdlib.h>

#include <type_traits>

#include "kernels.cuh"

namespace bfs200 {

typedef unsigned long long ull;

#ifndef BFS200_EMIT_SMEM  // K3 emit pass: dense chunks' column offsets staged by async copies
#define BFS200_EMIT_SMEM 1
#endif
// the pipelined short-tile loop of K1 in P2 levels (short_tiles_p2; 0 = the staged loop)
#ifndef BFS200_SHORTPIPE
#define BFS200_SHORTPIPE 1
#endif
// row slots of the pipelined long-tile loop of K1 (long_tiles_p2; 0 = the double-buffered loop):
// one row segment (1 x C = 1 graphs, SEG1) / several (C > 1: the probe's segment lookup costs
// registers; measured on a loopback 1x2 at s26: 3 slots 2.79 ms, 4 slots 2.88 ms per peak level)
#ifndef BFS200_K1PIPE
#define BFS200_K1PIPE 4
#endif
#ifndef BFS200_K1PIPE_SEGS
#define BFS200_K1PIPE_SEGS 3
#endif

// ------------------------------------------------------------------ small helpers
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}


__device__ __forceinline__ void red_or(uint32_t* p, uint32_t m) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(m) : "memory");
}

// predicated forms (no branch, no reconvergence point): the destination keeps its input value
// when the predicate is false
__device__ __forceinline__ void ld_stream_u32_if(bool p, const uint32_t* a, uint32_t& v) {
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.L1::no_allocate.u32 %0, [%1]; }"
               : "+r"(v) : "l"(a), "r"((int)p));
}
// predicated loads whose destinations are undefined when the predicate is false (no register
// initialisation; every use is guarded by the same predicate)
__device__ __forceinline__ void ld_stream_u32_p(bool p, const uint32_t* a, uint32_t& v) {
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.nc.L1::no_allocate.u32 %0, [%1]; }"
      : "=r"(v) : "l"(a), "r"((int)p));
}
// visited word (L2 only: the bitmap changes during the kernel), undefined when p is false
__device__ __forceinline__ void ld_cg_u32_p(bool p, const uint32_t* a, uint32_t& x) {
  asm("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cg.u32 %0, [%1]; }" : "=r"(x) : "l"(a), "r"((int)p));
}
__device__ __forceinline__ void red_or_if(bool p, uint32_t* a, uint32_t m) {
  asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q red.relaxed.gpu.global.or.b32 [%0], %1; }"
               ::"l"(a), "r"(m), "r"((int)p));
}

// Bounds checks (a BFS200_CHECKS=1 build; compute-sanitizer is not available on the GPU pool):
// an index outside its array traps the kernel, which the caller sees as BFS_ECUDA.  Capacities
// come from LevelInfo (set by alloc_state).  Off in production builds.
#ifndef BFS200_CHECKS
#define BFS200_CHECKS 0
#endif
#if BFS200_CHECKS
#define BCHECK(c)     \
  do {                \
    if (!(c)) __trap(); \
  } while (0)
#else
#define BCHECK(c) \
  do {            \
  } while (0)
#endif

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ------------------------------------------------------------------ init (Alg.2 lines 1-10)
__global__ void k_seed_root(uint32_t* vis, uint32_t* vold, uint32_t* all_front, int32_t* level, uint32_t* pred, uint8_t* winner,
                            int fused,
                            const uint32_t* fwd_own, uint64_t t0, uint64_t block, int i, uint32_t root, int j) {
  const uint64_t t = fwd_own[t0];  // relabeled offset of the root in its block
  const uint64_t row_local = (uint64_t)j * block + t, col_local = (uint64_t)i * block + t;
  vis[row_local >> 5] |= 1u << (row_local & 31);   // bmap[LOCAL_ROW(r)] <- 1
  if (!fused) vold[row_local >> 5] |= 1u << (row_local & 31);  // fused: level 1's count pass takes it
  all_front[col_local >> 5] |= 1u << (col_local & 31);  // front[0] <- LOCAL_COL(r)
  level[t] = 0;                                          // level[LOCAL_ROW(r)] <- 0
  pred[row_local] = root;                                // pred[LOCAL_ROW(r)] <- r
  if (winner) winner[t] = (uint8_t)j;
}

// level[] and pred[] need no reset: both are written for a vertex when it is reached, and every
// reader masks with the visited bit (unreached -> -1).
cudaError_t launch_init(const Geom& g, Rank& rk, bool owner, uint64_t root, bool fused, cudaStream_t s) {
  const uint64_t rw = g.nrows() / 32, cw = g.ncols() / 32;
  cudaError_t e = cudaMemsetAsync(rk.vis, 0, rw * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(rk.vold, 0, rw * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(rk.all_front, 0, cw * 4, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(&rk.info->disc_total, 0, sizeof(ull), s);
  if (e != cudaSuccess) return e;
  if (owner) {
    const uint64_t t = root - (uint64_t)rk.r * g.block;
    k_seed_root<<<1, 1, 0, s>>>(rk.vis, rk.vold, rk.all_front, rk.level, rk.pred, rk.winner, fused ? 1 : 0, rk.fwd_own, t, g.block, rk.i,
                                (uint32_t)root, rk.j);
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K3: unpack + degree scan
// Frontier columns are split by degree d (E = edges per thread, TILE = 32*E):
//   short (0 < d < TILE/2): listed in ascending order with their row offsets and the exclusive
//     scan of their degrees `cumul`; the expansion maps threads to their edges by
//     the scan + binary search of P:455-470 over tiles of TILE consecutive short edges, and K3
//     also emits the first column of every such tile (tile_k);
//   long (d >= TILE/2): cut into ceil(d/TILE) column-aligned tiles whose (row position, length,
//     column) records are emitted directly (tileA): the mapping of those edges is the identity
//     inside one column, which is where almost all edges of a dense level live.
// A warp owns a segment of kScanSegWords bitmap words; it walks the non-zero words 32 at a time
// and, per word, lane b handles bit b, so the col[] reads of one word are coalesced.
struct SegTot {
  unsigned int cs;  // short columns
  unsigned int na;  // long-column tiles
  unsigned int nh;  // hub entries: columns of > 8 long tiles, one entry per kHubChunk of their tiles (k_tile_fill)
  unsigned int pad;
  ull ss;           // short edges
  ull ls;           // long edges
};
static_assert(sizeof(SegTot) == 32, "engine.cu allocates 32 B per segment");
constexpr unsigned kHubChunk = 1024;  // long tiles per hub entry (the records one k_tile_fill warp writes)
__host__ __device__ constexpr unsigned hub_entries(unsigned nt) { return nt > 8 ? (nt + kHubChunk - 1) / kHubChunk : 0u; }
#ifndef BFS200_BLIND3
#define BFS200_BLIND3 1
#endif
constexpr bool kBlind3 = BFS200_BLIND3;

// Parent-claim mode thresholds (level_bookkeeping; measured at s26): P2 when a row's
// expected CSR scan is <= kP2Factor entries; mode 3 when the P1 candidate edges are >= rows / kM3Factor.
constexpr ull kP2Factor = 8;
constexpr ull kM3Factor = 4;

// K3 scan of the per-CTA totals of the count pass, one CTA (the totals are few: one per 32 K
// columns), fused with the level bookkeeping: seg_off[k] = exclusive scan of seg_tot[0..nseg)
// (here: the CTA totals; seg_off[nseg] = the level's totals), then the per-level counters and the
// parent-claim mode.  Pass k scans segments
// [1024k, 1024k + 1024): warp inclusive scans by shuffles, the 32 warp totals scanned by warp 0
// through shared memory, a running carry; the next pass's totals are loaded during this one.
constexpr int kSegScanThreads = 1024;
struct SegAcc {  // the scanned fields (pad is never summed)
  unsigned cs, na, nh;
  ull ss, ls;
};
__device__ __forceinline__ SegAcc seg_add(const SegAcc& a, const SegAcc& b) {
  return SegAcc{a.cs + b.cs, a.na + b.na, a.nh + b.nh, a.ss + b.ss, a.ls + b.ls};
}
__device__ __forceinline__ SegAcc seg_sub(const SegAcc& a, const SegAcc& b) {
  return SegAcc{a.cs - b.cs, a.na - b.na, a.nh - b.nh, a.ss - b.ss, a.ls - b.ls};
}
__device__ __forceinline__ SegAcc seg_shfl_up(const SegAcc& a, int d) {
  return SegAcc{__shfl_up_sync(0xFFFFFFFFu, a.cs, d), __shfl_up_sync(0xFFFFFFFFu, a.na, d),
                __shfl_up_sync(0xFFFFFFFFu, a.nh, d), __shfl_up_sync(0xFFFFFFFFu, a.ss, d),
                __shfl_up_sync(0xFFFFFFFFu, a.ls, d)};
}
__device__ __forceinline__ SegAcc seg_load(const SegTot* p, uint64_t k, uint64_t n) {
  if (k >= n) return SegAcc{0u, 0u, 0u, 0ull, 0ull};
  const SegTot t = p[k];
  return SegAcc{t.cs, t.na, t.nh, t.ss, t.ls};
}

constexpr int kSegItems = 2;  // consecutive totals per thread and pass (2048 per pass)
// exclusive scan of tot[0..n) into off[0..n], by the NT threads of one CTA; returns the total
template <int NT>
__device__ __forceinline__ SegAcc block_scan_totals(const SegTot* tot, uint64_t n, SegTot* off, SegAcc* s_warp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  SegAcc carry{0u, 0u, 0u, 0ull, 0ull};
  for (uint64_t base = 0; base < n; base += (uint64_t)NT * kSegItems) {
    const uint64_t k0 = base + (uint64_t)threadIdx.x * kSegItems;
    SegAcc v[kSegItems];
#pragma unroll
    for (int q = 0; q < kSegItems; ++q) v[q] = seg_load(tot, k0 + q, n);  // all in flight
    SegAcc mine{0u, 0u, 0u, 0ull, 0ull};
#pragma unroll
    for (int q = 0; q < kSegItems; ++q) mine = seg_add(mine, v[q]);
    SegAcc inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const SegAcc y = seg_shfl_up(inc, d);
      if (lane >= d) inc = seg_add(inc, y);
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const SegAcc w = lane < NT / 32 ? s_warp[lane] : SegAcc{0u, 0u, 0u, 0ull, 0ull};
      SegAcc wi = w;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const SegAcc y = seg_shfl_up(wi, d);
        if (lane >= d) wi = seg_add(wi, y);
      }
      if (lane < NT / 32) s_warp[lane] = seg_sub(wi, w);  // exclusive over the warps
      if (lane == 31) s_warp[NT / 32] = wi;               // the pass total
    }
    __syncthreads();
    SegAcc ex = seg_add(carry, seg_add(s_warp[wid], seg_sub(inc, mine)));
#pragma unroll
    for (int q = 0; q < kSegItems; ++q) {
      if (k0 + q < n) off[k0 + q] = SegTot{ex.cs, ex.na, ex.nh, 0u, ex.ss, ex.ls};
      ex = seg_add(ex, v[q]);
    }
    carry = seg_add(carry, s_warp[NT / 32]);
    __syncthreads();  // s_warp is rewritten by the next pass
  }
  return carry;
}

__global__ void __launch_bounds__(kSegScanThreads) k_seg_scan(const SegTot* __restrict__ seg_tot, uint64_t nseg,
                                                               SegTot* seg_off, LevelInfo* info, void* cumul, int narrow,
                                                               ull nnz,
                                                               ull p2_factor, ull nz_rows, ull m3_factor, ull nrows) {
  __shared__ SegAcc s_warp[kSegScanThreads / 32 + 1];
  const SegAcc carry = block_scan_totals<kSegScanThreads>(seg_tot, nseg, seg_off, s_warp);
  if (threadIdx.x != 0) return;
  const SegAcc c = carry;
  seg_off[nseg] = SegTot{c.cs, c.na, c.nh, 0u, c.ss, c.ls};
  // level totals; resets the per-level counters
  info->n = c.cs;
  info->sedges = c.ss;
  info->nA = c.na;
  info->edges = c.ss + c.ls;
  info->ncols = c.cs;
  info->newv = 0;
  // Parent-claim mode of this level.  A discovered row's CSR scan stops at its first frontier
  // neighbour, after ~nnz/edges entries on average (edges = entries leaving the frontier), so
  // the scan (P2) is used when that is <= p2_factor (default 8); otherwise (small frontiers,
  // e.g. the first levels) the expansion does atomicMin per candidate edge (P1).  P2 also when
  // few rows remain to be discovered (the scans are then few, whatever their length):
  // remaining = rows with entries - rows discovered so far (an estimate on this rank).
  const ull edges = c.ss + c.ls, seen = info->disc_total;
  const ull remaining = nz_rows > seen ? nz_rows - seen : 0ull;
  info->mode = (edges * p2_factor >= nnz || remaining * 64ull <= edges) ? 2ull : 1ull;
  // P1 with many candidate edges (mode 3): the expansion only claims (atomicMin); the parent
  // pass derives the discovered words from pmin in one pass over the rows (cheaper than a
  // RED.OR and a probe per edge once edges * m3_factor >= rows)
  if (info->mode == 1 && m3_factor && edges * m3_factor >= nrows) info->mode = 3ull;
  // mode 3 while at most 1/16 of the rows are visited (the first dense level): the visited
  // probe of a non-hot row almost never finds the bit set, so the claim goes out without it
  info->blind = (info->mode == 3 && kBlind3 && seen * 16ull <= nz_rows) ? 1ull : 0ull;
  info->nlong = c.nh;  // hub columns, listed by k_scan_emit at scan positions
  info->nlongcols = 0;
  if (narrow) static_cast<uint32_t*>(cumul)[c.cs] = (uint32_t)c.ss;
  else static_cast<ull*>(cumul)[c.cs] = c.ss;
}

// Count pass: a warp owns a segment of kScanSegWords bitmap words; lane l takes word 32c + l of
// chunk c and walks its set bits, their degrees read from the saturated byte copy deg8 (a quarter
// of the bytes of col32, read as whole 32-B runs: no dependent per-column loads).
// Fused frontier update of a 1x1 graph (no exchange between K4 and K3): K2 does not run; the
// count pass of the NEXT level takes the frontier as the rows discovered in the previous level,
// f = vis & ~vold, writes it to the frontier bitmap (read by the emit pass and K4), advances
// vold and writes the rows' level (ctrl->lvl - 1).  The root is seeded into vis only.
struct FusedUpd {
  const uint32_t* vis;
  uint32_t* vold;
  uint32_t* front;  // the frontier bitmap written here (== the bm the emit pass reads)
  int32_t* level;
  const LevelCtrl* ctrl;
};

template <typename Col, bool FUSED>
__device__ __forceinline__ SegTot count_seg(const uint32_t* __restrict__ bm, uint64_t nwords, uint64_t seg,
                                            const Col* __restrict__ col, const uint8_t* __restrict__ deg8,
                                            int tile_shift, const FusedUpd& fu) {
  const int lane = threadIdx.x & 31;
  const uint64_t w0 = seg * kScanSegWords;
  const uint64_t w1 = min(w0 + kScanSegWords, nwords);
  const ull half = 1ull << (tile_shift - 1), tm = (1ull << tile_shift) - 1;
  SegTot t{0u, 0u, 0ull, 0ull};
  uint32_t xw[kScanSegWords / 32];  // the segment's words, lane l: word w0 + 32c + l
  {  // all words of the segment in one round trip; an empty segment (sparse levels) ends here
    uint32_t any = 0;
#pragma unroll
    for (int c = 0; c < kScanSegWords / 32; ++c) {
      const uint64_t w = w0 + 32 * c + lane;
      if (FUSED) {
        const uint32_t vn = (w < w1) ? fu.vis[w] : 0u, vo = (w < w1) ? fu.vold[w] : 0u;
        xw[c] = vn & ~vo;
        if (w < w1) {
          fu.front[w] = xw[c];
          if (xw[c]) fu.vold[w] = vn;
        }
      } else {
        xw[c] = (w < w1) ? __ldg(bm + w) : 0u;
      }
      any |= xw[c];
    }
    if (FUSED) {  // levels of the new frontier, lane l writing vertex 32k + l of word k (coalesced)
      const int32_t lv = (int32_t)fu.ctrl->lvl - 1;
#pragma unroll
      for (int c = 0; c < kScanSegWords / 32; ++c) {
        unsigned nz = __ballot_sync(0xFFFFFFFFu, xw[c] != 0u);
        while (nz) {
          const int k = __ffs(nz) - 1;
          nz &= nz - 1;
          const uint32_t nb = __shfl_sync(0xFFFFFFFFu, xw[c], k);
          if ((nb >> lane) & 1u) fu.level[(w0 + 32 * c + k) * 32 + lane] = lv;
        }
      }
    }
    if (!__any_sync(0xFFFFFFFFu, any != 0u)) return SegTot{0u, 0u, 0u, 0u, 0ull, 0ull};
  }
  auto add_col = [&](ull d) {
    if (d >= half) {
      const unsigned nt = (unsigned)((d + tm) >> tile_shift);
      t.na += nt;
      t.nh += hub_entries(nt);
      t.ls += d;
    } else if (d) {
      t.cs += 1u;
      t.ss += d;
    }
  };
  // Lane l takes word w of chunk c (w = w0 + 32c + l) and the saturated degrees of its 32 columns,
  // deg8[32w .. 32w + 32) (two 16-B loads; a warp reads 1 KB contiguous, two chunks in flight);
  // the exact degree comes from col[] only for a saturated byte (degree >= 255).
  auto add_word = [&](uint32_t x, const uint4& lo, const uint4& hi, uint64_t w) {
    const uint32_t dw[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    uint32_t sat = 0;  // frontier columns of saturated degree (hubs): exact degree from col[]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      for (uint32_t bits = (x >> (4 * j)) & 0xFu; bits; bits &= bits - 1) {
        const int bb = __ffs(bits) - 1;
        const uint32_t d = (dw[j] >> (8 * bb)) & 0xFFu;
        if (d == 255u) sat |= 1u << (4 * j + bb);
        else add_col(d);
      }
    }
    while (sat) {  // 4 at a time: their col[] loads in flight together (hub words of the first levels)
      ull dd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int b = sat ? __ffs(sat) - 1 : -1;
        sat &= sat ? sat - 1 : 0u;
        const uint64_t u = w * 32 + (b < 0 ? 0 : b);
        dd[q] = b < 0 ? 0ull : (ull)(__ldg(col + u + 1) - __ldg(col + u));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) add_col(dd[q]);
    }
  };
  const uint4* __restrict__ d16 = reinterpret_cast<const uint4*>(deg8);
#pragma unroll
  for (int c = 0; c < kScanSegWords / 32; c += 2) {
    uint4 dg[2][2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t w = w0 + 32 * (c + k) + lane;
      dg[k][0] = dg[k][1] = make_uint4(0u, 0u, 0u, 0u);
      if (xw[c + k]) {  // zero past w1
        dg[k][0] = __ldg(d16 + 2 * w);
        dg[k][1] = __ldg(d16 + 2 * w + 1);
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) add_word(xw[c + k], dg[k][0], dg[k][1], w0 + 32 * (c + k) + lane);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    t.cs += __shfl_xor_sync(0xFFFFFFFFu, t.cs, o);
    t.na += __shfl_xor_sync(0xFFFFFFFFu, t.na, o);
    t.nh += __shfl_xor_sync(0xFFFFFFFFu, t.nh, o);
    t.ss += __shfl_xor_sync(0xFFFFFFFFu, t.ss, o);
    t.ls += __shfl_xor_sync(0xFFFFFFFFu, t.ls, o);
  }
  return t;
}

// Per-segment totals (seg_tot[seg]) and per-CTA totals of the kScanThreads/32 segments of a CTA
// (cta_tot[b]): the single-CTA scan (k_seg_scan) then only scans the few CTA totals, and the
// emit pass adds the in-CTA prefix itself.
template <typename Col, bool FUSED>
__global__ void __launch_bounds__(kScanThreads) k_scan_count(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                              uint64_t nseg, const Col* __restrict__ col,
                                                              const uint8_t* __restrict__ deg8, SegTot* seg_tot,
                                                              SegTot* cta_tot, int tile_shift, FusedUpd fu) {
  __shared__ SegTot s_t[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t seg = (uint64_t)blockIdx.x * (kScanThreads / 32) + wid;
  const SegTot t =
      seg < nseg ? count_seg<Col, FUSED>(bm, nwords, seg, col, deg8, tile_shift, fu) : SegTot{0u, 0u, 0u, 0u, 0ull, 0ull};
  if (lane == 0) {
    if (seg < nseg) seg_tot[seg] = t;
    s_t[wid] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    SegTot c{0u, 0u, 0u, 0u, 0ull, 0ull};
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w)
      c = SegTot{c.cs + s_t[w].cs, c.na + s_t[w].na, c.nh + s_t[w].nh, 0u, c.ss + s_t[w].ss, c.ls + s_t[w].ls};
    cta_tot[blockIdx.x] = c;
  }
}

// Emit pass: same word ownership.  Sparse chunks (< 96 set bits in 32 words): each lane totals
// its word, one warp exclusive scan per chunk gives the lane its list / edge / long-tile / hub
// positions, then the lane writes its columns in ascending order.  Dense chunks: word by word,
// lane b handles bit b (coalesced col reads and list writes), col loads of 4 words in flight.
// NARROW (every CSC position < 2^32): the row offsets and the scan are stored as 32-bit values
// (12 B per short column instead of 20, written here and read by K1).
template <bool NARROW>
__global__ void __launch_bounds__(kScanThreads) k_scan_emit(const uint32_t* __restrict__ bm, uint64_t nwords,
                                                             uint64_t nseg,
                                                             const typename std::conditional<NARROW, uint32_t, ull>::type*
                                                                 __restrict__ col,
                                                             const SegTot* seg_tot, const SegTot* cta_off,
                                                             uint32_t* flist, void* rowoff_v, void* cumul_v,
                                                             uint32_t* tile_k, uint4* tileA,
                                                             int tile_shift, uint4* longlist, LevelInfo* info) {
  typedef typename std::conditional<NARROW, uint32_t, ull>::type Off;
  Off* rowoff = static_cast<Off*>(rowoff_v);
  Off* cumul = static_cast<Off*>(cumul_v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t seg = (uint64_t)blockIdx.x * (kScanThreads / 32) + wid;
  if (seg >= nseg) return;
  const uint64_t w0 = seg * kScanSegWords;
  const uint64_t w1 = min(w0 + kScanSegWords, nwords);
  SegTot o = cta_off[blockIdx.x];  // + the totals of this CTA's earlier segments
  for (int w2 = 0; w2 < wid; ++w2) {
    const SegTot q = seg_tot[(uint64_t)blockIdx.x * (kScanThreads / 32) + w2];
    o = SegTot{o.cs + q.cs, o.na + q.na, o.nh + q.nh, 0u, o.ss + q.ss, o.ls + q.ls};
  }
  {  // nothing to emit (no column of non-zero degree in the segment): skip the bitmap
    const SegTot mine = seg_tot[seg];
    if (mine.cs == 0 && mine.na == 0) return;
  }
  uint64_t k = o.cs;  // next short list position
  ull e = o.ss;       // next short edge position
  uint64_t a = o.na;  // next long-tile position
  uint64_t h = o.nh;  // next hub slot
  const ull half = 1ull << (tile_shift - 1), tm = (1ull << tile_shift) - 1;
  const unsigned lt = lanemask_lt();
  unsigned nlongcols = 0;
  __shared__ uint16_t s_lists[kScanThreads / 32][1024];
  uint16_t* s_list = s_lists[threadIdx.x >> 5];
  // NARROW: the column offsets of a dense chunk (1024 columns + the end), one slice per warp
  constexpr bool kEmitSmem = NARROW && BFS200_EMIT_SMEM;
  __shared__ __align__(16) uint32_t s_cols[kEmitSmem ? kScanThreads / 32 : 1][kEmitSmem ? 1024 : 4];
  // compact 8-byte long-tile records (position, length) in P2 levels of the pipelined loop (the
  // column is only needed by the P1 claims): half the record traffic of K3 and K1
  const bool compact = NARROW && BFS200_K1PIPE > 0 && info->mode == 2 && tile_shift <= 8;
  const bool need_flist = info->mode != 2;  // the column ids of short columns: P1 claims only
  auto emit_long = [&](uint64_t u, ull c0, ull d, uint64_t pa, unsigned nt, uint64_t hub) {
    if (nt <= 8) {
      for (unsigned q = 0; q < nt; ++q) {
        const ull pos = c0 + ((ull)q << tile_shift);
        const ull len = min(d - ((ull)q << tile_shift), tm + 1);
        BCHECK(pa + q < info->cap_tiles && pos + len <= info->cap_nnz);
        if (compact) reinterpret_cast<uint2*>(tileA)[pa + q] = make_uint2((uint32_t)pos, (uint32_t)len);
        else tileA[pa + q] = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)len, (uint32_t)u);
      }
    } else {  // hub column: its tiles are written by k_tile_fill, kHubChunk per entry
      for (unsigned k = 0; k < hub_entries(nt); ++k) {
        const ull q0 = (ull)k * kHubChunk, pk = pa + q0, ck = c0 + (q0 << tile_shift), dk = d - (q0 << tile_shift);
        const unsigned nk = min(nt - (unsigned)q0, kHubChunk);
        BCHECK(2 * (hub + k) + 1 < info->cap_long && c0 + d <= info->cap_nnz);
        longlist[2 * (hub + k)] = make_uint4((uint32_t)pk, nk, (uint32_t)u, (uint32_t)(pk >> 32));
        longlist[2 * (hub + k) + 1] = make_uint4((uint32_t)ck, (uint32_t)(ck >> 32), (uint32_t)dk, (uint32_t)(dk >> 32));
      }
    }
  };
  for (uint64_t wb = w0; wb < w1; wb += 32) {
    const uint64_t w = wb + lane;
    const uint32_t x = (w < w1) ? __ldg(bm + w) : 0u;
    const unsigned nbits = __reduce_add_sync(0xFFFFFFFFu, (unsigned)__popc(x));
    if (nbits >= 96) {
      // dense chunk: compact its set bits (column offsets in the chunk, ascending) into this
      // warp's shared list, then emit 32 frontier columns per step with every lane busy
      // (NARROW: the chunk's 1025 column offsets are first copied into the warp's shared slice
      // with 16-B asynchronous copies -- one round trip, overlapping the compaction -- so the
      // steps read no global memory; else the col loads of two steps are in flight together)
      const uint64_t cw1 = min(wb + 32, w1);  // the chunk's words are [wb, cw1)
      if constexpr (kEmitSmem) {
        uint32_t* s_c = s_cols[wid];
        const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_c);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t piece = 32u * k + lane;  // columns 4*piece .. 4*piece+3 of the chunk (word piece/8)
          if (wb + piece / 8 < cw1)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sbase + 16u * piece),
                         "l"(col + wb * 32 + 4ull * piece));
        }
        asm volatile("cp.async.commit_group;\n" ::);
      }
      // the end offset of the chunk's last column
      const uint32_t cend = kEmitSmem ? (uint32_t)__ldg(col + cw1 * 32) : 0u;
      const unsigned ccols = (unsigned)(cw1 - wb) * 32;
      const unsigned c = __popc(x);
      unsigned incl = c;
#pragma unroll
      for (int s2 = 1; s2 < 32; s2 <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, incl, s2);
        if (lane >= s2) incl += y;
      }
      unsigned p = incl - c;
      for (uint32_t y = x; y; y &= y - 1) s_list[p++] = (uint16_t)(lane * 32 + __ffs(y) - 1);
      if constexpr (kEmitSmem) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      __syncwarp();
      // one step: lane = frontier column u (c0, d) of the compacted list, valid = inside the list
      auto emit_step = [&](uint64_t u, ull c0, ull d, bool valid) {
        const bool isl = valid && d >= half;
        const unsigned ds = (valid && !isl) ? (unsigned)d : 0u;  // short degree < TILE/2
        const unsigned na = isl ? (unsigned)((d + tm) >> tile_shift) : 0u;
        const unsigned smask = __ballot_sync(0xFFFFFFFFu, ds != 0);
        const unsigned ne = hub_entries(na);
        unsigned inc = ds, ia = na, ih = ne;  // inclusive warp scans
#pragma unroll
        for (int s2 = 1; s2 < 32; s2 <<= 1) {
          const unsigned y1 = __shfl_up_sync(0xFFFFFFFFu, inc, s2);
          const unsigned y2 = __shfl_up_sync(0xFFFFFFFFu, ia, s2);
          const unsigned y3 = __shfl_up_sync(0xFFFFFFFFu, ih, s2);
          if (lane >= s2) {
            inc += y1;
            ia += y2;
            ih += y3;
          }
        }
        if (ds) {
          const uint64_t pos = k + __popc(smask & lt);
          const ull eb = e + inc - ds;
          BCHECK(pos < info->cap_ncols && u < info->cap_ncols && c0 + ds <= info->cap_nnz);
          if (need_flist) flist[pos] = (uint32_t)u;
          rowoff[pos] = (Off)c0;
          cumul[pos] = (Off)eb;
          for (ull t = (eb + tm) >> tile_shift; (t << tile_shift) < eb + ds; ++t) {
            BCHECK(t < info->cap_nnz / 32 + 2);
            tile_k[t] = (uint32_t)pos;
          }
        }
        if (isl) {
          emit_long(u, c0, d, a + ia - na, na, h + ih - ne);
          ++nlongcols;
        }
        k += __popc(smask);
        h += __shfl_sync(0xFFFFFFFFu, ih, 31);
        e += __shfl_sync(0xFFFFFFFFu, inc, 31);
        a += __shfl_sync(0xFFFFFFFFu, ia, 31);
      };
      if constexpr (kEmitSmem) {
        const uint32_t* s_c = s_cols[wid];
        for (unsigned g = 0; g < nbits; g += 32) {
          const unsigned idx = g + lane;
          const bool valid = idx < nbits;
          const unsigned off = valid ? s_list[idx] : 0u;
          const uint32_t c0 = s_c[off], c1 = off + 1 < ccols ? s_c[off + 1] : cend;
          emit_step(wb * 32 + off, (ull)c0, (ull)(c1 - c0), valid);
        }
      } else {
        for (unsigned g = 0; g < nbits; g += 64) {
          ull c0b[2], c1b[2];
          uint64_t ub[2];
#pragma unroll
          for (int b = 0; b < 2; ++b) {  // col loads of two groups in flight together
            const unsigned idx = g + 32 * b + lane;
            const bool valid = idx < nbits;
            ub[b] = wb * 32 + (valid ? s_list[idx] : 0u);
            c0b[b] = valid ? (ull)__ldg(col + ub[b]) : 0ull;
            c1b[b] = valid ? (ull)__ldg(col + ub[b] + 1) : 0ull;
          }
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            if (g + 32 * b >= nbits) break;  // warp-uniform
            emit_step(ub[b], c0b[b], c1b[b] - c0b[b], g + 32 * b + lane < nbits);
          }
        }
      }
      __syncwarp();  // the list (and the offsets) are rewritten by the next chunk
      continue;
    }
    // sparse chunk: lane totals of its word (4 set bits at a time)
    unsigned cs = 0, na = 0, nh = 0;
    ull ss = 0;
    for (uint32_t y = x; y;) {
      ull dd[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int b = y ? __ffs(y) - 1 : -1;
        y &= y ? y - 1 : 0u;
        const uint64_t u = w * 32 + (b < 0 ? 0 : b);
        dd[q] = b < 0 ? 0ull : (ull)(__ldg(col + u + 1) - __ldg(col + u));
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const ull d = dd[q];
        if (d >= half) {
          const unsigned nt = (unsigned)((d + tm) >> tile_shift);
          na += nt;
          nh += hub_entries(nt);
        } else if (d) {
          cs += 1u;
          ss += d;
        }
      }
    }
    // warp exclusive scans of the lane totals
    unsigned ics = cs, ina = na, inh = nh;
    ull iss = ss;
#pragma unroll
    for (int s2 = 1; s2 < 32; s2 <<= 1) {
      const unsigned y1 = __shfl_up_sync(0xFFFFFFFFu, ics, s2);
      const unsigned y2 = __shfl_up_sync(0xFFFFFFFFu, ina, s2);
      const unsigned y4 = __shfl_up_sync(0xFFFFFFFFu, inh, s2);
      const ull y3 = __shfl_up_sync(0xFFFFFFFFu, iss, s2);
      if (lane >= s2) {
        ics += y1;
        ina += y2;
        inh += y4;
        iss += y3;
      }
    }
    uint64_t kk = k + ics - cs;
    ull ee = e + iss - ss;
    uint64_t aa = a + ina - na;
    uint64_t hh = h + inh - nh;
    for (uint32_t y = x; y;) {
      const int b = __ffs(y) - 1;
      y &= y - 1;
      const uint64_t u = w * 32 + b;
      const ull c0 = (ull)__ldg(col + u), d = (ull)__ldg(col + u + 1) - c0;
      if (d >= half) {
        const unsigned nt = (unsigned)((d + tm) >> tile_shift);
        emit_long(u, c0, d, aa, nt, hh);
        aa += nt;
        hh += hub_entries(nt);
        ++nlongcols;
      } else if (d) {
        BCHECK(kk < info->cap_ncols && u < info->cap_ncols && c0 + d <= info->cap_nnz);
        if (need_flist) flist[kk] = (uint32_t)u;
        rowoff[kk] = (Off)c0;
        cumul[kk] = (Off)ee;
        for (ull t = (ee + tm) >> tile_shift; (t << tile_shift) < ee + d; ++t) {
          BCHECK(t < info->cap_nnz / 32 + 2);
          tile_k[t] = (uint32_t)kk;
        }
        ++kk;
        ee += d;
      }
    }
    k += __shfl_sync(0xFFFFFFFFu, ics, 31);
    e += __shfl_sync(0xFFFFFFFFu, iss, 31);
    a += __shfl_sync(0xFFFFFFFFu, ina, 31);
    h += __shfl_sync(0xFFFFFFFFu, inh, 31);
  }
#pragma unroll
  for (int s2 = 16; s2; s2 >>= 1) nlongcols += __shfl_xor_sync(0xFFFFFFFFu, nlongcols, s2);
  if (lane == 0 && nlongcols) atomicAdd(&info->nlongcols, (ull)nlongcols);
}

// long-tile records of hub columns: one warp per hub entry (a hub of more than kHubChunk tiles
// is listed as several entries by k_scan_emit, so no warp writes more than kHubChunk records)
__global__ void k_tile_fill(const uint4* longlist, const LevelInfo* info, uint4* tileA, int tile_shift, int narrow) {
  const int lane = threadIdx.x & 31;
  const bool compact = narrow && BFS200_K1PIPE > 0 && info->mode == 2 && tile_shift <= 8;  // as in k_scan_emit
  const ull nl = info->nlong;
  const ull tm = (1ull << tile_shift) - 1;
  for (ull r = ((ull)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nl; r += ((ull)gridDim.x * blockDim.x) >> 5) {
    const uint4 h = longlist[2 * r], b = longlist[2 * r + 1];
    const ull pa = (ull)h.x | ((ull)h.w << 32);
    const ull c0 = (ull)b.x | ((ull)b.y << 32), d = (ull)b.z | ((ull)b.w << 32);
    BCHECK(h.y <= (uint32_t)kHubChunk);
    for (uint32_t q = lane; q < h.y; q += 32) {
      const ull pos = c0 + ((ull)q << tile_shift);
      const ull len = min(d - ((ull)q << tile_shift), tm + 1);
      BCHECK(pa + q < info->cap_tiles && pos + len <= info->cap_nnz);
      if (compact) reinterpret_cast<uint2*>(tileA)[pa + q] = make_uint2((uint32_t)pos, (uint32_t)len);
      else tileA[pa + q] = make_uint4((uint32_t)pos, (uint32_t)(pos >> 32), (uint32_t)len, h.z);
    }
  }
}

cudaError_t launch_scan(const Geom& g, Rank& rk, uint32_t tile_edges, bool narrow, const LevelCtrl* ctrl,
                        cudaStream_t s) {
  const uint64_t nwords = g.ncols() / 32;
  const uint64_t nseg = (nwords + kScanSegWords - 1) / kScanSegWords;
  const unsigned grid = (unsigned)((nseg + kScanThreads / 32 - 1) / (kScanThreads / 32));
  const int ts = __builtin_ctz(tile_edges);
  SegTot* st = static_cast<SegTot*>(rk.seg_tot);
  SegTot* ct = static_cast<SegTot*>(rk.seg_off);  // [grid] CTA totals, then [grid + 1] their scan
  SegTot* co = ct + grid;
  // narrow: the 32-bit copy of the column offsets (half the bytes of the col[] reads)
  const FusedUpd fu{rk.vis, rk.vold, rk.all_front, rk.level, ctrl};
  if (ctrl) {  // fused update (1x1): narrow or not
    if (narrow)
      k_scan_count<uint32_t, true><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col32, rk.deg8, st, ct, ts, fu);
    else
      k_scan_count<ull, true><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col, rk.deg8, st, ct, ts, fu);
  } else if (narrow) {
    k_scan_count<uint32_t, false><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col32, rk.deg8, st, ct, ts, fu);
  } else {
    k_scan_count<ull, false><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col, rk.deg8, st, ct, ts, fu);
  }

  // exclusive scan of the CTA totals (co[grid] = level total) + the level's counters
  k_seg_scan<<<1, kSegScanThreads, 0, s>>>(ct, grid, co, rk.info, rk.cumul, narrow ? 1 : 0, (ull)rk.nnz, kP2Factor,
                                          (ull)rk.nz_rows, kM3Factor, (ull)g.nrows());
  if (narrow)
    k_scan_emit<true><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col32, st, co, rk.flist, rk.rowoff,
                                                    rk.cumul, rk.tile_k, rk.tileA, ts, rk.longlist, rk.info);
  else
    k_scan_emit<false><<<grid, kScanThreads, 0, s>>>(rk.all_front, nwords, nseg, rk.col, st, co, rk.flist, rk.rowoff,
                                                     rk.cumul, rk.tile_k, rk.tileA, ts, rk.longlist, rk.info);
  k_tile_fill<<<g.nsm * 8, 256, 0, s>>>(rk.longlist, rk.info, rk.tileA, ts, narrow ? 1 : 0);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K1: frontier expansion
// Persistent grid, one CTA of THREADS threads per SM; every WARP independently walks warp
// tiles of TILE = 32*E consecutive frontier edges (grid-stride), so no CTA barrier ever waits
// on the slowest memory access.  A warp stages its tile's columns (<= TILE+1: edge begin within
// the tile, row offset, and in P1 levels the parent's original global id) in its own shared
// memory slice from the K3 tile table; each lane maps its first edge by binary search there and
// the next E-1 by linear advance.  The E row loads are issued together,
// then the visited tests: rows in the hot (relabeled, highest-degree) prefix of each row segment
// are tested against a CTA-wide shared-memory copy of their visited bits taken at kernel start;
// the others with one 8-byte load of the visited|discovered pair.  Then one RED.OR per row
// neither visited nor already discovered; in P1 levels also compare-then-atomicMin of the
// parent's global id.
constexpr ull kHotMinEdges = 1ull << 22;  // stage the hot visited prefix only for big levels
constexpr size_t kSmemBudget = 227 * 1024;
#ifndef BFS200_SMEM_KB
#define BFS200_SMEM_KB 160
#endif
constexpr size_t kSmemTarget = (size_t)BFS200_SMEM_KB * 1024;  // K1 dynamic shared memory (staging + hot copy)
// per-warp chunk before the hot-copy region: the warp's short-tile staging (s_off, s_beg)
template <int E>
__host__ __device__ constexpr size_t expand_warp_bytes(bool pos32) {
  return 16 * (((32 * E + 2) * ((pos32 ? 4 : 8) + 4) + 15) / 16);
}
template <int E, int THREADS>
__host__ __device__ constexpr size_t expand_stage_bytes(bool pos32) {
  return (THREADS / 32) * expand_warp_bytes<E>(pos32);
}

// Visited word of row v in the shared-memory hot copy.  Layout: per row segment hw words of the
// hot prefix and one zero sentinel (word hw), so rows past the prefix need no range test: their
// lookup lands on the sentinel and they take the L2 probe.
template <bool SEG1>
__device__ __forceinline__ uint32_t hot_word(const uint32_t* s_hot, uint32_t v, bool ok, uint32_t hw, int bl,
                                             uint32_t bmask) {
  if (SEG1) return s_hot[min(v >> 5, hw)];  // one segment: v is the offset (any v stays in bounds)
  const uint32_t idx = (v >> bl) * (hw + 1) + min((v & bmask) >> 5, hw);
  return s_hot[ok ? idx : hw];
}

// Visited test of one row of a P2 level, hand-scheduled (the hot loop of K1): probe the hot copy
// (32-bit shared address sa, SEG1 layout: hw words + sentinel), then, if the row is neither hot
// and visited nor invalid (pos >= len), one 8-byte L2 load of its visited|discovered pair.
// Outputs: need (0/1), the bit mask m, the pair x|y and the pair's address for the RED.
// `vis` holds the visited bits of the level start ORed with the rows discovered so far in this
// level (the RED.ORs go into the same word), so one 4-byte load both tests "visited" and
// de-duplicates the REDs; `vold` keeps the level-start bits (K4 / K2 take the discovered word as
// vis & ~vold).  A 128-byte line covers 1024 rows: lanes probing nearby rows of one column share
// L2 requests (the L2 tag rate bounds the peak level).
struct Probe {
  uint32_t x, need, m;
  uint32_t* a;
};
__device__ __forceinline__ void probe_seg1(Probe& p, uint32_t v, uint32_t pos, uint32_t len, uint32_t hw, uint32_t sa,
                                           uint32_t* vis) {
  asm("{\n"
      " .reg .pred pok, pn;\n"
      " .reg .b32 wi, hi, hv;\n"
      " setp.lt.u32 pok, %5, %6;\n"
      " shr.b32 wi, %4, 5;\n"
      " min.u32 hi, wi, %7;\n"
      " shl.b32 hi, hi, 2;\n"
      " add.u32 hi, hi, %8;\n"
      " ld.shared.u32 hv, [hi];\n"
      " shf.l.wrap.b32 %2, 0, 1, %4;\n"
      " and.b32 hv, hv, %2;\n"
      " setp.eq.and.b32 pn, hv, 0, pok;\n"
      " mad.wide.u32 %3, wi, 4, %9;\n"
      " @pn ld.global.cg.u32 %0, [%3];\n"
      " selp.u32 %1, 1, 0, pn;\n"
      "}"
      : "=r"(p.x), "=r"(p.need), "=r"(p.m), "=l"(p.a)
      : "r"(v), "r"(pos), "r"(len), "r"(hw), "r"(sa), "l"(vis));
}
// general layout (C row segments of hw words + sentinel each)
__device__ __forceinline__ void probe_segs(Probe& p, uint32_t v, uint32_t pos, uint32_t len, uint32_t hw, uint32_t sa,
                                           uint32_t* vis, int bl, uint32_t bmask) {
  asm("{\n"
      " .reg .pred pok, pn;\n"
      " .reg .b32 wi, hi, hv, sg, off;\n"
      " setp.lt.u32 pok, %5, %6;\n"
      " shr.b32 wi, %4, 5;\n"
      " shr.b32 sg, %4, %10;\n"
      " and.b32 off, %4, %11;\n"
      " shr.b32 off, off, 5;\n"
      " min.u32 off, off, %7;\n"
      " add.u32 hv, %7, 1;\n"
      " mad.lo.u32 hi, sg, hv, off;\n"
      " selp.u32 hi, hi, %7, pok;\n"
      " shl.b32 hi, hi, 2;\n"
      " add.u32 hi, hi, %8;\n"
      " ld.shared.u32 hv, [hi];\n"
      " shf.l.wrap.b32 %2, 0, 1, %4;\n"
      " and.b32 hv, hv, %2;\n"
      " setp.eq.and.b32 pn, hv, 0, pok;\n"
      " mad.wide.u32 %3, wi, 4, %9;\n"
      " @pn ld.global.cg.u32 %0, [%3];\n"
      " selp.u32 %1, 1, 0, pn;\n"
      "}"
      : "=r"(p.x), "=r"(p.need), "=r"(p.m), "=l"(p.a)
      : "r"(v), "r"(pos), "r"(len), "r"(hw), "r"(sa), "l"(vis), "r"(bl), "r"(bmask));
}
// RED.OR of the row's bit if the probe was needed and found it neither visited nor discovered
// (Alg.3 line 7)
__device__ __forceinline__ void probe_red(const Probe& p) {
  asm volatile("{\n"
               " .reg .pred pn, pr;\n"
               " .reg .b32 t;\n"
               " setp.ne.b32 pn, %2, 0;\n"
               " and.b32 t, %0, %1;\n"
               " setp.eq.and.b32 pr, t, 0, pn;\n"
               " @pr red.relaxed.gpu.global.or.b32 [%3], %1;\n"
               "}" ::"r"(p.x), "r"(p.m), "r"(p.need), "l"(p.a));
}

// One warp tile's edges after their row ids v[] are loaded: the visited test (hot rows against
// the shared-memory copy, the others with one 4-byte load), then the RED.OR of the row's bit and,
// in P1 levels, the parent claim.  P1 levels test the LEVEL-START bits (vold): every frontier
// neighbour of a row not visited before the level must claim it (the minimum decides), even when
// another edge discovered the row earlier in this level; their RED.ORs into vis are then not
// de-duplicated (P1 levels are the sparse ones).  P2 levels test vis (visited or discovered).
// claim3 (P1 levels with a dense claim, mode 3): the claim alone, atomicMin of pmin; rows of the
// hot prefix need no probe (their visited bit is exact in shared memory) and no bit is set here
// -- k_parent derives the discovered words from pmin.
template <int WV, bool P1, bool SEG1>
__device__ __forceinline__ void expand_edges(const uint32_t (&v)[WV], const uint32_t (&ug)[WV], uint32_t* vis,
                                             const uint32_t* vold, uint32_t* pmin, const uint32_t* s_hot,
                                             uint32_t bmask, int bl, uint32_t hw, bool claim3 = false,
                                             bool blind3 = false) {
  uint32_t wx[WV];
  bool need[WV], probe[WV];
#pragma unroll
  for (int q = 0; q < WV; ++q) {
    const bool ok = v[q] != 0xFFFFFFFFu;
    const uint32_t m = 1u << (v[q] & 31);
    need[q] = ok;
    probe[q] = ok;
    if (!P1 || claim3) {
      need[q] = ok && !(hot_word<SEG1>(s_hot, v[q], ok, hw, bl, bmask) & m);
      const uint32_t off = SEG1 ? v[q] : (v[q] & bmask);
      // claim3: hot rows are decided already; blind3: the other rows claim without a probe
      probe[q] = need[q] && !(claim3 && (blind3 || off < hw * 32u));
    }
    ld_cg_u32_p(probe[q], (P1 ? vold : vis) + (v[q] >> 5), wx[q]);
  }
#pragma unroll
  for (int q = 0; q < WV; ++q) {
    const uint32_t m = 1u << (v[q] & 31);
    const bool cand = need[q] && !(probe[q] && (wx[q] & m));  // not visited (Alg.3 lines 5-6)
    if (P1 && cand) atomicMin(pmin + v[q], ug[q]);  // parent claim: minimum original id (R1)
    if (!claim3) red_or_if(cand, vis + (v[q] >> 5), m);  // Alg.3 line 7
  }
}

// Long-column tiles of a P2 level, software-pipelined (the hot loop of the peak level).  A warp
// walks its tiles q = 0, 1, ... (tile id t0 + q*stride) through NS register slots.  Phase q: the
// `row` loads of tile q+AHEAD (into a slot already tested and RED'ed), the record of tile
// q+AHEAD+NS, then the visited tests of tile q -- hot copy in shared memory, else one L2 probe of
// the visited word -- and the RED.ORs of tile q (Alg.3 lines 4-7).  So every tile's rows have AHEAD phases to arrive from
// HBM and no phase waits for a record.  Slots are compile-time indices of a loop unrolled NS times
// (no register moves between slots: a moved register waits for its load).  A row id of 0xFFFFFFFF
// marks a lane past the tile's end (partial last tile of a column, or past the warp's last tile).
// The probe keeps one register per row (probe_lean: the loaded word, 0xFFFFFFFF when no RED is
// due; the RED recomputes bit and address from the row id).  Not inlined: its registers are
// allocated apart from the rest of k_expand (inlined, the short-tile state live across it made
// both spill).
// Measured at s26, peak level (tools/ab_expand.py, same box, two runs each): the round-1
// double-buffered loop 3.19 ms; this loop with NS = 2 / 3 / 4 (AHEAD = NS-1) and a probe keeping
// the need flag, mask and address (5 registers per row): 3.20 / 3.08 / 4.24 ms (NS = 4 spills);
// the REDs deferred (NS = 2): 3.34 ms; a warp-uniform full-tile branch without per-lane bounds:
// 3.46 ms.  Later (profiles/r02_long_lean_ab.log): the lean probe at NS = 3 / 4 / 5 (AHEAD =
// NS-1): 2.78 → 2.69 / 2.69 / 2.83 ms per peak level; the REDs of tile q deferred behind tile
// q+1's probes (one more slot of rows and probed words) spill at NS = 4 and 5 (not measured).
// Register-lean probe / RED for the pipelined loops (no room for a need flag, mask and address
// per row next to their pipeline state): the probe leaves x = 0xFFFFFFFF when no RED is due (hot and
// visited, or no row), else the loaded visited word; the RED recomputes the bit and the word
// address from v.  Two live registers per row instead of five.
template <bool SEG1>
__device__ __forceinline__ uint32_t probe_lean(uint32_t v, uint32_t hw, uint32_t sa, const uint32_t* vis, int bl,
                                               uint32_t bmask) {
  uint32_t x;
  if (SEG1) {
    asm("{\n"
        " .reg .pred pok, pn;\n"
        " .reg .b32 wi, hi, hv, m;\n"
        " .reg .b64 a;\n"
        " setp.ne.u32 pok, %1, 0xFFFFFFFF;\n"
        " shr.b32 wi, %1, 5;\n"
        " min.u32 hi, wi, %2;\n"
        " shl.b32 hi, hi, 2;\n"
        " add.u32 hi, hi, %3;\n"
        " ld.shared.u32 hv, [hi];\n"
        " shf.l.wrap.b32 m, 0, 1, %1;\n"
        " and.b32 hv, hv, m;\n"
        " setp.eq.and.b32 pn, hv, 0, pok;\n"
        " mov.b32 %0, 0xFFFFFFFF;\n"
        " mad.wide.u32 a, wi, 4, %4;\n"
        " @pn ld.global.cg.u32 %0, [a];\n"
        "}"
        : "=r"(x)
        : "r"(v), "r"(hw), "r"(sa), "l"(vis));
  } else {
    asm("{\n"
        " .reg .pred pok, pn;\n"
        " .reg .b32 wi, hi, hv, m, sg, off;\n"
        " .reg .b64 a;\n"
        " setp.ne.u32 pok, %1, 0xFFFFFFFF;\n"
        " shr.b32 wi, %1, 5;\n"
        " shr.b32 sg, %1, %5;\n"
        " and.b32 off, %1, %6;\n"
        " shr.b32 off, off, 5;\n"
        " min.u32 off, off, %2;\n"
        " add.u32 hv, %2, 1;\n"
        " mad.lo.u32 hi, sg, hv, off;\n"
        " selp.u32 hi, hi, %2, pok;\n"
        " shl.b32 hi, hi, 2;\n"
        " add.u32 hi, hi, %3;\n"
        " ld.shared.u32 hv, [hi];\n"
        " shf.l.wrap.b32 m, 0, 1, %1;\n"
        " and.b32 hv, hv, m;\n"
        " setp.eq.and.b32 pn, hv, 0, pok;\n"
        " mov.b32 %0, 0xFFFFFFFF;\n"
        " mad.wide.u32 a, wi, 4, %4;\n"
        " @pn ld.global.cg.u32 %0, [a];\n"
        "}"
        : "=r"(x)
        : "r"(v), "r"(hw), "r"(sa), "l"(vis), "r"(bl), "r"(bmask));
  }
  return x;
}
__device__ __forceinline__ void red_lean(uint32_t x, uint32_t v, uint32_t* vis) {
  asm volatile("{\n"
               " .reg .pred pr;\n"
               " .reg .b32 m, t, wi;\n"
               " .reg .b64 a;\n"
               " shf.l.wrap.b32 m, 0, 1, %1;\n"
               " and.b32 t, %0, m;\n"
               " setp.eq.b32 pr, t, 0;\n"
               " shr.b32 wi, %1, 5;\n"
               " mad.wide.u32 a, wi, 4, %2;\n"
               " @pr red.relaxed.gpu.global.or.b32 [a], m;\n"
               "}" ::"r"(x), "r"(v), "l"(vis));
}

template <int E, bool SEG1, bool POS32, int NS, int AHEAD>
__device__ __noinline__ void long_tiles_p2(const uint32_t* __restrict__ row, const uint4* __restrict__ tileA,
                                           uint32_t nA, uint32_t t0, uint32_t stride, uint32_t* vis, uint32_t hw,
                                           uint32_t sa, int bl, uint32_t bmask, int lane, const LevelInfo* info) {
  static_assert(AHEAD >= 1 && AHEAD <= NS - 1, "row slots: AHEAD tiles in flight + the tested one");
  typedef typename std::conditional<POS32, uint32_t, ull>::type Pos;
  uint32_t v[NS][E];  // row ids of the tiles in flight; 0xFFFFFFFF past a tile's end
  uint32_t x[NS][E];  // probed visited words (probe_lean; 0xFFFFFFFF: no RED due)
  Pos rpos[NS];       // prefetched records: position, length (0 past the warp's last tile)
  uint32_t rlen[NS];
  auto rec_load = [&](int slot, uint32_t t) {
    rlen[slot] = 0u;
    rpos[slot] = 0;
    if (t < nA) {
      if (POS32) {  // compact records (k_scan_emit: narrow, P2, E <= 8)
        const uint2 r = reinterpret_cast<const uint2*>(tileA)[t];
        BCHECK((ull)r.x + r.y <= info->cap_nnz && r.y <= 32u * E);
        rpos[slot] = (Pos)r.x;
        rlen[slot] = r.y;
      } else {
        const uint4 r = tileA[t];
        BCHECK(((ull)r.x | ((ull)r.y << 32)) + r.z <= info->cap_nnz && r.z <= 32u * E);
        rpos[slot] = (Pos)((ull)r.x | ((ull)r.y << 32));
        rlen[slot] = r.z;
      }
    }
  };
  auto rows_issue = [&](int slot) {  // from the record in the same slot
    const uint32_t* rp = row + rpos[slot] + lane;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      v[slot][e] = 0xFFFFFFFFu;
      ld_stream_u32_if(32u * e + lane < rlen[slot], rp + 32 * e, v[slot][e]);  // Alg.3 line 4
    }
  };
  auto reds = [&](int slot) {  // Alg.3 line 7
#pragma unroll
    for (int e = 0; e < E; ++e) red_lean(x[slot][e], v[slot][e], vis);
  };
  // prologue: rows of tiles 0 .. AHEAD-1 issued; records of tiles AHEAD .. AHEAD+NS-1 prefetched
  // (the warp's tile q is t0 + q*stride; tile ids and counts fit in 32 bits: tileA holds < 2^32)
#pragma unroll
  for (int k = 0; k < AHEAD; ++k) {
    rec_load(k, t0 + (uint32_t)k * stride);
    rows_issue(k);
  }
#pragma unroll
  for (int k = AHEAD; k < NS; ++k) rec_load(k, t0 + (uint32_t)k * stride);
#pragma unroll
  for (int k = 0; k < AHEAD; ++k) rec_load(k, t0 + (uint32_t)(NS + k) * stride);
  const uint32_t ahead = (uint32_t)(AHEAD + NS) * stride;
  // The exit test breaks out of the loop instead of returning from inside it: a RET waits for
  // every load in flight (the caller may read any register), so a predicated RET at the top of
  // each phase made every phase wait for the rows and records prefetched for the next ones.
  for (uint32_t t = t0; t < nA;) {
#pragma unroll
    for (int p = 0; p < NS; ++p) {
      if (t >= nA) break;  // warp-uniform
      const int sr = (p + AHEAD) % NS;  // slot of tile q+AHEAD (its record is loaded)
      rows_issue(sr);
      rec_load(sr, t + ahead);  // overflow past 2^32 cannot reach back below nA: nA + ahead < 2^32
#pragma unroll
      for (int e = 0; e < E; ++e) {  // Alg.3 lines 5-6
        BCHECK(v[p][e] == 0xFFFFFFFFu || v[p][e] < info->cap_nrows);
        x[p][e] = probe_lean<SEG1>(v[p][e], hw, sa, vis, bl, bmask);
      }
      reds(p);
      t += stride;
    }
  }
}

// Edge -> column mapping of one 32-edge window of a short tile, in registers (the paper's
// binary search of the scan, P:455-470 / Alg.3 line 2).  Lane l holds CS of the tile's columns,
// l + 32c: beg = the column's first edge relative to the tile (0 for a column begun in an
// earlier tile; TILE for lanes past the tile's last column) and base = its row offset minus its
// scan value (row position of short edge g of the column = base + g, modular when Pos is 32-bit).
// Columns have distinct starts (a short column has degree >= 1), so edge lo + lane belongs to
// column k = #(columns starting before the window) + #(columns starting in the window at or
// before the edge) - 1: one ballot and one OR-reduction of start bits per column set, a popcount,
// then a shuffle of base from the lane holding column k.
template <int CS, typename Pos>
__device__ __forceinline__ Pos short_map(const uint32_t (&beg)[CS], const Pos (&base)[CS], uint32_t lo, int lane) {
  uint32_t sb = 0, before = 0;
#pragma unroll
  for (int c = 0; c < CS; ++c) {
    const uint32_t r = beg[c] - lo;  // in the window when r < 32 (unsigned)
    sb |= __reduce_or_sync(0xFFFFFFFFu, r < 32u ? 1u << r : 0u);
    before += __popc(__ballot_sync(0xFFFFFFFFu, beg[c] < lo));
  }
  const uint32_t k = before + __popc(sb & (0xFFFFFFFFu >> (31 - lane))) - 1u;
  Pos b = __shfl_sync(0xFFFFFFFFu, base[0], (int)(k & 31u));
#pragma unroll
  for (int c = 1; c < CS; ++c) {
    const Pos bc = __shfl_sync(0xFFFFFFFFu, base[c], (int)(k & 31u));
    b = (k >> 5) == (uint32_t)c ? bc : b;
  }
  return b;
}

// One short tile of more than 32 columns (runs of degree-1..3 columns) of a P2 level: its table
// entries, columns (E sets per lane, short_map) and rows loaded in one go, then the visited tests
// and RED.ORs.  Not inlined: its column registers would otherwise be allocated on top of the whole
// pipeline state of short_tiles_p2 (which then spilled the row slots).
template <int E, bool SEG1, bool POS32>
__device__ __noinline__ void short_wide_tile(const uint32_t* __restrict__ row, const uint32_t* __restrict__ tile_k,
                                             const void* __restrict__ rowoff_v, const void* __restrict__ cumul_v,
                                             uint32_t n, ull total, uint32_t ntiles, uint32_t t, uint32_t* vis,
                                             uint32_t hw, uint32_t sa, int bl, uint32_t bmask, int lane,
                                             const LevelInfo* info) {
  typedef typename std::conditional<POS32, uint32_t, ull>::type Pos;
  constexpr int TILE = 32 * E;
  const Pos* __restrict__ rowoff = static_cast<const Pos*>(rowoff_v);
  const Pos* __restrict__ cumul = static_cast<const Pos*>(cumul_v);
  const uint32_t klo = tile_k[t];
  const uint32_t cnt = (t + 1 < ntiles ? tile_k[t + 1] : n - 1) - klo + 1u;
  BCHECK(cnt > 32u && cnt <= (uint32_t)TILE + 1 && klo + cnt <= n);
  const Pos tb = (Pos)t * TILE;
  uint32_t beg[E];
  Pos base[E];
#pragma unroll
  for (int c = 0; c < E; ++c) {
    const uint32_t idx = 32u * c + lane;
    Pos rc = ~(Pos)0, ro = 0;
    if (idx < cnt) {
      rc = cumul[klo + idx];
      ro = rowoff[klo + idx];
    }
    beg[c] = rc > tb ? (uint32_t)min(rc - tb, (Pos)TILE) : 0u;
    base[c] = (Pos)(ro - rc);
  }
  uint32_t vv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const Pos g = tb + 32u * e + lane;
    const Pos b = short_map<E, Pos>(beg, base, 32u * e, lane);
    vv[e] = 0xFFFFFFFFu;
    ld_stream_u32_if(g < (Pos)total, row + (Pos)(b + g), vv[e]);  // Alg.3 line 4
  }
  uint32_t x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {  // Alg.3 lines 5-6
    BCHECK(vv[e] == 0xFFFFFFFFu || vv[e] < info->cap_nrows);
    x[e] = probe_lean<SEG1>(vv[e], hw, sa, vis, bl, bmask);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) red_lean(x[e], vv[e], vis);  // Alg.3 line 7
}

// Short-column tiles of a P2 level, software-pipelined like long_tiles_p2.  Warp tile q (tile id
// t0 + q*stride) covers short edges [32E*tile, 32E*tile + 32E) of the level's scan; its columns
// are klo .. khi of the short list (tile_k), cnt <= 32E of them.  Tiles of cnt <= 32 columns (the
// bulk of the edges: short columns average more than 4 edges) keep one column per lane and run
// four stages one phase apart -- phase q: the tile-table entries of tile q+3, the column loads
// (scan value, row offset) of tile q+2, the mapping (short_map) and row loads of tile q+1, the
// visited tests and RED.ORs of tile q (Alg.3 lines 4-7) -- so no load is waited on in the phase
// that issues it.  Slots are compile-time indices of a loop unrolled four times.  A tile of more
// than 32 columns (runs of degree-1..3 columns) is loaded, mapped (all E column sets per lane)
// and tested in its own phase, outside the pipeline.
template <int E, bool SEG1, bool POS32>
__device__ __noinline__ void short_tiles_p2(const uint32_t* __restrict__ row, const uint32_t* __restrict__ tile_k,
                                            const void* __restrict__ rowoff_v, const void* __restrict__ cumul_v,
                                            uint32_t n, ull total, uint32_t ntiles, uint32_t t0, uint32_t stride,
                                            uint32_t* vis, uint32_t hw, uint32_t sa, int bl, uint32_t bmask, int lane,
                                            const LevelInfo* info) {
  typedef typename std::conditional<POS32, uint32_t, ull>::type Pos;  // also edge counts (total < 2^32 when POS32)
  constexpr int TILE = 32 * E;
  constexpr int NS = 4;
  constexpr uint32_t kWide = 0xFFFFFFFEu;  // v[s][0] of a tile of > 32 columns (never a row id: rows < 2^32 - 1)
  const Pos* __restrict__ rowoff = static_cast<const Pos*>(rowoff_v);
  const Pos* __restrict__ cumul = static_cast<const Pos*>(cumul_v);
  const Pos tot = (Pos)total;
  uint32_t mklo[NS], mcnt[NS];  // table entries: first column, column count (0 past the warp's last tile)
  Pos crc[NS], cro[NS];         // the lane's column: scan value, row offset (raw loads)
  uint32_t v[NS][E];            // row ids; 0xFFFFFFFF past the tile's end; kWide: a tile of > 32 columns
  auto meta_load = [&](int s, uint32_t t) {
    mcnt[s] = 0u;
    mklo[s] = 0u;
    if (t < ntiles) {
      const uint32_t klo = tile_k[t];
      const uint32_t khi = t + 1 < ntiles ? tile_k[t + 1] : n - 1;
      BCHECK(klo <= khi && khi < n && khi - klo < (uint32_t)TILE + 1);
      mklo[s] = klo;
      mcnt[s] = khi - klo + 1u;
    }
  };
  auto cols_load = [&](int s) {
    crc[s] = ~(Pos)0;  // no column: beg clamps to TILE
    cro[s] = 0;
    if (mcnt[s] <= 32u && (uint32_t)lane < mcnt[s]) {
      crc[s] = cumul[mklo[s] + lane];
      cro[s] = rowoff[mklo[s] + lane];
    }
  };
  auto tile_beg = [&](Pos c, Pos tb) -> uint32_t {  // column start relative to the tile, clamped to [0, TILE]
    return c > tb ? (uint32_t)min(c - tb, (Pos)TILE) : 0u;
  };
  auto rows_issue = [&](int s, uint32_t t) {
#pragma unroll
    for (int e = 0; e < E; ++e) v[s][e] = 0xFFFFFFFFu;
    if (mcnt[s] > 32u) v[s][0] = kWide;
    if (mcnt[s] == 0u || mcnt[s] > 32u) return;  // warp-uniform
    const Pos tb = (Pos)t * TILE;
    const uint32_t beg[1] = {tile_beg(crc[s], tb)};
    const Pos base[1] = {(Pos)(cro[s] - crc[s])};
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const Pos g = tb + 32u * e + lane;
      const Pos b = short_map<1, Pos>(beg, base, 32u * e, lane);
      ld_stream_u32_if(g < tot, row + (Pos)(b + g), v[s][e]);  // Alg.3 line 4
    }
  };
  auto test_red = [&](const uint32_t (&vv)[E]) {
    uint32_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {  // Alg.3 lines 5-6
      BCHECK(vv[e] == 0xFFFFFFFFu || vv[e] < info->cap_nrows);
      x[e] = probe_lean<SEG1>(vv[e], hw, sa, vis, bl, bmask);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) red_lean(x[e], vv[e], vis);  // Alg.3 line 7
  };
  // prologue: tables of tiles 0..2, columns of tiles 0..1, rows of tile 0
  meta_load(0, t0);
  meta_load(1, t0 + stride);
  meta_load(2, t0 + 2 * stride);
  cols_load(0);
  cols_load(1);
  rows_issue(0, t0);
  // (leaving by break as in long_tiles_p2 costs this loop registers: 32-64 B of spills, slower)
  for (uint32_t t = t0;;) {
#pragma unroll
    for (int p = 0; p < NS; ++p) {
      if (t >= ntiles) return;  // warp-uniform
      meta_load((p + 3) % NS, t + 3 * stride);  // ntiles + 3*stride < 2^32 (checked by the caller)
      cols_load((p + 2) % NS);
      rows_issue((p + 1) % NS, t + stride);
      if (v[p][0] == kWide)  // warp-uniform
        short_wide_tile<E, SEG1, POS32>(row, tile_k, rowoff_v, cumul_v, n, total, ntiles, t, vis, hw, sa, bl, bmask,
                                        lane, info);
      else test_red(v[p]);
      t += stride;
    }
  }
}


template <int E, int THREADS, bool P1, bool SEG1, bool POS32>
__device__ __forceinline__ void expand_body(const uint32_t* __restrict__ row, const uint32_t* __restrict__ flist,
                                            const void* __restrict__ rowoff_v, const void* __restrict__ cumul_v,
                                            const uint32_t* __restrict__ tile_k, const uint4* __restrict__ tileA,
                                            ull nA, ull n, ull total, ull all_edges, uint32_t* vis,
                                            const uint32_t* __restrict__ vold, uint32_t* pmin,
                                            const uint32_t* __restrict__ inv_col, uint32_t hot_words, int C,
                                            uint64_t W, int blog, uint32_t region_words, bool claim3,
                                            bool blind3, const LevelInfo* info) {
  constexpr int TILE = 32 * E;
  BCHECK(nA <= info->cap_tiles && total <= info->cap_nnz && n <= info->cap_ncols);
  constexpr int WARPS = THREADS / 32;
  constexpr int SLOT = TILE + 2;
  constexpr int WV = E < 4 ? E : 4;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // staged row positions: 32-bit when every CSC position fits (nnz < 2^32; modular arithmetic
  // below stays exact), which leaves more of the SM's unified L1/shared memory to L1
  typedef typename std::conditional<POS32, uint32_t, ull>::type Pos;
  // K3's row offsets and degree scan are 32-bit in the same case (k_scan_emit<NARROW>)
  const Pos* __restrict__ rowoff = static_cast<const Pos*>(rowoff_v);
  const Pos* __restrict__ cumul = static_cast<const Pos*>(cumul_v);
  unsigned char* wchunk = smem + (size_t)wid * expand_warp_bytes<E>(POS32);
  Pos* s_off = reinterpret_cast<Pos*>(wchunk);
  uint32_t* s_beg = reinterpret_cast<uint32_t*>(s_off + SLOT);
  // the region after the staging holds either the parents' ids (P1) or the hot visited bits
  uint32_t* s_region = reinterpret_cast<uint32_t*>(smem + expand_stage_bytes<E, THREADS>(POS32));
  // P1: the per-warp parents' ids sit at the end of the region, the hot copy (P2, mode 3) at its start
  uint32_t* s_u = s_region + (region_words - WARPS * SLOT) + wid * SLOT;
  const uint32_t* s_hot = s_region;
  uint32_t hw = 0;
  if (!P1 && all_edges >= kHotMinEdges && blog >= 0) hw = hot_words;
  if (P1 && claim3 && blog >= 0) {  // mode 3: the hot copy shares the region with s_u
    const uint32_t room = (region_words - WARPS * SLOT) / (uint32_t)C;
    hw = room > 1 ? min(hot_words, room - 1) : 0u;
  }
  if (!P1 || claim3) {  // hot prefix of every row segment + its zero sentinel (hw = 0: sentinels only)
    const uint32_t hs = hw + 1;
    for (uint32_t k = threadIdx.x; k < (uint32_t)C * hs; k += THREADS) {
      const uint32_t m = k / hs, w = k - m * hs;
      s_region[k] = w < hw ? vold[(uint64_t)m * W + w] : 0u;  // level-start visited bits
    }
  }
  __syncthreads();
  // 32-bit shared address of the hot copy, opaque to the compiler so it stays in a register
  uint32_t sa = (uint32_t)__cvta_generic_to_shared(s_hot);
  asm volatile("" : "+r"(sa));
  const uint32_t bmask = (blog >= 0) ? ((1u << blog) - 1u) : 0u;
  const ull stride = (ull)gridDim.x * WARPS;
  // ---- long columns: column-aligned tiles, positions pos + e, no mapping work
  const int bl = blog >= 0 ? blog : 31;  // blog < 0 (no hot copy): every row maps to sentinel 0
  {
    constexpr int LWV = E <= 8 ? E : 8;  // all loads of a wave in flight together
    // Double-buffered: the next tile's row loads are issued before this tile's visited tests,
    // so each warp keeps two tiles of row data in flight (the level streams `row` from HBM).
    static_assert(E <= 16, "E");
    constexpr int LE = E;
    auto load_rows = [&](const uint4& r, bool valid, uint32_t (&v)[LE]) {
      const uint32_t* rp = row + ((ull)r.x | ((ull)r.y << 32)) + lane;
      const uint32_t len = valid ? r.z : 0u;
#pragma unroll
      for (int q = 0; q < LE; ++q) {
        if (P1) {  // P1 tests validity by the id; P2 by the position
          v[q] = 0xFFFFFFFFu;
          ld_stream_u32_if(32u * q + lane < len, rp + 32 * q, v[q]);  // Alg.3 line 4
        } else {
          ld_stream_u32_p(32u * q + lane < len, rp + 32 * q, v[q]);
        }
      }
    };
    auto process = [&](const uint4& r, const uint32_t (&v)[LE], uint32_t ug0) {
#pragma unroll
      for (int wv = 0; wv < E / LWV; ++wv) {
        uint32_t vw[LWV];
#pragma unroll
        for (int q = 0; q < LWV; ++q) vw[q] = v[LWV * wv + q];
        if (P1) {
          uint32_t ug[LWV];
#pragma unroll
          for (int q = 0; q < LWV; ++q) ug[q] = ug0;
          expand_edges<LWV, true, SEG1>(vw, ug, vis, vold, pmin, s_hot, bmask, bl, hw, claim3, blind3);
        } else {
          Probe pr[LWV];
#pragma unroll
          for (int q = 0; q < LWV; ++q) {  // Alg.3 lines 5-6
            if (SEG1) probe_seg1(pr[q], vw[q], 32u * (LWV * wv + q) + lane, r.z, hw, sa, vis);
            else probe_segs(pr[q], vw[q], 32u * (LWV * wv + q) + lane, r.z, hw, sa, vis, bl, bmask);
          }
#pragma unroll
          for (int q = 0; q < LWV; ++q) probe_red(pr[q]);
        }
      }
    };
    ull t = (ull)blockIdx.x * WARPS + wid;
    if constexpr (!P1 && BFS200_K1PIPE > 0 && E <= 8) {
      constexpr int NS = SEG1 ? BFS200_K1PIPE : BFS200_K1PIPE_SEGS;
      long_tiles_p2<E, SEG1, POS32, NS, NS - 1>(
          row, tileA, (uint32_t)nA, (uint32_t)t, (uint32_t)stride, vis, hw, sa, bl, bmask, lane, info);
    } else {
    uint4 rec = t < nA ? tileA[t] : make_uint4(0, 0, 0, 0);
    ull t1 = t + stride;
    uint4 rec1 = t1 < nA ? tileA[t1] : make_uint4(0, 0, 0, 0);
    // P1: the parent's original id of the tile's column (prefetched with the rows)
    auto col_id = [&](const uint4& r, bool valid) -> uint32_t { return (P1 && valid) ? inv_col[r.w] : 0u; };
    if (E <= 8) {
      uint32_t v[LE];
      load_rows(rec, t < nA, v);
      uint32_t ug = col_id(rec, t < nA);
      while (t < nA) {
        const ull t2 = t1 + stride;
        const uint4 rec2 = t2 < nA ? tileA[t2] : make_uint4(0, 0, 0, 0);
        uint32_t vn[LE];
        load_rows(rec1, t1 < nA, vn);
        const uint32_t ugn = col_id(rec1, t1 < nA);
        process(rec, v, ug);
#pragma unroll
        for (int q = 0; q < LE; ++q) v[q] = vn[q];
        ug = ugn;
        rec = rec1;
        rec1 = rec2;
        t = t1;
        t1 = t2;
      }
    } else {
      while (t < nA) {
        uint32_t v[LE];
        load_rows(rec, true, v);
        process(rec, v, col_id(rec, true));
        rec = rec1;
        t = t1;
        t1 = t + stride;
        rec1 = t1 < nA ? tileA[t1] : make_uint4(0, 0, 0, 0);
      }
    }
    }
  }
  // ---- short columns: tiles of TILE consecutive short edges, scan + binary-search mapping
  const ull ntiles = (total + TILE - 1) / TILE;
  if constexpr (!P1 && BFS200_K1PIPE > 0 && BFS200_SHORTPIPE && E <= 4) {  // E = 8 would spill
    if (ntiles + 4 * stride < (1ull << 32)) {  // tile ids stay 32-bit
      short_tiles_p2<E, SEG1, POS32>(row, tile_k, rowoff_v, cumul_v, (uint32_t)n, total, (uint32_t)ntiles,
                                     (uint32_t)((ull)blockIdx.x * WARPS + wid), (uint32_t)stride, vis, hw, sa, bl,
                                     bmask, lane, info);
      return;
    }
  }
  // software pipeline: the tile-table entries and the first 32 staged columns of the NEXT tile
  // are loaded while the current tile's row loads and visited tests are in flight.
  ull tile = (ull)blockIdx.x * WARPS + wid;
  uint32_t klo = 0, khi = 0;
  ull rc = 0, ro = 0;
  uint32_t ru = 0;
  if (tile < ntiles) {
    klo = tile_k[tile];
    khi = (tile + 1 < ntiles) ? tile_k[tile + 1] : (uint32_t)(n - 1);
    if (lane <= khi - klo) {
      rc = cumul[klo + lane];
      ro = rowoff[klo + lane];
      if (P1) ru = inv_col[flist[klo + lane]];
    }
  }
  while (tile < ntiles) {
    const ull t0 = tile * TILE;
    BCHECK(klo <= khi && khi < n);
    const uint32_t len = (uint32_t)min((ull)TILE, total - t0);
    const uint32_t cnt = khi - klo + 1;
    // stage this tile's columns
    if (lane < cnt) {
      const uint32_t beg = rc > t0 ? (uint32_t)(rc - t0) : 0u;
      s_beg[lane] = beg;
      s_off[lane] = (Pos)(ro + (t0 + beg - rc));
      if (P1) s_u[lane] = ru;
    }
    for (uint32_t idx = 32 + lane; idx < cnt; idx += 32) {  // tiles of many short columns
      const ull c = cumul[klo + idx];
      const uint32_t beg = c > t0 ? (uint32_t)(c - t0) : 0u;
      s_beg[idx] = beg;
      s_off[idx] = (Pos)(rowoff[klo + idx] + (t0 + beg - c));
      if (P1) s_u[idx] = inv_col[flist[klo + idx]];
    }
    if (lane == 0) s_beg[cnt] = 0xFFFFFFFFu;
    __syncwarp();
    // next tile's table entries (in flight during this tile)
    const ull next = tile + stride;
    uint32_t nklo = 0, nkhi = 0;
    if (next < ntiles) {
      nklo = tile_k[next];
      nkhi = (next + 1 < ntiles) ? tile_k[next + 1] : (uint32_t)(n - 1);
    }
    bool rnext = false;
    auto prefetch_next = [&]() {  // next tile's first 32 staged columns
      if (next < ntiles && lane <= nkhi - nklo) {
        rc = cumul[nklo + lane];
        ro = rowoff[nklo + lane];
        if (P1) ru = inv_col[flist[nklo + lane]];
        rnext = true;
      }
    };
    if (!P1 && cnt == 1 && len == TILE) {
      // lean path (the bulk of a dense level): a full tile inside one column, positions base + e,
      // every lane valid; branch-free visited test, predicated probe and RED.
      const uint32_t* rp = row + s_off[0] + lane;
      constexpr int LWV = E <= 8 ? E : 8;  // all loads of the wave in flight together
#pragma unroll
      for (int wv = 0; wv < E / LWV; ++wv) {
        uint32_t v[LWV];
#pragma unroll
        for (int q = 0; q < LWV; ++q) v[q] = ld_stream_u32(rp + 32 * (LWV * wv + q));  // Alg.3 line 4
        if (wv == 0) prefetch_next();
        Probe pr[LWV];
#pragma unroll
        for (int q = 0; q < LWV; ++q) {  // Alg.3 lines 5-6
          if (SEG1) probe_seg1(pr[q], v[q], 0u, 1u, hw, sa, vis);
          else probe_segs(pr[q], v[q], 0u, 1u, hw, sa, vis, bl, bmask);
        }
#pragma unroll
        for (int q = 0; q < LWV; ++q) probe_red(pr[q]);
      }
    } else if (cnt == 1) {
      // the whole tile lies in one column: positions are base + e, no mapping work
      const Pos base = s_off[0];
      const uint32_t u0 = P1 ? s_u[0] : 0u;
#pragma unroll
      for (int wv = 0; wv < E / WV; ++wv) {
        uint32_t v[WV], ug[WV];
#pragma unroll
        for (int q = 0; q < WV; ++q) {
          const uint32_t e = 32u * (WV * wv + q) + lane;
          v[q] = 0xFFFFFFFFu;
          ld_stream_u32_if(e < len, row + (Pos)(base + e), v[q]);  // Alg.3 line 4
          ug[q] = u0;
        }
        if (wv == 0) prefetch_next();
        expand_edges<WV, P1, SEG1>(v, ug, vis, vold, pmin, s_hot, bmask, bl, hw, claim3, blind3);
      }
    } else {
      // lane-interleaved edges e = 32q + lane; lane state: the staged column idx holding its
      // current edge, that column's end within the tile and base = row position of tile edge 0
      uint32_t idx = 0;
      if (cnt > 2) {  // binsearch_maxle for the lane's first edge (Alg.3 line 2)
        uint32_t lo = 0, hi = cnt - 1;
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (s_beg[mid] <= (uint32_t)lane) lo = mid; else hi = mid - 1;
        }
        idx = lo;
      } else {
        idx = (uint32_t)lane >= s_beg[1] ? 1u : 0u;
      }
      uint32_t cur_end = s_beg[idx + 1];
      Pos base = s_off[idx] - s_beg[idx];
#pragma unroll
      for (int wv = 0; wv < E / WV; ++wv) {
        uint32_t v[WV], ug[WV];
#pragma unroll
        for (int q = 0; q < WV; ++q) {
          const uint32_t e = 32u * (WV * wv + q) + lane;
          const bool ok = e < len;
          {  // linear advance: one step branch-free, more steps (short columns) looped
            const bool adv = ok && e >= cur_end;
            idx += adv ? 1u : 0u;
            const uint32_t nb = s_beg[idx], ne = s_beg[idx + 1];
            const Pos no = s_off[idx];
            if (adv) {
              cur_end = ne;
              base = no - nb;
            }
          }
          if (__any_sync(0xFFFFFFFFu, ok && e >= cur_end)) {  // a lane crossed more than one column
            while (ok && e >= cur_end) {
              ++idx;
              cur_end = s_beg[idx + 1];
              base = s_off[idx] - s_beg[idx];
            }
          }
          v[q] = 0xFFFFFFFFu;
          ld_stream_u32_if(ok, row + (Pos)(base + e), v[q]);  // Alg.3 line 4 (modular when Pos is 32-bit)
          ug[q] = P1 ? s_u[idx] : 0u;
        }
        if (wv == 0) prefetch_next();
        expand_edges<WV, P1, SEG1>(v, ug, vis, vold, pmin, s_hot, bmask, bl, hw, claim3, blind3);
      }
    }
    if (!rnext) {
      rc = 0;
      ro = 0;
    }
    __syncwarp();  // all lanes done with this tile's staging
    tile = next;
    klo = nklo;
    khi = nkhi;
  }
}

template <int E, int THREADS, bool SEG1, bool POS32>
__global__ void __launch_bounds__(THREADS, 1) k_expand(const uint32_t* __restrict__ row,
                                                       const uint32_t* __restrict__ flist,
                                                       const void* __restrict__ rowoff,
                                                       const void* __restrict__ cumul,
                                                       const uint32_t* __restrict__ tile_k,
                                                       const uint4* __restrict__ tileA,
                                                       const LevelInfo* __restrict__ info, uint32_t* vis,
                                                       const uint32_t* __restrict__ vold,
                                                       uint32_t* pmin, const uint32_t* __restrict__ inv_col,
                                                       uint32_t hot_words, int C, uint64_t W, int blog,
                                                       uint32_t region_words) {
  const ull n = info->n, total = info->sedges, nA = info->nA, all_edges = info->edges;
  if (all_edges == 0) return;
  if (info->mode != 2)
    expand_body<E, THREADS, true, SEG1, POS32>(row, flist, rowoff, cumul, tile_k, tileA, nA, n, total, all_edges, vis,
                                               vold, pmin, inv_col, hot_words, C, W, blog, region_words, info->mode == 3,
                                               info->blind != 0, info);
  else
    expand_body<E, THREADS, false, SEG1, POS32>(row, flist, rowoff, cumul, tile_k, tileA, nA, n, total, all_edges,
                                                vis, vold, pmin, inv_col, hot_words, C, W, blog, region_words, false, false,
                                                info);
}

template <int E, int THREADS>
static cudaError_t launch_expand_t(const Geom& g, Rank& rk, uint64_t hot_h, bool force_pos64, cudaStream_t s) {
  constexpr int SLOT = 32 * E + 2;
  constexpr size_t WARPS = THREADS / 32;
  const bool pos32 = rk.nnz < (1ull << 32) && !force_pos64;  // every CSC position fits in 32 bits
  const size_t staging = expand_stage_bytes<E, THREADS>(pos32);
  const size_t s_u_bytes = WARPS * SLOT * 4;
  // hot visited words per row segment: the relabeled prefix, as far as shared memory allows
  int blog = -1;
  if (g.block && (g.block & (g.block - 1)) == 0) {
    blog = 0;
    while ((1ull << blog) < g.block) ++blog;
  }
  uint64_t hw = hot_h / 32;
  // The hot copy fills the shared memory up to kSmemTarget in all: a larger carve-out costs L1
  // capacity, which holds the in-flight row loads and probes (measured at s26, peak level:
  // 162 KB of shared memory 3.67 ms, 178 KB 4.28 ms, 210 KB 6.9 ms).
  const size_t hot_smem = kSmemTarget > staging + 16 + 64 ? kSmemTarget - staging - 16 - 64 : 4;
  const uint64_t budget = hot_smem < kSmemBudget - staging - 16 ? hot_smem : kSmemBudget - staging - 16;
  const uint64_t cap = budget / 4 / (uint64_t)g.C - 1;  // + one sentinel word per segment
  if (hw > cap) hw = cap;
  if (blog < 0) hw = 0;
  size_t region = (size_t)g.C * (hw + 1) * 4;
  // P1 levels keep s_u at the end of the region and (mode 3) at least the C sentinels before it
  if (region < s_u_bytes + (size_t)g.C * 4) region = s_u_bytes + (size_t)g.C * 4;
  const size_t smem = staging + region + 16;
  auto kern = g.C == 1 ? (pos32 ? k_expand<E, THREADS, true, true> : k_expand<E, THREADS, true, false>)
                       : (pos32 ? k_expand<E, THREADS, false, true> : k_expand<E, THREADS, false, false>);
  kern<<<g.nsm, THREADS, smem, s>>>(rk.row, rk.flist, rk.rowoff, rk.cumul, rk.tile_k, rk.tileA, rk.info, rk.vis, rk.vold,
                                        rk.pmin, rk.inv_col, (uint32_t)hw, g.C, g.words_block(), blog,
                                        (uint32_t)(region / 4));
  return cudaGetLastError();
}

uint32_t expand_tile_edges(int E) { return 32u * (uint32_t)E; }

template <int E, int THREADS>
static cudaError_t expand_attrs() {
  const int b = (int)kSmemBudget;
  cudaError_t e = cudaFuncSetAttribute(k_expand<E, THREADS, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_expand<E, THREADS, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_expand<E, THREADS, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_expand<E, THREADS, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
  return e;
}



cudaError_t launch_expand(const Geom& g, Rank& rk, int E, uint64_t hot_h, bool force_pos64, cudaStream_t s) {
  switch (E) {
    case 1: return launch_expand_t<1, 1024>(g, rk, hot_h, force_pos64, s);
    case 2: return launch_expand_t<2, 1024>(g, rk, hot_h, force_pos64, s);
    case 4: return launch_expand_t<4, 1024>(g, rk, hot_h, force_pos64, s);
    case 8: return launch_expand_t<8, 1024>(g, rk, hot_h, force_pos64, s);
    case 16: return launch_expand_t<16, 512>(g, rk, hot_h, force_pos64, s);
    default: return cudaErrorInvalidValue;
  }
}

// ------------------------------------------------------------------ K4: parent claim
// For every row discovered in this level (discovered words exclude visited rows):
//   P1 levels: pred[r] = pmin[r] (the atomicMin result of the expansion); pmin[r] = UINT32_MAX.
//   P2 levels: pred[r] = the minimum frontier column adjacent to r on this rank = the first
//     entry of its ascending CSR row set in the frontier bitmap being expanded (all_front).
//     Lanes scan their own rows 4 entries at a time for up to kShortScan entries; rows without a
//     hit by then are finished by the whole warp, 32 entries per step (ballot -> first lane).
// A warp takes 32 consecutive words and queues their rows in shared memory.  With C > 1 the
// discovered words are also packed contiguously as the fold message.
constexpr int kParentThreads = 1024;
constexpr int kShortScan = 32;
#ifndef BFS200_LANE_STEP
#define BFS200_LANE_STEP 4
#endif
constexpr int kLaneStep = BFS200_LANE_STEP;  // CSR entries per lane step (loads in flight together)
#ifndef BFS200_PAR_ROWS
#define BFS200_PAR_ROWS 2
#endif
constexpr int kParRows = BFS200_PAR_ROWS;  // P2 rows scanned together per lane
constexpr size_t kParentHotSmem = 64 * 1024;  // hot prefix of the frontier bitmap (P2 levels)

// Ptr: the CSR row offsets, the 32-bit copy when nnz < 2^32 (half the pointer bytes: every
// discovered row of a P2 level reads its pair)
template <typename Ptr>
__global__ void __launch_bounds__(kParentThreads, 1) k_parent(uint32_t* vis, const uint32_t* __restrict__ vold,
                                                               uint64_t nwords,
                                                               const Ptr* __restrict__ csr_ptr,
                                                               const uint32_t* __restrict__ csr_col,
                                                               const uint32_t* __restrict__ front, uint32_t* pred,
                                                               uint32_t* pmin, uint32_t* sendbuf,
                                                               const uint32_t* __restrict__ inv_col,
                                                               LevelInfo* info, uint32_t hot_words, int R,
                                                               uint64_t Wc, int blog,
                                                               uint32_t* const* __restrict__ fold_dst, int fused,
                                                               uint32_t* const* __restrict__ pred_dst, int jcol,
                                                               uint64_t block) {
  extern __shared__ __align__(16) unsigned char psmem[];
  uint32_t (*queue)[1024] = reinterpret_cast<uint32_t (*)[1024]>(psmem);
  uint32_t* s_hot = reinterpret_cast<uint32_t*>(psmem) + (kParentThreads / 32) * 1024;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool p1 = info->mode == 1, m3 = info->mode == 3, blind = m3 && info->blind;
  // parent candidate of local row r.  (Measured: the owned rows' candidates interleaved with
  // their levels, so k_finalize gathers one 8-byte record per vertex: finalize -0.03 ms but the
  // stride-2 writes of K4 and K2 +0.1 ms per BFS at s26 -- partial sectors; not kept.)
  // With the peer exchange (C > 1) the candidate of a row of another column block c goes
  // straight into the owner's answer slot for this column (pred_dst[c] = respin of P_ic +
  // jcol*block, indexed by the owned offset): the owner's finalize then reads the winner
  // column's candidate there, and no end-of-search request/answer round runs.  A stale candidate
  // (this column reaching the row at a later level than the winner) lands in a slot the owner
  // never reads: the winner is the lowest column that reached the row at its first level.
  auto put_pred = [&](uint64_t r, uint32_t val) {
    if (pred_dst) {
      const uint64_t c = blog >= 0 ? (r >> blog) : r / block;
      if ((int)c != jcol) {
        pred_dst[c][r - c * block] = val;
        return;
      }
    }
    pred[r] = val;
  };
  unsigned ndisc = 0;
  // P2: frontier bits of the hot (relabeled, highest-degree) column prefix of each of the R
  // column segments, so most frontier tests of the CSR scans stay in shared memory
  const uint32_t hw = (!p1 && !m3 && blog >= 0) ? hot_words : 0u;
  for (uint32_t k = threadIdx.x; k < (uint32_t)R * hw; k += kParentThreads) {
    const uint32_t m = k / hw, w = k - m * hw;
    s_hot[k] = front[(uint64_t)m * Wc + w];
  }
  __syncthreads();
  const uint32_t hot_bits = hw * 32, bmask = (blog >= 0) ? ((1u << blog) - 1u) : 0u;
  const int bl = blog > 0 ? blog : 0;
  auto in_front = [&](uint32_t u) -> bool {
    const uint32_t off = u & bmask;
    if (off < hot_bits) return (s_hot[(u >> bl) * hw + (off >> 5)] >> (off & 31)) & 1u;
    return (__ldg(front + (u >> 5)) >> (u & 31)) & 1u;
  };
  const uint64_t nchunks = (nwords + 31) / 32;
  const uint64_t cstride = (uint64_t)gridDim.x * (kParentThreads / 32);
  const uint64_t first = (uint64_t)blockIdx.x * (kParentThreads / 32) + wid;
  if (m3) {
    for (uint64_t ch = first; ch < nchunks; ch += cstride) {
      const uint64_t w = ch * 32 + lane;
      // mode 3: the rows claimed in pmin are the discovered ones; lane l handles row 32k + l of
      // the chunk's word k (coalesced), the ballot is word k's discovered bits
      uint32_t myd = 0;
      const int nk = (int)min((uint64_t)32, nwords - ch * 32);
      // visited words of the chunk (blind claims may have reached visited rows: not discovered)
      const uint32_t visw = (blind && w < nwords) ? vold[w] : 0u;
      // 16 rows' pmin loads in flight per lane (a streaming pass: bytes in flight set its speed)
#pragma unroll 1
      for (int k0 = 0; k0 < nk; k0 += 16) {
        uint32_t pm[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          pm[q] = (k0 + q < nk) ? pmin[(ch * 32 + k0 + q) * 32 + lane] : 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const int k = k0 + q;
          const uint64_t r = (ch * 32 + k) * 32 + lane;
          const uint32_t vk = __shfl_sync(0xFFFFFFFFu, visw, k);
          const bool c = pm[q] != 0xFFFFFFFFu;
          const bool f = c && !((vk >> lane) & 1u);
          const unsigned dd = __ballot_sync(0xFFFFFFFFu, f);
          if (f) put_pred(r, pm[q]);
          if (c) pmin[r] = 0xFFFFFFFFu;
          if (lane == k) myd = dd;
        }
      }
      if (w < nwords) {
        vis[w] = vold[w] | myd;  // mode 3 sets no bit in K1: the level's discoveries enter here
        if (sendbuf) sendbuf[w] = myd;
        if (fold_dst) {  // peer exchange: the fold message goes straight into the owner's recv
          const uint64_t c = w / Wc;
          if (fold_dst[c]) fold_dst[c][w - c * Wc] = myd;
        }
      }
      ndisc += __popc(myd);
    }
  } else {
    // P1 / P2: the chunk's rows discovered in this level (lane l: word ch*32 + l), their parents
    auto process_chunk = [&](uint64_t w, uint32_t d) {
      if (p1) {
        uint32_t b = d;
        while (b) {
          const int bit = __ffs(b) - 1;
          b &= b - 1;
          const uint64_t r = w * 32 + bit;
          put_pred(r, pmin[r]);
          pmin[r] = 0xFFFFFFFFu;
        }
        return;
      }
      // exclusive prefix of popcounts across lanes -> queue positions
      const unsigned c = __popc(d);
      unsigned inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned total = __shfl_sync(0xFFFFFFFFu, inc, 31);
      unsigned pos = inc - c;
      uint32_t b = d;
      while (b) {
        const int bit = __ffs(b) - 1;
        b &= b - 1;
        queue[wid][pos++] = (uint32_t)(w * 32 + bit);
      }
      __syncwarp();
      unsigned nlong = 0;  // lane-local count of deferred rows (written at slots lane, lane+32, ...)
      // kParRows rows per lane at a time: their dependent chains (row pointers -> first CSR entries
      // -> frontier tests -> inv_col) overlap, so more random loads are in flight per lane
      for (unsigned q0 = lane; q0 < total; q0 += 32 * kParRows) {
        uint32_t r[kParRows], best[kParRows];
        ull p[kParRows], stop[kParRows];
#pragma unroll
        for (int i = 0; i < kParRows; ++i) r[i] = (q0 + 32 * i < total) ? queue[wid][q0 + 32 * i] : 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < kParRows; ++i) {
          const bool v = r[i] != 0xFFFFFFFFu;
          const ull beg = v ? (ull)csr_ptr[r[i]] : 0ull, end = v ? (ull)csr_ptr[r[i] + 1] : 0ull;
          p[i] = beg;
          stop[i] = min(end, beg + kShortScan);
          best[i] = 0xFFFFFFFFu;
        }
        bool more = true;
        while (more) {  // every row still searching takes one lane step, all rows' loads together
          uint32_t u[kParRows][kLaneStep];
#pragma unroll
          for (int i = 0; i < kParRows; ++i) {
            const bool act = best[i] == 0xFFFFFFFFu && p[i] < stop[i];
#pragma unroll
            for (int k = 0; k < kLaneStep; ++k)
              u[i][k] = (act && p[i] + k < stop[i]) ? __ldg(csr_col + p[i] + k) : 0xFFFFFFFFu;
          }
          more = false;
#pragma unroll
          for (int i = 0; i < kParRows; ++i) {
            bool f[kLaneStep];
#pragma unroll
            for (int k = 0; k < kLaneStep; ++k) f[k] = (u[i][k] != 0xFFFFFFFFu) && in_front(u[i][k]);
#pragma unroll
            for (int k = kLaneStep - 1; k >= 0; --k)
              if (f[k]) best[i] = u[i][k];
            p[i] += kLaneStep;
            more |= best[i] == 0xFFFFFFFFu && p[i] < stop[i];
          }
        }
        uint32_t pv[kParRows];
#pragma unroll
        for (int i = 0; i < kParRows; ++i)
          pv[i] = (r[i] != 0xFFFFFFFFu && best[i] != 0xFFFFFFFFu) ? inv_col[best[i]] : 0u;
#pragma unroll
        for (int i = 0; i < kParRows; ++i) {
          if (r[i] == 0xFFFFFFFFu) continue;
          BCHECK(r[i] < nwords * 32 && (best[i] == 0xFFFFFFFFu || best[i] < info->cap_ncols));
          if (best[i] != 0xFFFFFFFFu) {
            put_pred(r[i], pv[i]);
          } else {  // defer to the whole warp; slot lane+32*nlong <= q0+32i was already read
            queue[wid][lane + 32 * nlong] = r[i];
            ++nlong;
          }
        }
      }
      __syncwarp();
      // cooperative scan of the deferred rows: lane l's k-th row sits at slot l + 32k
      unsigned maxlong = nlong;
#pragma unroll
      for (int o = 16; o; o >>= 1) maxlong = max(maxlong, __shfl_xor_sync(0xFFFFFFFFu, maxlong, o));
      for (unsigned k = 0; k < maxlong; ++k) {
        unsigned has = __ballot_sync(0xFFFFFFFFu, k < nlong);
        while (has) {
          const int src = __ffs(has) - 1;
          has &= has - 1;
          const uint32_t r = queue[wid][src + 32 * k];
          const ull end = (ull)csr_ptr[r + 1];
          uint32_t best = 0xFFFFFFFFu;
          for (ull p = (ull)csr_ptr[r] + kShortScan; p < end; p += 32) {
            const uint32_t u = (p + lane < end) ? __ldg(csr_col + p + lane) : 0xFFFFFFFFu;
            const bool f = (u != 0xFFFFFFFFu) && in_front(u);
            const unsigned m = __ballot_sync(0xFFFFFFFFu, f);
            if (m) {
              best = __shfl_sync(0xFFFFFFFFu, u, __ffs(m) - 1);
              break;
            }
          }
          BCHECK(best < info->cap_ncols);  // a discovered row has a frontier neighbour in its CSR row
          if (lane == 0) put_pred(r, inv_col[best]);
        }
      }
      __syncwarp();
    };
    // Chunks in groups of 32 per warp: pass 1 loads the discovered words of the group (8 chunks'
    // loads in flight), writes the fold message and marks the non-empty chunks; pass 2 runs the
    // parent claims of those only -- sparse levels end after pass 1's round trips.
    for (uint64_t g0 = first; g0 < nchunks; g0 += 32 * cstride) {
      unsigned mask = 0;
      for (int q0 = 0; q0 < 32; q0 += 8) {
        uint32_t dv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t ch = g0 + (uint64_t)(q0 + q) * cstride, w = ch * 32 + lane;
          dv[q] = (ch < nchunks && w < nwords) ? (vis[w] & ~vold[w]) : 0u;  // rows discovered in this level
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint64_t ch = g0 + (uint64_t)(q0 + q) * cstride, w = ch * 32 + lane;
          if (ch >= nchunks) break;  // warp-uniform
          const uint32_t d = dv[q];
          if (sendbuf && w < nwords) sendbuf[w] = d;
          if (fold_dst && w < nwords) {  // peer exchange (NVLink stores): segment c -> recv of P_ic
            const uint64_t c = w / Wc;
            if (fold_dst[c]) fold_dst[c][w - c * Wc] = d;
          }
          ndisc += __popc(d);
          if (__any_sync(0xFFFFFFFFu, d != 0)) mask |= 1u << (q0 + q);
        }
      }
      while (mask) {
        const int q = __ffs(mask) - 1;
        mask &= mask - 1;
        const uint64_t ch = g0 + (uint64_t)q * cstride, w = ch * 32 + lane;
        process_chunk(w, (w < nwords) ? (vis[w] & ~vold[w]) : 0u);
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ndisc += __shfl_xor_sync(0xFFFFFFFFu, ndisc, o);
  if (lane == 0 && ndisc) {
    atomicAdd(&info->disc_total, (ull)ndisc);
    if (fused) atomicAdd(&info->newv, (ull)ndisc);  // no K2 (1x1): the level's new vertices, counted here
  }
  if (fold_dst) {  // the CTA's peer stores, then one system-scope fence (cumulative) before the flag
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

cudaError_t launch_parent(const Geom& g, Rank& rk, bool fused, bool force_ptr64, cudaStream_t s) {
  const uint64_t nwords = g.nrows() / 32;
  const uint64_t nchunks = (nwords + 31) / 32;
  uint64_t grid = (nchunks + kParentThreads / 32 - 1) / (kParentThreads / 32);
  const uint64_t cap = (uint64_t)g.nsm;
  if (grid > cap) grid = cap;
  int blog = -1;
  if (g.block && (g.block & (g.block - 1)) == 0) {
    blog = 0;
    while ((1ull << blog) < g.block) ++blog;
  }
  uint64_t hw = kParentHotSmem / 4 / (uint64_t)g.R;
  if (hw > g.words_block()) hw = g.words_block();
  if (blog < 0) hw = 0;
  const size_t smem = (size_t)(kParentThreads / 32) * 1024 * 4 + (size_t)(g.R * hw > 4 ? g.R * hw : 4) * 4;
  // peer exchange: fold bitmaps and the parent candidates of other columns' rows as peer stores
  uint32_t* const* fold = g.C > 1 ? rk.fold_dst : nullptr;
  uint32_t* const* pdst = fold ? rk.respin_dst : nullptr;
  if (rk.csr_ptr32 && !force_ptr64)
    k_parent<uint32_t><<<(unsigned)grid, kParentThreads, smem, s>>>(
        rk.vis, rk.vold, nwords, rk.csr_ptr32, rk.csr_col, rk.all_front, rk.pred, rk.pmin,
        g.C > 1 ? rk.sendbuf : nullptr, rk.inv_col, rk.info, (uint32_t)hw, g.R, g.words_block(), blog, fold,
        fused ? 1 : 0, pdst, rk.j, g.block);
  else
    k_parent<ull><<<(unsigned)grid, kParentThreads, smem, s>>>(
        rk.vis, rk.vold, nwords, rk.csr_ptr, rk.csr_col, rk.all_front, rk.pred, rk.pmin,
        g.C > 1 ? rk.sendbuf : nullptr, rk.inv_col, rk.info, (uint32_t)hw, g.R, g.words_block(), blog, fold,
        fused ? 1 : 0, pdst, rk.j, g.block);
  return cudaGetLastError();
}

// Per-device launch attributes (the opt-in shared-memory sizes of K1 and K4).  The attribute
// belongs to the current device's context, so every graph sets it for its own device at creation
// (no process-wide "already set" flag).
cudaError_t kernels_init_device() {
  cudaError_t e = expand_attrs<1, 1024>();
  if (e == cudaSuccess) e = expand_attrs<2, 1024>();
  if (e == cudaSuccess) e = expand_attrs<4, 1024>();
  if (e == cudaSuccess) e = expand_attrs<8, 1024>();
  if (e == cudaSuccess) e = expand_attrs<16, 512>();
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_parent<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_parent<ull>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(227 * 1024));
  return e;
}

// ------------------------------------------------------------------ K2: frontier update
// Thread per (segment m, word w) of the local rows.  Owned segment m == j: new vertices are the
// rows received from any column (own discoveries included) that are not yet visited; the
// lowest sending column is recorded as the parent's column (winner).  Other segments: mark the
// rows this rank discovered as visited so they are sent at most once.
constexpr int kUpdWords = 4;  // words per thread of K2 (their loads in flight together)
__global__ void __launch_bounds__(256) k_update(uint32_t* vis, uint32_t* vold, const uint32_t* recv,
                                                uint32_t* front_seg,
                                                int32_t* level, uint8_t* winner, LevelInfo* info, uint64_t W, int C,
                                                int j, const LevelCtrl* ctrl, uint32_t* const* __restrict__ exp_dst,
                                                int R) {
  // grid: x strides over the words of one segment (kUpdWords groups of 256 words per CTA and
  // step), y = segment m
  const int lvl = (int)ctrl->lvl;  // the level being assigned (device-side: the loop may be a graph)
  const int m = (int)blockIdx.y;
  const int lane = threadIdx.x & 31;
  unsigned cnt = 0;
  const uint64_t step = (uint64_t)gridDim.x * blockDim.x * kUpdWords;
  for (uint64_t wb0 = (uint64_t)blockIdx.x * blockDim.x * kUpdWords; wb0 < W; wb0 += step) {
    uint32_t vo[kUpdWords], vn[kUpdWords];
#pragma unroll
    for (int q = 0; q < kUpdWords; ++q) {  // all the thread's words in one round trip
      const uint64_t w = wb0 + (uint64_t)q * blockDim.x + threadIdx.x;
      const uint64_t gid = (uint64_t)m * W + w;
      vo[q] = w < W ? vold[gid] : 0u;
      vn[q] = w < W ? vis[gid] : 0u;
    }
#pragma unroll
    for (int q = 0; q < kUpdWords; ++q) {
      const uint64_t wb = wb0 + (uint64_t)q * blockDim.x;
      if (wb >= W) break;  // CTA-uniform
      const uint64_t w = wb + threadIdx.x;
      const uint64_t gid = (uint64_t)m * W + w;
      uint32_t newbits = 0;
      uint32_t wbits[8];  // winner column c's share of newbits (C <= 8 per row of the grid is typical)
      if (m == j && w < W) {
        const uint32_t own = vn[q] & ~vo[q];  // own discoveries (vo: the level-start bits)
        uint32_t claimed = 0;
        for (int c = 0; c < C; ++c) {
          const uint32_t x = ((c == j) ? own : recv[(uint64_t)c * W + w]) & ~vo[q] & ~claimed;
          if (c < 8) wbits[c] = x;
          if (x && winner && c >= 8) {  // wide grids: per-bit winner stores
            uint32_t b = x;
            while (b) {
              const int bit = __ffs(b) - 1;
              b &= b - 1;
              winner[w * 32 + bit] = (uint8_t)c;
            }
          }
          claimed |= x;
        }
        newbits = claimed;  // includes own (own discoveries were not visited at the level start)
        if (newbits) vis[gid] = vold[gid] = vo[q] | newbits;
        front_seg[w] = newbits;
        if (exp_dst)  // peer exchange (NVLink stores): the next frontier segment into the column peers
          for (int i2 = 0; i2 < R; ++i2)
            if (exp_dst[i2]) exp_dst[i2][w] = newbits;
      } else if (w < W) {  // rows of other owners discovered here stay visited on this rank
        if (vn[q] != vo[q]) vold[gid] = vn[q];
      }
      // levels (and winners) of the new vertices: the warp walks its 32 words, lane l writing
      // vertex 32k + l of word k (coalesced stores instead of per-bit scattered ones)
      if (m == j) {
        const uint64_t wbase = w - lane;
        unsigned nz = __ballot_sync(0xFFFFFFFFu, newbits != 0);
        while (nz) {
          const int k = __ffs(nz) - 1;
          nz &= nz - 1;
          const uint32_t nb = __shfl_sync(0xFFFFFFFFu, newbits, k);
          const uint64_t v = (wbase + k) * 32 + lane;
          if ((nb >> lane) & 1u) level[v] = lvl;
          if (winner) {
            const int cmax = C < 8 ? C : 8;
            for (int c = 0; c < cmax; ++c) {
              const uint32_t x = __shfl_sync(0xFFFFFFFFu, wbits[c], k);
              if ((x >> lane) & 1u) winner[v] = (uint8_t)c;
            }
          }
        }
      }
      cnt += __popc(newbits);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&info->newv, (ull)cnt);
  if (exp_dst) {
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
  }
}

cudaError_t launch_update(const Geom& g, Rank& rk, const LevelCtrl* ctrl, cudaStream_t s) {
  const uint64_t W = g.words_block();
  uint64_t gx = (W + 256 * kUpdWords - 1) / (256 * kUpdWords);
  // peer stores: each CTA ends with a system-scope fence, so a capped grid strides instead
  const uint64_t cap = (uint64_t)g.nsm * 8 / (uint64_t)g.C;
  if (g.R > 1 && rk.exp_dst && gx > cap) gx = cap ? cap : 1;
  const dim3 grid((unsigned)gx, (unsigned)g.C);
  k_update<<<grid, 256, 0, s>>>(rk.vis, rk.vold, rk.recv, rk.all_front + (uint64_t)rk.i * W, rk.level,
                                g.C > 1 ? rk.winner : nullptr, rk.info, W, g.C, rk.j, ctrl,
                                g.R > 1 ? rk.exp_dst : nullptr, g.R);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ level control
// End of a level: termination test on the total of new vertices (all local ranks; with NCCL the
// update counter of rank 0's info has been all-reduced first), per-level statistics, lvl + 1,
// and -- when the level loop is a CUDA-graph WHILE node -- the loop condition.
__global__ void k_level_end(LevelCtrl* ctrl, const LevelInfo* infos, int nlocal, int distributed,
                            cudaGraphConditionalHandle cond, int use_cond) {
  if (threadIdx.x != 0) return;
  ull total = 0, fr = 0, ed = 0;
  for (int k = 0; k < nlocal; ++k) {
    total += distributed ? (k == 0 ? infos[0].newv : 0ull) : infos[k].newv;
    fr += infos[k].n + infos[k].nlongcols;
    ed += infos[k].edges;
  }
  const uint32_t l = ctrl->nlev;
  if (l < kMaxLevels) {
    ctrl->lvl_frontier[l] = fr;
    ctrl->lvl_edges[l] = ed;
  }
  ctrl->sum_frontier += fr;
  ctrl->sum_edges += ed;
  ctrl->nlev = l + 1;
  ctrl->lvl += 1;
  ctrl->total_new = total;
  // a BFS ends after at most nverts levels; per-level statistics are kept for the first
  // kMaxLevels levels only (deeper graphs, e.g. long paths, keep iterating)
  const bool done = total == 0;
  ctrl->done = done ? 1u : 0u;
  if (use_cond) cudaGraphSetConditional(cond, done ? 0u : 1u);
}

__global__ void k_level_begin(LevelCtrl* ctrl) {
  ctrl->lvl = 1;
  ctrl->nlev = 0;
  ctrl->done = 0;
  ctrl->total_new = 0;
  ctrl->sum_frontier = 0;
  ctrl->sum_edges = 0;
}

cudaError_t launch_level_begin(LevelCtrl* ctrl, cudaStream_t s) {
  k_level_begin<<<1, 1, 0, s>>>(ctrl);
  return cudaGetLastError();
}

cudaError_t launch_level_end(LevelCtrl* ctrl, const LevelInfo* infos, int nlocal, bool distributed,
                             cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t s) {
  k_level_end<<<1, 32, 0, s>>>(ctrl, infos, nlocal, distributed ? 1 : 0, cond, use_cond ? 1 : 0);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ outputs
// For owned t: unreached (visited bit clear) -> level -1, parent -1; reached with the winner
// column == own column (always when C == 1) -> parent = pred of the own row segment; other
// reached vertices take the answers of the resolution exchange (see k_finalize).
// t indexes the ORIGINAL owned offsets (outputs, written coalesced); p = fwd_own[t] the relabeled
// one (state; identity outside the relabeled prefix and the slots it displaced).  Four outputs
// per thread with 16-byte loads and stores (block is a multiple of 32).  With C > 1 a vertex
// whose winner column c differs from j takes its parent from the answers of P_ic: position =
// rank of its bit among the requests sent to c (exclusive popcount scan off_req + in-word popc).
struct FinalizeArgs {
  const uint32_t* vis_own;
  const int32_t* level;
  const uint32_t* pred_own;
  const uint8_t* winner;  // null when C == 1
  const uint32_t* fwd_own;
  const uint32_t* req;      // [C*W] request bitmaps
  const uint32_t* off_req;  // exclusive popcount scan of req
  const uint32_t* respin;   // answers, segment c at c*block
  int direct;               // peer exchange: respin[c*block + p] is column c's candidate (pushed by K4)
  int j;
  uint64_t block, W;
};

__global__ void k_finalize(FinalizeArgs a, int64_t* parent_out, int32_t* level_out) {
  const uint64_t t0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (t0 >= a.block) return;
  const uint4 p4 = *reinterpret_cast<const uint4*>(a.fwd_own + t0);
  const uint32_t pp[4] = {p4.x, p4.y, p4.z, p4.w};
  int64_t q[4];
  int32_t l[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t p = pp[k];
    BCHECK(p < a.block);
    const bool reached = (a.vis_own[p >> 5] >> (p & 31)) & 1u;
    int64_t v = -1;
    if (reached && parent_out) {  // without a parent output the resolution did not run
      const int c = a.winner ? (int)a.winner[p] : a.j;
      if (c == a.j) {
        v = (int64_t)a.pred_own[p];
      } else if (a.direct) {
        v = (int64_t)a.respin[(uint64_t)c * a.block + p];
      } else {
        const uint64_t wi = (uint64_t)c * a.W + (p >> 5);
        const uint32_t below = a.req[wi] & ((1u << (p & 31)) - 1u);
        const uint64_t pos = a.off_req[wi] - a.off_req[(uint64_t)c * a.W] + __popc(below);
        v = (int64_t)a.respin[(uint64_t)c * a.block + pos];
      }
    }
    q[k] = v;
    l[k] = reached ? a.level[p] : -1;
  }
  if (parent_out) {
    longlong2* po = reinterpret_cast<longlong2*>(parent_out + t0);
    po[0] = make_longlong2(q[0], q[1]);
    po[1] = make_longlong2(q[2], q[3]);
  }
  if (level_out) *reinterpret_cast<int4*>(level_out + t0) = make_int4(l[0], l[1], l[2], l[3]);
}

cudaError_t launch_finalize(const Geom& g, Rank& rk, int64_t* parent_out, int32_t* level_out, bool direct,
                            cudaStream_t s) {
  FinalizeArgs a;
  a.direct = direct ? 1 : 0;
  a.vis_own = rk.vis + (uint64_t)rk.j * g.words_block();
  a.level = rk.level;
  a.pred_own = rk.pred + (uint64_t)rk.j * g.block;
  a.winner = (g.C > 1 && parent_out) ? rk.winner : nullptr;  // parents of other columns need resolution
  a.fwd_own = rk.fwd_own;
  a.req = rk.req;
  a.off_req = rk.off_req;
  a.respin = rk.respin;
  a.j = rk.j;
  a.block = g.block;
  a.W = g.words_block();
  const unsigned grid = (unsigned)((g.block / 4 + 255) / 256);
  k_finalize<<<grid, 256, 0, s>>>(a, parent_out, level_out);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ parent resolution (C > 1)
// request bitmaps: req[c] has bit t for owned reached t whose winner column is c != j.  A warp
// takes 32 consecutive words; for word k lane l reads the winner of vertex 32k + l (coalesced) and
// one ballot per column builds the word (C <= 8; wider grids take the per-bit loop).
__global__ void k_req_build(const uint32_t* vis_own, const uint8_t* winner, uint32_t* req, uint64_t W, int C, int j) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t vb = w < W ? vis_own[w] : 0u;  // visited word
  if (C > 8) {
    if (w >= W) return;
    for (int c = 0; c < C; ++c) req[(uint64_t)c * W + w] = 0u;
    uint32_t b = vb;
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      const int c = winner[w * 32 + bit];
      if (c != j) req[(uint64_t)c * W + w] |= 1u << bit;
    }
    return;
  }
  const uint64_t w0 = w - lane;
  uint32_t r[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // lane l: request word of w0 + l per column
  unsigned nz = __ballot_sync(0xFFFFFFFFu, vb != 0u);
  while (nz) {
    const int k = __ffs(nz) - 1;
    nz &= nz - 1;
    const uint32_t bk = __shfl_sync(0xFFFFFFFFu, vb, k);
    const bool reached = (bk >> lane) & 1u;
    const int c = reached ? (int)winner[(w0 + k) * 32 + lane] : j;
#pragma unroll
    for (int c2 = 0; c2 < 8; ++c2) {
      if (c2 >= C) break;
      const unsigned m = __ballot_sync(0xFFFFFFFFu, c == c2 && c2 != j);
      if (lane == k) r[c2] = m;
    }
  }
  if (w < W)
#pragma unroll
    for (int c2 = 0; c2 < 8; ++c2)
      if (c2 < C) req[(uint64_t)c2 * W + w] = r[c2];
}

cudaError_t launch_req_build(const Geom& g, Rank& rk, cudaStream_t s) {
  const uint64_t W = g.words_block();
  k_req_build<<<(unsigned)((W + 255) / 256), 256, 0, s>>>(rk.vis + (uint64_t)rk.j * W, rk.winner, rk.req, W,
                                                           g.C, rk.j);
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
// in ascending order into resp[c*block ...].  A warp takes 32 consecutive request words of one
// segment; for word k lane l moves row 32k + l (coalesced pred read, contiguous writes at the
// word's scan offset + the requested rows below it).
__global__ void k_resp_pack(const uint32_t* reqin, const uint32_t* off, const uint32_t* pred, uint32_t* resp,
                            uint64_t W, uint64_t block, int C, int j) {
  const int lane = threadIdx.x & 31;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = gid < W * (uint64_t)C;
  const int c = in ? (int)(gid / W) : j;
  const uint32_t b = (in && c != j) ? reqin[gid] : 0u;
  const uint64_t pos = b ? off[gid] - off[(uint64_t)c * W] : 0ull;
  const uint64_t w = in ? gid - (uint64_t)c * W : 0ull;
  const unsigned lt = lanemask_lt();
  unsigned nz = __ballot_sync(0xFFFFFFFFu, b != 0u);
  while (nz) {
    const int k = __ffs(nz) - 1;
    nz &= nz - 1;
    const uint32_t bk = __shfl_sync(0xFFFFFFFFu, b, k);
    const uint64_t pk = __shfl_sync(0xFFFFFFFFu, pos, k);
    const uint64_t wk = __shfl_sync(0xFFFFFFFFu, w, k);
    const int ck = __shfl_sync(0xFFFFFFFFu, c, k);
    if ((bk >> lane) & 1u)
      resp[(uint64_t)ck * block + pk + __popc(bk & lt)] = pred[(uint64_t)ck * block + wk * 32 + lane];
  }
}

cudaError_t launch_resp_pack(const Geom& g, Rank& rk, cudaStream_t s) {
  const uint64_t W = g.words_block();
  const uint64_t n = W * g.C;
  k_resp_pack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(rk.reqin, rk.off_in, rk.pred, rk.resp, W, g.block, g.C,
                                                          rk.j);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ m_comp, degree
__global__ void __launch_bounds__(256) k_mcomp(const uint32_t* vis_own, const uint32_t* tdeg, const uint32_t* fwd_own,
                                               uint64_t block, ull* out) {
  typedef cub::BlockReduce<ull, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  ull acc = 0;
  for (uint64_t t = (uint64_t)blockIdx.x * 256 + threadIdx.x; t < block; t += (uint64_t)gridDim.x * 256)
    if ((vis_own[fwd_own[t] >> 5] >> (fwd_own[t] & 31)) & 1u) acc += tdeg[t];
  ull tot = BR(tmp).Sum(acc);
  if (threadIdx.x == 0 && tot) atomicAdd(out, tot);
}

cudaError_t launch_mcomp(const Geom& g, Rank& rk, ull* out, cudaStream_t s) {
  k_mcomp<<<g.nsm * 4, 256, 0, s>>>(rk.vis + (uint64_t)rk.j * g.words_block(), rk.tdeg, rk.fwd_own, g.block,
                                         out);
  return cudaGetLastError();
}

// degree of ORIGINAL global vertex v held by this rank's column block (ncols columns)
__global__ void k_degree(const ull* col, const uint32_t* perm_fwd, uint64_t v, uint64_t ncols, ull* out) {
  const uint64_t u = (uint64_t)perm_fwd[v] % ncols;
  *out += col[u + 1] - col[u];
}

cudaError_t launch_degree(const Geom& g, Rank& rk, const uint32_t* perm_fwd, uint64_t v, ull* out, cudaStream_t s) {
  k_degree<<<1, 1, 0, s>>>(rk.col, perm_fwd, v, g.ncols(), out);
  return cudaGetLastError();
}

}  // namespace bfs200

namespace bfs200 {
// totals[c] = popcount of segment c of a bitmap whose exclusive popcount scan is off
__global__ void k_seg_totals(const uint32_t* off, uint64_t W, int C, unsigned long long* totals) {
  const int c = threadIdx.x;
  if (c < C) totals[c] = off[(uint64_t)(c + 1) * W] - off[(uint64_t)c * W];
}
// ------------------------------------------------------------------ peer exchange (NEXT-2)
// Cross-GPU barrier over NVLink peer memory: every rank stores (value, epoch) into its slot of
// every peer's signal array (release, system scope), then waits until every peer's slot of its
// own array carries the epoch (acquire).  Epochs come from a device counter that every rank
// advances identically, so the barrier also works inside the CUDA-graph level loop.  With
// sum_newv the values are the ranks' new-vertex counts and the sum replaces info->newv (the
// termination reduction).  A bounded spin sets *err instead of hanging.
__global__ void k_xbarrier(XSig* local, XSig* const* peers, int nranks, int me, ull* epoch_ctr, LevelInfo* info,
                           int sum_newv, int* err) {
  if (threadIdx.x != 0) return;
  const ull epoch = ++(*epoch_ctr);
  if (*(volatile int*)err) {  // an earlier barrier timed out: end the level loop (newv = 0)
    if (sum_newv) info->newv = 0;
    return;
  }
  const ull mine = sum_newv ? info->newv : 0ull;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  for (int p = 0; p < nranks; ++p) {
    if (p == me) continue;
    XSig* dst = peers[p] + me;
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(&dst->val), "l"(mine) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(&dst->flag), "l"(epoch) : "memory");
  }
  ull total = mine;
  const long long t0 = clock64();
  for (int p = 0; p < nranks; ++p) {
    if (p == me) continue;
    ull f = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(f) : "l"(&local[p].flag) : "memory");
      if (f >= epoch) break;
      if (clock64() - t0 > (1ll << 35)) {  // ~17 s at 2 GHz: a peer is gone
        atomicExch(err, 1);
        if (sum_newv) info->newv = 0;
        return;
      }
    }
    ull v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(&local[p].val) : "memory");
    total += v;
  }
  if (sum_newv) info->newv = total;
}

cudaError_t launch_xbarrier(XSig* local, XSig* const* peers, int nranks, int me, ull* epoch_ctr, LevelInfo* info,
                            bool sum_newv, int* err, cudaStream_t s) {
  k_xbarrier<<<1, 32, 0, s>>>(local, peers, nranks, me, epoch_ctr, info, sum_newv ? 1 : 0, err);
  return cudaGetLastError();
}

// the root's frontier bit in the all-gathered bitmap of a column peer of its owner (what the
// first expand exchange would deliver)
__global__ void k_seed_col(uint32_t* all_front, const uint32_t* perm_fwd, uint64_t root, uint64_t block, int i_owner) {
  const uint64_t t = (uint64_t)perm_fwd[root] - (root / block) * block;
  const uint64_t col_local = (uint64_t)i_owner * block + t;
  all_front[col_local >> 5] |= 1u << (col_local & 31);
}

cudaError_t launch_seed_col(uint32_t* all_front, const uint32_t* perm_fwd, uint64_t root, uint64_t block, int i_owner,
                            cudaStream_t s) {
  k_seed_col<<<1, 1, 0, s>>>(all_front, perm_fwd, root, block, i_owner);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ list exchange
// count of set bits of each of nseg segments of W words (grid.y = segment)
__global__ void k_seg_popc(const uint32_t* __restrict__ bm, uint64_t W, ull* cnt) {
  const uint64_t base = (uint64_t)blockIdx.y * W;
  unsigned c = 0;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < W; w += (uint64_t)gridDim.x * blockDim.x)
    c += __popc(bm[base + w]);
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt + blockIdx.y, (ull)c);
}


cudaError_t launch_seg_popc(const uint32_t* bm, uint64_t W, int nseg, ull* cnt, uint64_t* launches, cudaStream_t s) {
  if (!W || nseg <= 0) return cudaSuccess;
  ++*launches;
  const uint64_t blocks = (W + 255) / 256;
  k_seg_popc<<<dim3((unsigned)(blocks < 1024 ? blocks : 1024), (unsigned)nseg), 256, 0, s>>>(bm, W, cnt);
  return cudaGetLastError();
}

// list of segment k (ascending local indices) at list[k*lstride + ...]; off = exclusive popcount
// scan over all nseg*W words
__global__ void k_list_write(const uint32_t* __restrict__ bm, const uint32_t* __restrict__ off, uint64_t W,
                             uint64_t nwords, uint64_t lstride, uint32_t* list) {
  for (uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gid < nwords;
       gid += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = bm[gid];
    if (!b) continue;
    const uint64_t k = gid / W, w = gid - k * W;
    uint64_t pos = k * lstride + (off[gid] - off[k * W]);
    while (b) {
      const int bit = __ffs(b) - 1;
      b &= b - 1;
      list[pos++] = (uint32_t)(w * 32 + bit);
    }
  }
}

size_t list_encode_tmp_bytes(uint64_t nwords) {
  size_t bytes = 0;
  cub::TransformInputIterator<uint32_t, PopcOp, const uint32_t*> it(nullptr, PopcOp());
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (uint32_t*)nullptr, nwords, (cudaStream_t)0);
  return bytes;
}

cudaError_t launch_list_encode(const uint32_t* bm, uint64_t W, int nseg, uint32_t* off, void* tmp, size_t tmp_bytes,
                               uint32_t* list, uint64_t lstride, int nsm, uint64_t* launches, cudaStream_t s) {
  const uint64_t nwords = W * (uint64_t)nseg;
  if (!nwords) return cudaSuccess;
  cub::TransformInputIterator<uint32_t, PopcOp, const uint32_t*> it(bm, PopcOp());
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, it, off, nwords, s);
  if (e != cudaSuccess) return e;
  ++*launches;
  k_list_write<<<nsm * 8, 256, 0, s>>>(bm, off, W, nwords, lstride, list);
  return cudaGetLastError();
}

__global__ void k_list_scatter(const uint32_t* __restrict__ list, uint64_t n, uint32_t* bm) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = list[t];
    atomicOr(bm + (x >> 5), 1u << (x & 31));
  }
}

cudaError_t launch_list_scatter(const uint32_t* list, uint64_t n, uint32_t* bm, int nsm, uint64_t* launches,
                               cudaStream_t s) {
  if (!n) return cudaSuccess;
  ++*launches;
  const uint64_t blocks = (n + 255) / 256;
  k_list_scatter<<<(unsigned)(blocks < (uint64_t)nsm * 8 ? blocks : (uint64_t)nsm * 8), 256, 0, s>>>(
      list, n, bm);
  return cudaGetLastError();
}

cudaError_t launch_seg_totals(const uint32_t* off, uint64_t W, int C, unsigned long long* totals, cudaStream_t s) {
  k_seg_totals<<<1, 64, 0, s>>>(off, W, C, totals);
  return cudaGetLastError();
}
}  // namespace bfs200
