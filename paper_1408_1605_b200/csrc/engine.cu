// engine.cu -- libbfs200 C ABI: graph lifetime, the Alg.2 level loop, the expand / fold /
// termination transport (loopback copies or NCCL over NVLink) and the deferred parent exchange.
//
// Level loop (Alg.2), per level lvl = 1, 2, ...:
//   expand_comm   column all-gather of the owned frontier bitmaps
//   scan          K3 unpack + degree exclusive scan
//   expand        K1 frontier expansion                                       (Alg.3)
//   fold_comm     row exchange of the discovered-row bitmap segments
//   update        K2 OR / filter / level / next frontier
//   allreduce     termination: total new vertices; stop when 0
// After the loop the parents discovered by other grid columns are fetched once (P:47-49,
// P:625-627): the owner requests, by bitmap, the rows whose lowest sending
// column was c from P_ic, which answers with its pred[] entries in ascending row order.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "engine.h"
#include "kernels.cuh"

namespace bfs200 {

typedef unsigned long long ull;

// NVTX ranges (host-side enqueue phases: graph construction, level loop, parent resolution,
// outputs) for Nsight timelines; no cost when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// head of LevelCtrl read by the host each level (everything before the per-level arrays)
constexpr size_t kCtrlHead = offsetof(LevelCtrl, lvl_frontier);

static thread_local std::string tl_err;

int set_err(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  tl_err = buf;
  return status;
}

int cuda_fail(Graph& G, cudaError_t e, const char* what, const char* file, int line) {
  G.broken = true;
  return set_err(e == cudaErrorMemoryAllocation ? BFS_ENOMEM : BFS_ECUDA, "CUDA error %s (%s) at %s:%d: %s",
                 cudaGetErrorName(e), cudaGetErrorString(e), file, line, what);
}

int nccl_fail(Graph& G, ncclResult_t r, const char* what, const char* file, int line) {
  G.broken = true;
  return set_err(BFS_ENCCL, "NCCL error %d (%s) at %s:%d: %s", (int)r, ncclGetErrorString(r), file, line, what);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int G_alloc(Graph& G, void** p, size_t bytes) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    *p = nullptr;
    return set_err(BFS_ENOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  }
  G.allocs.push_back(q);
  G.device_bytes += bytes;
  *p = q;
  return BFS_OK;
}

// ------------------------------------------------------------------ NCCL transport helpers
int comm_allreduce_int_max(Graph& G, int* v) {
  int* d = reinterpret_cast<int*>(G.dscratch);
  CKR(cudaMemcpyAsync(d, v, sizeof(int), cudaMemcpyHostToDevice, G.stream));
  NKR(ncclAllReduce(d, d, 1, ncclInt32, ncclMax, G.world, G.stream));
  CKR(cudaMemcpyAsync(v, d, sizeof(int), cudaMemcpyDeviceToHost, G.stream));
  CKR(cudaStreamSynchronize(G.stream));
  return BFS_OK;
}

int comm_exchange_counts(Graph& G, const ull* send_counts, ull* recv_counts) {
  const int P = G.world_size;
  NKR(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    NKR(ncclSend(send_counts + q, 1, ncclUint64, q, G.world, G.stream));
    NKR(ncclRecv(recv_counts + q, 1, ncclUint64, q, G.world, G.stream));
  }
  NKR(ncclGroupEnd());
  return BFS_OK;
}

int comm_alltoallv_u64(Graph& G, const ull* send, const ull* soff, const ull* scnt, ull* recv, const ull* roff,
                       const ull* rcnt) {
  const int P = G.world_size, me = G.world_rank;
  if (scnt[me]) CKR(cudaMemcpyAsync(recv + roff[me], send + soff[me], scnt[me] * sizeof(ull), cudaMemcpyDeviceToDevice,
                                    G.stream));
  NKR(ncclGroupStart());
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    if (scnt[q]) NKR(ncclSend(send + soff[q], scnt[q], ncclUint64, q, G.world, G.stream));
    if (rcnt[q]) NKR(ncclRecv(recv + roff[q], rcnt[q], ncclUint64, q, G.world, G.stream));
  }
  NKR(ncclGroupEnd());
  return BFS_OK;
}

int comm_allreduce_u32_sum(Graph& G, uint32_t* buf, uint64_t n) {
  NKR(ncclAllReduce(buf, buf, n, ncclUint32, ncclSum, G.world, G.stream));
  return BFS_OK;
}

int comm_reduce_scatter_u32(Graph& G, const uint32_t* full, uint32_t* mine, uint64_t block) {
  NKR(ncclReduceScatter(full, mine, block, ncclUint32, ncclSum, G.world, G.stream));
  return BFS_OK;
}

// ------------------------------------------------------------------ per-level exchanges
// expand: every rank of grid column j receives the owned-frontier segment of every other rank
// of the column; segment i of all_front = frontier of P_ij (local column order).
static int expand_exchange(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  if (g.R == 1) return BFS_OK;
  if (G.world_size == 1) {
    for (Rank& dst : G.ranks)
      for (int i2 = 0; i2 < g.R; ++i2) {
        if (i2 == dst.i) continue;
        const Rank& src = G.ranks[dst.j * g.R + i2];
        CKR(cudaMemcpyAsync(dst.all_front + i2 * W, src.all_front + i2 * W, W * 4, cudaMemcpyDeviceToDevice,
                            G.stream));
      }
  } else {
    Rank& rk = G.ranks[0];
    NKR(ncclAllGather(rk.all_front + (uint64_t)rk.i * W, rk.all_front, W, ncclUint32, G.colc, G.stream));
  }
  return BFS_OK;
}

// fold: P_ij receives from every P_ic (c != j) the segment j of its discovered-row bitmap
// (the rows it owns); the OR and the winner are taken by K2.
static int fold_exchange(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  if (g.C == 1) return BFS_OK;
  if (G.world_size == 1) {
    for (Rank& dst : G.ranks)
      for (int c = 0; c < g.C; ++c) {
        if (c == dst.j) continue;
        const Rank& src = G.ranks[c * g.R + dst.i];
        CKR(cudaMemcpyAsync(dst.recv + c * W, src.sendbuf + (uint64_t)dst.j * W, W * 4, cudaMemcpyDeviceToDevice,
                            G.stream));
      }
  } else {
    Rank& rk = G.ranks[0];
    NKR(ncclGroupStart());
    for (int c = 0; c < g.C; ++c) {
      if (c == rk.j) continue;
      NKR(ncclSend(rk.sendbuf + (uint64_t)c * W, W, ncclUint32, c, G.rowc, G.stream));
      NKR(ncclRecv(rk.recv + (uint64_t)c * W, W, ncclUint32, c, G.rowc, G.stream));
    }
    NKR(ncclGroupEnd());
  }
  return BFS_OK;
}

// ------------------------------------------------------------------ graph lifetime
static int alloc_state(Graph& G, Rank& rk) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  const uint64_t rw = g.nrows() / 32, cw = g.ncols() / 32;
  const uint64_t nseg = (cw + kScanSegWords - 1) / kScanSegWords;
  int rc;
#define AL(ptr, bytes)                                  \
  if ((rc = G_alloc(G, (void**)&(ptr), (bytes))) != 0) \
    return rc;
  AL(rk.vis, rw * 4);
  AL(rk.vold, rw * 4);
  AL(rk.all_front, cw * 4);
  AL(rk.pred, g.nrows() * 4);
  AL(rk.pmin, g.nrows() * 4);
  CKR(cudaMemsetAsync(rk.pmin, 0xFF, g.nrows() * 4, G.stream));
  AL(rk.level, g.block * 4);
  AL(rk.flist, g.ncols() * 4);
  AL(rk.rowoff, g.ncols() * 8);
  AL(rk.cumul, (g.ncols() + 1) * 8);
  AL(rk.tile_k, (rk.nnz / 32 + 2) * 4);          // short-edge tiles have >= 32 edges
  AL(rk.tileA, (3 * (rk.nnz / 32) + 64) * 16);    // long tiles: <= nnz/TILE + #long columns (d >= TILE/2)
  // hub entries: <= one per column of > 8 tiles of >= 32 edges, + one per kHubChunk (1024) tiles
  const uint64_t nhub = rk.nnz / 256 + rk.nnz / (32 * 1024) + 64;
  AL(rk.longlist, 2 * nhub * 16);
  AL(rk.seg_tot, (nseg + 1) * 32);
  AL(rk.seg_off, (nseg + 8) * 32);  // CTA totals (nseg/8 + 1) and their scan (nseg/8 + 2)
  CKR(cudaMemsetAsync(rk.seg_tot, 0, (nseg + 1) * 32, G.stream));  // entry nseg stays zero
  AL(rk.parent_tmp, g.block * 8);
  AL(rk.level_tmp, g.block * 4);
  AL(rk.scratch, 64 * 8);
  {  // array capacities for the bounds checks of a BFS200_CHECKS build (kernels.cu)
    const unsigned long long caps[5] = {rk.nnz, g.ncols(), g.nrows(), 3 * (rk.nnz / 32) + 64, 2 * nhub};
    CKR(cudaMemcpyAsync(&rk.info->cap_nnz, caps, sizeof caps, cudaMemcpyHostToDevice, G.stream));
  }
  if (g.C > 1) {
    AL(rk.sendbuf, rw * 4);
    AL(rk.recv, (uint64_t)g.C * W * 4);
    AL(rk.winner, g.block);
    AL(rk.req, ((uint64_t)g.C * W + 32) * 4);
    AL(rk.reqin, ((uint64_t)g.C * W + 32) * 4);
    AL(rk.off_in, ((uint64_t)g.C * W + 32) * 4);
    AL(rk.off_req, ((uint64_t)g.C * W + 32) * 4);
    AL(rk.resp, g.nrows() * 4);
    AL(rk.respin, g.nrows() * 4);
    rk.scan_tmp_bytes = popc_scan_tmp_bytes((uint64_t)g.C * W);
    AL(rk.scan_tmp, rk.scan_tmp_bytes);
    CKR(cudaMemsetAsync(rk.req, 0, ((uint64_t)g.C * W + 32) * 4, G.stream));
    CKR(cudaMemsetAsync(rk.reqin, 0, ((uint64_t)g.C * W + 32) * 4, G.stream));
  }
#undef AL
  return BFS_OK;
}

static void drop_graph(Graph& G);

// release every resource held by *G (the Graph object itself is owned by bfs_graph)
static void release_graph(Graph* G) {
  if (!G) return;
  cudaSetDevice(G->device);
  if (G->stream) cudaStreamSynchronize(G->stream);
  for (void* p : G->ipc_opened) cudaIpcCloseMemHandle(p);
  G->ipc_opened.clear();
  for (void* p : G->allocs) cudaFree(p);
  G->allocs.clear();
  for (cudaEvent_t e : G->ev) cudaEventDestroy(e);
  G->ev.clear();
  for (cudaEvent_t e : G->tail_ev) cudaEventDestroy(e);
  G->tail_ev.clear();
  if (G->copy_stream) {
    cudaStreamSynchronize(G->copy_stream);
    cudaStreamDestroy(G->copy_stream);
    G->copy_stream = nullptr;
  }
  for (int k = 0; k < 2; ++k) {
    if (G->fin_ev[k]) cudaEventDestroy(G->fin_ev[k]);
    if (G->copy_ev[k]) cudaEventDestroy(G->copy_ev[k]);
    G->fin_ev[k] = G->copy_ev[k] = nullptr;
  }
  drop_graph(*G);
  if (G->h_infos) cudaFreeHost(G->h_infos);
  if (G->h_ctrl) cudaFreeHost(G->h_ctrl);
  G->h_ctrl = nullptr;
  if (G->h_scratch) cudaFreeHost(G->h_scratch);
  if (G->rowc) ncclCommDestroy(G->rowc);
  if (G->colc) ncclCommDestroy(G->colc);
  if (G->world) ncclCommDestroy(G->world);
  if (G->owns_stream && G->stream) cudaStreamDestroy(G->stream);
  G->stream = nullptr;
  G->h_infos = nullptr;
  G->h_scratch = nullptr;
  G->rowc = G->colc = G->world = nullptr;
}

static int check_opts(const bfs_opts* o) {
  if (!o) return BFS_OK;
  const int E = o->edges_per_thread;
  if (E != 0 && E != 1 && E != 2 && E != 4 && E != 8 && E != 16)
    return set_err(BFS_EINVAL, "edges_per_thread must be 1, 2, 4, 8 or 16 (got %d)", E);
  if (o->exchange < BFS_XCHG_BITMAP || o->exchange > BFS_XCHG_AUTO)
    return set_err(BFS_EINVAL, "exchange must be 0 (bitmap), 1 (list) or 2 (auto) (got %d)", o->exchange);
  if (o->peer_exchange != 0 && o->peer_exchange != 1)
    return set_err(BFS_EINVAL, "peer_exchange must be 0 or 1 (got %d)", o->peer_exchange);
  if (o->debug_flags & ~BFS_DEBUG_POS64) return set_err(BFS_EINVAL, "unknown debug_flags 0x%x", o->debug_flags);
  if (o->peer_exchange && o->exchange != BFS_XCHG_BITMAP)
    return set_err(BFS_EINVAL, "peer_exchange needs exchange = 0 (bitmap messages)");
  return BFS_OK;
}

static void apply_opts(Graph& G, const bfs_opts* o) {
  bfs_opts d{};
  if (o) d = *o;
  if (!d.edges_per_thread) d.edges_per_thread = 4;
  G.opts = d;
}

static int create(const uint64_t* src, const uint64_t* dst, uint64_t nedges, uint64_t nverts, int R, int C,
                  const bfs_comm* comm, const bfs_opts* opts, Graph* Gp) {
  Graph& G = *Gp;
  bfs_comm cm{};
  if (comm) {
    cm = *comm;
  } else {
    cm.loopback = 1;
    cm.nranks = 1;
    cudaGetDevice(&cm.device);
  }
  const int P = R * C;
  if (!cm.loopback && P != cm.nranks) return set_err(BFS_EINVAL, "R*C=%d != nranks=%d", P, cm.nranks);
  if (!cm.loopback && (cm.rank < 0 || cm.rank >= cm.nranks)) return set_err(BFS_EINVAL, "bad rank %d", cm.rank);
  G.device = cm.device;
  CKR(cudaSetDevice(G.device));
  G.loopback = cm.loopback || P == 1;
  G.world_rank = G.loopback ? 0 : cm.rank;
  G.world_size = G.loopback ? 1 : cm.nranks;
  apply_opts(G, opts);
  if (G.opts.stream) {
    G.stream = (cudaStream_t)G.opts.stream;
  } else {
    CKR(cudaStreamCreateWithFlags(&G.stream, cudaStreamNonBlocking));
    G.owns_stream = true;
  }
  // geometry: pad N to a multiple of 32*R*C; ids must fit u32 below the sentinel
  const uint64_t q = 32ull * (uint64_t)P;
  G.g.nverts = nverts;
  G.g.npad = (nverts + q - 1) / q * q;
  if (G.g.npad >= 0xFFFFFFFFull) return set_err(BFS_EINVAL, "nverts too large: padded %llu >= 2^32", (ull)G.g.npad);
  G.g.R = R;
  G.g.C = C;
  G.g.block = G.g.npad / P;
  // degree-ordered relabeling of every whole vertex block
  G.hot_h = G.g.block;
  {
    int nsm = 0;
    CKR(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, G.device));
    G.g.nsm = nsm > 0 ? nsm : 148;
  }
  CKR(kernels_init_device());
  G.ntuples = nedges;
  CKR(cudaMallocHost(&G.h_scratch, 16 * sizeof(ull)));
  {
    int rc = G_alloc(G, (void**)&G.dscratch, 16 * sizeof(ull));
    if (rc) return rc;
  }
  if (!G.loopback) {
    ncclUniqueId id;
    memcpy(&id, cm.nccl_id, sizeof id);
    NKR(ncclCommInitRank(&G.world, cm.nranks, id, cm.rank));
    const int i = cm.rank % R, j = cm.rank / R;
    NKR(ncclCommSplit(G.world, i, j, &G.rowc, nullptr));  // grid row i, ordered by column j
    NKR(ncclCommSplit(G.world, j, i, &G.colc, nullptr));  // grid column j, ordered by row i
  }
  const int nlocal = G.loopback ? P : 1;
  G.ranks.resize(nlocal);
  for (int k = 0; k < nlocal; ++k) {
    Rank& rk = G.ranks[k];
    rk.r = G.loopback ? k : cm.rank;
    rk.i = rk.r % R;
    rk.j = rk.r / R;
  }
  int rc = build_graph(G, src, dst, nedges);
  if (rc) return rc;
  rc = G_alloc(G, (void**)&G.infos, nlocal * sizeof(LevelInfo));
  if (rc) return rc;
  rc = G_alloc(G, (void**)&G.d_ctrl, sizeof(LevelCtrl));
  if (rc) return rc;
  CKR(cudaMallocHost(&G.h_ctrl, sizeof(LevelCtrl)));
  CKR(cudaMallocHost(&G.h_infos, nlocal * sizeof(LevelInfo)));
  for (int k = 0; k < nlocal; ++k) {
    G.ranks[k].info = G.infos + k;
    rc = alloc_state(G, G.ranks[k]);
    if (rc) return rc;
  }
  CKR(cudaStreamSynchronize(G.stream));
  return BFS_OK;
}

// ------------------------------------------------------------------ phase events
static int ev_prepare(Graph& G, int level) {
  const size_t need = (size_t)(level + 1) * kPhaseEvents;
  while (G.ev.size() < need) {
    cudaEvent_t e;
    CKR(cudaEventCreate(&e));
    G.ev.push_back(e);
  }
  return BFS_OK;
}

static inline int ev_rec(Graph& G, int level, int p) {
  if (!G.opts.phase_timing || level >= kMaxLevels) return BFS_OK;  // per-level records stop at kMaxLevels
  int rc = ev_prepare(G, level);
  if (rc) return rc;
  CKR(cudaEventRecord(G.ev[(size_t)level * kPhaseEvents + p], G.stream));
  return BFS_OK;
}

// ------------------------------------------------------------------ peer exchange (NEXT-2)
// CUDA IPC handles of every rank's recv, all_front and signal array are all-gathered over the
// world communicator and opened; each rank then holds device tables of the peer pointers its
// kernels store into (fold: recv of P_ic; expand: all_front of P_(i2)j) and of the signal arrays.
static bool peer_active(const Graph& G) {
  return G.opts.peer_exchange && G.world_size > 1 && G.opts.exchange == BFS_XCHG_BITMAP;
}

static int setup_peer(Graph& G) {
  if (G.peer_ready) return BFS_OK;
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  const int P = G.world_size, me = G.world_rank;
  cudaStream_t s = G.stream;
  Rank& rk = G.ranks[0];
  int rc;
  // Every step up to the agreement below is collective-safe: a local failure is recorded (not
  // returned), the rank still takes part in the handle all-gather, and the failure flag is then
  // all-reduced, so every rank returns the same error instead of some ranks waiting forever in
  // a collective that a failed rank never joins.
  int local_fail = 0;
  std::string why;
  auto fail = [&](const char* what, cudaError_t e) {
    if (!local_fail) why = std::string(what) + ": " + cudaGetErrorString(e);
    local_fail = 1;
    cudaGetLastError();
  };
  if ((rc = G_alloc(G, (void**)&G.xsig, 64 * sizeof(XSig)))) return rc;
  if ((rc = G_alloc(G, (void**)&G.d_epoch, 8))) return rc;
  if ((rc = G_alloc(G, (void**)&G.d_xerr, 8))) return rc;
  // C == 1: no fold / resolution buffers; dummies keep the handle layout uniform
  if (!rk.recv && (rc = G_alloc(G, (void**)&rk.recv, 16))) return rc;
  if (!rk.respin && (rc = G_alloc(G, (void**)&rk.respin, 16))) return rc;
  CKR(cudaMemset(G.xsig, 0, 64 * sizeof(XSig)));
  CKR(cudaMemset(G.d_epoch, 0, 8));
  CKR(cudaMemset(G.d_xerr, 0, 8));
  constexpr int NH = 4;
  cudaIpcMemHandle_t mine[NH];
  memset(mine, 0, sizeof mine);
  void* const bufs[NH] = {rk.recv, rk.all_front, G.xsig, rk.respin};
  for (int k = 0; k < NH && !local_fail; ++k) {
    const cudaError_t e = cudaIpcGetMemHandle(&mine[k], bufs[k]);
    if (e != cudaSuccess) fail("peer_exchange: cudaIpcGetMemHandle", e);
  }
  const size_t hb = sizeof(mine);
  Scratch sc;
  unsigned char* dbuf = nullptr;
  CKR(sc.alloc(&dbuf, hb * (P + 1)));
  CKR(cudaMemcpy(dbuf, mine, hb, cudaMemcpyHostToDevice));
  NKR(ncclAllGather(dbuf, dbuf + hb, hb, ncclUint8, G.world, s));
  std::vector<cudaIpcMemHandle_t> all((size_t)P * NH);
  CKR(cudaMemcpyAsync(all.data(), dbuf + hb, hb * P, cudaMemcpyDeviceToHost, s));
  CKR(cudaStreamSynchronize(s));
  std::vector<std::vector<void*>> of(NH, std::vector<void*>(P, nullptr));  // [buffer][rank]
  for (int p = 0; p < P && !local_fail; ++p) {
    for (int k = 0; k < NH && !local_fail; ++k) {
      if (p == me) {
        of[k][p] = bufs[k];
        continue;
      }
      void* ptr = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&ptr, all[(size_t)p * NH + k], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        fail("peer_exchange: cudaIpcOpenMemHandle (no CUDA IPC / peer access between the ranks' GPUs?)", e);
        break;
      }
      G.ipc_opened.push_back(ptr);
      of[k][p] = ptr;
    }
  }
  {  // agreement: any rank's failure fails every rank (the graph is then unusable everywhere)
    int any = local_fail;
    if ((rc = comm_allreduce_int_max(G, &any))) return rc;
    if (any) {
      G.broken = true;
      return set_err(BFS_ECUDA, "%s", local_fail ? why.c_str() : "peer_exchange: setup failed on another rank");
    }
  }
  const std::vector<void*>&recv_of = of[0], &front_of = of[1], &sig_of = of[2], &respin_of = of[3];
  // tables: fold_dst[c] = recv of P_ic + j*W; exp_dst[i2] = all_front of P_(i2)j + i*W;
  // respin_dst[c] = respin of P_ic + j*block (K4's parent candidates for the rows P_ic owns)
  std::vector<uint32_t*> fold((size_t)g.C, nullptr), expd((size_t)g.R, nullptr), rsd((size_t)g.C, nullptr);
  for (int c = 0; c < g.C; ++c)
    if (c != rk.j) {
      fold[c] = static_cast<uint32_t*>(recv_of[c * g.R + rk.i]) + (uint64_t)rk.j * W;
      rsd[c] = static_cast<uint32_t*>(respin_of[c * g.R + rk.i]) + (uint64_t)rk.j * g.block;
    }
  for (int i2 = 0; i2 < g.R; ++i2)
    if (i2 != rk.i) expd[i2] = static_cast<uint32_t*>(front_of[rk.j * g.R + i2]) + (uint64_t)rk.i * W;
  std::vector<XSig*> sigs(P);
  for (int p = 0; p < P; ++p) sigs[p] = static_cast<XSig*>(sig_of[p]);
  if ((rc = G_alloc(G, (void**)&rk.fold_dst, g.C * sizeof(uint32_t*)))) return rc;
  if ((rc = G_alloc(G, (void**)&rk.exp_dst, g.R * sizeof(uint32_t*)))) return rc;
  if ((rc = G_alloc(G, (void**)&G.d_sig_peers, P * sizeof(XSig*)))) return rc;
  CKR(cudaMemcpy(rk.fold_dst, fold.data(), g.C * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  CKR(cudaMemcpy(rk.exp_dst, expd.data(), g.R * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  if ((rc = G_alloc(G, (void**)&rk.respin_dst, g.C * sizeof(uint32_t*)))) return rc;
  CKR(cudaMemcpy(rk.respin_dst, rsd.data(), g.C * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  CKR(cudaMemcpy(G.d_sig_peers, sigs.data(), P * sizeof(XSig*), cudaMemcpyHostToDevice));
  // the peers' arrays must be zero (epochs start at 0) before anyone signals
  NKR(ncclAllReduce(G.d_xerr, G.d_xerr, 1, ncclInt, ncclSum, G.world, s));
  CKR(cudaStreamSynchronize(s));
  G.peer_ready = true;
  return BFS_OK;
}

// ------------------------------------------------------------------ list exchange (NEXT-1)
// The paper's per-phase choice between a list of indices and a bitmap: a message of
// n indices over an index space of L = block vertices is a list iff n <= T = L/32 words (the
// bitmap's size, strict ">" for the bitmap).  Message sizes depend on counts,
// so both phases first exchange the counts and read them on the host (host-driven level loop).
static int alloc_xchg(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  const uint64_t S = (uint64_t)(g.R > g.C ? g.R : g.C);
  int rc;
  for (Rank& rk : G.ranks) {
    if (rk.xsend) continue;
    // a list holds up to `block` indices (forced list mode on a dense level)
    if ((rc = G_alloc(G, (void**)&rk.xsend, S * g.block * 4 + 16))) return rc;
    if ((rc = G_alloc(G, (void**)&rk.xrecv, S * g.block * 4 + 16))) return rc;
    if ((rc = G_alloc(G, (void**)&rk.xoff, S * W * 4 + 16))) return rc;
    if ((rc = G_alloc(G, (void**)&rk.xcnt, 64 * 8))) return rc;
    rk.xtmp_bytes = list_encode_tmp_bytes(S * W);
    if ((rc = G_alloc(G, &rk.xtmp, rk.xtmp_bytes ? rk.xtmp_bytes : 16))) return rc;
  }
  return BFS_OK;
}

static bool use_list(const Graph& G, uint64_t n) {
  return G.opts.exchange == BFS_XCHG_LIST || (G.opts.exchange == BFS_XCHG_AUTO && n <= G.g.words_block());
}

// column phase: the R owned frontier segments of a grid column, gathered into all_front
static int expand_exchange_x(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  cudaStream_t s = G.stream;
  if (g.R == 1) return BFS_OK;
  // counts of every rank of each local column, on the host: h[i] for column rank i
  std::vector<ull> cnt((size_t)G.ranks.size() * 64, 0);
  for (Rank& rk : G.ranks) {
    CKR(cudaMemsetAsync(rk.xcnt, 0, 64 * 8, s));
    CKR(launch_seg_popc(rk.all_front + (uint64_t)rk.i * W, W, 1, rk.xcnt, &G.xlaunches, s));
  }
  if (G.world_size > 1) {
    Rank& rk = G.ranks[0];
    NKR(ncclAllGather(rk.xcnt, rk.xcnt + 1, 1, ncclUint64, G.colc, s));  // R <= 63 counts
    CKR(cudaMemcpyAsync(cnt.data(), rk.xcnt + 1, g.R * 8, cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  } else {
    for (size_t k = 0; k < G.ranks.size(); ++k)
      CKR(cudaMemcpyAsync(&cnt[k * 64], G.ranks[k].xcnt, 8, cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  }
  auto n_of = [&](const Rank& dst, int i2) -> ull {  // count of column rank i2 of dst's column
    if (G.world_size > 1) return cnt[i2];
    for (size_t k = 0; k < G.ranks.size(); ++k)
      if (G.ranks[k].j == dst.j && G.ranks[k].i == i2) return cnt[k * 64];
    return 0;
  };
  // one encoding per phase and column (an all-gather has one message size): the largest count
  for (Rank& dst : G.ranks) {
    ull maxn = 0;
    for (int i2 = 0; i2 < g.R; ++i2) maxn = n_of(dst, i2) > maxn ? n_of(dst, i2) : maxn;
    if (!use_list(G, maxn)) {
      if (G.world_size > 1) {
        NKR(ncclAllGather(dst.all_front + (uint64_t)dst.i * W, dst.all_front, W, ncclUint32, G.colc, s));
      } else {
        for (int i2 = 0; i2 < g.R; ++i2) {
          if (i2 == dst.i) continue;
          const Rank& src = G.ranks[dst.j * g.R + i2];
          CKR(cudaMemcpyAsync(dst.all_front + i2 * W, src.all_front + i2 * W, W * 4, cudaMemcpyDeviceToDevice, s));
        }
      }
      G.xbytes += (ull)(g.R - 1) * W * 4;
      continue;
    }
    G.xlists += (ull)(g.R - 1);
    if (G.world_size > 1) {
      CKR(launch_list_encode(dst.all_front + (uint64_t)dst.i * W, W, 1, dst.xoff, dst.xtmp, dst.xtmp_bytes, dst.xsend,
                             g.block, g.nsm, &G.xlaunches, s));
      if (maxn) NKR(ncclAllGather(dst.xsend, dst.xrecv, maxn, ncclUint32, G.colc, s));
    } else {
      for (int i2 = 0; i2 < g.R; ++i2) {
        if (i2 == dst.i) continue;
        Rank& src = G.ranks[dst.j * g.R + i2];
        CKR(launch_list_encode(src.all_front + (uint64_t)i2 * W, W, 1, src.xoff, src.xtmp, src.xtmp_bytes, src.xsend,
                               g.block, g.nsm, &G.xlaunches, s));
        const ull n = n_of(dst, i2);
        if (n) CKR(cudaMemcpyAsync(dst.xrecv + i2 * maxn, src.xsend, n * 4, cudaMemcpyDeviceToDevice, s));
      }
    }
    for (int i2 = 0; i2 < g.R; ++i2) {
      if (i2 == dst.i) continue;
      const ull n = n_of(dst, i2);
      G.xbytes += n * 4;
      CKR(cudaMemsetAsync(dst.all_front + i2 * W, 0, W * 4, s));
      CKR(launch_list_scatter(dst.xrecv + i2 * maxn, n, dst.all_front + i2 * W, g.nsm, &G.xlaunches, s));
    }
  }
  return BFS_OK;
}

// row phase: P_ij sends its discovered rows of block (i,c) to P_ic, one message per pair, each
// encoded by its own count
static int fold_exchange_x(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  cudaStream_t s = G.stream;
  if (g.C == 1) return BFS_OK;
  const size_t nl = G.ranks.size();
  // cnt[k*64 + c] = rows of segment c discovered by local rank k
  std::vector<ull> cnt(nl * 64, 0), rcnt(64, 0);
  for (Rank& rk : G.ranks) {
    CKR(cudaMemsetAsync(rk.xcnt, 0, 64 * 8, s));
    CKR(launch_seg_popc(rk.sendbuf, W, g.C, rk.xcnt, &G.xlaunches, s));
  }
  if (G.world_size > 1) {
    Rank& rk = G.ranks[0];
    NKR(ncclGroupStart());  // counts: xcnt[c] = mine for c, xcnt[32 + c] = c's for me (C <= 32)
    for (int c = 0; c < g.C; ++c) {
      if (c == rk.j) continue;
      NKR(ncclSend(rk.xcnt + c, 1, ncclUint64, c, G.rowc, s));
      NKR(ncclRecv(rk.xcnt + 32 + c, 1, ncclUint64, c, G.rowc, s));
    }
    NKR(ncclGroupEnd());
    std::vector<ull> h(64);
    CKR(cudaMemcpyAsync(h.data(), rk.xcnt, 64 * 8, cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
    for (int c = 0; c < g.C; ++c) {
      cnt[c] = h[c];
      rcnt[c] = h[32 + c];
    }
  } else {
    for (size_t k = 0; k < nl; ++k) CKR(cudaMemcpyAsync(&cnt[k * 64], G.ranks[k].xcnt, g.C * 8, cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  }
  // encode every outgoing segment as a list (segments sent as bitmaps ignore theirs)
  for (Rank& rk : G.ranks)
    CKR(launch_list_encode(rk.sendbuf, W, g.C, rk.xoff, rk.xtmp, rk.xtmp_bytes, rk.xsend, g.block, g.nsm, &G.xlaunches, s));
  if (G.world_size > 1) {
    Rank& rk = G.ranks[0];
    NKR(ncclGroupStart());
    for (int c = 0; c < g.C; ++c) {
      if (c == rk.j) continue;
      const ull n = cnt[c], nr = rcnt[c];
      if (use_list(G, n)) {
        if (n) NKR(ncclSend(rk.xsend + (uint64_t)c * g.block, n, ncclUint32, c, G.rowc, s));
        G.xbytes += n * 4;
        ++G.xlists;
      } else {
        NKR(ncclSend(rk.sendbuf + (uint64_t)c * W, W, ncclUint32, c, G.rowc, s));
        G.xbytes += W * 4;
      }
      if (use_list(G, nr)) {
        if (nr) NKR(ncclRecv(rk.xrecv + (uint64_t)c * g.block, nr, ncclUint32, c, G.rowc, s));
      } else {
        NKR(ncclRecv(rk.recv + (uint64_t)c * W, W, ncclUint32, c, G.rowc, s));
      }
    }
    NKR(ncclGroupEnd());
    for (int c = 0; c < g.C; ++c) {
      if (c == rk.j || !use_list(G, rcnt[c])) continue;
      CKR(cudaMemsetAsync(rk.recv + (uint64_t)c * W, 0, W * 4, s));
      CKR(launch_list_scatter(rk.xrecv + (uint64_t)c * g.block, rcnt[c], rk.recv + (uint64_t)c * W, g.nsm, &G.xlaunches, s));
    }
  } else {
    for (size_t kd = 0; kd < nl; ++kd) {
      Rank& dst = G.ranks[kd];
      for (int c = 0; c < g.C; ++c) {
        if (c == dst.j) continue;
        const size_t ks = (size_t)c * g.R + dst.i;
        const Rank& src = G.ranks[ks];
        const ull n = cnt[ks * 64 + dst.j];
        if (use_list(G, n)) {
          G.xbytes += n * 4;
          ++G.xlists;
          if (n)
            CKR(cudaMemcpyAsync(dst.xrecv + (uint64_t)c * g.block, src.xsend + (uint64_t)dst.j * g.block, n * 4,
                                cudaMemcpyDeviceToDevice, s));
          CKR(cudaMemsetAsync(dst.recv + (uint64_t)c * W, 0, W * 4, s));
          CKR(launch_list_scatter(dst.xrecv + (uint64_t)c * g.block, n, dst.recv + (uint64_t)c * W, g.nsm, &G.xlaunches, s));
        } else {
          G.xbytes += W * 4;
          CKR(cudaMemcpyAsync(dst.recv + (uint64_t)c * W, src.sendbuf + (uint64_t)dst.j * W, W * 4,
                              cudaMemcpyDeviceToDevice, s));
        }
      }
    }
  }
  return BFS_OK;
}

// ------------------------------------------------------------------ parent resolution (C > 1)
static int resolve_parents(Graph& G) {
  const Geom& g = G.g;
  const uint64_t W = g.words_block();
  const int C = g.C;
  cudaStream_t s = G.stream;
  // NEXT-2 peer exchange: nothing to do -- every K4 stored the candidates of other columns' rows
  // in their owners' answer slots during the search (kernels.cu k_parent), and the last level's
  // barrier made them visible; k_finalize reads them directly
  if (peer_active(G)) return BFS_OK;
  for (Rank& rk : G.ranks) CKR(launch_req_build(g, rk, s));
  // requests: rank (i,j) sends req segment c to (i,c), which stores it as reqin segment j
  if (G.world_size == 1) {
    for (Rank& dst : G.ranks)
      for (int c = 0; c < C; ++c) {
        if (c == dst.j) continue;
        const Rank& src = G.ranks[c * g.R + dst.i];
        CKR(cudaMemcpyAsync(dst.reqin + (uint64_t)c * W, src.req + (uint64_t)dst.j * W, W * 4,
                            cudaMemcpyDeviceToDevice, s));
      }
  } else {
    Rank& rk = G.ranks[0];
    NKR(ncclGroupStart());
    for (int c = 0; c < C; ++c) {
      if (c == rk.j) continue;
      NKR(ncclSend(rk.req + (uint64_t)c * W, W, ncclUint32, c, G.rowc, s));
      NKR(ncclRecv(rk.reqin + (uint64_t)c * W, W, ncclUint32, c, G.rowc, s));
    }
    NKR(ncclGroupEnd());
  }
  // popcount scans of requests received / sent, segment totals to the host
  const size_t nl = G.ranks.size();
  std::vector<ull> h_tot(nl * 2 * 64);
  for (size_t k = 0; k < nl; ++k) {
    Rank& rk = G.ranks[k];
    CKR(launch_popc_scan(rk.reqin, rk.off_in, (uint64_t)C * W, rk.scan_tmp, rk.scan_tmp_bytes, s));
    CKR(launch_popc_scan(rk.req, rk.off_req, (uint64_t)C * W, rk.scan_tmp, rk.scan_tmp_bytes, s));
    CKR(launch_seg_totals(rk.off_in, W, C, rk.scratch, s));
    CKR(launch_seg_totals(rk.off_req, W, C, rk.scratch + 64 / 2, s));
    CKR(launch_resp_pack(g, rk, s));
    CKR(cudaMemcpyAsync(&h_tot[k * 128], rk.scratch, 64 * sizeof(ull), cudaMemcpyDeviceToHost, s));
  }
  CKR(cudaStreamSynchronize(s));
  // answers: (i,c) sends resp segment j (count = popc(reqin_j)) to (i,j) -> respin segment c
  if (G.world_size == 1) {
    for (size_t k = 0; k < nl; ++k) {
      Rank& dst = G.ranks[k];
      for (int c = 0; c < C; ++c) {
        if (c == dst.j) continue;
        const ull cnt = h_tot[k * 128 + 32 + c];  // popc(req segment c) of the owner
        if (!cnt) continue;
        const Rank& src = G.ranks[c * g.R + dst.i];
        CKR(cudaMemcpyAsync(dst.respin + (uint64_t)c * g.block, src.resp + (uint64_t)dst.j * g.block, cnt * 4,
                            cudaMemcpyDeviceToDevice, s));
      }
    }
  } else {
    Rank& rk = G.ranks[0];
    NKR(ncclGroupStart());
    for (int c = 0; c < C; ++c) {
      if (c == rk.j) continue;
      const ull scnt = h_tot[c], rcnt = h_tot[32 + c];
      if (scnt) NKR(ncclSend(rk.resp + (uint64_t)c * g.block, scnt, ncclUint32, c, G.rowc, s));
      if (rcnt) NKR(ncclRecv(rk.respin + (uint64_t)c * g.block, rcnt, ncclUint32, c, G.rowc, s));
    }
    NKR(ncclGroupEnd());
  }
  return BFS_OK;  // k_finalize reads the answers (no separate scatter)
}

// ------------------------------------------------------------------ one BFS
// One level of Alg.2, enqueued on the graph's stream without host synchronisation:
// expand exchange, K3 scan, K1 expansion, K4 parent claim, fold exchange, K2 update,
// termination all-reduce and the device-side level bookkeeping.  use_cond: the call is being
// captured into the body of the CUDA-graph WHILE node (no phase events then).
// 32-bit K3/K1 offsets when every CSC position of the rank fits (the same test as K1's POS32
// variant; the test-only BFS_DEBUG_POS64 flag forces the 64-bit path in both)
// 1x1 graph with the level loop on one stream: K2's frontier update moves into the next level's
// count pass (kernels.cu FusedUpd) and K4 counts the new vertices
static bool fused_of(const Graph& G) { return G.g.R == 1 && G.g.C == 1 && G.ranks.size() == 1; }

static bool narrow_of(const Graph& G, const Rank& rk) {
  return rk.nnz < (1ull << 32) && !(G.opts.debug_flags & BFS_DEBUG_POS64);
}

static int enqueue_level(Graph& G, bool use_cond, int nlev) {
  const Geom& g = G.g;
  cudaStream_t s = G.stream;
  const int E = G.opts.edges_per_thread;
  const uint32_t tile_edges = expand_tile_edges(E);
  const bool ev = !use_cond;
  int rc;
  if (peer_active(G)) {
    // NEXT-2: the column all-gather happened in the previous level's K2 (peer stores), the fold
    // in K4; two flag barriers replace the collectives (the second sums the new-vertex counts)
    Rank& rk = G.ranks[0];
    if (ev && (rc = ev_rec(G, nlev, 0))) return rc;
    if (ev && (rc = ev_rec(G, nlev, 1))) return rc;
    CKR(launch_scan(g, rk, tile_edges, narrow_of(G, rk), fused_of(G) ? G.d_ctrl : nullptr, s));
    if (ev && (rc = ev_rec(G, nlev, 2))) return rc;
    CKR(launch_expand(g, rk, E, G.hot_h, (G.opts.debug_flags & BFS_DEBUG_POS64) != 0, s));
    if (ev && (rc = ev_rec(G, nlev, 3))) return rc;
    CKR(launch_parent(g, rk, fused_of(G), (G.opts.debug_flags & BFS_DEBUG_POS64) != 0, s));
    if (ev && (rc = ev_rec(G, nlev, 4))) return rc;
    // barrier 1: every fold store has landed, and every rank is done reading its frontier bitmap
    // (K2's peer stores below overwrite it)
    CKR(launch_xbarrier(G.xsig, G.d_sig_peers, G.world_size, G.world_rank, G.d_epoch, G.infos, false, G.d_xerr, s));
    if (ev && (rc = ev_rec(G, nlev, 5))) return rc;
    CKR(launch_update(g, rk, G.d_ctrl, s));
    if (ev && (rc = ev_rec(G, nlev, 6))) return rc;
    CKR(launch_xbarrier(G.xsig, G.d_sig_peers, G.world_size, G.world_rank, G.d_epoch, G.infos, true, G.d_xerr, s));
    CKR(launch_level_end(G.d_ctrl, G.infos, 1, true, G.cond, use_cond, s));
    if (ev && (rc = ev_rec(G, nlev, 7))) return rc;
    return BFS_OK;
  }
  if (ev && (rc = ev_rec(G, nlev, 0))) return rc;
  const bool xl = G.opts.exchange != BFS_XCHG_BITMAP;  // never inside a graph capture
  if ((rc = xl ? expand_exchange_x(G) : expand_exchange(G))) return rc;
  if (ev && (rc = ev_rec(G, nlev, 1))) return rc;
  for (Rank& rk : G.ranks) CKR(launch_scan(g, rk, tile_edges, narrow_of(G, rk), fused_of(G) ? G.d_ctrl : nullptr, s));
  if (ev && (rc = ev_rec(G, nlev, 2))) return rc;
  for (Rank& rk : G.ranks) CKR(launch_expand(g, rk, E, G.hot_h, (G.opts.debug_flags & BFS_DEBUG_POS64) != 0, s));
  if (ev && (rc = ev_rec(G, nlev, 3))) return rc;
  for (Rank& rk : G.ranks) CKR(launch_parent(g, rk, fused_of(G), (G.opts.debug_flags & BFS_DEBUG_POS64) != 0, s));
  if (ev && (rc = ev_rec(G, nlev, 4))) return rc;
  if ((rc = xl ? fold_exchange_x(G) : fold_exchange(G))) return rc;
  if (ev && (rc = ev_rec(G, nlev, 5))) return rc;
  if (!fused_of(G))
    for (Rank& rk : G.ranks) CKR(launch_update(g, rk, G.d_ctrl, s));
  if (ev && (rc = ev_rec(G, nlev, 6))) return rc;
  if (G.world_size > 1) NKR(ncclAllReduce(&G.infos[0].newv, &G.infos[0].newv, 1, ncclUint64, ncclSum, G.world, s));
  CKR(launch_level_end(G.d_ctrl, G.infos, (int)G.ranks.size(), G.world_size > 1, G.cond, use_cond, s));
  if (ev && (rc = ev_rec(G, nlev, 7))) return rc;
  return BFS_OK;
}

static void drop_graph(Graph& G) {
  if (G.gexec) cudaGraphExecDestroy(G.gexec);
  if (G.graph) cudaGraphDestroy(G.graph);
  G.gexec = nullptr;
  G.graph = nullptr;
}

// The level loop as one CUDA graph: a WHILE conditional node whose body is one captured level;
// k_level_end sets the condition (no host round trip per level).
static int build_level_graph(Graph& G) {
  drop_graph(G);
  CKR(cudaGraphCreate(&G.graph, 0));
  CKR(cudaGraphConditionalHandleCreate(&G.cond, G.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = G.cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CKR(cudaGraphAddNode(&node, G.graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CKR(cudaStreamBeginCaptureToGraph(G.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  int rc = enqueue_level(G, true, 0);
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(G.stream, &captured);
  if (rc) return rc;
  CKR(e);
  CKR(cudaGraphInstantiate(&G.gexec, G.graph, 0));
  G.graph_stream = G.stream;
  G.graph_E = G.opts.edges_per_thread;
  G.graph_peer = peer_active(G);
  return BFS_OK;
}

// bfs_run_batch resources, created on the first batch with host outputs: the second staging pair
// of every local rank, the copy stream and the slot events
static int batch_setup(Graph& G) {
  if (G.copy_stream) return BFS_OK;
  int rc;
  for (Rank& rk : G.ranks) {
    if ((rc = G_alloc(G, (void**)&rk.parent_tmp2, G.g.block * 8))) return rc;
    if ((rc = G_alloc(G, (void**)&rk.level_tmp2, G.g.block * 4))) return rc;
  }
  for (int k = 0; k < 2; ++k) {
    CKR(cudaEventCreateWithFlags(&G.fin_ev[k], cudaEventDisableTiming));
    CKR(cudaEventCreateWithFlags(&G.copy_ev[k], cudaEventDisableTiming));
  }
  CKR(cudaStreamCreateWithFlags(&G.copy_stream, cudaStreamNonBlocking));
  return BFS_OK;
}

static int run(Graph& G, uint64_t root, int64_t* parent, int32_t* level, bfs_stats* stats) {
  const Geom& g = G.g;
  cudaStream_t s = G.stream;
  const uint64_t W = g.words_block();
  const uint64_t owner = root / g.block;
  bool owner_local = false;
  int rcp;
  if (peer_active(G)) {
    if ((rcp = setup_peer(G))) return rcp;
    // Rendezvous on the stream before the first cross-GPU flag barrier: NCCL waits for a late
    // rank without a timeout, so a caller that reaches bfs_run long after its peers (e.g. after
    // validating the previous result on the host) is not mistaken for a dead peer by the bounded
    // spin of k_xbarrier.  The max also spreads any earlier barrier error to every rank.
    NKR(ncclAllReduce(G.d_xerr, G.d_xerr, 1, ncclInt, ncclMax, G.world, s));
  }
  for (Rank& rk : G.ranks) {
    owner_local |= (uint64_t)rk.r == owner;
    CKR(launch_init(g, rk, (uint64_t)rk.r == owner, root, fused_of(G), s));
    // peer exchange: no all-gather before level 1, so the owner's column peers seed the bit
    const int owner_i = (int)(owner % (uint64_t)g.R), owner_j = (int)(owner / (uint64_t)g.R);
    if (peer_active(G) && (uint64_t)rk.r != owner && rk.j == owner_j)
      CKR(launch_seed_col(rk.all_front, G.perm_fwd, root, g.block, owner_i, s));
  }
  CKR(launch_level_begin(G.d_ctrl, s));
  int rc;
  // graph mode: no phase events, and not on the very first run (which initialises the kernels'
  // launch attributes outside of any capture)
  bool use_graph = !G.opts.phase_timing && !G.graph_failed && G.runs > 0 && G.opts.exchange == BFS_XCHG_BITMAP;
  G.xbytes = G.xlists = G.xlaunches = 0;
  if (G.opts.exchange != BFS_XCHG_BITMAP && (rc = alloc_xchg(G))) return rc;
  if (use_graph && (!G.gexec || G.graph_stream != s || G.graph_E != G.opts.edges_per_thread ||
                    G.graph_peer != peer_active(G))) {
    if (build_level_graph(G) != BFS_OK) {
      // Capture or instantiation of the level graph failed (e.g. a driver without conditional
      // nodes): fall back to the host-driven loop, which runs the same kernels.  Only errors of
      // the capture itself are forgiven: the (non-sticky) error is cleared, and the device must
      // then still synchronise cleanly -- a sticky error leaves the graph broken.
      G.graph_failed = true;
      drop_graph(G);
      use_graph = false;
      cudaGetLastError();
      const cudaError_t e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_fail(G, e, "device unhealthy after a failed level-graph capture", __FILE__, __LINE__);
      G.broken = false;
    }
  }
  NvtxRange r_loop(use_graph ? "bfs200: level loop (CUDA graph)" : "bfs200: level loop (host-driven)");
  if (use_graph) {
    CKR(cudaGraphLaunch(G.gexec, s));
  } else {
    for (int nlev = 0;; ++nlev) {
      if ((rc = enqueue_level(G, false, nlev))) return rc;
      CKR(cudaMemcpyAsync(G.h_ctrl, G.d_ctrl, kCtrlHead, cudaMemcpyDeviceToHost, s));
      CKR(cudaStreamSynchronize(s));
      if (G.h_ctrl->done) break;
    }
  }
  if (peer_active(G)) {  // a barrier that timed out leaves the level loop undefined
    int xerr = 0;
    CKR(cudaMemcpyAsync(&xerr, G.d_xerr, sizeof(int), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
    if (xerr) {
      G.broken = true;
      return set_err(BFS_ENCCL, "peer_exchange: a cross-GPU barrier timed out (a peer stopped)");
    }
  }
  // outputs
  const size_t nl = G.ranks.size();
  // the finalize kernel writes 16-byte vectors: unaligned device outputs go through the staging
  // buffers like host outputs (then one copy)
  const bool par_is_dev = is_device_ptr(parent) && (((uintptr_t)parent & 15) == 0);
  const bool lev_is_dev = is_device_ptr(level) && (((uintptr_t)level & 15) == 0);
  std::vector<int64_t*> par_dev(nl, nullptr);
  if (G.opts.phase_timing) {
    for (int q = (int)G.tail_ev.size(); q < 3; ++q) {
      cudaEvent_t ev;
      CKR(cudaEventCreate(&ev));
      G.tail_ev.push_back(ev);
    }
    CKR(cudaEventRecord(G.tail_ev[0], s));
  }
  if (g.C > 1 && parent) {
    NvtxRange r_res("bfs200: parent resolution");
    if ((rc = resolve_parents(G))) return rc;
  }
  if (G.opts.phase_timing) CKR(cudaEventRecord(G.tail_ev[1], s));
  // bfs_run_batch: staging pair of this root's slot, free once the copies of root k-2 are done;
  // the host copies then run on the copy stream, overlapping the next root's search
  const int slot = G.batch_slot;
  const bool staged = (parent && !par_is_dev) || (level && !lev_is_dev);
  const bool async_copy = slot >= 0 && staged;
  if (async_copy) {
    if ((rc = batch_setup(G))) return rc;
    CKR(cudaStreamWaitEvent(s, G.copy_ev[slot], 0));
  }
  for (size_t k = 0; k < nl; ++k) {
    Rank& rk = G.ranks[k];
    int64_t* ptmp = slot == 1 ? rk.parent_tmp2 : rk.parent_tmp;
    int32_t* ltmp = slot == 1 ? rk.level_tmp2 : rk.level_tmp;
    par_dev[k] = parent ? (par_is_dev ? parent + k * g.block : ptmp) : nullptr;  // no parent: not computed
    CKR(launch_finalize(g, rk, par_dev[k], level ? (lev_is_dev ? level + k * g.block : ltmp) : nullptr,
                        peer_active(G), s));
  }
  if (G.opts.phase_timing) CKR(cudaEventRecord(G.tail_ev[2], s));
  // host copies of the staged outputs: on the stream (bfs_run), or on the copy stream once this
  // run's small statistics reads are done (bfs_run_batch; a D2H copy engine serves its queue in
  // order, so a statistics read queued behind this root's 0.5 GB copy would hold the host until
  // the copy ends and nothing would overlap)
  auto host_copies = [&](cudaStream_t cs) -> int {
    for (size_t k = 0; k < nl; ++k) {
      Rank& rk = G.ranks[k];
      if (parent && !par_is_dev)
        CKR(cudaMemcpyAsync(parent + k * g.block, par_dev[k], g.block * 8, cudaMemcpyDefault, cs));
      if (level && !lev_is_dev)
        CKR(cudaMemcpyAsync(level + k * g.block, slot == 1 ? rk.level_tmp2 : rk.level_tmp, g.block * 4,
                            cudaMemcpyDefault, cs));
    }
    return BFS_OK;
  };
  if (!async_copy && (rc = host_copies(s))) return rc;
  CKR(cudaStreamSynchronize(s));
  if (peer_active(G)) {  // the resolution's barriers
    int xerr = 0;
    CKR(cudaMemcpy(&xerr, G.d_xerr, sizeof(int), cudaMemcpyDeviceToHost));
    if (xerr) {
      G.broken = true;
      return set_err(BFS_ENCCL, "peer_exchange: a cross-GPU barrier timed out (a peer stopped)");
    }
  }
  // per-level statistics of the device-side loop
  CKR(cudaMemcpyAsync(G.h_ctrl, G.d_ctrl, kCtrlHead, cudaMemcpyDeviceToHost, s));
  CKR(cudaStreamSynchronize(s));
  const int nlev = (int)G.h_ctrl->nlev;
  const int nrec = nlev < kMaxLevels ? nlev : kMaxLevels;  // per-level records kept
  CKR(cudaMemcpyAsync(G.h_ctrl->lvl_frontier, G.d_ctrl->lvl_frontier, nrec * sizeof(ull), cudaMemcpyDeviceToHost, s));
  CKR(cudaMemcpyAsync(G.h_ctrl->lvl_edges, G.d_ctrl->lvl_edges, nrec * sizeof(ull), cudaMemcpyDeviceToHost, s));
  CKR(cudaStreamSynchronize(s));
  G.last_levels = nlev;
  G.lvl_frontier.assign(G.h_ctrl->lvl_frontier, G.h_ctrl->lvl_frontier + nrec);
  G.lvl_edges.assign(G.h_ctrl->lvl_edges, G.h_ctrl->lvl_edges + nrec);
  const ull bytes = (ull)nlev * G.ranks.size() * ((ull)(g.R - 1) + (ull)(g.C - 1)) * W * 4;
  G.has_run = true;
  ++G.runs;
  if (stats) {
    memset(stats, 0, sizeof *stats);
    stats->nlevels = nlev;
    stats->edges_scanned = G.h_ctrl->sum_edges;
    stats->frontier_columns = G.h_ctrl->sum_frontier;
    stats->bytes_exchanged = G.opts.exchange == BFS_XCHG_BITMAP ? bytes : G.xbytes;
    stats->list_messages = G.xlists;
    if (G.opts.phase_timing) {  // the stream is synchronised: reading the events costs nothing
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, G.tail_ev[0], G.tail_ev[1]);
      cudaEventElapsedTime(&b, G.tail_ev[1], G.tail_ev[2]);
      stats->resolve_ms = a;
      stats->finalize_ms = b;
    }
    stats->reached = 0;
    // own kernels: seed (owner only), level_begin, per level level_end and per local rank
    // scan(4) + expand + parent + update (no update on a fused 1x1 graph), then finalize; with C > 1 the resolution adds
    // req_build, 2 seg_totals and resp_pack.
    const uint64_t nl = G.ranks.size();
    const bool peer = peer_active(G);
    const int owner_j = (int)(owner / (uint64_t)g.R);
    stats->kernel_launches =
        (owner_local ? 1 : 0) + 1 + nlev + nl * ((fused_of(G) ? 6ull : 7ull) * nlev + 1) + ((g.C > 1 && parent) ? nl * (peer ? 6 : 4) : 0) +
        G.xlaunches +
        (peer ? 2ull * nlev + ((G.ranks[0].j == owner_j && !owner_local) ? 1 : 0) : 0);
  }
  if (async_copy) {  // after the statistics reads: root k's copies overlap root k+1's search
    CKR(cudaEventRecord(G.fin_ev[slot], s));
    CKR(cudaStreamWaitEvent(G.copy_stream, G.fin_ev[slot], 0));
    if ((rc = host_copies(G.copy_stream))) return rc;
    CKR(cudaEventRecord(G.copy_ev[slot], G.copy_stream));
  }
  return BFS_OK;
}

}  // namespace bfs200

using namespace bfs200;

struct bfs_graph {
  Graph G;
};

#define ENTER(gp)                                                        \
  if (!(gp)) return set_err(BFS_EINVAL, "null graph");                   \
  Graph& G = (gp)->G;                                                    \
  if (G.broken) return set_err(BFS_ESTATE, "graph unusable after an earlier fatal error"); \
  if (cudaSetDevice(G.device) != cudaSuccess) return cuda_fail(G, cudaGetLastError(), "cudaSetDevice", __FILE__, __LINE__);

extern "C" {

int bfs_nccl_unique_id(unsigned char* out128) {
  if (!out128) return set_err(BFS_EINVAL, "null output");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return set_err(BFS_ENCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return BFS_OK;
}

int bfs_graph_create(const uint64_t* src, const uint64_t* dst, uint64_t nedges, uint64_t nverts, int R, int C,
                     const bfs_comm* comm, const bfs_opts* opts, bfs_graph** out) {
  if (!out) return set_err(BFS_EINVAL, "null out");
  *out = nullptr;
  if (nedges && (!src || !dst)) return set_err(BFS_EINVAL, "null edge arrays");
  if (nverts < 1) return set_err(BFS_EINVAL, "nverts must be >= 1");
  if (R < 1 || C < 1 || R * C > 64) return set_err(BFS_EINVAL, "grid %dx%d not supported (1 <= R*C <= 64)", R, C);
  if (C > 32) return set_err(BFS_EINVAL, "C must be <= 32");
  int rc = check_opts(opts);
  if (rc) return rc;
  bfs_graph* gp = nullptr;
  try {
    gp = new bfs_graph();
  } catch (std::bad_alloc&) {
    return set_err(BFS_ENOMEM, "host allocation failed");
  }
  try {
    NvtxRange r_create("bfs200: bfs_graph_create");
    rc = create(src, dst, nedges, nverts, R, C, comm, opts, &gp->G);
  } catch (std::bad_alloc&) {
    rc = set_err(BFS_ENOMEM, "host allocation failed");
  }
  if (rc) {
    std::string keep = bfs_last_error();
    release_graph(&gp->G);
    delete gp;
    tl_err = keep;
    return rc;
  }
  *out = gp;
  return BFS_OK;
}

int bfs_graph_info(const bfs_graph* gp, bfs_info* info) {
  if (!gp || !info) return set_err(BFS_EINVAL, "null argument");
  const Graph& G = gp->G;
  memset(info, 0, sizeof *info);
  info->nverts = G.g.nverts;
  info->npad = G.g.npad;
  info->block = G.g.block;
  info->R = G.g.R;
  info->C = G.g.C;
  info->rank = G.ranks.empty() ? 0 : G.ranks[0].r;
  info->nlocal = (int)G.ranks.size();
  info->first_vertex = (uint64_t)info->rank * G.g.block;
  info->nout = (uint64_t)info->nlocal * G.g.block;
  for (const Rank& rk : G.ranks) info->nnz_local += rk.nnz;
  info->ntuples = G.ntuples;
  info->device_bytes = G.device_bytes;
  return BFS_OK;
}

int bfs_set_opts(bfs_graph* gp, const bfs_opts* opts) {
  ENTER(gp);
  int rc = check_opts(opts);
  if (rc) return rc;
  cudaStream_t old = G.stream;
  bool owned = G.owns_stream;
  apply_opts(G, opts);
  if (G.opts.stream) {
    if (owned && old != (cudaStream_t)G.opts.stream) {
      cudaStreamSynchronize(old);
      cudaStreamDestroy(old);
    }
    G.stream = (cudaStream_t)G.opts.stream;
    G.owns_stream = false;
  } else {
    G.opts.stream = owned ? (void*)old : nullptr;
    if (!owned) {
      CKR(cudaStreamCreateWithFlags(&G.stream, cudaStreamNonBlocking));
      G.owns_stream = true;
    }
  }
  return BFS_OK;
}

int bfs_degree(bfs_graph* gp, uint64_t v, uint64_t* degree) {
  ENTER(gp);
  if (!degree) return set_err(BFS_EINVAL, "null output");
  if (v >= G.g.nverts) return set_err(BFS_ERANGE, "vertex %llu >= nverts", (ull)v);
  const uint64_t jv = v / G.g.ncols();  // relabeling stays inside vertex blocks, so columns too
  CKR(cudaMemsetAsync(G.dscratch, 0, sizeof(ull), G.stream));
  for (Rank& rk : G.ranks)
    if ((uint64_t)rk.j == jv) CKR(launch_degree(G.g, rk, G.perm_fwd, v, G.dscratch, G.stream));
  if (G.world_size > 1) NKR(ncclAllReduce(G.dscratch, G.dscratch, 1, ncclUint64, ncclSum, G.world, G.stream));
  CKR(cudaMemcpyAsync(G.h_scratch, G.dscratch, sizeof(ull), cudaMemcpyDeviceToHost, G.stream));
  CKR(cudaStreamSynchronize(G.stream));
  *degree = G.h_scratch[0];
  return BFS_OK;
}

int bfs_run(bfs_graph* gp, uint64_t root, int64_t* parent, int32_t* level, bfs_stats* stats) {
  ENTER(gp);
  NvtxRange r_run("bfs200: bfs_run");
  if (root >= G.g.nverts) return set_err(BFS_ERANGE, "root %llu >= nverts %llu", (ull)root, (ull)G.g.nverts);
  try {
    return run(G, root, parent, level, stats);
  } catch (std::bad_alloc&) {
    return set_err(BFS_ENOMEM, "host allocation failed");
  }
}

int bfs_run_batch(bfs_graph* gp, const uint64_t* roots, int n, int64_t* const* parent, int32_t* const* level,
                  bfs_stats* stats) {
  ENTER(gp);
  NvtxRange r_run("bfs200: bfs_run_batch");
  if (n < 0 || (n > 0 && !roots)) return set_err(BFS_EINVAL, "bad roots / n");
  for (int k = 0; k < n; ++k)
    if (roots[k] >= G.g.nverts)
      return set_err(BFS_ERANGE, "roots[%d] = %llu >= nverts %llu", k, (ull)roots[k], (ull)G.g.nverts);
  int rc = BFS_OK;
  try {
    for (int k = 0; k < n && rc == BFS_OK; ++k) {
      G.batch_slot = k & 1;
      rc = run(G, roots[k], parent ? parent[k] : nullptr, level ? level[k] : nullptr, stats ? stats + k : nullptr);
    }
  } catch (std::bad_alloc&) {
    rc = set_err(BFS_ENOMEM, "host allocation failed");
  }
  G.batch_slot = -1;
  if (G.copy_stream) {  // every host output complete
    const cudaError_t e = cudaStreamSynchronize(G.copy_stream);
    if (e != cudaSuccess && rc == BFS_OK) rc = cuda_fail(G, e, "bfs_run_batch: host copies", __FILE__, __LINE__);
  }
  return rc;
}

int bfs_mcomp(bfs_graph* gp, uint64_t* m_comp) {
  ENTER(gp);
  if (!m_comp) return set_err(BFS_EINVAL, "null output");
  if (!G.has_run) return set_err(BFS_ESTATE, "no BFS has run on this graph");
  CKR(cudaMemsetAsync(G.dscratch, 0, sizeof(ull), G.stream));
  for (Rank& rk : G.ranks) CKR(launch_mcomp(G.g, rk, G.dscratch, G.stream));
  if (G.world_size > 1) NKR(ncclAllReduce(G.dscratch, G.dscratch, 1, ncclUint64, ncclSum, G.world, G.stream));
  CKR(cudaMemcpyAsync(G.h_scratch, G.dscratch, sizeof(ull), cudaMemcpyDeviceToHost, G.stream));
  CKR(cudaStreamSynchronize(G.stream));
  *m_comp = G.h_scratch[0];
  return BFS_OK;
}

int bfs_gather(bfs_graph* gp, const int64_t* parent, const int32_t* level, int64_t* parent_all, int32_t* level_all) {
  ENTER(gp);
  const Geom& g = G.g;
  const uint64_t nout = (uint64_t)G.ranks.size() * g.block;  // this process's slice
  const bool root = G.world_rank == 0;
  cudaStream_t s = G.stream;
  if (root && ((parent && !parent_all) || (level && !level_all)))
    return set_err(BFS_EINVAL, "rank 0 needs parent_all / level_all for every non-NULL input");
  try {
    if (G.world_size == 1) {  // one process holds every rank: the slice is the whole vertex range
      if (parent) CKR(cudaMemcpyAsync(parent_all, parent, nout * 8, cudaMemcpyDefault, s));
      if (level) CKR(cudaMemcpyAsync(level_all, level, nout * 4, cudaMemcpyDefault, s));
      CKR(cudaStreamSynchronize(s));
      return BFS_OK;
    }
    // one process per rank: rank r's slice is global [r*block, (r+1)*block); point-to-point sends
    // to rank 0 over the world communicator (device staging where the caller's buffers are host)
    const int P = G.world_size;
    auto gather_one = [&](const void* mine, void* all, size_t esz, ncclDataType_t dt) -> int {
      Scratch sc;
      const void* src = mine;
      if (!is_device_ptr(mine)) {
        void* st = nullptr;
        CKR(sc.alloc(&st, nout * esz));
        CKR(cudaMemcpyAsync(st, mine, nout * esz, cudaMemcpyHostToDevice, s));
        src = st;
      }
      void* dst = nullptr;
      if (root) {
        if (is_device_ptr(all)) {
          dst = all;
        } else {
          CKR(sc.alloc(&dst, (size_t)P * nout * esz));
        }
      }
      NKR(ncclGroupStart());
      if (root) {
        for (int q = 1; q < P; ++q)
          NKR(ncclRecv(static_cast<char*>(dst) + (size_t)q * nout * esz, nout, dt, q, G.world, s));
      } else {
        NKR(ncclSend(src, nout, dt, 0, G.world, s));
      }
      NKR(ncclGroupEnd());
      if (root) {
        CKR(cudaMemcpyAsync(dst, src, nout * esz, cudaMemcpyDeviceToDevice, s));
        if (dst != all) CKR(cudaMemcpyAsync(all, dst, (size_t)P * nout * esz, cudaMemcpyDeviceToHost, s));
      }
      CKR(cudaStreamSynchronize(s));
      return BFS_OK;
    };
    int rc;
    if (parent && (rc = gather_one(parent, parent_all, 8, ncclInt64))) return rc;
    if (level && (rc = gather_one(level, level_all, 4, ncclInt32))) return rc;
    return BFS_OK;
  } catch (std::bad_alloc&) {
    return set_err(BFS_ENOMEM, "host allocation failed");
  }
}

int bfs_level_times(bfs_graph* gp, bfs_level_record* out, int max_levels, int* nlevels) {
  ENTER(gp);
  if (!nlevels) return set_err(BFS_EINVAL, "null nlevels");
  if (!G.has_run) return set_err(BFS_ESTATE, "no BFS has run on this graph");
  if (!G.opts.phase_timing) return set_err(BFS_ESTATE, "phase_timing was off for the last run");
  *nlevels = G.last_levels < kMaxLevels ? G.last_levels : kMaxLevels;  // records kept (first kMaxLevels levels)
  const int n = *nlevels < max_levels ? *nlevels : max_levels;
  if (n > 0 && !out) return set_err(BFS_EINVAL, "null output");
  for (int l = 0; l < n; ++l) {
    float t[kPhaseEvents - 1];
    for (int p = 0; p < kPhaseEvents - 1; ++p) {
      CKR(cudaEventSynchronize(G.ev[(size_t)l * kPhaseEvents + p + 1]));
      CKR(cudaEventElapsedTime(&t[p], G.ev[(size_t)l * kPhaseEvents + p], G.ev[(size_t)l * kPhaseEvents + p + 1]));
    }
    out[l].expand_comm = t[0];
    out[l].scan = t[1];
    out[l].expand = t[2];
    out[l].parent = t[3];
    out[l].fold_comm = t[4];
    out[l].update = t[5];
    out[l].allreduce = t[6];
    out[l].frontier = G.lvl_frontier[l];
    out[l].edges = G.lvl_edges[l];
  }
  return BFS_OK;
}

void bfs_destroy(bfs_graph* gp) {
  if (!gp) return;
  release_graph(&gp->G);
  delete gp;
}

const char* bfs_strerror(int status) {
  switch (status) {
    case BFS_OK: return "ok";
    case BFS_EINVAL: return "invalid argument";
    case BFS_ERANGE: return "vertex id out of range";
    case BFS_ENOMEM: return "out of memory";
    case BFS_ECUDA: return "CUDA error";
    case BFS_ENCCL: return "NCCL error";
    case BFS_ESTATE: return "graph in unusable state";
    case BFS_EPARSE: return "edge-list parse error";
    default: return "unknown status";
  }
}

const char* bfs_last_error(void) { return tl_err.c_str(); }

}  // extern "C"
