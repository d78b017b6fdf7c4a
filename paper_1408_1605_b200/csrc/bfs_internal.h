// bfs_internal.h -- internal data structures of libbfs200 (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/bfs200.h"

namespace bfs200 {

constexpr uint32_t kNoPred = 0xFFFFFFFFu;  // "no candidate" sentinel in pred[] (R11)
constexpr int kScanSegWords = 128;         // bitmap words per warp segment of the unpack/scan (4096 vertices)
constexpr int kScanThreads = 256;          // 8 warps = 8 segments per CTA
constexpr int kExpandThreads = 256;
constexpr int kMaxLevels = 4096;
constexpr int kPhaseEvents = 8;  // event boundaries per level (bfs_level_record phases + 1)

// Device-side per-level counters written by the scan kernels (read by the expansion kernel,
// so the host never needs the frontier size to launch it).
struct LevelInfo {
  unsigned long long n;       // short frontier columns (0 < local degree < TILE/2), listed in flist
  unsigned long long edges;   // all CSC entries leaving the frontier (short + long)
  unsigned long long newv;    // vertices discovered by the update (this rank)
  unsigned long long mode;    // parent claim of this level: 1 = atomicMin in the expansion (P1),
                              // 2 = CSR scan of the discovered rows (P2), 3 = P1 with the
                              // discovered words derived from pmin; see k_seg_scan
  unsigned long long nlong;   // hub columns whose long-tile records are written by k_tile_fill
  unsigned long long sedges;  // edges of the short columns = cumul[n]
  unsigned long long nA;      // long-column tiles (tileA records)
  unsigned long long ncols;   // short columns (stats)
  unsigned long long nlongcols;  // long columns (stats)
  unsigned long long disc_total;  // rows discovered by this rank so far in this search (K4 counts)
  unsigned long long blind;   // mode 3 with few rows visited: claims without the visited probe
                              // for rows past the hot prefix (K4 masks the visited rows)
  // capacities of this rank's arrays, for the bounds checks of a BFS200_CHECKS build (kernels.cu)
  unsigned long long cap_nnz, cap_ncols, cap_nrows, cap_tiles, cap_long;
};
static_assert(sizeof(LevelInfo) == 128, "LevelInfo layout");

// One slot of the peer-exchange signal array (one slot per sending rank).
struct XSig {
  unsigned long long flag;  // epoch of the sender's last barrier
  unsigned long long val;   // the sender's value for that barrier (new-vertex count)
};

// Device-side level loop state (the loop may run as a CUDA-graph WHILE node).
struct LevelCtrl {
  uint32_t lvl;   // level being assigned (1 for the root's neighbours)
  uint32_t nlev;  // levels executed
  uint32_t done;
  uint32_t pad;
  unsigned long long total_new;  // vertices discovered by the last level (all ranks)
  unsigned long long sum_frontier, sum_edges;  // over all levels (the arrays below stop at kMaxLevels)
  unsigned long long lvl_frontier[kMaxLevels];
  unsigned long long lvl_edges[kMaxLevels];
};

// Geometry of the 2D partition (index maps SPEC.md S:109-148).
struct Geom {
  uint64_t nverts, npad, block;
  int R, C;
  int nsm = 148;  // SMs of the graph's device (persistent grids are sized by it)
  uint64_t ncols() const { return (uint64_t)R * block; }  // N/C local columns
  uint64_t nrows() const { return (uint64_t)C * block; }  // N/R local rows
  uint64_t words_block() const { return block / 32; }
};

// One P_ij.  All pointers are device pointers on the graph's device.
struct Rank {
  int r, i, j;        // r = j*R + i
  uint64_t nnz = 0;   // CSC entries
  uint64_t nz_rows = 0;  // local rows with at least one entry (for the parent-mode heuristic)
  unsigned long long* col = nullptr;  // [ncols+1] column offsets (u64: nnz can exceed 2^32)
  uint32_t* col32 = nullptr;          // [ncols+1] the same as u32 when nnz < 2^32 (read by K3)
  uint8_t* deg8 = nullptr;            // [ncols] min(column degree, 255) (K3 count pass; 16-B aligned)
  uint32_t* row = nullptr;    // [nnz] local row ids, ascending within each column
  // CSR view of the same local matrix (row -> ascending local columns) for the parent pass;
  // with R = C = 1 the matrix is symmetric and these alias col/row.
  unsigned long long* csr_ptr = nullptr;  // [nrows+1]
  uint32_t* csr_ptr32 = nullptr;          // [nrows+1] the same as u32 when nnz < 2^32 (read by K4)
  uint32_t* csr_col = nullptr;            // [nnz]
  uint32_t* tdeg = nullptr;   // [block] input tuples whose source is the owned vertex (m_comp), ORIGINAL offsets
  // hot-prefix relabeling maps (build_graph.cu): owned offsets original <-> relabeled, and the
  // ORIGINAL global id of every relabeled local column (the value stored as a parent)
  uint32_t* fwd_own = nullptr;  // [block]
  uint32_t* inv_own = nullptr;  // [block]
  uint32_t* inv_col = nullptr;  // [ncols]
  // per-search state
  // visited bitmap over ALL local rows: vis = visited at the level start
  // OR rows discovered by this rank in the level (the expansion's RED.ORs), so one 4-byte probe
  // tests "visited or already discovered"; vold = the level-start bits (discovered = vis & ~vold).
  // Equal between levels.
  uint32_t* vis = nullptr;       // [nrows/32]
  uint32_t* vold = nullptr;      // [nrows/32]
  uint32_t* sendbuf = nullptr;   // [nrows/32] discovered rows packed contiguously (fold message, C>1)
  uint32_t* recv = nullptr;      // [C * block/32] fold receive buffer (segment c from P_ic); C>1 only
  uint32_t* all_front = nullptr; // [ncols/32] gathered frontier bitmap; own segment i = own frontier
  uint32_t* pred = nullptr;      // [nrows] min parent candidate (global id) per local row
  uint32_t* pmin = nullptr;      // [nrows] atomicMin scratch of P1 levels; all UINT32_MAX between levels
  int32_t* level = nullptr;      // [block] owned levels
  uint8_t* winner = nullptr;     // [block] grid column that supplied the parent (C>1 only)
  uint32_t* flist = nullptr;     // [ncols] frontier columns with degree>0, ascending
  unsigned long long* rowoff = nullptr;  // [ncols] col[flist[k]]
  unsigned long long* cumul = nullptr;   // [ncols+1] exclusive scan of degrees
  uint32_t* tile_k = nullptr;            // [nnz/32 + 2] first frontier index of every expansion tile
  uint4* longlist = nullptr;             // [2 * (nnz/256 + nnz/32768 + 64)] hub entries (kernels.cu kHubChunk)
  void* seg_tot = nullptr;               // [nseg] per-segment totals (SegTot, kernels.cu)
  void* seg_off = nullptr;               // [nseg+1] K3 scratch: per-CTA totals of the count pass and their scan
  uint4* tileA = nullptr;                // [nnz/(TILE/2) + ncols] long-column tile records
  LevelInfo* info = nullptr;             // [1]
  int64_t* parent_tmp = nullptr;         // [block] parent staging for host outputs / resolution
  int32_t* level_tmp = nullptr;          // [block] level staging for host outputs
  int64_t* parent_tmp2 = nullptr;        // bfs_run_batch: the second staging pair (odd roots),
  int32_t* level_tmp2 = nullptr;         //   allocated on the first batch with host outputs
  // parent resolution (C>1)
  uint32_t* req = nullptr;       // [C * block/32] request bitmaps: rows whose parent lives at P_ic
  uint32_t* reqin = nullptr;     // [C * block/32] requests received from P_ic (rows of segment c)
  uint32_t* off_in = nullptr;    // [C*block/32 + 1] exclusive popcount scan of reqin
  uint32_t* off_req = nullptr;   // [C*block/32 + 1] exclusive popcount scan of req
  void* scan_tmp = nullptr;      // CUB temp for the popcount scans
  size_t scan_tmp_bytes = 0;
  uint32_t* resp = nullptr;      // [nrows] compacted responses (sent)
  uint32_t* respin = nullptr;    // [nrows] segment c: column c's answers (compacted; peer exchange: by owned offset)
  // list exchange (opts.exchange != 0), allocated on first use; S = max(R, C) segments of W words
  uint32_t* xsend = nullptr;     // [S*W] outgoing index lists, segment k at k*W
  uint32_t* xrecv = nullptr;     // [S*W] incoming index lists
  uint32_t* xoff = nullptr;      // [S*W] exclusive popcount scan of the segments being encoded
  void* xtmp = nullptr;          // CUB temporary storage of that scan
  size_t xtmp_bytes = 0;
  unsigned long long* xcnt = nullptr;  // [64] per-segment counts (device)
  // peer exchange (opts.peer_exchange): device arrays of peer pointers, null when inactive
  uint32_t** fold_dst = nullptr;  // [C] recv of P_ic + j*W (null for c == j)
  uint32_t** exp_dst = nullptr;   // [R] all_front of P_(i2)j + i*W (null for i2 == i)
  uint32_t** respin_dst = nullptr;  // [C] respin of P_ic + j*block (null for c == j): K4's parent candidates
  unsigned long long* scratch = nullptr;  // small reduction scratch
};

struct Graph {
  Geom g{};
  int device = 0;
  int loopback = 1;
  int world_rank = 0, world_size = 1;
  bool owns_stream = false;
  cudaStream_t stream = nullptr;
  bfs_opts opts{};
  bool broken = false;
  std::vector<Rank> ranks;  // local ranks (all R*C with loopback)
  std::vector<void*> allocs;  // graph-lifetime device allocations
  uint64_t hot_h = 0;         // degree-ordered prefix per vertex block (vertices; the whole block)
  uint32_t* perm_fwd = nullptr;  // [npad] original -> relabeled global id
  LevelInfo* infos = nullptr; // [nlocal] device, one per local rank
  LevelInfo* h_infos = nullptr; // pinned mirror
  unsigned long long* dscratch = nullptr; // [16] device scratch for reductions
  // NCCL (loopback == 0 and R*C > 1)
  ncclComm_t world = nullptr, rowc = nullptr, colc = nullptr;
  unsigned long long* h_scratch = nullptr;  // pinned [16]
  uint64_t ntuples = 0;
  uint64_t device_bytes = 0;
  int last_levels = 0;
  bool has_run = false;
  // phase-timing events: [level][phase boundary]
  std::vector<cudaEvent_t> ev;
  std::vector<cudaEvent_t> tail_ev;  // finalize / parent-resolution events (phase_timing)
  // level loop as a CUDA graph (one WHILE node whose body is one level), built on first use
  LevelCtrl* d_ctrl = nullptr;
  LevelCtrl* h_ctrl = nullptr;  // pinned mirror
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphConditionalHandle cond = 0;
  cudaStream_t graph_stream = nullptr;
  int graph_E = 0;
  bool graph_peer = false;  // the captured level used the peer exchange
  bool graph_failed = false;
  int runs = 0;
  int ev_levels = 0;
  std::vector<uint64_t> lvl_frontier, lvl_edges;
  uint64_t xbytes = 0, xlists = 0;  // list exchange: bytes sent and list messages in this run
  uint64_t xlaunches = 0;           // list exchange: kernels launched in this run
  // peer exchange (NEXT-2): NVLink peer mappings of every rank's signal array, set up on first use
  bool peer_ready = false;
  XSig* xsig = nullptr;               // [64] this rank's signal array (slot = sender world rank)
  XSig** d_sig_peers = nullptr;       // [world] device array: every rank's signal array (mapped)
  unsigned long long* d_epoch = nullptr;
  int* d_xerr = nullptr;
  std::vector<void*> ipc_opened;      // cudaIpcOpenMemHandle mappings to close
  // bfs_run_batch: host copies of root k on copy_stream while root k+1 searches on `stream`;
  // batch_slot = k & 1 selects the staging pair (-1 outside a batch)
  int batch_slot = -1;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t fin_ev[2] = {nullptr, nullptr};   // finalize of the slot's root done (on stream)
  cudaEvent_t copy_ev[2] = {nullptr, nullptr};  // the slot's host copies done (on copy_stream)
};

}  // namespace bfs200
