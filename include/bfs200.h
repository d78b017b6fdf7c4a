/*
 * bfs200.h -- C ABI of libbfs200.so: level-synchronous top-down BFS over a 2D (R x C)
 * partitioned adjacency matrix, B200 (sm_100a) native.  arXiv 1408.1605 ("the paper").
 *
 * Problem (Alg.2): given an undirected graph as a list of
 * input tuples ("We turn the graph undirected by adding, for each edge, its
 * opposite") and a root r, compute for every vertex v its BFS level (hop distance from r,
 * -1 if unreachable) and its BFS-tree parent,
 * the parent being fixed as the MINIMUM-id neighbour one level up (the deterministic parent
 * claim of BASELINE.json's north_star; reading R1).
 *
 * Partition: R*C ranks form an R x C grid; rank r = j*R + i is P_ij; it owns the
 * vertex block [r*block, (r+1)*block), block = Npad/(R*C), and stores the edge blocks
 * (m*R+i, j), m = 0..C-1, as one CSC matrix of (Npad/R) x (Npad/C).
 *
 * Conventions for every call:
 *   - Return value: BFS_OK (0) or a negative bfs_status.  bfs_last_error() gives a
 *     thread-local detail string for the last failure on the calling thread.
 *   - Pointers documented as "host or device" are classified with cudaPointerGetAttributes;
 *     device pointers must be on the graph's device.
 *   - All calls taking a bfs_graph* are COLLECTIVE over the R*C ranks when the graph was
 *     created with the NCCL transport (every rank calls them in the same order with the same
 *     scalar arguments).  With the loopback transport one process holds all R*C logical ranks
 *     on one GPU and the calls are ordinary.
 *   - A CUDA or NCCL failure is fatal for the graph: it returns BFS_ECUDA / BFS_ENCCL and
 *     every later call on that graph returns BFS_ESTATE.
 *   - No global mutable state besides the thread-local error string (launch attributes and SM
 *     counts are set / read per graph on its own device); distinct graphs may be used from
 *     distinct threads.  One graph must not be used from two threads at once.
 */
#ifndef BFS200_H
#define BFS200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BFS_OK = 0,
  BFS_EINVAL = -1, /* bad argument: null pointer, R*C mismatch, nverts too large, ...        */
  BFS_ERANGE = -2, /* a vertex id (root, edge endpoint, query) is >= nverts                  */
  BFS_ENOMEM = -3, /* device or host allocation failed                                       */
  BFS_ECUDA = -4,  /* CUDA runtime error (graph becomes unusable)                            */
  BFS_ENCCL = -5,  /* NCCL error (graph becomes unusable)                                    */
  BFS_ESTATE = -6, /* graph unusable after an earlier fatal error, or call out of order      */
  BFS_EPARSE = -7  /* edge-list file does not parse (bfs_load_edges; the detail names the line) */
} bfs_status;

typedef struct bfs_graph bfs_graph; /* opaque; owned by the library until bfs_destroy */

/* Transport.  loopback != 0: this process emulates all R*C ranks on `device` (collectives
 * become device-to-device copies; for tests of the 2D logic on one GPU).  loopback == 0:
 * one rank per process; `rank`/`nranks` are this process's place in the R*C grid and
 * nccl_id is the ncclUniqueId made by rank 0 (bfs_nccl_unique_id) and broadcast by the
 * caller (e.g. with torch.distributed).  R = C = 1 with loopback = 0 needs no NCCL. */
typedef struct {
  int rank;
  int nranks;
  int device;
  int loopback;
  unsigned char nccl_id[128];
} bfs_comm;

/* Tuning / execution options; zero-initialised means defaults. */
typedef struct {
  int edges_per_thread; /* E, consecutive edges per expansion thread; 0 -> 4;
                           allowed 1, 2, 4, 8, 16 */
  int phase_timing;     /* != 0: record CUDA events around every phase of every level; read
                           them afterwards with bfs_level_times (does not synchronise) */
  void* stream;         /* cudaStream_t all work is issued on; NULL -> a library-owned stream */
  int exchange;         /* encoding of the per-level messages:
                           0 BFS_XCHG_BITMAP: every message is the L/32-word bitmap (default; the
                             level loop runs as one CUDA graph);
                           1 BFS_XCHG_LIST: every message is its count n of raw local indices;
                           2 BFS_XCHG_AUTO: per phase and level, a message is a list iff
                             n <= T = L/32 (strict ">" for the bitmap), L = block.
                           1 and 2 size the messages on the host each level (host-driven loop, one
                           count exchange + device-to-host read per phase). Values are otherwise
                           BFS_EINVAL. Results are identical in every mode. */
  int peer_exchange;    /* 1: per-level exchanges over NVLink peer memory instead of NCCL
                           collectives (§8(f) NEXT-2): the parent pass (K4) stores the fold
                           message straight into the owners' receive buffers, the update (K2)
                           stores the next frontier segment into the column peers' frontier
                           bitmaps, and two cross-GPU flag barriers per level (the second also
                           sums the new-vertex counts) replace the all-gather, the send/recv and
                           the all-reduce.  Needs CUDA IPC / peer access between the ranks' GPUs
                           (set up collectively on the first run) and exchange = 0; ignored by
                           loopback and 1x1.  0 (default): NCCL collectives.  At the start of
                           every bfs_run the ranks meet in one 4-byte NCCL all-reduce, so a rank
                           may reach bfs_run arbitrarily long after its peers; within a run a peer
                           that stops for ~17 s makes the run fail with BFS_ENCCL. */
  int debug_flags;      /* testing only; 0 in production.  BFS_DEBUG_POS64: the expansion stages
                           64-bit row positions and the parent pass reads the 64-bit CSR row
                           offsets even when every position fits in 32 bits (the kernel variants
                           otherwise used only when a rank holds >= 2^32 entries). */
} bfs_opts;

enum { BFS_DEBUG_POS64 = 1 };

enum { BFS_XCHG_BITMAP = 0, BFS_XCHG_LIST = 1, BFS_XCHG_AUTO = 2 };

/* Shape of this process's part of the partition. */
typedef struct {
  uint64_t nverts;       /* as passed to bfs_graph_create */
  uint64_t npad;         /* nverts rounded up to a multiple of 32*R*C (padding = isolated)  */
  uint64_t block;        /* npad / (R*C): vertices owned per rank                           */
  int R, C;
  int rank;              /* first rank held by this process (0 with loopback)               */
  int nlocal;            /* ranks held by this process (R*C with loopback, else 1)          */
  uint64_t first_vertex; /* rank * block: global id of output element 0                     */
  uint64_t nout;         /* nlocal * block: length of the parent/level outputs of bfs_run   */
  uint64_t nnz_local;    /* CSC entries held by this process (after dedup, no self-loops)   */
  uint64_t ntuples;      /* input tuples seen by this process's create call                 */
  uint64_t device_bytes; /* device memory held by the graph                                 */
} bfs_info;

/* Per-run counters (cheap; filled by bfs_run when stats != NULL). Sums over local ranks. */
typedef struct {
  int nlevels;               /* BFS levels executed (including the final empty one)        */
  uint64_t edges_scanned;    /* CSC entries expanded (sum over levels of cumul[n])         */
  uint64_t frontier_columns; /* frontier columns with local degree > 0, summed over levels  */
  uint64_t reached;          /* owned vertices reached (level >= 0)                        */
  uint64_t bytes_exchanged;  /* bytes sent by this process's ranks over the transport
                                (per-level messages; counts and the end-of-search resolution
                                excluded)                                                    */
  uint64_t list_messages;    /* per-level messages sent as index lists (exchange 1 / 2)     */
  uint64_t kernel_launches;  /* libbfs200 kernels launched by the call (CUB/NCCL excluded)  */
  double finalize_ms;        /* output write (phase_timing only, else 0)                   */
  double resolve_ms;         /* end-of-search parent exchange, C > 1 (phase_timing only)   */
} bfs_stats;

/* Per-level phase times (milliseconds, CUDA events) of the last run with phase_timing. */
typedef struct {
  double expand_comm; /* column all-gather of the frontier bitmap        */
  double scan;        /* frontier unpack + degree exclusive scan    */
  double expand;      /* frontier expansion kernel                         (Alg.3)        */
  double parent;      /* parent claim of the rows discovered in the level  (Alg.3 l.17)   */
  double fold_comm;   /* row exchange of discovered-vertex bitmaps        */
  double update;      /* frontier update + pack    */
  double allreduce;   /* termination reduction + host read        */
  uint64_t frontier;  /* frontier columns with degree > 0 (all local ranks) */
  uint64_t edges;     /* CSC entries expanded (all local ranks)            */
} bfs_level_record;

/* ncclGetUniqueId into out[128] (call on rank 0 only). */
int bfs_nccl_unique_id(unsigned char* out128);

/* Build the partitioned graph.
 *   src, dst  : host or device arrays of nedges global vertex ids (the tuples this process
 *               contributes; with NCCL any split of the global list over ranks is allowed).
 *               Borrowed for the duration of the call only.  Tuples are undirected: both
 *               orientations are inserted; self-loops and duplicates are dropped
 *               from the CSC but counted for m_comp.
 *   nverts    : number of vertices, 1 <= nverts and npad < 2^32 (ids are stored as u32;
 *               UINT32_MAX is the "no parent candidate" sentinel). Same on every rank.
 *   R, C      : grid; R*C must equal comm->nranks (NCCL) -- with loopback any R, C >= 1.
 *   comm      : transport (see bfs_comm); NULL means single GPU, device 0, R = C = 1.
 *   opts      : NULL for defaults; copied.
 *   out       : receives the graph.
 * Errors: BFS_EINVAL (bad shape/args), BFS_ERANGE (endpoint >= nverts), BFS_ENOMEM,
 *         BFS_ECUDA, BFS_ENCCL.  On error *out is NULL. */
int bfs_graph_create(const uint64_t* src, const uint64_t* dst, uint64_t nedges, uint64_t nverts, int R, int C,
                     const bfs_comm* comm, const bfs_opts* opts, bfs_graph** out);

int bfs_graph_info(const bfs_graph* g, bfs_info* info);

/* Replace the options (E, phase timing, stream) used by later runs. */
int bfs_set_opts(bfs_graph* g, const bfs_opts* opts);

/* Degree of global vertex v in the simple undirected graph (distinct neighbours other than v).
 * Used by the harness to sample roots with degree >= 1. BFS_ERANGE if v >= nverts. */
int bfs_degree(bfs_graph* g, uint64_t v, uint64_t* degree);

/* One BFS from `root` (Alg.2).  Writes info.nout entries of parent[] (int64 global ids) and
 * level[] (int32), element t describing global vertex info.first_vertex + t; either may be a
 * host or a device pointer (or NULL to skip).  Unreached vertices (and padding vertices) get
 * level = -1, parent = -1; parent[root] = root.  Outputs are written only on success.
 * BFS_ERANGE if root >= nverts (outputs untouched).  Every rank passes the same root.
 * Returns after the outputs are complete (the stream is synchronised). */
int bfs_run(bfs_graph* g, uint64_t root, int64_t* parent, int32_t* level, bfs_stats* stats);

/* n BFS back to back (the Graph500 loop over sampled roots): root k = roots[k]
 * (host array) writes its outputs to parent[k] / level[k], each an array like bfs_run's (host
 * or device; parent / level themselves may be NULL, or any entry NULL, to skip that output).
 * With host outputs, root k's device-to-host copies run on a second stream while root k+1
 * searches (two device staging buffers per local rank, allocated on the first such batch; the
 * copies only overlap if the host buffers are page-locked, e.g. cudaHostRegister / pinned).
 * Entries may repeat a buffer: its contents are then those of the last root written to it.
 * stats: NULL or an array of n records.  Returns after every output is complete; on an error
 * the outputs of the failing root and any later root are undefined.  BFS_ERANGE if any root >=
 * nverts (nothing run), BFS_EINVAL if n < 0 or roots is NULL with n > 0.  Every rank passes the
 * same roots (COLLECTIVE like bfs_run). */
int bfs_run_batch(bfs_graph* g, const uint64_t* roots, int n, int64_t* const* parent, int32_t* const* level,
                  bfs_stats* stats);

/* m_comp of the last run: number of input tuples whose source was reached, duplicates and
 * self-loops included (the TEPS numerator).  Summed over all ranks. */
int bfs_mcomp(bfs_graph* g, uint64_t* m_comp);

/* Per-level phase times of the last run (requires opts.phase_timing). Writes up to
 * max_levels records and the number of recorded levels to *nlevels: every level of the run,
 * except that records stop after the first 4096 levels (a deeper BFS, e.g. on a long path, runs
 * to completion; bfs_stats.nlevels and its totals cover every level).  Synchronises on the
 * recorded events. */
int bfs_level_times(bfs_graph* g, bfs_level_record* out, int max_levels, int* nlevels);

/* Gather the outputs of every rank on rank 0 (untimed, for validation).
 * COLLECTIVE over the R*C ranks (NCCL point-to-point sends to world rank 0); with the loopback
 * transport the process already holds every rank and the call is a copy.
 *   parent, level        : this process's bfs_run outputs (info.nout entries each; host or
 *                          device), or NULL to skip -- NULL-ness must agree on every rank.
 *   parent_all, level_all: on world rank 0 only (ignored elsewhere, may be NULL there):
 *                          info.npad entries each (host or device), entry t = global vertex t
 *                          (rank r's slice lands at r*block; padding vertices are -1 / -1).
 * Errors: BFS_EINVAL (rank 0 misses an output for a non-NULL input), BFS_ENOMEM, BFS_ECUDA,
 * BFS_ENCCL (the latter two are fatal for the graph). */
int bfs_gather(bfs_graph* g, const int64_t* parent, const int32_t* level, int64_t* parent_all, int32_t* level_all);

/* NULL-safe, idempotent for NULL.  Collective with NCCL. */
void bfs_destroy(bfs_graph* g);

/* Edge-list files (the paper's real-world graphs from the Stanford Large
 * Network Dataset Collection), for bfs_graph_create:
 *   BFS_FMT_SNAP_TEXT    lines of two whitespace-separated decimal ids (extra fields ignored);
 *                        lines starting with '#' or '%' and blank lines are skipped;
 *   BFS_FMT_BINARY_PAIRS consecutive 16-byte records of two little-endian u64 ids.
 * Host only (no GPU).  On success *src / *dst are malloc'ed arrays of *nedges tuples in file
 * order (duplicates and self-loops kept: they count for m_comp) owned by the caller (release with
 * bfs_free_edges), and *nverts = max id + 1 (0 for an empty file; bfs_graph_create pads it).
 * Errors (nothing allocated, outputs zeroed): BFS_EINVAL (null argument, unknown format, file
 * cannot be opened), BFS_EPARSE (malformed line -- bfs_last_error names file:line -- or a binary
 * file whose size is not a multiple of 16), BFS_ERANGE (an id >= 2^48), BFS_ENOMEM. */
enum { BFS_FMT_SNAP_TEXT = 0, BFS_FMT_BINARY_PAIRS = 1 };
int bfs_load_edges(const char* path, int format, uint64_t** src, uint64_t** dst, uint64_t* nedges, uint64_t* nverts);
void bfs_free_edges(uint64_t* src, uint64_t* dst);

const char* bfs_strerror(int status);
const char* bfs_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* BFS200_H */
