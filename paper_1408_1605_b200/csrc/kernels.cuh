// kernels.cuh -- launchers for the hot-path kernels (sm_100a).  See kernels.cu.
#pragma once
#include "bfs_internal.h"

namespace bfs200 {

// Launch attributes of the hot-path kernels on the current device (call once per graph).
cudaError_t kernels_init_device();

// Alg.2 init lines P:334-343: reset per-search state of one rank and seed the root on its owner.
// fused: the frontier update of a 1x1 graph runs in the next level's count pass (no K2; see
// FusedUpd in kernels.cu): the root is seeded into vis only
cudaError_t launch_init(const Geom& g, Rank& rk, bool owner, uint64_t root, bool fused, cudaStream_t s);

// K3: frontier bitmap (ncols bits) -> ascending list of columns with degree > 0, their row
// offsets and the exclusive scan of their degrees.
// narrow: every CSC position of the rank fits in 32 bits and K1 runs its POS32 variant (the row
// offsets and the degree scan are then written as 32-bit values)
// ctrl != null: fused frontier update of a 1x1 graph (the count pass builds the frontier from
// vis & ~vold, advances vold, writes the previous level's levels)
cudaError_t launch_scan(const Geom& g, Rank& rk, uint32_t tile_edges, bool narrow, const LevelCtrl* ctrl,
                        cudaStream_t s);

// K1: top-down frontier expansion (Alg.3, grouped edges P:565-586).
cudaError_t launch_expand(const Geom& g, Rank& rk, int edges_per_thread, uint64_t hot_h, bool force_pos64,
                          cudaStream_t s);
uint32_t expand_tile_edges(int edges_per_thread);

// K4: parent claim for the rows discovered in this level (+ pack of the fold message, C > 1).
cudaError_t launch_parent(const Geom& g, Rank& rk, bool fused, bool force_ptr64, cudaStream_t s);

// K2: frontier update + pack; lvl is the level being assigned.
cudaError_t launch_update(const Geom& g, Rank& rk, const LevelCtrl* ctrl, cudaStream_t s);

// Level control: reset (lvl = 1) and end-of-level bookkeeping / termination.
cudaError_t launch_level_begin(LevelCtrl* ctrl, cudaStream_t s);
cudaError_t launch_level_end(LevelCtrl* ctrl, const LevelInfo* infos, int nlocal, bool distributed,
                             cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t s);

// Finalize: parent/level outputs for owned vertices whose parent is local.
cudaError_t launch_finalize(const Geom& g, Rank& rk, int64_t* parent_out, int32_t* level_out, bool direct,
                            cudaStream_t s);

// Parent resolution (C > 1): build request bitmaps and answer requests (k_finalize reads them).
cudaError_t launch_req_build(const Geom& g, Rank& rk, cudaStream_t s);
cudaError_t launch_popc_scan(const uint32_t* bits, uint32_t* off, uint64_t nwords, void* tmp, size_t tmp_bytes,
                             cudaStream_t s);
size_t popc_scan_tmp_bytes(uint64_t nwords);
cudaError_t launch_resp_pack(const Geom& g, Rank& rk, cudaStream_t s);
// peer exchange variants (stores into the peers' reqin / respin through rk.reqin_dst / respin_dst)

cudaError_t launch_seg_totals(const uint32_t* off, uint64_t W, int C, unsigned long long* totals, cudaStream_t s);

// List exchange (opts.exchange): per-segment set-bit counts (added into cnt[k]),
// bitmap segments -> ascending local index lists (list segment k at k*lstride), and lists -> bits
// (OR into a zeroed bitmap segment).
cudaError_t launch_seg_popc(const uint32_t* bm, uint64_t W, int nseg, unsigned long long* cnt, uint64_t* launches,
                            cudaStream_t s);
size_t list_encode_tmp_bytes(uint64_t nwords);
cudaError_t launch_list_encode(const uint32_t* bm, uint64_t W, int nseg, uint32_t* off, void* tmp, size_t tmp_bytes,
                               uint32_t* list, uint64_t lstride, int nsm, uint64_t* launches, cudaStream_t s);
cudaError_t launch_list_scatter(const uint32_t* list, uint64_t n, uint32_t* bm, int nsm, uint64_t* launches,
                               cudaStream_t s);

// Peer exchange (opts.peer_exchange): cross-GPU flag barrier over NVLink peer memory (optionally
// summing the ranks' new-vertex counts into info->newv), and the root bit for column peers.
cudaError_t launch_xbarrier(XSig* local, XSig* const* peers, int nranks, int me, unsigned long long* epoch_ctr,
                            LevelInfo* info, bool sum_newv, int* err, cudaStream_t s);
cudaError_t launch_seed_col(uint32_t* all_front, const uint32_t* perm_fwd, uint64_t root, uint64_t block, int i_owner,
                            cudaStream_t s);

// m_comp: sum of tdeg over reached owned vertices into *out (device u64).
cudaError_t launch_mcomp(const Geom& g, Rank& rk, unsigned long long* out, cudaStream_t s);

// Degree of local column u summed into *out (device u64).
cudaError_t launch_degree(const Geom& g, Rank& rk, const uint32_t* perm_fwd, uint64_t v, unsigned long long* out,
                          cudaStream_t s);

}  // namespace bfs200
