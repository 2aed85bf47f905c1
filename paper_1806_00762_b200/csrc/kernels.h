// Host-callable launchers for the sm_100a kernels in kernels.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_types.h"

namespace seraph {

// K1 / K7: dense pull relaxation over a set of tile segments.
void launch_pull(int algo, int gate, bool det, const PullArgs& a, int grid, cudaStream_t s);
// K2: reentry runs of one page set in one cooperative launch (false: the
// grid does not fit co-resident -- the caller launches the runs itself).
bool launch_pull_reentry(int algo, int gate, const PullArgs& a, const ReentryArgs& r, int grid,
                         cudaStream_t s);
// Deterministic mode commit: values[v] = next[v] for v in [lo, hi).
void launch_commit(uint32_t* values, const uint32_t* next, uint32_t lo, uint32_t hi,
                   cudaStream_t s);
// K8: PageRank pull-sum + hub finalize.
// Kernels launched so far by the calling thread (all launch_* wrappers).
uint64_t kernel_launch_count();
void launch_pr_pull(const PrArgs& a, int grid, cudaStream_t s);
int pr_hot_warps();
int pr_hot_blocks_per_sm(uint32_t n_hot);
uint32_t pr_hot_table_max();
// K8 hot-source staging (pr_pull_kernel<true>): per-iteration compaction of
// the hot contributions, threshold count, slot assignment, source encoding.
void launch_pr_hot_gather(const uint32_t* hot_vertex, uint32_t n_hot, const float* contrib,
                          float* hot_contrib, cudaStream_t s);
void launch_count_deg_ge(const uint32_t* deg, uint32_t n, uint32_t d, unsigned long long* out,
                         cudaStream_t s);
// out <- sum of counter slots [from, to) (the per-round aggregate a world reduces)
void launch_sum_ctr_slots(const RunCtr* slots, uint32_t from, uint32_t to, RunCtr* out,
                          cudaStream_t s);

void launch_hot_assign(const uint32_t* deg, uint32_t n, uint32_t d, uint32_t cap,
                       unsigned* counter, uint32_t* slot_of, uint32_t* hot_vertex, cudaStream_t s);
void launch_hot_encode(const uint32_t* in, uint32_t* out, uint64_t words, const uint32_t* slot_of,
                       uint32_t n, cudaStream_t s);
// Sparse push enumerated from the CSC pages (push adjacency not derived):
// relaxes the in-edges whose source is in a.list (n_list entries).
void launch_push_scan(int algo, const PushArgs& a, const PageDesc* pages, uint32_t n_pages,
                      uint32_t* fbits, uint32_t n, int grid, cudaStream_t s);
void launch_pr_hub_finalize(const uint32_t* hub_vertex, uint32_t n_hubs, float* hub_sum,
                            float* rank_out, float* contrib_out, const float* inv_outdeg,
                            float base, float damp, cudaStream_t s);
void launch_pr_init(float* rank, float* contrib, const float* inv_outdeg, uint32_t n,
                    float init, cudaStream_t s);
void launch_inv_outdeg(const unsigned long long* out_offsets, uint32_t n, float* inv,
                       cudaStream_t s);
// K3: sparse push over the compacted frontier.
void launch_push(int algo, bool det, const PushArgs& a, int grid, cudaStream_t s);
// Persistent sparse stage (cooperative launch): occupancy and launcher.
// Deterministic push commit: for changed v with next[v] < values[v].
void launch_push_commit(uint32_t* values, const uint32_t* next, const uint8_t* changed,
                        uint32_t n, RunCtr* ctr, Census* c, cudaStream_t s);
// K4/K5: per-pass census (+ weak DFA step, prediction log, status histogram).
constexpr uint32_t kCensusBlockVerts = 4096;
// pub.done != null: the census's last block also publishes the census and
// pub.n_ctr run counters into the mapped pinned buffers (launch_publish fused)
struct Publish {
  Census* cz_host;
  const RunCtr* ctr;
  RunCtr* ctr_host;
  uint32_t n_ctr;
  unsigned* done;  // zeroed block ticket (the last block resets it)
  unsigned* seq_host = nullptr;  // pinned: `seq` stored last, after a system fence
  unsigned seq = 0;
};
void launch_census(uint32_t n, const uint8_t* changed, uint8_t* status, uint8_t* logstate,
                   const uint32_t* outdeg, int pass_kind, uint32_t own_lo,
                   uint32_t own_hi, uint32_t* blk_cnt, unsigned long long* blk_edges,
                   unsigned long long* part, Census* c, const Publish& pub, cudaStream_t s);
void launch_scan_blocks(uint32_t nblocks, uint32_t* blk_cnt, unsigned long long* blk_edges,
                        cudaStream_t s);
void launch_compact(uint32_t n, uint32_t own_lo, uint32_t own_hi, uint8_t* changed,
                    const uint32_t* outdeg, const uint32_t* blk_off,
                    const unsigned long long* blk_eoff, uint32_t* list, unsigned long long* pref,
                    uint32_t* chunk_start, uint32_t shift, cudaStream_t s);
// Multi-GPU: flag vertices improved by any rank during the round.
void launch_mark_changed(uint32_t n, const uint32_t* values, const uint32_t* snap,
                         uint8_t* changed, cudaStream_t s);
// Streaming: point a page descriptor at the slot now holding the page.
void launch_set_page_desc(PageDesc* d, uint32_t page, const uint32_t* offs, const uint32_t* src,
                          const uint32_t* w, cudaStream_t s);
// K6: strong CC threshold (net label-population change since the last refresh).
// Device-side CSR adjacency from resident CSC pages; out-degrees (u32).
void launch_csr_from_pages(const uint4* tiles, const uint32_t* tile_page, const PageDesc* pages,
                           uint32_t tile_lo, uint32_t tile_hi, unsigned long long* cursor,
                           uint32_t* out_nbr, uint32_t* out_w, int grid, cudaStream_t s);
void launch_outdeg(const unsigned long long* off, uint32_t n, uint32_t* deg, cudaStream_t s);
// Source-blocked page split for PageRank locality (count / scan / scatter)
// and the per-iteration finalize of the accumulated partial sums.
void launch_src_block(int mode, const uint4* tiles, const uint32_t* tile_page,
                      const PageDesc* pages, uint32_t tile_lo, uint32_t tile_hi, uint32_t n,
                      uint32_t blk_verts, uint32_t n_pages, uint32_t* cnt,
                      unsigned long long* goff, uint32_t* out_src, uint32_t* out_w, int grid,
                      cudaStream_t s);
// Page-major per-page build of the sub-pages of page p (after its count):
// scan, sub-page bases, u32 local offsets and absolute scatter cursors.
void launch_src_block_page(const uint32_t* cnt, unsigned long long* goff, const PageDesc* pages,
                           uint32_t p, uint32_t vb, uint32_t range, uint32_t n, uint32_t cap,
                           uint32_t n_pages, uint32_t n_blocks, unsigned long long page_base,
                           unsigned long long* bp_edges, unsigned long long* bp_base,
                           uint32_t* offs, unsigned long long* part, cudaStream_t s);
// chunk-sum temporaries launch_src_block_page needs for pages of <= cap vertices
uint32_t src_block_scan_parts(uint32_t cap, uint32_t n_blocks);

// Tile cut of the source-blocked sub-pages on the device, one 128-destination
// window per thread: mode 0 writes the tile count of every window to cnt
// (sub_tile_windows entries, block-major); mode 1 writes the tiles at the
// exclusive scan `at` of those counts.
uint64_t sub_tile_windows(uint32_t cap, uint32_t n_pages, uint32_t n_blocks);
void launch_sub_tiles(int mode, uint32_t n, uint32_t cap, uint32_t n_pages, uint32_t n_blocks,
                      uint32_t own_lo, uint32_t own_hi, const uint32_t* offs, uint32_t* cnt,
                      const uint32_t* at, uint4* tiles, uint32_t* tile_page, cudaStream_t s);
constexpr uint32_t kDegHistCap = 1024;  // degrees >= cap share the last histogram bucket
void launch_degree_hist(const uint32_t* outdeg, uint32_t n, unsigned long long* hist_v,
                        unsigned long long* hist_e, cudaStream_t s);
// Frontier queue (q entries) -> exclusive out-degree prefix (q+1 entries)
// and push-chunk starts, the inputs of launch_push.
// census + n_ctr run counters -> mapped pinned host memory (one kernel)
void launch_publish(const Census* cz, Census* cz_host, const RunCtr* ctr, RunCtr* ctr_host,
                    uint32_t n_ctr, unsigned* seq_host, unsigned seq, cudaStream_t s);
// consecutive small-frontier sparse passes in one single-block launch
void launch_tail_loop(int algo, const TailArgs& a, cudaStream_t s);
void launch_seed_queue(uint32_t source, const uint32_t* outdeg, uint32_t* list, Census* cz,
                       cudaStream_t s);
size_t queue_prep_temp_bytes(uint32_t max_q);
void launch_queue_prep(const uint32_t* list, uint32_t q, const uint32_t* outdeg,
                       unsigned long long* pref, uint32_t* chunk_start, uint32_t shift,
                       uint64_t total_edges, void* tmp, size_t tmp_bytes, cudaStream_t s);
size_t exclusive_scan_u32_temp_bytes(size_t count);
void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t count, void* tmp,
                               size_t tmp_bytes, cudaStream_t s);


void launch_pr_block_finalize(uint32_t lo, uint32_t hi, float* acc, float* rank_out,
                              float* contrib_out, const float* inv_outdeg, float base, float damp,
                              cudaStream_t s);
// Values initialisation (VertexProgram::init, programs.hpp:20-28).
void launch_init_values(int algo, uint32_t source, uint32_t n, uint32_t* values,
                        cudaStream_t s);
void launch_init_hub_stamp(uint32_t* stamp, uint32_t n, cudaStream_t s);
// Fixpoint-law verifier.
void launch_verify(int algo, uint32_t lo, uint32_t hi, const unsigned long long* out_offsets,
                   const uint32_t* nbr, const uint32_t* w, const uint32_t* values,
                   unsigned long long* violations, cudaStream_t s);

int pull_blocks_per_sm(int algo, int gate, bool det);

}  // namespace seraph
