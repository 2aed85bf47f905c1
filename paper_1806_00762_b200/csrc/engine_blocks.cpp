// Source-blocked sweeps (K1 and K8 over per-source-block sub-pages, the
// persisting-L2 window, the blocking heuristics) and the PageRank driver.
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace seraph {

// ---------------------------------------------------------------------------
// Source-blocked sub-pages for PageRank: when the contrib array outgrows the
// L2, every iteration sweeps the sub-pages block by block so the gathers of
// one sweep stay inside a blk_verts slice (PageRank: SERAPH_PR_BLOCK_VERTS,
// default 32 Mi vertices = 128 MB of f32; K1: pull_block_verts; 0 disables).
// ---------------------------------------------------------------------------
bool Engine::build_src_blocks(uint64_t blk) {
  if (sb_.built && sb_.blk_verts == blk) return true;
  if (!sb_begin(blk)) return false;
  for (uint32_t p = 0; p < pages_.size(); ++p) sb_page(p);
  return sb_finish();
}

// Page-major layout: sub-page (p, b) at page_base[p] + sum_{b'<b} pad8(edges(p, b')),
// page_base[p] = sum_{q<p} (pad8(edges(q)) + 8 * n_blocks), all 32 B aligned
// (K1/K8 read aligned uint4 runs): every page's sub-pages are
// built from that page alone (sb_page), so sr_run_graph builds them page by
// page while the rest of the page set is still crossing the host link.
bool Engine::sb_begin(uint64_t blk) {
  sb_.built = false;
  sb_.pending = false;
  if (pr_hot_.blocked) pr_hot_.built = false;
  if (!all_resident_) return false;  // sharded ranks block their own destinations
  if (blk == 0 || n_ <= blk || page_n_ != n_) return false;
  const uint32_t np = uint32_t(pages_.size());
  for (uint32_t p = 0; p < np; ++p)
    if (pages_[p].vb != uint64_t(p) * cap_) return false;  // uniform cut (graph.cpp:75-92)
  const uint32_t nb = uint32_t((n_ + blk - 1) / blk);
  sb_.page_base.assign(np, 0);
  unsigned long long at = 0;
  for (uint32_t p = 0; p < np; ++p) {
    sb_.page_base[p] = at;
    if (pages_[p].tile_end > pages_[p].tile_begin) at += pad8(pages_[p].edges) + 8ull * nb;
  }
  sb_.t_cnt.reserve(size_t(nb) * n_);
  sb_.t_goff.reserve(size_t(nb) * n_);
  sb_.bp_edges.reserve(size_t(nb) * np);
  sb_.bp_base.reserve(size_t(nb) * np);
  sb_.t_part.reserve(std::max<uint32_t>(src_block_scan_parts(cap_, nb), 1));
  SR_CUDA(cudaMemsetAsync(sb_.bp_edges.p, 0, size_t(nb) * np * 8, cs_));
  SR_CUDA(cudaMemsetAsync(sb_.bp_base.p, 0, size_t(nb) * np * 8, cs_));
  sb_.src.reserve(at + 8);
  if (weighted_) sb_.w.reserve(at + 8);
  else sb_.w.release();
  const size_t per_block = size_t(n_) + np;
  sb_.offs.reserve(size_t(nb) * per_block);
  sb_.blk_verts = uint32_t(blk);
  sb_.n_blocks = nb;
  sb_.pending = true;
  return true;
}

void Engine::sb_page(uint32_t p) {
  const PageMeta& pm = pages_[p];
  if (pm.tile_end <= pm.tile_begin) return;  // not this rank's / no in-edges
  const uint32_t nb = sb_.n_blocks, np = uint32_t(pages_.size());
  const uint32_t range = pm.ve - pm.vb;
  // 1) counts per (block, destination) of this page
  SR_CUDA(cudaMemset2DAsync(sb_.t_cnt.p + pm.vb, size_t(n_) * 4, 0, size_t(range) * 4, nb, cs_));
  launch_src_block(0, tiles_.p, tile_page_.p, page_desc_.p, pm.tile_begin, pm.tile_end, n_,
                   sb_.blk_verts, np, sb_.t_cnt.p, nullptr, nullptr, nullptr, sm_count_ * 8, cs_);
  // 2) page-local offsets, sub-page sizes and bases, u32 offsets, cursors
  launch_src_block_page(sb_.t_cnt.p, sb_.t_goff.p, page_desc_.p, p, pm.vb, range, n_, cap_, np,
                        nb, sb_.page_base[p], sb_.bp_edges.p, sb_.bp_base.p, sb_.offs.p,
                        sb_.t_part.p, cs_);
  // 3) scatter the sources (one atomic per edge on the cursors)
  launch_src_block(1, tiles_.p, tile_page_.p, page_desc_.p, pm.tile_begin, pm.tile_end, n_,
                   sb_.blk_verts, np, nullptr, sb_.t_goff.p, sb_.src.p,
                   weighted_ ? sb_.w.p : nullptr, sm_count_ * 8, cs_);
}

bool Engine::sb_finish() {
  if (!sb_.pending) return sb_.built;
  sb_.pending = false;
  const uint32_t nb = sb_.n_blocks, np = uint32_t(pages_.size());
  const bool timing = std::getenv("SERAPH_TIMING") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<unsigned long long> edges_h(size_t(nb) * np), base_h(size_t(nb) * np);
  SR_CUDA(cudaMemcpyAsync(edges_h.data(), sb_.bp_edges.p, edges_h.size() * 8,
                          cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaMemcpyAsync(base_h.data(), sb_.bp_base.p, base_h.size() * 8, cudaMemcpyDeviceToHost,
                          cs_));
  // the tile cut on the device (per 128-destination window of every sub-page)
  const size_t K = sub_tile_windows(cap_, np, nb);
  const size_t K_blk = K / nb;  // windows per block
  DBuf<uint32_t>& tcnt = sb_.t_tcnt;
  DBuf<uint32_t>& tat = sb_.t_tat;
  tcnt.reserve(K + 1);
  tat.reserve(K + 1);
  SR_CUDA(cudaMemsetAsync(tcnt.p + K, 0, 4, cs_));
  launch_sub_tiles(0, n_, cap_, np, nb, own_lo_, own_hi_, sb_.offs.p, tcnt.p, nullptr, nullptr,
                   nullptr, cs_);
  sb_.t_scan.reserve(exclusive_scan_u32_temp_bytes(K + 1));
  launch_exclusive_scan_u32(tcnt.p, tat.p, K + 1, sb_.t_scan.p, sb_.t_scan.n, cs_);
  sb_.block_tile_begin.assign(nb + 1, 0);
  for (uint32_t b = 0; b <= nb; ++b)
    SR_CUDA(cudaMemcpyAsync(&sb_.block_tile_begin[b], tat.p + size_t(b) * K_blk, 4,
                            cudaMemcpyDeviceToHost, cs_));
  // first tile of every sub-page (b, p) (windows are block-major, page-major
  // inside a block): the diagonal-first launch order of pull_blocked_pass
  const size_t wpp = K_blk / std::max<uint32_t>(np, 1);
  sb_.sub_tile_begin.assign(size_t(nb) * np + 1, 0);
  for (size_t k = 0; k <= size_t(nb) * np; ++k)
    SR_CUDA(cudaMemcpyAsync(&sb_.sub_tile_begin[k], tat.p + k * wpp, 4, cudaMemcpyDeviceToHost,
                            cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  const uint32_t n_sub_tiles = sb_.block_tile_begin[nb];
  sb_.tiles.reserve(std::max<size_t>(n_sub_tiles, 1));
  sb_.tile_page.reserve(std::max<size_t>(n_sub_tiles, 1));
  launch_sub_tiles(1, n_, cap_, np, nb, own_lo_, own_hi_, sb_.offs.p, nullptr, tat.p, sb_.tiles.p,
                   sb_.tile_page.p, cs_);
  SR_CUDA(cudaGetLastError());
  const size_t per_block = size_t(n_) + np;
  std::vector<PageDesc> desc(size_t(nb) * np);
  for (uint32_t b = 0; b < nb; ++b)
    for (uint32_t p = 0; p < np; ++p) {
      PageDesc& d = desc[size_t(b) * np + p];
      d.vertex_begin = pages_[p].vb;
      d.range = pages_[p].ve - pages_[p].vb;
      d.edge_count = edges_h[size_t(b) * np + p];
      d.offs = sb_.offs.p + size_t(b) * per_block + size_t(p) * cap_ + p;
      d.src = sb_.src.p + base_h[size_t(b) * np + p];
      d.w = weighted_ ? sb_.w.p + base_h[size_t(b) * np + p] : nullptr;
    }
  sb_.desc.reserve(desc.size());
  SR_CUDA(cudaMemcpyAsync(sb_.desc.p, desc.data(), desc.size() * sizeof(PageDesc),
                          cudaMemcpyHostToDevice, cs_));
  sb_.acc.reserve(n_);
  SR_CUDA(cudaMemsetAsync(sb_.acc.p, 0, size_t(n_) * 4, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  if (timing)
    std::fprintf(stderr, "[seraph] src blocks finish (after the last page): %.1f ms\n",
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                     .count());
  sb_.built = true;
  return true;
}

// Source-blocked dense pull (K1): when the vertex array outgrows the L2,
// a baseline-schedule dense pass sweeps the source-blocked sub-pages block by
// block, so every launch gathers from one blk-vertex slice that stays in
// L2 instead of 32-byte DRAM sectors spread over the whole array.
// SERAPH_PULL_BLOCK_VERTS: block size (0 = off; default 16 Mi vertices =
// 64 MB of values, used when the array exceeds half the L2).  Values are
// unchanged (min-combine is order independent; every destination sees
// every in-edge once per pass).  Attempts/skips are counted on block 0,
// edges on every block, valid updates = destinations changed in the pass.
//
// Blocking pays only when the unblocked gathers have no L2 locality: by
// default it is used when the vertex array exceeds half the L2 AND the
// sources that fit there (the L2/8 highest out-degree vertices) carry less
// than half of the edges -- true for uniform graphs (C4: ~15 %), false for
// RMAT, whose hubs stay L2-resident anyway (RMAT-26 SSSP: 10.1 ms unblocked
// vs 10.9 ms blocked; uniform-27 CC: 122 ms vs 22 ms).
uint64_t Engine::pull_block_verts() {
  uint64_t blk = 16ull << 20;
  const char* env = std::getenv("SERAPH_PULL_BLOCK_VERTS");
  if (env) blk = std::strtoull(env, nullptr, 10);
  if (blk == 0 || n_ <= blk) return 0;
  if (env) return blk;
  if (uint64_t(n_) * 4 <= uint64_t(l2_bytes_) / 2) return 0;
  return hot_source_coverage(uint64_t(l2_bytes_) / 8) < 0.5 ? blk : 0;
}

uint64_t Engine::pr_block_verts() const {
  uint64_t pr_blk = 32ull << 20;  // tools/pr_blocks.py: 32 Mi best on RMAT-26, smaller lose
  if (const char* e = std::getenv("SERAPH_PR_BLOCK_VERTS")) pr_blk = std::strtoull(e, nullptr, 10);
  return pr_blk < n_ ? pr_blk : 0;
}

// Fraction of the edges whose source is among the k highest out-degree
// vertices (degree histogram on the device; cached per CSR).
double Engine::hot_source_coverage(uint64_t k) {
  if (coverage_k_ == k && coverage_ >= 0) return coverage_;
  DBuf<unsigned long long> hv, he;
  hv.reserve(kDegHistCap + 1);
  he.reserve(kDegHistCap + 1);
  SR_CUDA(cudaMemsetAsync(hv.p, 0, (kDegHistCap + 1) * 8, cs_));
  SR_CUDA(cudaMemsetAsync(he.p, 0, (kDegHistCap + 1) * 8, cs_));
  launch_degree_hist(outdeg_.p, n_, hv.p, he.p, cs_);
  std::vector<unsigned long long> v(kDegHistCap + 1), e(kDegHistCap + 1);
  SR_CUDA(cudaMemcpyAsync(v.data(), hv.p, v.size() * 8, cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaMemcpyAsync(e.data(), he.p, e.size() * 8, cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  uint64_t total = 0;
  for (auto x : e) total += x;
  double covered = 0;
  uint64_t left = k;
  for (int d = int(kDegHistCap); d >= 0 && left; --d) {
    const uint64_t take = std::min<uint64_t>(left, v[d]);
    if (v[d]) covered += double(e[d]) * double(take) / double(v[d]);
    left -= take;
  }
  coverage_k_ = k;
  coverage_ = total ? covered / double(total) : 1.0;
  return coverage_;
}

// Pin the gathered slice of a source block in L2 for the launches that
// follow on the compute stream (cudaAccessPolicyWindow, persisting lines;
// the streamed page arrays are loaded evict-first).  bytes == 0 clears it.
// SERAPH_L2_PERSIST=0 disables.  Measured: uniform-27 CC 22.3 -> 21.8 ms;
// PageRank's 128 MB contribution blocks exceed the carve-out (105.9 vs
// 103.2 ms with it), so K8 does not use it.
void Engine::l2_window(const void* base, size_t bytes) {
  if (l2_persist_max_ < 0) {
    int mx = 0;
    l2_persist_max_ =
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev_) == cudaSuccess ? mx : 0;
  }
  const char* e = std::getenv("SERAPH_L2_PERSIST");
  if (e && std::atoi(e) == 0) bytes = 0;
  if (!l2_persist_max_ || (bytes == 0 && !l2_window_set_)) return;
  // the persisting carve-out shrinks the normal L2 for everything else: it
  // exists only while a window is set
  if (bytes && !l2_window_set_)
    SR_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, size_t(l2_persist_max_)));
  cudaStreamAttrValue attr{};
  attr.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  attr.accessPolicyWindow.num_bytes = bytes;
  attr.accessPolicyWindow.hitRatio =
      bytes ? float(std::min(1.0, double(l2_persist_max_) / double(bytes))) : 0.f;
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  SR_CUDA(cudaStreamSetAttribute(cs_, cudaStreamAttributeAccessPolicyWindow, &attr));
  l2_window_set_ = bytes != 0;
  if (!bytes) {
    SR_CUDA(cudaCtxResetPersistingL2Cache());
    SR_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0));
  }
}

bool Engine::pull_blocked_pass(int gate, RunCtr* ctr, bool count_valid) {
  const uint64_t blk = pull_block_verts();
  if (!blk || !build_src_blocks(blk)) return false;
  const uint32_t run_id = ++run_id_;
  uint32_t last_b = sb_.n_blocks;  // the last block with tiles gets its own counter slot
  for (uint32_t b = 0; b < sb_.n_blocks; ++b)
    if (sb_.block_tile_begin[b + 1] > sb_.block_tile_begin[b]) last_b = b;
  RunCtr* last_ctr = nullptr;
  if (last_b > 0 && last_b < sb_.n_blocks && size_t(ctr_used_) + 1 <= ctr_.n) {
    last_ctr = alloc_ctr(1);
    sb_last_slot_ = int(last_ctr - ctr_.p);
  }
  // LIST variant for a block launch expected to gather little: the previous
  // block's probe (or, for block 0, the previous pass) gathered for < 30 %
  double prev_frac = last_block_gather_frac_;
  bool list = false, root_done = false;
  auto make_args = [&](const Segments& seg, RunCtr* slot, bool count_dest, bool count_v,
                       uint32_t rid) {
    PullArgs a{};
    a.list = list ? 1u : 0u;
    a.work = next_work_counter();
    a.tiles = sb_.tiles.p;
    a.tile_page = sb_.tile_page.p;
    a.pages = sb_.desc.p;
    a.seg = seg;
    a.values = values_.p;
    a.next = values_.p;
    a.changed = changed_.p;
    a.status = status_.p;
    a.hub_stamp = hub_stamp_.p;
    a.run_id = rid;
    a.ctr = slot;
    a.census = census_.p;
    a.count_dest = count_dest ? 1u : 0u;
    a.count_valid = count_v ? 1u : 0u;
    a.peers = peer_list();
    a.n_peers = n_peers_;
    a.k_bfs = k_bfs_;
    a.s_cc = s_cc_;
    a.l_sssp = l_sssp_;
    a.src_floor = floor_sssp_;
    a.floor_step = weights_ge1_ ? 1u : 0u;
    return a;
  };
  auto grid_of = [&](const Segments& seg) {
    const uint32_t tasks = seg.task_prefix[seg.n];
    return std::max(1, int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                              (uint64_t(tasks) + kWarpsPerBlock - 1) /
                                                  kWarpsPerBlock)));
  };
  auto launch_range = [&](const Segments& seg, RunCtr* slot, bool count_dest, bool count_v,
                          uint32_t rid) {
    PullArgs a = make_args(seg, slot, count_dest, count_v, rid);
    const int grid = grid_of(seg);
    // sub-page tiles are small and numerous: big launches grab 8 tiles
    // (CC uniform-26: 4 -> 8, 9.0 -> 8.6 ms); a sharded rank's clipped
    // blocks get the same per-launch share rule as launch_pages
    a.grab = k1_grab(seg.task_prefix[seg.n], grid, "SERAPH_K1_GRAB_BLOCKED");
    auto* evp = relax_begin();
    launch_pull(algo_, gate, false, a, grid, cs_);
    SR_CUDA(cudaGetLastError());
    if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
  };
  // K2 over the diagonal: up to `runs` sweeps in ONE cooperative launch that
  // stops at the first quiet sweep (false: not co-resident -> host loop)
  auto diag_loop_device = [&](const Segments& seg, int runs, bool count_dest) {
    if (size_t(ctr_used_) + size_t(runs) > ctr_.n) return false;
    if (!work_.p || work_used_ + size_t(runs) > work_.n) {
      next_work_counter();
      if (work_used_ + size_t(runs) > work_.n) {
        SR_CUDA(cudaMemsetAsync(work_.p, 0, work_.n * sizeof(unsigned), cs_));
        work_used_ = 0;
      }
    }
    unsigned* work = work_.p + work_used_;
    if (!runs_done_.p) runs_done_.reserve(1);
    PullArgs a = make_args(seg, nullptr, count_dest, true, run_id_ + 1);
    const int grid = grid_of(seg);
    a.grab = k1_grab(seg.task_prefix[seg.n], grid, "SERAPH_K1_GRAB_BLOCKED");
    ReentryArgs r{work, ctr_.p + ctr_used_, 1u, uint32_t(runs), runs_done_.p, 0u};
    auto* evp = relax_begin();
    if (!launch_pull_reentry(algo_, gate, a, r, grid, cs_)) {
      if (evp) --relax_ev_used_;
      return false;
    }
    SR_CUDA(cudaGetLastError());
    if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
    work_used_ += size_t(runs);
    ctr_used_ += uint32_t(runs);
    run_id_ += uint32_t(runs);
    return true;
  };
  const int diag_iters = diag_local_iterations();
  int root_reps = algo_ == SR_ALGO_CC ? kRootDiagReps : 1;
  if (const char* e = std::getenv("SERAPH_ROOT_DIAG_REPS")) root_reps = std::max(1, std::min(64, std::atoi(e)));
  for (uint32_t b = 0; b < sb_.n_blocks; ++b) {
    const uint32_t t0 = sb_.block_tile_begin[b], t1 = sb_.block_tile_begin[b + 1];
    if (t1 <= t0) continue;
    l2_window(values_.p + uint64_t(b) * blk, std::min<uint64_t>(blk, n_ - uint64_t(b) * blk) * 4);
    // every block but the last counts into its own slot: the probe below
    // reads each block's gathers / edges
    RunCtr* slot = (b == last_b && last_ctr) ? last_ctr
                   : (b == 0 || size_t(ctr_used_) + 1 > ctr_.n) ? ctr
                                                                : alloc_ctr(1);
    uint32_t d0 = 0, d1 = 0;
    // (after the CC root block's sweeps carried label 0 out, the later
    // blocks' launches find most destinations at the floor: LIST too)
    list = list_ok() && (prev_frac < list_frac() || (b > 0 && root_done));
    if (diag_iters > 1 && diag_range(b, t0, t1, d0, d1)) {
      // Local convergence of the block's own subgraph (Seraph's multi-pass
      // subgraph iteration): the diagonal sub-pages -- edges whose source AND
      // destination lie in block b, values L2-resident -- are swept until a
      // sweep changes nothing (capped), then the block's other sub-pages once.
      const bool on_device = !std::getenv("SERAPH_DIAG_HOST_LOOP") &&
                             diag_loop_device(range_segments(d0, d1, 0, 0), diag_iters, b == 0);
      for (int it = 0; !on_device && it < diag_iters; ++it) {
        if (size_t(ctr_used_) + 1 > ctr_.n) break;
        RunCtr* ds = alloc_ctr(1);
        launch_range(range_segments(d0, d1, 0, 0), ds, b == 0 && it == 0, true, ++run_id_);
        if (it + 1 == diag_iters) break;
        SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ds, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
        SR_CUDA(cudaStreamSynchronize(cs_));
        if (ctr_h_.p[0].valid == 0) break;  // locally converged
      }
      launch_range(range_segments(t0, d0, d1, t1), slot, b == 0, count_valid, run_id);
    } else if (root_reps > 1 && b == 0 && diag_range(b, t0, t1, d0, d1)) {
      // Connected components: block 0 -- it holds vertex 0, the global
      // minimum label -- sweeps its own subgraph (the diagonal sub-pages,
      // labels L2-resident) root_reps times before its cross-block edges
      // carry label 0 to every other destination (local iteration of the
      // resident subgraph).  One launch per sweep: K1's phase C stores
      // assume one writer per destination per launch.  Measured: C4 15.45 ->
      // 10.0 ms (2 passes instead of 3); BFS on uniform-27 from the source's
      // block 58.2 -> 59.1 ms, so CC only.
      for (int r = 0; r < root_reps; ++r)
        launch_range(range_segments(d0, d1, 0, 0), slot, r == 0, count_valid, run_id);
      launch_range(range_segments(t0, d0, d1, t1), slot, true, count_valid, run_id);
      root_done = true;
    } else {
      // Diagonal first: the sub-pages whose destinations are this block's own
      // sources go first, so the labels / levels / distances they improve are
      // already visible to the rest of the launch's gathers (async, a15)
      launch_range(diag_first_segments(b, t0, t1), slot, b == 0, count_valid, run_id);
    }
    if (b < last_b && (b == 0 || probe_every_block())) {
      // Probe: blocking pays for gathers only.  If this block gathered for
      // < 5 % of its edges (converged labels/levels skip theirs), finish the
      // pass with one unblocked sweep -- destinations at the floor read no
      // edges there -- instead of more block launches that each scan every
      // destination (the relaxations are idempotent; the pass's counters
      // restart).  (Measured and dropped: finishing unblocked when < 1 % of
      // the destinations are still above the floor after block 0 -- on C4
      // that never fired, and its count + sync cost 0.2 ms.)
      SR_CUDA(cudaMemcpyAsync(ctr_h_.p, slot, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
      SR_CUDA(cudaStreamSynchronize(cs_));
      const RunCtr& c0 = ctr_h_.p[0];
      if (c0.edges > 0) prev_frac = double(c0.gathers) / double(c0.edges);
      if (c0.edges > 0 && double(c0.gathers) < 0.05 * double(c0.edges)) {
        // the reference's per-pass counters (attempts, valid, skipped,
        // edges_read) restart with the unblocked sweep; the work counters
        // (gathers, edges streamed, destinations scanned) keep what the
        // blocked launches did
        const size_t from = size_t(ctr - ctr_.p), k = size_t(ctr_used_) - from;
        SR_CUDA(cudaMemset2DAsync(ctr, sizeof(RunCtr), 0, 4 * sizeof(unsigned long long), k, cs_));
        sb_last_slot_ = -1;
        fallback_frac_ = double(c0.gathers) / double(c0.edges);
        l2_window(nullptr, 0);
        return false;
      }
    }
  }
  l2_window(nullptr, 0);
  return true;
}

// SERAPH_PROBE_BLOCKS=0: probe block 0 only (the round-1 rule).
bool Engine::probe_every_block() const {
  const char* e = std::getenv("SERAPH_PROBE_BLOCKS");
  return !e || std::atoi(e) != 0;
}

// SERAPH_DIAG_ITERS: sweeps of a block's diagonal before its other
// sub-pages (1 = the diagonal once, first in the block's launch).
int Engine::diag_local_iterations() const {
  int it = kDiagIters;
  if (const char* e = std::getenv("SERAPH_DIAG_ITERS")) it = std::max(1, std::min(64, std::atoi(e)));
  return it;
}

// Tiles of the sub-pages (b, p) whose destinations lie in block b.
bool Engine::diag_range(uint32_t b, uint32_t t0, uint32_t t1, uint32_t& d0, uint32_t& d1) const {
  const uint32_t np = uint32_t(pages_.size());
  if (sb_.sub_tile_begin.size() != size_t(sb_.n_blocks) * np + 1 || cap_ == 0) return false;
  const uint64_t lo = uint64_t(b) * sb_.blk_verts;
  const uint64_t hi = std::min<uint64_t>(lo + sb_.blk_verts, n_);
  if (hi <= lo) return false;
  const uint32_t p_lo = uint32_t(lo / cap_), p_hi = uint32_t(std::min<uint64_t>((hi - 1) / cap_ + 1, np));
  d0 = sb_.sub_tile_begin[size_t(b) * np + p_lo];
  d1 = sb_.sub_tile_begin[size_t(b) * np + p_hi];
  return d0 >= t0 && d1 <= t1 && d1 > d0;
}

// Up to two tile ranges [a0, a1) and [b0, b1) as launch segments.
Segments Engine::range_segments(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) const {
  Segments seg{};
  seg.task_prefix[0] = 0;
  const uint32_t r[2][2] = {{a0, a1}, {b0, b1}};
  for (const auto& x : r) {
    if (x[1] <= x[0]) continue;
    seg.tile_begin[seg.n] = x[0];
    seg.task_prefix[seg.n + 1] = seg.task_prefix[seg.n] + (x[1] - x[0]);
    ++seg.n;
  }
  return seg;
}

Segments Engine::diag_first_segments(uint32_t b, uint32_t t0, uint32_t t1) const {
  uint32_t d0 = 0, d1 = 0;
  if (std::getenv("SERAPH_NO_DIAG_FIRST") || !diag_range(b, t0, t1, d0, d1))
    return range_segments(t0, t1, 0, 0);
  Segments seg = range_segments(d0, d1, t0, d0);  // the diagonal, then the tiles before it
  if (d1 < t1) {                                  // and the tiles after it
    seg.tile_begin[seg.n] = d1;
    seg.task_prefix[seg.n + 1] = seg.task_prefix[seg.n] + (t1 - d1);
    ++seg.n;
  }
  return seg;
}

std::pair<cudaEvent_t, cudaEvent_t>* Engine::relax_begin() {
  if (!profile_kernels_) return nullptr;
  if (relax_ev_used_ == relax_ev_.size()) {
    std::pair<cudaEvent_t, cudaEvent_t> e;
    SR_CUDA(cudaEventCreate(&e.first));
    SR_CUDA(cudaEventCreate(&e.second));
    relax_ev_.push_back(e);
  }
  auto* evp = &relax_ev_[relax_ev_used_++];
  SR_CUDA(cudaEventRecord(evp->first, cs_));
  return evp;
}

void Engine::pr_blocked_pass(float base, float damp) {
  for (uint32_t b = 0; b < sb_.n_blocks; ++b) {
    const uint32_t t0 = sb_.block_tile_begin[b], t1 = sb_.block_tile_begin[b + 1];
    if (t1 <= t0) continue;
    PrArgs a{};
    a.work = next_work_counter();
    a.tiles = sb_.tiles.p;
    a.tile_page = sb_.tile_page.p;
    a.pages = sb_.desc.p;
    a.seg.n = 1;
    a.seg.tile_begin[0] = t0;
    a.seg.task_prefix[0] = 0;
    a.seg.task_prefix[1] = t1 - t0;
    a.contrib_in = contrib_a_.p;
    a.rank_out = rank_b_.p;
    a.contrib_out = contrib_b_.p;
    a.inv_outdeg = inv_outdeg_.p;
    a.hub_sum = hub_sum_.p;
    a.acc = sb_.acc.p;
    a.ctr = nullptr;
    a.base = base;
    a.damp = damp;
    int grid = int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                      (uint64_t(t1 - t0) + kWarpsPerBlock - 1) / kWarpsPerBlock));
    if (pr_hot_.built && pr_hot_.blocked) {
      a.pages = pr_hot_.desc.p;
      a.hot_contrib = pr_hot_.hot_contrib.p;
      a.n_hot = pr_hot_.n_hot;
      grid = int(std::min<uint64_t>(uint64_t(sm_count_) * pr_hot_.blocks_per_sm,
                                    (uint64_t(t1 - t0) + pr_hot_warps() - 1) / pr_hot_warps()));
    }
    std::pair<cudaEvent_t, cudaEvent_t>* evp = nullptr;
    if (profile_kernels_) {
      if (relax_ev_used_ == relax_ev_.size()) {
        std::pair<cudaEvent_t, cudaEvent_t> e;
        SR_CUDA(cudaEventCreate(&e.first));
        SR_CUDA(cudaEventCreate(&e.second));
        relax_ev_.push_back(e);
      }
      evp = &relax_ev_[relax_ev_used_++];
      SR_CUDA(cudaEventRecord(evp->first, cs_));
    }
    launch_pr_pull(a, std::max(grid, 1), cs_);
    SR_CUDA(cudaGetLastError());
    if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
  }
  launch_pr_block_finalize(own_lo_, own_hi_, sb_.acc.p, rank_b_.p, contrib_b_.p, inv_outdeg_.p,
                           base, damp, cs_);
}

// ---------------------------------------------------------------------------
// K8 hot-source staging.  Hot set = every vertex whose out-degree is at least
// the smallest threshold D that admits <= H of them (H = kHotDefault, or
// SERAPH_PR_HOT entries up to what the block shape holds; default on when
// |V| > 1 Mi, i.e. when the contribution array outgrows what the L1s serve).
// The encoded source copy costs 4 B/edge of HBM; without room for it K8 runs
// unstaged.
// ---------------------------------------------------------------------------
bool Engine::prepare_pr_hot(bool blocked) {
  uint64_t cap = n_ > (1u << 20) ? kHotDefault : 0;
  if (const char* e = std::getenv("SERAPH_PR_HOT")) cap = std::strtoull(e, nullptr, 10);
  cap = std::min<uint64_t>(cap, pr_hot_table_max());
  if (cap == 0 || !all_resident_ || !has_csr_ || n_ == 0) return false;
  const uint32_t* key = blocked ? sb_.src.p : arena_src_.p;
  const uint64_t words = blocked ? sb_.src.n : arena_src_.n;
  if (pr_hot_.built && pr_hot_.blocked == blocked && pr_hot_.key == key) return true;
  pr_hot_.built = false;
  size_t free_b = 0, total_b = 0;
  SR_CUDA(cudaMemGetInfo(&free_b, &total_b));
  const uint64_t need = (words + 4) * 4 + uint64_t(n_) * 4 + (256ull << 20);
  if (pr_hot_.enc.n < words + 4 && free_b + pr_hot_.enc.n * 4 < need) return false;
  // 1) threshold: smallest D >= 1 with |{v : deg(v) >= D}| <= cap
  pr_hot_.cnt.reserve(1);
  auto count_ge = [&](uint32_t d) {
    SR_CUDA(cudaMemsetAsync(pr_hot_.cnt.p, 0, 8, cs_));
    launch_count_deg_ge(outdeg_.p, n_, d, pr_hot_.cnt.p, cs_);
    unsigned long long k = 0;
    SR_CUDA(cudaMemcpyAsync(&k, pr_hot_.cnt.p, 8, cudaMemcpyDeviceToHost, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
    return uint64_t(k);
  };
  uint32_t lo = 1, hi = 0xffffffffu;  // count_ge(hi) == 0 <= cap
  if (count_ge(1) <= cap) hi = 1;
  while (lo < hi) {  // invariant: count_ge(hi) <= cap, and count_ge(d) > cap for d < lo
    const uint32_t mid = lo + (hi - lo) / 2;
    if (count_ge(mid) <= cap) hi = mid;
    else lo = mid + 1;
  }
  const uint32_t d = hi;
  // 2) slots
  pr_hot_.slot_of.reserve(n_);
  pr_hot_.hot_vertex.reserve(cap);
  pr_hot_.hot_contrib.reserve((cap + 3) & ~uint64_t(3));
  SR_CUDA(cudaMemsetAsync(pr_hot_.cnt.p, 0, 8, cs_));
  launch_hot_assign(outdeg_.p, n_, d, uint32_t(cap), reinterpret_cast<unsigned*>(pr_hot_.cnt.p),
                    pr_hot_.slot_of.p, pr_hot_.hot_vertex.p, cs_);
  unsigned long long nh = 0;
  SR_CUDA(cudaMemcpyAsync(&nh, pr_hot_.cnt.p, 8, cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  pr_hot_.n_hot = uint32_t(std::min<unsigned long long>(nh, cap));
  if (pr_hot_.n_hot == 0) return false;
  pr_hot_.blocks_per_sm = pr_hot_blocks_per_sm(pr_hot_.n_hot);
  // 3) encoded source copy + descriptors pointing into it
  pr_hot_.enc.reserve(words + 4);
  launch_hot_encode(key, pr_hot_.enc.p, words & ~uint64_t(3), pr_hot_.slot_of.p, n_, cs_);
  std::vector<PageDesc> desc;
  if (blocked) {
    desc.resize(size_t(sb_.n_blocks) * pages_.size());
    SR_CUDA(cudaMemcpyAsync(desc.data(), sb_.desc.p, desc.size() * sizeof(PageDesc),
                            cudaMemcpyDeviceToHost, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
  } else {
    desc = page_desc_h_;
  }
  for (PageDesc& pd : desc)
    if (pd.src) pd.src = pr_hot_.enc.p + (pd.src - key);
  pr_hot_.desc.reserve(std::max<size_t>(desc.size(), 1));
  SR_CUDA(cudaMemcpyAsync(pr_hot_.desc.p, desc.data(), desc.size() * sizeof(PageDesc),
                          cudaMemcpyHostToDevice, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  pr_hot_.slot_of.release();
  if (std::getenv("SERAPH_TIMING"))
    std::fprintf(stderr, "[seraph] pr hot set: %u sources (out-degree >= %u)\n", pr_hot_.n_hot, d);
  pr_hot_.blocked = blocked;
  pr_hot_.key = key;
  pr_hot_.built = true;
  return true;
}

// ---------------------------------------------------------------------------
// PageRank (new algorithm; conventions pinned in DESIGN.md §2)
// ---------------------------------------------------------------------------
void Engine::run_pagerank(const sr_run_config& cfg, float* ranks_out, sr_metrics& m,
                          std::vector<sr_pass_stats>& passes) {
  const bool blocked = build_src_blocks(pr_block_verts());
  const bool hot = prepare_pr_hot(blocked);
  const auto wall0 = std::chrono::steady_clock::now();
  SR_CUDA(cudaEventRecord(ev_start_, cs_));
  launch_inv_outdeg(out_off_.p, n_, inv_outdeg_.p, cs_);
  launch_pr_init(rank_a_.p, contrib_a_.p, inv_outdeg_.p, n_, n_ ? float(1.0 / double(n_)) : 0.f, cs_);
  if (n_hubs_) SR_CUDA(cudaMemsetAsync(hub_sum_.p, 0, n_hubs_ * 4, cs_));
  // The iterations are enqueued back to back with no host sync in between
  // (the copy stream prefetches the next iteration's pages while the current
  // one computes); each iteration's counters get their own slice of the
  // counter arena, read back once at the end.
  ctr_used_ = 0;
  SR_CUDA(cudaMemsetAsync(ctr_.p, 0, ctr_.n * sizeof(RunCtr), cs_));
  std::vector<uint32_t> ctr_begin;
  std::vector<int> pr_agg;  // per iteration: the all-reduced aggregate slot (worlds) or -1
  for (uint32_t it = 0; it < cfg.pr_iterations; ++it) {
    ctr_begin.push_back(ctr_used_);
    if (attached()) {
      SR_CUDA(cudaMemsetAsync(rank_b_.p, 0, size_t(n_) * 4, cs_));
      SR_CUDA(cudaMemsetAsync(contrib_b_.p, 0, size_t(n_) * 4, cs_));
    }
    PassOut po;
    const float base = float((1.0 - cfg.pr_damping) / double(n_));
    if (hot)
      launch_pr_hot_gather(pr_hot_.hot_vertex.p, pr_hot_.n_hot, contrib_a_.p,
                           pr_hot_.hot_contrib.p, cs_);
    if (blocked) {
      pr_blocked_pass(base, float(cfg.pr_damping));
      po.kernel_runs = sb_.n_blocks * pages_.size();
      if (!first_touch_done_) {
        for (const auto& pm : pages_) {
          po.pages_transferred += 1;
          po.bytes_transferred += pm.bytes;
        }
        first_touch_done_ = true;
      }
    } else {
      po = dense_pass_wall(cfg, kGateOff, false, it, true);
      launch_pr_hub_finalize(hub_vertex_.p, n_hubs_, hub_sum_.p, rank_b_.p, contrib_b_.p,
                             inv_outdeg_.p, base, float(cfg.pr_damping), cs_);
    }
    exchange_round(true, ctr_begin.back());
    pr_agg.push_back(agg_slot_);
    sr_pass_stats st{};
    st.pass_index = it;
    st.kind = SR_PASS_DENSE_PULL;
    if (blocked) {  // every destination and edge once per iteration
      st.attempts = n_;
      st.edges_read = page_edges_total_;
      gathers_total_ += page_edges_total_;
    }
    st.changed_vertices = n_;
    m.pages_transferred += po.pages_transferred;
    m.bytes_transferred += po.bytes_transferred;
    m.kernel_runs += po.kernel_runs;
    m.passes += 1;
    m.dense_passes += 1;
    if (blocked) {
      m.update_attempts += st.attempts;
      m.edges_read += st.edges_read;
    }
    passes.push_back(st);
    std::swap(rank_a_.p, rank_b_.p);
    std::swap(contrib_a_.p, contrib_b_.p);
  }
  SR_CUDA(cudaEventRecord(ev_stop_, cs_));
  if (ranks_out) stager_.d2h_sync(ranks_out, rank_a_.p, size_t(n_) * 4, cs_);
  if (ctr_used_)
    SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr_.p, size_t(ctr_used_) * sizeof(RunCtr),
                            cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  ctr_begin.push_back(ctr_used_);
  for (size_t it = 0; it + 1 < ctr_begin.size(); ++it) {
    if (blocked) continue;  // counted analytically above
    sr_pass_stats& st = passes[passes.size() - (ctr_begin.size() - 1) + it];
    const int ag = it < pr_agg.size() ? pr_agg[it] : -1;  // a world's reduced aggregate
    for (uint32_t i = ctr_begin[it]; i < ctr_begin[it + 1]; ++i) {
      if (int(i) == ag) continue;
      gathers_total_ += ctr_h_.p[i].gathers;
      if (ag >= 0) continue;
      st.attempts += ctr_h_.p[i].attempts;
      st.edges_read += ctr_h_.p[i].edges;
    }
    if (ag >= 0) {
      st.attempts += ctr_h_.p[ag].attempts;
      st.edges_read += ctr_h_.p[ag].edges;
    }
    m.update_attempts += st.attempts;
    m.edges_read += st.edges_read;
  }
  float ms = 0;
  SR_CUDA(cudaEventElapsedTime(&ms, ev_start_, ev_stop_));
  m.device_seconds = ms * 1e-3;
  if (ranks_out) m.d2h_bytes = uint64_t(n_) * 4;
  m.wall_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
}

}  // namespace seraph
