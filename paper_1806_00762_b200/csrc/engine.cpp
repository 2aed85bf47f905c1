// Host engine of libseraph: graph residency, the density-switched pass loop
// and the transfer scheduler.  The loop follows the reference Runner
// (proj/src/engine.cpp:225-416) decision for decision; all per-vertex work
// runs in the sm_100a kernels of kernels.cu.
#include "engine.h"
#include "loopback.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <thread>

#include "kernels.h"
#include "devgraph.h"
#include "nccl_dyn.h"

namespace seraph {

namespace {

int host_threads() {
  unsigned h = std::thread::hardware_concurrency();
  return h ? int(std::min(h, 64u)) : 8;
}

template <typename F>
void parallel_for(size_t n, F&& f, int threads = 0) {
  if (threads <= 0) threads = host_threads();
  if (n == 0) return;
  if (threads == 1 || n == 1) {
    for (size_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> pool;
  std::atomic<size_t> next{0};
  const int t = int(std::min<size_t>(threads, n));
  for (int k = 0; k < t; ++k)
    pool.emplace_back([&] {
      for (size_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& th : pool) th.join();
}

uint64_t page_bytes_rule(uint32_t range, uint64_t edges, bool weighted) {
  // graph.cpp:96-100: (offset entries + source entries [+ weight entries]) * 4
  return (uint64_t(range) + 1 + edges * (weighted ? 2 : 1)) * 4ull;
}

struct TileJob {
  uint32_t page, lo, hi;  // page-local destination range
  std::vector<uint4> tiles;
  std::vector<uint32_t> hubs;  // global vertex ids, local hub numbering
};

// Greedy cut of [lo, hi) into warp tiles (device_types.h).
void cut_tiles(const uint32_t* offs, uint32_t vb, TileJob& job) {
  uint32_t i = job.lo;
  while (i < job.hi) {
    const uint32_t deg = offs[i + 1] - offs[i];
    if (deg > kHubChunk) {
      const uint32_t hub = uint32_t(job.hubs.size());
      job.hubs.push_back(vb + i);
      for (uint32_t e = offs[i]; e < offs[i + 1]; e += kHubChunk)
        job.tiles.push_back(make_uint4(e, std::min(e + kHubChunk, offs[i + 1]), i, kHubFlag | hub));
      ++i;
      continue;
    }
    uint32_t j = i;
    uint32_t edges = 0;
    while (j < job.hi && j - i < kTileMaxDests) {
      const uint32_t d = offs[j + 1] - offs[j];
      if (d > kHubChunk) break;
      if (j > i && edges + d > kTileEdgeBudget) break;
      edges += d;
      ++j;
    }
    job.tiles.push_back(make_uint4(offs[i], offs[j], i, j));
    i = j;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
Engine::Engine(int device, uint64_t budget) : dev_(device), budget_(budget) {
  SR_CUDA(cudaSetDevice(dev_));
  SR_CUDA(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, dev_));
  SR_CUDA(cudaDeviceGetAttribute(&l2_bytes_, cudaDevAttrL2CacheSize, dev_));
  SR_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  SR_CUDA(cudaStreamCreateWithFlags(&xs_, cudaStreamNonBlocking));
  SR_CUDA(cudaEventCreate(&ev_start_));
  SR_CUDA(cudaEventCreate(&ev_stop_));
  SR_CUDA(cudaEventCreateWithFlags(&ev_step_, cudaEventDisableTiming));
  SR_CUDA(cudaEventCreateWithFlags(&ev_tiles_, cudaEventDisableTiming));
  blocks_per_sm_ = pull_blocks_per_sm(kSssp, kGateOff, false);
  census_.reserve(1);
  census_h_.reserve(1);
  pub_seq_h_.reserve(1);
  *pub_seq_h_.p = 0;
}

Engine::~Engine() {
  cudaSetDevice(dev_);
  for (void* p : ipc_ptrs_)
    if (p) cudaIpcCloseMemHandle(p);
  if (comm_) nccl().CommDestroy(comm_);
  for (cudaEvent_t e : page_events_) cudaEventDestroy(e);
  for (auto& s : slots_) {
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.freed) cudaEventDestroy(s.freed);
  }
  if (cs_) cudaStreamSynchronize(cs_);
  if (xs_) cudaStreamSynchronize(xs_);
  if (ev_start_) cudaEventDestroy(ev_start_);
  if (ev_stop_) cudaEventDestroy(ev_stop_);
  if (ev_step_) cudaEventDestroy(ev_step_);
  if (ev_tiles_) cudaEventDestroy(ev_tiles_);
  if (ev_csr_) cudaEventDestroy(ev_csr_);
  for (auto& e : relax_ev_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  for (cudaEvent_t e : wtrace_pool_) cudaEventDestroy(e);
  if (cs_) cudaStreamDestroy(cs_);
  if (xs_) cudaStreamDestroy(xs_);
}

// ---------------------------------------------------------------------------
// Graph upload
// ---------------------------------------------------------------------------
void Engine::load_csr(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                      const uint32_t* w, bool sync) {
  SR_CUDA(cudaSetDevice(dev_));
  if (!off) throw EngineError(SR_E_INPUT, "csr: out_offsets is null");
  if (off[0] != 0 || off[n] != m)
    throw EngineError(SR_E_INPUT, "csr: out_offsets must start at 0 and end at num_edges");
  const auto t0 = std::chrono::steady_clock::now();
  n_ = n;
  m_ = m;
  out_off_.reserve(size_t(n) + 1);
  stager_.h2d(out_off_.p, off, (size_t(n) + 1) * 8, xs_);
  uint64_t bytes = (uint64_t(n) + 1) * 8;
  has_csr_edges_ = nbr != nullptr;
  csr_weighted_ = false;
  adj_host_ = false;
  row_lo_ = 0;
  row_hi_ = n;
  nbr_base_ = 0;
  if (nbr && m && budget_ != 0) {
    // forced budget: stage the adjacency in pinned host memory; load_pages
    // decides where it lives (place_adjacency)
    out_nbr_.release();
    out_w_.release();
    host_nbr_.reserve(m);
    if (w) host_w_.reserve(m);
    auto on_dev = [](const void* p) {
      cudaPointerAttributes at{};
      return cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice;
    };
    if (on_dev(nbr) || (w && on_dev(w))) {
      SR_CUDA(cudaMemcpy(host_nbr_.p, nbr, m * 4, cudaMemcpyDefault));
      if (w) SR_CUDA(cudaMemcpy(host_w_.p, w, m * 4, cudaMemcpyDefault));
    } else {
      const uint64_t chunk = 16ull << 20;
      parallel_for((m + chunk - 1) / chunk, [&](size_t k) {
        const uint64_t a = k * chunk, b = std::min(m, a + chunk);
        std::memcpy(host_nbr_.p + a, nbr + a, (b - a) * 4);
        if (w) std::memcpy(host_w_.p + a, w + a, (b - a) * 4);
      });
    }
    adj_host_ = true;
    csr_weighted_ = w != nullptr;
  } else if (nbr && m) {
    out_nbr_.reserve(m);
    stager_.h2d(out_nbr_.p, nbr, m * 4, xs_);
    bytes += m * 4;
    if (w) {
      out_w_.reserve(m);
      stager_.h2d(out_w_.p, w, m * 4, xs_);
      bytes += m * 4;
      csr_weighted_ = true;
    }
  } else if (nbr && w) {
    csr_weighted_ = true;  // weighted graph without edges
  }
  finish_csr(sync);
  last_upload_bytes += bytes;
  last_upload_seconds +=
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::finish_csr(bool sync) {
  coverage_ = -1;  // hot_source_coverage follows the out-degrees
  const size_t npad = (size_t(n_) + kCensusBlockVerts) / kCensusBlockVerts * kCensusBlockVerts + 16;
  outdeg_.reserve(npad);
  SR_CUDA(cudaMemsetAsync(outdeg_.p, 0, npad * 4, xs_));
  launch_outdeg(out_off_.p, n_, outdeg_.p, xs_);
  // unsynchronised only inside sr_run_graph, whose load_pages follows on the
  // same copy stream and synchronises it before returning
  if (sync) SR_CUDA(cudaStreamSynchronize(xs_));
  has_csr_ = true;
  csr_derived_ = false;
}

// Defer the push adjacency derivation of a one-shot sr_run_graph when the
// run will need it only for a few small sparse passes: connected components
// (the initial frontier is every vertex, so its sparse passes come last) on
// >= 2^30 edges.  BFS/SSSP start with sparse passes from the source and keep
// the derivation overlapped with the upload (SSSP RMAT-26: 198 ms per call
// eager vs 311 ms deferred).  SERAPH_DEFER_CSR_EDGES=<edges> forces the
// threshold for every algorithm (0 = never defer).
bool Engine::defer_csr(uint64_t m, int algo) const {
  if (const char* e = std::getenv("SERAPH_DEFER_CSR_EDGES")) {
    const uint64_t v = std::strtoull(e, nullptr, 10);
    return v != 0 && m >= v;
  }
  return algo == SR_ALGO_CC && m >= (1ull << 30);
}

void Engine::drop_csr() {
  has_csr_ = has_csr_edges_ = csr_weighted_ = csr_derived_ = csr_deferred_ = false;
  adj_host_ = false;
  nbr_base_ = 0;
  row_lo_ = row_hi_ = 0;
  out_nbr_.release();
  out_w_.release();
  host_nbr_.release();
  host_w_.release();
}

void Engine::load_csr_shard(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                            const uint32_t* w) {
  SR_CUDA(cudaSetDevice(dev_));
  if (!pages_loaded_ || page_n_ != n)
    throw EngineError(SR_E_CONFIG, "load_csr_shard needs this rank's page set loaded first");
  if (!off || off[0] != 0 || off[n] != m)
    throw EngineError(SR_E_INPUT, "csr: out_offsets must start at 0 and end at num_edges");
  const auto t0 = std::chrono::steady_clock::now();
  n_ = n;
  m_ = m;
  out_off_.reserve(size_t(n) + 1);
  stager_.h2d(out_off_.p, off, (size_t(n) + 1) * 8, xs_);
  uint64_t bytes = (uint64_t(n) + 1) * 8;
  row_lo_ = own_lo_;
  row_hi_ = own_hi_;
  const uint64_t e0 = off[row_lo_], e1 = off[row_hi_], me = e1 - e0;
  nbr_base_ = e0;
  has_csr_edges_ = nbr != nullptr;
  csr_weighted_ = nbr && w;
  adj_host_ = false;
  out_nbr_.release();
  out_w_.release();
  if (nbr) {
    uint64_t pages_dev = 0;
    for (const PageMeta& pm : pages_) pages_dev += pm.on_device ? pm.bytes : 0;
    const uint64_t ab = me * 4 * (w ? 2 : 1);
    if (budget_ != 0 && (all_resident_ ? pages_dev : budget_) + ab > budget_) {
      host_nbr_.reserve(std::max<uint64_t>(me, 1));  // zero-copy rows in pinned host memory
      std::memcpy(host_nbr_.p, nbr + e0, me * 4);
      if (w) {
        host_w_.reserve(std::max<uint64_t>(me, 1));
        std::memcpy(host_w_.p, w + e0, me * 4);
      }
      adj_host_ = true;
    } else {
      out_nbr_.reserve(std::max<uint64_t>(me, 1));
      stager_.h2d(out_nbr_.p, nbr + e0, me * 4, xs_);
      if (w) {
        out_w_.reserve(std::max<uint64_t>(me, 1));
        stager_.h2d(out_w_.p, w + e0, me * 4, xs_);
      }
      bytes += ab;
    }
  }
  finish_csr(true);
  stager_.sync();
  last_upload_bytes += bytes;
  last_upload_seconds +=
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::derive_csr_now() {
  csr_deferred_ = false;
  maybe_derive_csr();
}

void Engine::place_adjacency(uint64_t used, PassOut* po) {
  if (budget_ == 0) {
    page_budget_ = 0;
    return;
  }
  const uint64_t ab = has_csr_edges_ && !csr_derived_ ? m_ * 4 * (csr_weighted_ ? 2 : 1) : 0;
  const bool fit = used + ab <= budget_;
  if (ab && fit && adj_host_) {  // both fit: the adjacency goes to HBM
    out_nbr_.reserve(m_);
    SR_CUDA(cudaMemcpyAsync(out_nbr_.p, host_nbr_.p, m_ * 4, cudaMemcpyHostToDevice, xs_));
    if (csr_weighted_) {
      out_w_.reserve(m_);
      SR_CUDA(cudaMemcpyAsync(out_w_.p, host_w_.p, m_ * 4, cudaMemcpyHostToDevice, xs_));
    }
    SR_CUDA(cudaStreamSynchronize(xs_));
    last_upload_bytes += ab;
    adj_host_ = false;
    host_nbr_.release();
    host_w_.release();
  } else if (ab && !fit && !adj_host_) {  // device-built graph: move the adjacency out
    SR_CUDA(cudaDeviceSynchronize());
    host_nbr_.reserve(m_);
    SR_CUDA(cudaMemcpy(host_nbr_.p, out_nbr_.p, m_ * 4, cudaMemcpyDeviceToHost));
    if (csr_weighted_) {
      host_w_.reserve(m_);
      SR_CUDA(cudaMemcpy(host_w_.p, out_w_.p, m_ * 4, cudaMemcpyDeviceToHost));
    }
    out_nbr_.release();
    out_w_.release();
    adj_host_ = true;
  }
  (void)po;
  page_budget_ = budget_ - (ab && !adj_host_ ? ab : 0);
}

void Engine::maybe_derive_csr() {
  // sr_load_csr without out_neighbors + a resident page set: build the push
  // adjacency on the device instead of shipping it over the host link
  // (only when pages + adjacency fit a forced budget).
  if (csr_deferred_ || !has_csr_ || has_csr_edges_ || !pages_loaded_ || !all_resident_ ||
      world_ > 1)
    return;
  if (budget_ != 0 && page_bytes_total_ + m_ * 4 * (weighted_ ? 2 : 1) > budget_) return;
  if (n_ != page_n_ || m_ != page_edges_total_) return;
  if (m_ == 0) {
    has_csr_edges_ = true;
    csr_weighted_ = weighted_;
    csr_derived_ = true;
    return;
  }
  out_nbr_.reserve(m_);
  if (weighted_) out_w_.reserve(m_);
  csr_cursor_.reserve(n_);
  SR_CUDA(cudaMemcpyAsync(csr_cursor_.p, out_off_.p, size_t(n_) * 8, cudaMemcpyDeviceToDevice, cs_));
  for (const PageMeta& pm : pages_)
    launch_csr_from_pages(tiles_.p, tile_page_.p, page_desc_.p, pm.tile_begin, pm.tile_end,
                          csr_cursor_.p, out_nbr_.p, weighted_ ? out_w_.p : nullptr,
                          sm_count_ * 8, cs_);
  SR_CUDA(cudaGetLastError());
  has_csr_edges_ = true;
  csr_weighted_ = weighted_;
  csr_derived_ = true;
}

void Engine::build_tiles(uint32_t lo, uint32_t hi, cudaStream_t st) {
  // Jobs of at most 1M destinations so big pages cut in parallel.
  std::vector<TileJob> jobs;
  const uint32_t np = uint32_t(pages_.size());
  for (uint32_t p = 0; p < np; ++p) {
    const PageMeta& pm = pages_[p];
    const uint32_t a = std::max(pm.vb, lo), b = std::min(pm.ve, hi);
    if (a >= b) continue;
    for (uint32_t x = a - pm.vb; x < b - pm.vb; x += (1u << 20))
      jobs.push_back(TileJob{p, x, std::min(x + (1u << 20), b - pm.vb), {}, {}});
  }
  parallel_for(jobs.size(), [&](size_t j) {
    const PageMeta& pm = pages_[jobs[j].page];
    cut_tiles(pm.h_offs, pm.vb, jobs[j]);
  });
  hub_vertex_h_.clear();
  for (auto& pm : pages_) pm.tile_begin = pm.tile_end = 0;
  size_t total = 0;
  for (auto& j : jobs) total += j.tiles.size();
  if (total >= (1ull << 32)) throw EngineError(SR_E_CONFIG, "graph too large: tile count");
  tile_stage_.reserve(std::max<size_t>(total, 1));
  tile_page_stage_.reserve(std::max<size_t>(total, 1));
  size_t at = 0;
  for (auto& j : jobs) {
    PageMeta& pm = pages_[j.page];
    if (pm.tile_end == 0 && pm.tile_begin == 0) pm.tile_begin = uint32_t(at);
    const uint32_t hub_base = uint32_t(hub_vertex_h_.size());
    for (uint4 t : j.tiles) {
      if (t.w & kHubFlag) t.w = kHubFlag | ((t.w & ~kHubFlag) + hub_base);
      tile_stage_.p[at] = t;
      tile_page_stage_.p[at] = j.page;
      ++at;
    }
    hub_vertex_h_.insert(hub_vertex_h_.end(), j.hubs.begin(), j.hubs.end());
    pm.tile_end = uint32_t(at);
  }
  n_hubs_ = uint32_t(hub_vertex_h_.size());
  tiles_.reserve(std::max<size_t>(total, 1));
  tile_page_.reserve(std::max<size_t>(total, 1));
  if (total) {
    SR_CUDA(cudaMemcpyAsync(tiles_.p, tile_stage_.p, total * 16, cudaMemcpyHostToDevice, st));
    SR_CUDA(cudaMemcpyAsync(tile_page_.p, tile_page_stage_.p, total * 4, cudaMemcpyHostToDevice,
                            st));
  }
  hub_vertex_.reserve(std::max<uint32_t>(n_hubs_, 1));
  hub_stamp_.reserve(std::max<uint32_t>(n_hubs_, 1));
  hub_sum_.reserve(std::max<uint32_t>(n_hubs_, 1));
  if (n_hubs_) {
    hub_stage_.reserve(n_hubs_);
    std::memcpy(hub_stage_.p, hub_vertex_h_.data(), n_hubs_ * 4);
    SR_CUDA(cudaMemcpyAsync(hub_vertex_.p, hub_stage_.p, n_hubs_ * 4, cudaMemcpyHostToDevice, st));
    SR_CUDA(cudaMemsetAsync(hub_stamp_.p, 0, n_hubs_ * 4, st));
    SR_CUDA(cudaMemsetAsync(hub_sum_.p, 0, n_hubs_ * 4, st));
  }
  run_id_ = 0;
}

// Gather fraction below which a launch takes K1's LIST variant
// (SERAPH_LIST_FRAC overrides kListFrac; A/B knob).
double Engine::list_frac() const {
  static const double f = [] {
    const char* e = std::getenv("SERAPH_LIST_FRAC");
    return e ? std::atof(e) : kListFrac;
  }();
  return f;
}

// K1's LIST variant (SERAPH_K1_LIST=0 disables).
bool Engine::list_ok() const {
  const char* e = std::getenv("SERAPH_K1_LIST");
  return !e || std::atoi(e) != 0;
}

// K1 tiles per work-counter grab: about 1/16 of a warp's share of the
// launch, clamped to 1..cap; `env` overrides (1..64, A/B knob).
uint32_t k1_grab(uint64_t tiles, int grid, const char* env, uint32_t cap) {
  const uint64_t warps = uint64_t(std::max(grid, 1)) * kWarpsPerBlock;
  uint64_t g = std::max<uint64_t>(1, std::min<uint64_t>(cap, tiles / (warps * 16)));
  if (const char* e = std::getenv(env)) {
    char* end = nullptr;
    const unsigned long v = std::strtoul(e, &end, 10);
    if (end != e && *end == 0 && v >= 1 && v <= 64) g = v;
  }
  return uint32_t(g);
}

void Engine::load_pages(uint32_t n, uint32_t cap, bool weighted, const sr_page_view* views,
                        uint32_t np) {
  const int algo_hint = load_algo_;  // one load only (sr_run_graph sets it)
  load_algo_ = -1;
  SR_CUDA(cudaSetDevice(dev_));
  const auto t0 = std::chrono::steady_clock::now();
  if (np == 0 && n != 0) throw EngineError(SR_E_INPUT, "page set has no pages");
  // ---- validate the CscPage contract (graph.hpp:46-65) ----
  uint32_t expect = 0;
  for (uint32_t p = 0; p < np; ++p) {
    const sr_page_view& v = views[p];
    if (v.vertex_begin != expect || v.vertex_end <= v.vertex_begin || v.vertex_end > n)
      throw EngineError(SR_E_INPUT, "page " + std::to_string(p) +
                                        ": destination ranges must tile [0, num_vertices)");
    if (v.edge_count > 0xffffffffull)
      throw EngineError(SR_E_CONFIG, "page " + std::to_string(p) +
                                         " exceeds 2^32 edges (u32 local offsets, graph.hpp:49)");
    const uint32_t range = v.vertex_end - v.vertex_begin;
    if (!v.in_offsets || v.in_offsets[0] != 0 || v.in_offsets[range] != v.edge_count)
      throw EngineError(SR_E_INPUT, "page " + std::to_string(p) + ": bad in_offsets");
    if (v.edge_count && !v.in_sources)
      throw EngineError(SR_E_INPUT, "page " + std::to_string(p) + ": null in_sources");
    if (weighted && v.edge_count && !v.in_weights)
      throw EngineError(SR_E_INPUT, "page " + std::to_string(p) + ": weighted page without weights");
    expect = v.vertex_end;
  }
  if (expect != n) throw EngineError(SR_E_INPUT, "pages do not cover all vertices");

  page_n_ = n;
  cap_ = cap;
  weighted_ = weighted;
  pages_.assign(np, PageMeta{});
  page_bytes_total_ = 0;
  page_edges_total_ = 0;
  for (uint32_t p = 0; p < np; ++p) {
    PageMeta& pm = pages_[p];
    pm.vb = views[p].vertex_begin;
    pm.ve = views[p].vertex_end;
    pm.edges = views[p].edge_count;
    pm.bytes = page_bytes_rule(pm.ve - pm.vb, pm.edges, weighted);
    pm.h_offs = views[p].in_offsets;
    pm.h_src = views[p].in_sources;
    pm.h_w = weighted ? views[p].in_weights : nullptr;
    page_bytes_total_ += pm.bytes;
    page_edges_total_ += pm.edges;
  }
  if (world_ <= 1) {
    own_lo_ = 0;
    own_hi_ = n;
  } else {
    // edge-balanced contiguous destination cut (sr_shard_plan)
    std::vector<uint64_t> before(np + 1, 0);
    for (uint32_t p = 0; p < np; ++p) before[p + 1] = before[p] + views[p].edge_count;
    auto cut_at = [&](uint64_t target) -> uint32_t {
      if (target == 0) return 0;
      if (target >= before[np]) return n;
      // smallest vertex whose global in-edge prefix reaches target
      uint32_t p = uint32_t(std::lower_bound(before.begin() + 1, before.end(), target) -
                            (before.begin() + 1));
      const sr_page_view& v = views[p];
      const uint32_t range = v.vertex_end - v.vertex_begin;
      const uint64_t local = target - before[p];
      const uint32_t* o = v.in_offsets;
      const uint32_t k = uint32_t(std::lower_bound(o, o + range + 1, local) - o);
      return v.vertex_begin + std::min(k, range);
    };
    own_lo_ = cut_at(before[np] * uint64_t(rank_) / uint64_t(world_));
    own_hi_ = cut_at(before[np] * uint64_t(rank_ + 1) / uint64_t(world_));
    if (rank_ == world_ - 1) own_hi_ = n;
  }
  // ---- a sharded rank keeps only its own CSR rows (its pushes read no others)
  if (world_ > 1 && has_csr_edges_ && !adj_host_ && n_ == n && row_lo_ == 0 && row_hi_ == n &&
      m_ > 0) {
    unsigned long long e0 = 0, e1 = 0;
    SR_CUDA(cudaStreamSynchronize(xs_));
    SR_CUDA(cudaMemcpy(&e0, out_off_.p + own_lo_, 8, cudaMemcpyDeviceToHost));
    SR_CUDA(cudaMemcpy(&e1, out_off_.p + own_hi_, 8, cudaMemcpyDeviceToHost));
    DBuf<uint32_t> nb, wb;
    nb.reserve(std::max<uint64_t>(e1 - e0, 1));
    SR_CUDA(cudaMemcpy(nb.p, out_nbr_.p + e0, (e1 - e0) * 4, cudaMemcpyDeviceToDevice));
    if (csr_weighted_) {
      wb.reserve(std::max<uint64_t>(e1 - e0, 1));
      SR_CUDA(cudaMemcpy(wb.p, out_w_.p + e0, (e1 - e0) * 4, cudaMemcpyDeviceToDevice));
    }
    out_nbr_ = std::move(nb);
    out_w_ = std::move(wb);
    nbr_base_ = e0;
    row_lo_ = own_lo_;
    row_hi_ = own_hi_;
  }
  // ---- residency: the whole (owned) page set in HBM when it fits ----
  uint64_t used_bytes = 0;
  std::vector<char> used(np, 0);
  for (uint32_t p = 0; p < np; ++p) {
    used[p] = pages_[p].vb < own_hi_ && pages_[p].ve > own_lo_;
    if (used[p]) used_bytes += pages_[p].bytes;
  }
  place_adjacency(used_bytes, nullptr);
  all_resident_ = budget_ == 0 || used_bytes <= page_budget_;
  ring_reset();
  plan_window_ = 0;
  plan_cached_ = size_t(-1);
  sb_.built = false;
  pr_hot_.built = false;
  page_desc_h_.assign(np, PageDesc{});
  for (uint32_t p = 0; p < np; ++p) {
    page_desc_h_[p].vertex_begin = pages_[p].vb;
    page_desc_h_[p].range = pages_[p].ve - pages_[p].vb;
    page_desc_h_[p].edge_count = pages_[p].edges;
  }
  uint64_t upload = 0;
  if (all_resident_) {
    uint64_t off_total = 0, edge_total = 0;
    for (uint32_t p = 0; p < np; ++p) {
      if (!used[p]) continue;
      pages_[p].off_base = off_total;
      pages_[p].edge_base = edge_total;
      off_total += pages_[p].ve - pages_[p].vb + 1;
      edge_total += (pages_[p].edges + 7) & ~7ull;  // K1 reads 32 B-aligned runs
    }
    edge_total += 8;  // slack past the last page
    arena_offs_.reserve(std::max<uint64_t>(off_total, 1));
    arena_src_.reserve(edge_total);
    if (weighted) arena_w_.reserve(edge_total);
    // 1) page copies on the copy stream, one event per page; the largest
    //    page (RMAT page 0) goes first so tile cutting hides under its DMA
    while (page_events_.size() < np) {
      cudaEvent_t e;
      SR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      page_events_.push_back(e);
    }
    for (uint32_t p = 0; p < np; ++p) {
      PageMeta& pm = pages_[p];
      PageDesc& d = page_desc_h_[p];
      if (!used[p]) continue;
      d.offs = arena_offs_.p + pm.off_base;
      d.src = arena_src_.p + pm.edge_base;
      d.w = weighted ? arena_w_.p + pm.edge_base : nullptr;
    }
    auto copy_page = [&](uint32_t p) {
      PageMeta& pm = pages_[p];
      const PageDesc& d = page_desc_h_[p];
      // host (pinned/pageable: stager) or device (sr_build_graph) sources
      stager_.h2d(const_cast<uint32_t*>(d.offs), pm.h_offs, (size_t(d.range) + 1) * 4, xs_);
      if (pm.edges) {
        stager_.h2d(const_cast<uint32_t*>(d.src), pm.h_src, pm.edges * 4, xs_);
        if (weighted) stager_.h2d(const_cast<uint32_t*>(d.w), pm.h_w, pm.edges * 4, xs_);
      }
      SR_CUDA(cudaEventRecord(page_events_[p], xs_));
      pm.on_device = true;
      upload += pm.bytes;
    };
    uint32_t first = np;
    for (uint32_t p = 0; p < np && first == np; ++p)
      if (used[p]) first = p;
    if (!ev_csr_) SR_CUDA(cudaEventCreateWithFlags(&ev_csr_, cudaEventDisableTiming));
    SR_CUDA(cudaEventRecord(ev_csr_, xs_));  // load_csr's offsets + out-degrees (queued first)
    if (first < np) copy_page(first);
    // 2) cut tiles on the host while that DMA runs, then the small uploads
    build_tiles(own_lo_, own_hi_, xs_);
    page_desc_.reserve(std::max<uint32_t>(np, 1));
    desc_stage_.reserve(std::max<uint32_t>(np, 1));
    std::memcpy(desc_stage_.p, page_desc_h_.data(), np * sizeof(PageDesc));
    SR_CUDA(cudaMemcpyAsync(page_desc_.p, desc_stage_.p, np * sizeof(PageDesc),
                            cudaMemcpyHostToDevice, xs_));
    SR_CUDA(cudaEventRecord(ev_tiles_, xs_));
    // 3) per-page device work as each copy lands, enqueued between the copies
    //    (pageable inputs keep the host busy staging: the kernels of page p
    //    must already be queued while page p+1 is being staged): the push
    //    adjacency derivation and the source-blocked sub-pages
    if (csr_derived_) {
      has_csr_edges_ = false;
      csr_derived_ = false;
    }
    bool derive = has_csr_ && !has_csr_edges_ && world_ == 1 && n_ == n &&
                  m_ == page_edges_total_ && algo_hint != SR_ALGO_PAGERANK &&
                  (budget_ == 0 || used_bytes + m_ * 4 * (weighted ? 2 : 1) <= budget_);
    csr_deferred_ = false;
    runs_since_pages_ = 0;
    if (derive && defer_csr(m_, algo_hint)) {  // derived on demand (derive_csr_now)
      derive = false;
      csr_deferred_ = true;
      csr_weighted_ = weighted;  // what the derivation will produce
    }
    SR_CUDA(cudaStreamWaitEvent(cs_, ev_tiles_, 0));
    // source-blocked sub-pages for the run this load is for (sr_run_graph
    // names it): decided from the out-degrees, built page by page
    bool prebuild = false;
    if (algo_hint >= 0 && world_ == 1 && has_csr_ && n_ == n && !std::getenv("SERAPH_NO_PREBUILD")) {
      SR_CUDA(cudaStreamWaitEvent(cs_, ev_csr_, 0));
      const uint64_t blk = algo_hint == SR_ALGO_PAGERANK ? pr_block_verts() : pull_block_verts();
      prebuild = blk && sb_begin(blk);
    }
    const bool derive_now = derive && m_;
    if (derive_now) {
      out_nbr_.reserve(m_);
      if (weighted) out_w_.reserve(m_);
      csr_cursor_.reserve(n_);
      SR_CUDA(cudaMemcpyAsync(csr_cursor_.p, out_off_.p, size_t(n_) * 8,
                              cudaMemcpyDeviceToDevice, cs_));
    }
    for (uint32_t p = first; p < np; ++p) {
      if (!used[p]) continue;
      if (p != first) copy_page(p);
      if (!derive_now && !prebuild) continue;
      SR_CUDA(cudaStreamWaitEvent(cs_, page_events_[p], 0));
      if (derive_now)
        launch_csr_from_pages(tiles_.p, tile_page_.p, page_desc_.p, pages_[p].tile_begin,
                              pages_[p].tile_end, csr_cursor_.p, out_nbr_.p,
                              weighted ? out_w_.p : nullptr, sm_count_ * 8, cs_);
      if (prebuild) sb_page(p);
    }
    SR_CUDA(cudaGetLastError());
    if (derive) {
      has_csr_edges_ = true;
      csr_weighted_ = weighted;
      csr_derived_ = true;
    }
    // compute work on the pages is ordered after every copy
    for (uint32_t p = 0; p < np; ++p)
      if (used[p]) SR_CUDA(cudaStreamWaitEvent(cs_, page_events_[p], 0));
    weights_ge1_ = true;
    if (weighted) {  // one device scan of the resident weights (~0.15 ms per G edges)
      wflag_.reserve(1);
      SR_CUDA(cudaMemsetAsync(wflag_.p, 0, 4, cs_));
      for (uint32_t p = 0; p < np; ++p)
        if (used[p]) dg_weights_check_async(pages_[p].edges, page_desc_h_[p].w, wflag_.p, cs_);
      unsigned bad = 0;
      SR_CUDA(cudaMemcpyAsync(&bad, wflag_.p, 4, cudaMemcpyDeviceToHost, cs_));
      SR_CUDA(cudaStreamSynchronize(cs_));
      weights_ge1_ = bad == 0;
    }
    if (prebuild) sb_finish();
    SR_CUDA(cudaStreamSynchronize(xs_));  // host buffers are borrowed only for the call
    for (auto& pm : pages_) pm.h_offs = pm.h_src = pm.h_w = nullptr;
  } else {
    // Out-of-core: keep a pinned host copy of every used page (the source
    // of the copy-stream transfers); pages are admitted at run time.
    build_tiles(own_lo_, own_hi_, cs_);
    SR_CUDA(cudaStreamSynchronize(cs_));
    uint64_t words = 0;
    for (uint32_t p = 0; p < np; ++p)
      if (used[p]) words += stream_image_words(pages_[p], weighted);
    stage_.reserve(std::max<uint64_t>(words, 1));
    uint64_t at = 0;
    std::vector<std::pair<uint32_t, uint64_t>> place;
    for (uint32_t p = 0; p < np; ++p) {
      PageMeta& pm = pages_[p];
      PageDesc& d = page_desc_h_[p];
      d.vertex_begin = pm.vb;
      d.range = pm.ve - pm.vb;
      d.edge_count = pm.edges;
      pm.on_device = false;
      if (!used[p]) continue;
      place.push_back({p, at});
      at += stream_image_words(pm, weighted);
    }
    auto on_device = [](const void* p) {
      cudaPointerAttributes at{};
      return p && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
             at.type == cudaMemoryTypeDevice;
    };
    const bool dev_src = !place.empty() && on_device(pages_[place[0].first].h_src);
    std::vector<char> zero_w(place.size(), 0);
    parallel_for(place.size(), [&](size_t k) {
      PageMeta& pm = pages_[place[k].first];
      uint32_t* base = stage_.p + place[k].second;
      const size_t r1 = size_t(pm.ve - pm.vb) + 1, so = pad8(r1), wo = so + pad8(pm.edges);
      std::memset(base, 0, stream_image_words(pm, weighted) * 4);
      std::memcpy(base, pm.h_offs, r1 * 4);
      if (dev_src) {  // device-built graph under a forced budget: stage it on the host
        SR_CUDA(cudaMemcpy(base + so, pm.h_src, pm.edges * 4, cudaMemcpyDeviceToHost));
        if (weighted)
          SR_CUDA(cudaMemcpy(base + wo, pm.h_w, pm.edges * 4, cudaMemcpyDeviceToHost));
      } else {
        std::memcpy(base + so, pm.h_src, pm.edges * 4);
        if (weighted) std::memcpy(base + wo, pm.h_w, pm.edges * 4);
      }
      if (weighted) {
        const uint32_t* wp = base + wo;
        uint32_t mn = 1;
        for (uint64_t e = 0; e < pm.edges; ++e) mn = std::min(mn, wp[e]);
        zero_w[k] = mn < 1;
      }
    });
    weights_ge1_ = std::find(zero_w.begin(), zero_w.end(), 1) == zero_w.end();
    for (auto& [p, off] : place) {
      PageMeta& pm = pages_[p];
      const size_t r1 = size_t(pm.ve - pm.vb) + 1, so = pad8(r1), wo = so + pad8(pm.edges);
      pm.h_offs = stage_.p + off;
      pm.h_src = stage_.p + off + so;
      pm.h_w = weighted ? stage_.p + off + wo : nullptr;
    }
    for (auto& pm : pages_)
      if (!pm.h_offs) pm.h_src = pm.h_w = nullptr;
  }
  if (!all_resident_) {
    page_desc_.reserve(std::max<uint32_t>(np, 1));
    if (np)
      SR_CUDA(cudaMemcpyAsync(page_desc_.p, page_desc_h_.data(), np * sizeof(PageDesc),
                              cudaMemcpyHostToDevice, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
    SR_CUDA(cudaStreamSynchronize(xs_));  // a CSR upload queued by sr_run_graph
    if (csr_derived_) {  // the derived adjacency belonged to the previous page set
      has_csr_edges_ = false;
      csr_derived_ = false;
    }
  }
  pages_loaded_ = true;
  last_upload_bytes += upload;
  last_upload_seconds +=
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---------------------------------------------------------------------------
// Run configuration
// ---------------------------------------------------------------------------
void Engine::validate(const sr_run_config& c) const {
  // EngineConfig::validate (engine.cpp:43-49) + ScheduleMode::validate
  // (scheduler.cpp:40-47) + run()'s structure checks (engine.cpp:421-431).
  if (c.window_capacity < 2) throw EngineError(SR_E_CONFIG, "window capacity must be >= 2");
  if (!(c.density_threshold_fraction > 0.0 && c.density_threshold_fraction <= 1.0))
    throw EngineError(SR_E_CONFIG, "density threshold fraction must be in (0, 1]");
  if (c.bytes_per_time_unit <= 0.0 || c.edges_per_time_unit_per_worker <= 0.0)
    throw EngineError(SR_E_CONFIG, "transfer model rates must be positive");
  if (c.worker_count < 1) throw EngineError(SR_E_CONFIG, "worker_count must be >= 1");
  if (c.schedule < 0 || c.schedule > SR_SCHED_PIPELINED_FINE)
    throw EngineError(SR_E_CONFIG, "unknown scheduler mode");
  if (c.schedule == SR_SCHED_REENTRY && c.max_reentry_times < 1)
    throw EngineError(SR_E_CONFIG, "max reentry times must be >= 1");
  if (c.schedule == SR_SCHED_DOUBLE_BUFFER && c.buffer_repetitions < 1)
    throw EngineError(SR_E_CONFIG, "double-buffer repetitions must be >= 1");
  if (c.predictor < 0 || c.predictor > SR_PRED_WEAK)
    throw EngineError(SR_E_CONFIG, "unknown predictor mode");
  if (c.execution < 0 || c.execution > SR_EXEC_FORCE_DENSE)
    throw EngineError(SR_E_CONFIG, "unknown execution policy");
  if (c.algo < SR_ALGO_BFS || c.algo > SR_ALGO_PAGERANK)
    throw EngineError(SR_E_CONFIG, "unknown algorithm");
  if (!pages_loaded_) throw EngineError(SR_E_CONFIG, "no page set loaded");
  if (!has_csr_) throw EngineError(SR_E_CONFIG, "no csr loaded");
  if (n_ != page_n_) throw EngineError(SR_E_CONFIG, "csr and page set disagree on vertex count");
  if (c.algo == SR_ALGO_SSSP && (!csr_weighted_ || !weighted_))
    throw EngineError(SR_E_CONFIG, "sssp requires weighted graph structures");
  if ((c.algo == SR_ALGO_BFS || c.algo == SR_ALGO_SSSP) && c.source >= n_)
    throw EngineError(SR_E_CONFIG, "source vertex out of range");
  if (c.algo != SR_ALGO_PAGERANK && !has_csr_edges_ && !csr_deferred_ && m_ > 0)
    throw EngineError(SR_E_CONFIG, "traversal needs the csr adjacency (push stage)");
  if (c.algo == SR_ALGO_PAGERANK) {
    if (c.pr_iterations < 1) throw EngineError(SR_E_CONFIG, "pagerank iterations must be >= 1");
    if (!(c.pr_damping >= 0.0 && c.pr_damping < 1.0))
      throw EngineError(SR_E_CONFIG, "pagerank damping must be in [0, 1)");
  }
  if (c.clock == SR_CLOCK_VIRTUAL && c.algo != SR_ALGO_PAGERANK && attached())
    throw EngineError(SR_E_CONFIG, "virtual clock runs on a single device");
}

void Engine::alloc_run_state(const sr_run_config& c) {
  const size_t npad = (size_t(n_) + kCensusBlockVerts) / kCensusBlockVerts * kCensusBlockVerts + 16;
  const uint32_t nb = (n_ + kCensusBlockVerts - 1) / kCensusBlockVerts;
  if (c.algo == SR_ALGO_PAGERANK) {
    rank_a_.reserve(npad);
    rank_b_.reserve(npad);
    contrib_a_.reserve(npad);
    contrib_b_.reserve(npad);
    inv_outdeg_.reserve(npad);
  } else {
    values_.reserve(npad);
    changed_.reserve(npad);
    if (det_) next_.reserve(npad);
    if (c.predictor == SR_PRED_WEAK) {
      status_.reserve(npad);
      logstate_.reserve(npad);
    }
    list_.reserve(npad);
    pref_.reserve(npad);
    if (stamp_.n < npad) {  // frontier-queue dedup stamps (epochs never repeat)
      stamp_.reserve(npad);
      list2_.reserve(npad);
      scan_tmp_.reserve(queue_prep_temp_bytes(uint32_t(std::min<size_t>(npad, 0xfffffffeu))));
      SR_CUDA(cudaMemset(stamp_.p, 0, npad * 4));
      fq_epoch_ = 0;
    }
    chunk_start_.reserve(m_ / kPushChunk + uint64_t(sm_count_) * 48 * 2 + 2);
    blk_cnt_.reserve(nb + 1);
    blk_edges_.reserve(nb + 1);
    census_part_.reserve(size_t(nb + 1) * 13);
    if (attached()) round_snap_.reserve(npad);
  }
  const size_t np = std::max<size_t>(pages_.size(), 1);
  // counter entries per pass: gated (reentry) runs keep one entry per page
  // and run; every other launch aggregates into a single entry.
  size_t entries = size_t(std::max(1, c.max_reentry_times)) * np + np;
  entries += (np + 1) * size_t(std::max(1, c.buffer_repetitions)) + 4096 + 64;
  if (c.algo == SR_ALGO_PAGERANK)  // all iterations' counters stay in the arena (run_pagerank)
    entries = std::max(entries, (np + 2) * size_t(std::max<uint32_t>(c.pr_iterations, 1)) + 64);
  ctr_.reserve(entries);
  ctr_h_.reserve(entries);
}

unsigned* Engine::next_work_counter() {
  if (!work_.p) {
    work_.reserve(1 << 16);
    SR_CUDA(cudaMemsetAsync(work_.p, 0, work_.n * sizeof(unsigned), cs_));
    work_used_ = 0;
  }
  if (work_used_ == work_.n) {
    SR_CUDA(cudaMemsetAsync(work_.p, 0, work_.n * sizeof(unsigned), cs_));
    work_used_ = 0;
  }
  return work_.p + work_used_++;
}

RunCtr* Engine::alloc_ctr(size_t entries) {
  if (size_t(ctr_used_) + entries > ctr_.n)
    throw EngineError(SR_E_INTERNAL, "counter arena exhausted");
  RunCtr* r = ctr_.p + ctr_used_;
  ctr_used_ += uint32_t(entries);
  return r;
}

// ---------------------------------------------------------------------------
// Kernel launches over page sets
// ---------------------------------------------------------------------------
RunStats Engine::launch_pages(const std::vector<uint32_t>& pages, int gate, bool det, RunCtr* ctr,
                              const RunCtr* prev, bool per_page, bool pagerank) {
  Segments seg{};
  std::vector<uint32_t> seg_pages;
  auto flush = [&]() {
    if (seg.n == 0) return;
    const uint32_t tasks = seg.task_prefix[seg.n];
    int grid = int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                      (uint64_t(tasks) + kWarpsPerBlock - 1) / kWarpsPerBlock));
    grid = std::max(grid, 1);
    WallTraceRec* tr = nullptr;
    if (record_trace_ && !det) {
      wtrace_.push_back(WallTraceRec{trace_event(), trace_event(), seg_pages,
                                     trace_reentry_ ? SR_TRACE_REENTRY : SR_TRACE_KERNEL_START,
                                     cur_pass_});
      tr = &wtrace_.back();
      SR_CUDA(cudaEventRecord(tr->a, cs_));
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
    if (pagerank) {
      PrArgs a{};
      a.work = next_work_counter();
      a.tiles = tiles_.p;
      a.tile_page = tile_page_.p;
      a.pages = page_desc_.p;
      if (pr_hot_.built && !pr_hot_.blocked) {
        a.pages = pr_hot_.desc.p;
        a.hot_contrib = pr_hot_.hot_contrib.p;
        a.n_hot = pr_hot_.n_hot;
        grid = std::max(1, int(std::min<uint64_t>(
                               uint64_t(sm_count_) * pr_hot_.blocks_per_sm,
                               (uint64_t(tasks) + pr_hot_warps() - 1) / pr_hot_warps())));
      }
      a.seg = seg;
      a.contrib_in = contrib_a_.p;
      a.rank_out = rank_b_.p;
      a.contrib_out = contrib_b_.p;
      a.inv_outdeg = inv_outdeg_.p;
      a.hub_sum = hub_sum_.p;
      a.ctr = ctr;
      a.base = float((1.0 - pr_damp_) / double(n_));
      a.damp = float(pr_damp_);
      launch_pr_pull(a, grid, cs_);
    } else {
      PullArgs a{};
      a.work = next_work_counter();
      a.tiles = tiles_.p;
      a.tile_page = tile_page_.p;
      a.pages = page_desc_.p;
      a.seg = seg;
      a.values = values_.p;
      a.next = det ? next_.p : values_.p;
      a.changed = changed_.p;
      a.status = status_.p;
      a.hub_stamp = hub_stamp_.p;
      a.run_id = ++run_id_;
      a.ctr = ctr;
      a.prev_ctr = prev;
      a.ctr_per_page = per_page ? 1u : 0u;
      a.census = census_.p;
      a.count_dest = 1;
      a.count_valid = 1;
      a.peers = peer_list();
      a.n_peers = n_peers_;
      a.k_bfs = k_bfs_;
      a.s_cc = s_cc_;
      a.l_sssp = l_sssp_;
      a.src_floor = floor_sssp_;
      a.floor_step = weights_ge1_ ? 1u : 0u;
      {
        // tiles per work grab: about 1/16 of a warp's share of the launch,
        // 1..8 (measured best: C1 1, C2 2, SSSP RMAT-26 8 -- small launches
        // with big grabs leave warps idle, big ones amortise the atomic)
        // BFS/CC go up to 32: their grabs are gated whole first (the
        // grab-wide scan, 4 chunks per round trip), and a big converging
        // sweep is otherwise bound by the shared work counter's atomics plus
        // one round trip per 32 destinations (C4: 7.19 -> 6.91 ms)
        a.grab = k1_grab(seg.task_prefix[seg.n], grid, "SERAPH_K1_GRAB",
                         algo_ == SR_ALGO_SSSP ? 8u : 32u);
      }
      // a converging sweep: the previous pass gathered little, or this is
      // the unblocked finish of a blocked pass whose probe found gathers rare
      a.list = list_ok() && (dense_gather_frac_ < list_frac() || fallback_frac_ >= 0) ? 1u : 0u;
      launch_pull(algo_, gate, det, a, grid, cs_);
    }
    SR_CUDA(cudaGetLastError());
    if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
    if (tr) SR_CUDA(cudaEventRecord(tr->b, cs_));
    seg = Segments{};
    seg_pages.clear();
  };
  uint32_t last_end = 0xffffffffu;
  for (uint32_t p : pages) {
    const PageMeta& pm = pages_[p];
    if (pm.tile_end <= pm.tile_begin) continue;
    if (seg.n == kMaxSegments && !(pm.tile_begin == last_end)) flush();
    seg_pages.push_back(p);
    if (seg.n > 0 && pm.tile_begin == last_end) {
      seg.task_prefix[seg.n] += pm.tile_end - pm.tile_begin;
    } else {
      seg.tile_begin[seg.n] = pm.tile_begin;
      seg.task_prefix[seg.n + 1] = seg.task_prefix[seg.n] + (pm.tile_end - pm.tile_begin);
      ++seg.n;
    }
    last_end = pm.tile_end;
  }
  flush();
  return RunStats{};
}

// K2 launch: `runs` reentry runs of a resident page set in one cooperative
// kernel (pull_reentry_kernel).  False when the set needs more than one
// launch segment or the grid cannot be co-resident: the host loop runs it.
bool Engine::reentry_on_device(const std::vector<uint32_t>& pages, int gate, int runs,
                               bool per_page) {
  Segments seg{};
  uint32_t last_end = 0xffffffffu;
  for (uint32_t p : pages) {
    const PageMeta& pm = pages_[p];
    if (pm.tile_end <= pm.tile_begin) continue;
    if (seg.n > 0 && pm.tile_begin == last_end) {
      seg.task_prefix[seg.n] += pm.tile_end - pm.tile_begin;
    } else {
      if (seg.n == kMaxSegments) return false;
      seg.tile_begin[seg.n] = pm.tile_begin;
      seg.task_prefix[seg.n + 1] = seg.task_prefix[seg.n] + (pm.tile_end - pm.tile_begin);
      ++seg.n;
    }
    last_end = pm.tile_end;
  }
  if (seg.n == 0) return true;
  const uint32_t np = uint32_t(pages_.size());
  const size_t stride = per_page ? std::max<size_t>(np, 1) : 1;
  if (size_t(ctr_used_) + stride * runs > ctr_.n) return false;
  if (work_used_ + size_t(runs) > work_.n || !work_.p) {  // contiguous, zeroed counters
    next_work_counter();
    if (work_used_ + size_t(runs) > work_.n) {
      SR_CUDA(cudaMemsetAsync(work_.p, 0, work_.n * sizeof(unsigned), cs_));
      work_used_ = 0;
    }
  }
  unsigned* work = work_.p + work_used_;
  work_used_ += runs;
  if (!runs_done_.p) runs_done_.reserve(1);
  const uint32_t tasks = seg.task_prefix[seg.n];
  const int grid = std::max(1, int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                                      (uint64_t(tasks) + kWarpsPerBlock - 1) /
                                                          kWarpsPerBlock)));
  PullArgs a{};
  a.work = work;
  a.tiles = tiles_.p;
  a.tile_page = tile_page_.p;
  a.pages = page_desc_.p;
  a.seg = seg;
  a.values = values_.p;
  a.next = values_.p;
  a.changed = changed_.p;
  a.status = status_.p;
  a.hub_stamp = hub_stamp_.p;
  a.run_id = run_id_ + 1;
  a.ctr_per_page = per_page ? 1u : 0u;
  a.census = census_.p;
  a.count_dest = 1;
  a.count_valid = 1;
  a.peers = peer_list();
  a.n_peers = n_peers_;
  a.k_bfs = k_bfs_;
  a.s_cc = s_cc_;
  a.l_sssp = l_sssp_;
  a.src_floor = floor_sssp_;
  a.floor_step = weights_ge1_ ? 1u : 0u;
  a.grab = k1_grab(tasks, grid, "SERAPH_K1_GRAB");
  ReentryArgs r{work, ctr_.p + ctr_used_, uint32_t(stride), uint32_t(runs), runs_done_.p, 1u};
  auto* evp = relax_begin();
  if (!launch_pull_reentry(algo_, gate, a, r, grid, cs_)) {
    if (evp) --relax_ev_used_;
    return false;
  }
  SR_CUDA(cudaGetLastError());
  if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
  ctr_used_ += uint32_t(stride * runs);
  run_id_ += uint32_t(runs);
  return true;
}

// ---------------------------------------------------------------------------
// Dense pass, device-native schedule (ClockMode::Wall)
// ---------------------------------------------------------------------------
PassOut Engine::dense_pass_wall(const sr_run_config& cfg, int gate, bool recovery,
                                uint32_t pass_index, bool pagerank) {
  cur_pass_ = pass_index;
  PassOut po;
  // Double-buffer / pipelined(-fine) exist to overlap page transfers with
  // compute (their re-runs fill the window while the next page is in flight,
  // scheduler.cpp:293-390).  With the whole page set resident there is no
  // transfer to hide, so the device-native schedule is the resident fast path
  // (north_star: "becomes a resident-HBM fast path when partitions fit");
  // ClockMode::Virtual keeps the reference's exact schedule.  Reentry keeps
  // its meaning (re-run pages that still change: local convergence).
  const bool resident_fast = !streaming() && (cfg.schedule == SR_SCHED_DOUBLE_BUFFER ||
                                              cfg.schedule == SR_SCHED_PIPELINED ||
                                              cfg.schedule == SR_SCHED_PIPELINED_FINE);
  const int mode = (recovery || pagerank || resident_fast) ? SR_SCHED_BASELINE : cfg.schedule;
  const uint32_t B = cfg.window_capacity;
  // admission order: pages already on the device first (reference
  // scheduler.cpp:211-228), then the rest by id
  std::vector<uint32_t> order;
  std::vector<uint32_t> rest;
  for (uint32_t p = 0; p < pages_.size(); ++p) {
    if (pages_[p].tile_end <= pages_[p].tile_begin) continue;
    if (pages_[p].on_device || pages_[p].slot >= 0) order.push_back(p);
    else rest.push_back(p);
  }
  const size_t n_dev = order.size();
  order.insert(order.end(), rest.begin(), rest.end());
  const size_t n = order.size();

  struct Step {
    std::vector<uint32_t> pages;
    int reps;
    bool gated;
  };
  std::vector<Step> steps;
  auto slice = [&](size_t lo, size_t hi) {
    return std::vector<uint32_t>(order.begin() + lo, order.begin() + hi);
  };
  const bool stream = streaming();
  switch (mode) {
    case SR_SCHED_REENTRY:
      if (!stream) {
        steps.push_back({order, cfg.max_reentry_times, true});
      } else {
        if (n_dev) steps.push_back({slice(0, n_dev), cfg.max_reentry_times, true});
        for (size_t i = n_dev; i < n; ++i) steps.push_back({slice(i, i + 1), cfg.max_reentry_times, true});
      }
      break;
    case SR_SCHED_DOUBLE_BUFFER: {
      const size_t half = std::max<size_t>(1, B / 2);
      for (size_t lo = 0; lo < n; lo += half)
        steps.push_back({slice(lo, std::min(lo + half, n)), cfg.buffer_repetitions, false});
      break;
    }
    case SR_SCHED_PIPELINED:
    case SR_SCHED_PIPELINED_FINE: {
      const size_t cs = std::min<size_t>(B - 1, n);
      for (size_t j = 0; cs && j + cs <= n; ++j) steps.push_back({slice(j, j + cs), 1, false});
      break;
    }
    default:
      if (!stream) {
        steps.push_back({order, 1, false});
      } else if (n > n_dev) {
        // pages still in the streaming ring first (before newer transfers
        // evict them), then one step per streamed page with the permanently
        // cached pages spread evenly over those steps (their compute then
        // overlaps the transfers instead of stalling the link)
        std::vector<uint32_t> ring_pages, cached;
        for (size_t i = 0; i < n_dev; ++i)
          (pages_[order[i]].on_device ? cached : ring_pages).push_back(order[i]);
        if (!ring_pages.empty()) steps.push_back({ring_pages, 1, false});
        const size_t ns = n - n_dev, nc = cached.size();
        size_t next_c = 0;
        for (size_t i = n_dev; i < n; ++i) {
          std::vector<uint32_t> pg;
          for (const size_t upto = (i - n_dev + 1) * nc / ns; next_c < upto; ++next_c)
            pg.push_back(cached[next_c]);
          pg.push_back(order[i]);
          steps.push_back({pg, 1, false});
        }
      } else {
        steps.push_back({order, 1, false});
      }
      break;
  }

  const uint32_t np = uint32_t(pages_.size());
  std::vector<char> protect(np, 0);
  auto set_protect = [&](size_t a, size_t b) {
    std::fill(protect.begin(), protect.end(), 0);
    for (size_t s = a; s < std::min(b, steps.size()); ++s)
      for (uint32_t p : steps[s].pages) protect[p] = 1;
  };
  if (stream) ensure_slots(B, po);
  if (!stream && !first_touch_done_) {
    // resident window: every page admitted once per run (warm afterwards)
    for (uint32_t p : order) {
      po.pages_transferred += 1;
      po.bytes_transferred += pages_[p].bytes;
    }
    first_touch_done_ = true;
  }

  last_pass_blocked_ = false;
  // Source blocking pays for gathers only: once the previous dense pass
  // gathered for < 5 % of its edges (converged labels/levels skip theirs), the
  // per-block destination traffic would dominate -- sweep unblocked.
  // Resident reentry takes the same blocked sweeps: its re-runs of the
  // whole resident set (local convergence, scheduler.cpp:272-291) repeat the
  // blocked pass while the previous run still changed something, up to MRT.
  const bool reentry_res = mode == SR_SCHED_REENTRY && !stream;
  if ((mode == SR_SCHED_BASELINE || reentry_res) && !stream && !pagerank &&
      last_gather_frac_ >= 0.05 && last_block_gather_frac_ >= 0.05 && pull_block_verts()) {
    RunCtr* slot = alloc_ctr(1);
    if (pull_blocked_pass(gate, slot, reentry_res)) {
      last_pass_blocked_ = true;
      po.kernel_runs += order.size();
      for (int r = 1; reentry_res && r < cfg.max_reentry_times; ++r) {
        SR_CUDA(cudaMemcpyAsync(ctr_h_.p, slot, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
        SR_CUDA(cudaStreamSynchronize(cs_));
        if (ctr_h_.p[0].valid == 0) break;  // quiet: locally converged
        slot = alloc_ctr(1);
        trace_reentry_ = true;
        if (!pull_blocked_pass(gate, slot, true)) {  // probe: gathers are rare now
          slot = alloc_ctr(1);  // the blocked attempt released its slots (zeroed)
          launch_pages(order, gate, false, slot, nullptr, false, false);
        }
        trace_reentry_ = false;
        po.kernel_runs += order.size();
      }
      return po;
    }
    // (the probe zeroed the reference counters of this pass's blocked slots;
    // the unblocked steps below count the pass afresh)
    // a probed pass falls back after block 0 already applied some updates:
    // count valid updates as the destinations changed in the pass
    last_pass_blocked_ = sb_.built && pull_block_verts() != 0;
  }

  for (size_t si = 0; si < steps.size(); ++si) {
    const Step& st = steps[si];
    const long long step_id = ++step_counter_;
    if (stream) {
      set_protect(si, si + 1);
      for (uint32_t p : st.pages)
        if (!make_resident(p, step_id, protect, po))
          throw EngineError(SR_E_CONFIG, "streaming ring cannot hold one schedule step");
      for (uint32_t p : st.pages)
        if (pages_[p].slot >= 0) SR_CUDA(cudaStreamWaitEvent(cs_, slots_[pages_[p].slot].ready, 0));
    }
    const bool per_page = st.gated && st.pages.size() > 1;
    // K2 (SERAPH_K2=1): the reentry runs of a resident set loop on the device
    // in one cooperative launch that stops at the first quiet run.  Measured
    // on C2 reentry: 2.86 ms vs 2.58 ms for the host-enqueued runs (whose
    // device quiet-page gate already makes a converged re-run nearly free),
    // so the default stays the host-enqueued form.
    const char* k2e = std::getenv("SERAPH_K2");
    const bool k2 = k2e && std::atoi(k2e) != 0;
    if (k2 && st.gated && st.reps > 1 && !stream && !pagerank && !record_trace_ &&
        reentry_on_device(st.pages, gate, st.reps, per_page)) {
      po.kernel_runs += st.pages.size() * size_t(st.reps);
      continue;
    }
    RunCtr* prev = nullptr;
    for (int r = 0; r < st.reps; ++r) {
      RunCtr* slot = alloc_ctr(per_page ? std::max<size_t>(np, 1) : 1);
      trace_reentry_ = r > 0;
      launch_pages(st.pages, gate, false, slot, (st.gated && r > 0) ? prev : nullptr, per_page,
                   pagerank);
      trace_reentry_ = false;
      prev = slot;
      po.kernel_runs += st.pages.size();
    }
    if (stream) {
      for (uint32_t p : st.pages) {
        const int s = pages_[p].slot;
        if (s >= 0) {
          SR_CUDA(cudaEventRecord(slots_[s].freed, cs_));
          slots_[s].last_use = step_id;
        }
      }
      // prefetch the next step's pages into the ring (oldest images are
      // evicted first, never those of the current or the next step)
      if (si + 1 < steps.size()) {
        set_protect(si, si + 2);
        bool pending = false, admitted = true;
        cudaEvent_t last_ready = nullptr;
        for (uint32_t p : steps[si + 1].pages) {
          const bool was = pages_[p].on_device || pages_[p].slot >= 0;
          if (!make_resident(p, step_id, protect, po)) {
            admitted = false;
            break;
          }
          if (!was) {
            pending = true;
            last_ready = slots_[pages_[p].slot].ready;
          }
        }
        if (mode == SR_SCHED_PIPELINED_FINE && pending && !st.pages.empty()) {
          // fill_idle_slot (scheduler.cpp:153-158): while the stream is in
          // flight and compute is idle, re-run the lowest-id page of the set
          const uint32_t victim = *std::min_element(st.pages.begin(), st.pages.end());
          SR_CUDA(cudaEventRecord(ev_step_, cs_));
          int guard = 0;
          while (cudaEventQuery(last_ready) == cudaErrorNotReady && guard < 4000) {
            if (cudaEventQuery(ev_step_) == cudaSuccess) {
              if (size_t(ctr_used_) + 1 > ctr_.n) break;
              RunCtr* slot = alloc_ctr(1);
              trace_reentry_ = true;
              launch_pages({victim}, gate, false, slot, nullptr, false, pagerank);
              trace_reentry_ = false;
              po.kernel_runs += 1;
              SR_CUDA(cudaEventRecord(ev_step_, cs_));
              ++guard;
            } else {
              std::this_thread::yield();
            }
          }
          const int s = pages_[victim].slot;
          if (s >= 0) SR_CUDA(cudaEventRecord(slots_[s].freed, cs_));
        }
        // deeper lookahead: keep the copy engine busy while a long step (e.g.
        // the cached heavy pages) computes -- admit later steps' pages as long
        // as the ring has room that no step from here to there still needs
        if (mode != SR_SCHED_PIPELINED_FINE && admitted) {
          for (size_t sj = si + 2; sj < steps.size() && sj < si + 64; ++sj) {
            set_protect(si, sj + 1);
            bool all = true;
            for (uint32_t p : steps[sj].pages)
              if (!make_resident(p, step_id, protect, po)) {
                all = false;
                break;
              }
            if (!all) break;
          }
        }
      }
    }
  }
  return po;
}

// ---------------------------------------------------------------------------
// Dense pass, deterministic virtual-clock schedule (ClockMode::Virtual)
// ---------------------------------------------------------------------------
PassOut Engine::dense_pass_virtual(const sr_run_config& cfg, int gate, bool recovery,
                                   uint32_t pass_index) {
  if (streaming())
    throw EngineError(SR_E_CONFIG,
                      "virtual clock needs the page set resident (raise the hbm budget)");
  std::vector<uint64_t> bytes(pages_.size());
  for (size_t p = 0; p < pages_.size(); ++p) bytes[p] = pages_[p].bytes;
  const uint32_t np = uint32_t(pages_.size());
  VKernel kernel = [&](uint32_t page) -> RunStats {
    RunCtr* slot = ctr_.p;  // slot 0, synchronous
    SR_CUDA(cudaMemsetAsync(slot, 0, sizeof(RunCtr), cs_));
    launch_pages({page}, gate, true, slot, nullptr, false, false);
    launch_commit(values_.p, next_.p, pages_[page].vb, pages_[page].ve, cs_);
    SR_CUDA(cudaMemcpyAsync(ctr_h_.p, slot, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
    RunStats st;
    st.attempts = ctr_h_.p[0].attempts;
    st.valid = ctr_h_.p[0].valid;
    st.skipped = ctr_h_.p[0].skipped;
    st.edges = ctr_h_.p[0].edges;
    gathers_total_ += ctr_h_.p[0].gathers;
    streamed_total_ += ctr_h_.p[0].streamed;
    visits_total_ += ctr_h_.p[0].visits;
    return st;
  };
  (void)np;
  const int mode = recovery ? SR_SCHED_BASELINE : cfg.schedule;
  VPassResult r = vschedule_pass(bytes, mode, cfg.max_reentry_times, cfg.buffer_repetitions,
                                 vwin_, vclock_, vmodel_, kernel, pass_index,
                                 record_trace_ ? &trace : nullptr);
  PassOut po;
  po.totals = r.totals;
  po.kernel_runs = r.kernel_runs;
  po.pages_transferred = r.pages_transferred;
  po.bytes_transferred = r.bytes_transferred;
  return po;
}

// ---------------------------------------------------------------------------
// Per-pass bookkeeping
// ---------------------------------------------------------------------------
void Engine::census(int pass_kind) {
  SR_CUDA(cudaMemsetAsync(census_.p, 0, kCensusResetBytes, cs_));
  // every census is read right after (read_census): its last block publishes
  Publish pub{};
  if (ctr_used_ <= 64 && !std::getenv("SERAPH_NO_PUBLISH")) {
    if (!pub_done_.p) {
      pub_done_.reserve(1);
      SR_CUDA(cudaMemsetAsync(pub_done_.p, 0, 4, cs_));
    }
    pub = Publish{census_h_.p, ctr_.p, ctr_h_.p, ctr_used_, pub_done_.p, pub_seq_h_.p, ++pub_seq_};
    published_ = true;
  }
  launch_census(n_, changed_.p, predictor_ == SR_PRED_WEAK ? status_.p : nullptr,
                predictor_ == SR_PRED_WEAK ? logstate_.p : nullptr,
                has_csr_ ? outdeg_.p : nullptr, pass_kind, own_lo_, own_hi_, blk_cnt_.p,
                blk_edges_.p, census_part_.p, census_.p, pub, cs_);
}

void Engine::read_census() {
  if (published_) {  // the census kernel already wrote them into mapped memory
    published_ = false;
    wait_published(pub_seq_);
    return;
  } else if (ctr_used_ <= 64 && !std::getenv("SERAPH_NO_PUBLISH")) {
    // one kernel writes both into the mapped pinned buffers (UVA): no D2H DMAs
    launch_publish(census_.p, census_h_.p, ctr_.p, ctr_h_.p, ctr_used_, pub_seq_h_.p, ++pub_seq_,
                   cs_);
    wait_published(pub_seq_);
    return;
  } else {
    SR_CUDA(cudaMemcpyAsync(census_h_.p, census_.p, sizeof(Census), cudaMemcpyDeviceToHost, cs_));
    if (ctr_used_)
      SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr_.p, size_t(ctr_used_) * sizeof(RunCtr),
                              cudaMemcpyDeviceToHost, cs_));
  }
  SR_CUDA(cudaStreamSynchronize(cs_));
}

// The publishing kernel stores `seq` into pinned memory after a system-scope
// fence, behind the census and counters it wrote: the host spins on that word
// instead of a stream synchronize (whose wake-up costs several us per pass on
// small graphs), polling the stream now and then so that an idle stream (or
// an error, which the synchronize then throws) ends the wait.
// SERAPH_NO_SPIN=1: plain stream synchronize.
static bool spin_waits() {
  static const bool no_spin = [] {
    const char* e = std::getenv("SERAPH_NO_SPIN");
    return e && std::atoi(e) != 0;
  }();
  return !no_spin;
}

void Engine::wait_published(unsigned seq) {
  if (spin_waits()) {
    for (uint32_t it = 1;; ++it) {
      if (*reinterpret_cast<volatile unsigned*>(pub_seq_h_.p) == seq) {
        std::atomic_thread_fence(std::memory_order_acquire);
        return;
      }
      if ((it & 1023) == 0 && cudaStreamQuery(cs_) != cudaErrorNotReady) break;
    }
  }
  SR_CUDA(cudaStreamSynchronize(cs_));
}

// The same wait for a pinned word a kernel stores last (fenced): until it
// differs from `pending`.
void Engine::wait_word(const uint32_t* word, uint32_t pending) {
  if (spin_waits()) {
    for (uint32_t it = 1;; ++it) {
      if (*reinterpret_cast<const volatile uint32_t*>(word) != pending) {
        std::atomic_thread_fence(std::memory_order_acquire);
        return;
      }
      if ((it & 1023) == 0 && cudaStreamQuery(cs_) != cudaErrorNotReady) break;
    }
  }
  SR_CUDA(cudaStreamSynchronize(cs_));
}

// Edges per push warp task: enough tasks to give every resident warp one
// (a pass of a few hub sources would otherwise leave most SMs idle behind
// long per-warp chains), 32..kPushChunk, a power of two.
uint32_t Engine::push_chunk_shift(uint64_t total) const {
  const uint64_t warps = uint64_t(sm_count_) * 48;
  uint32_t shift = 5;
  while ((1ull << shift) < kPushChunk && (total >> shift) > warps) ++shift;
  return shift;
}

void Engine::build_push_list(uint32_t shift) {
  const uint32_t nb = (n_ + kCensusBlockVerts - 1) / kCensusBlockVerts;
  launch_scan_blocks(nb, blk_cnt_.p, blk_edges_.p, cs_);
  launch_compact(n_, own_lo_, own_hi_, changed_.p, outdeg_.p, blk_cnt_.p, blk_edges_.p,
                 list_.p, pref_.p, chunk_start_.p, shift, cs_);
}

// Sparse passes keep their frontier as a queue (O(frontier) work, no
// |V|-sized census or compaction) when the push is asynchronous, single-rank
// and no weak-predictor bookkeeping needs the changed flags; a queue pass
// starts from the compacted changed flags after a dense pass.
bool Engine::queue_mode() const {
  return !det_ && !attached() && world_ == 1 &&
         !std::getenv("SERAPH_NO_FRONTIER_QUEUE");
}

void Engine::push_pass(const sr_run_config& cfg, RunStats& st) {
  (void)cfg;
  const uint64_t n_list = census_h_.p->own_push;
  const uint64_t total = census_h_.p->own_edges;
  const bool queue = queue_mode();
  const uint32_t shift = push_chunk_shift(total);
  if (queue && fq_ready_) {
    launch_queue_prep(list_.p, uint32_t(n_list), outdeg_.p, pref_.p, chunk_start_.p, shift, total,
                      scan_tmp_.p, scan_tmp_.n, cs_);
  } else {
    build_push_list(shift);
  }
  if (queue) {
    SR_CUDA(cudaMemsetAsync(census_.p, 0, kCensusResetBytes, cs_));
    if (++fq_epoch_ == 0xffffffffu) {  // epochs exhausted: restart the stamps
      SR_CUDA(cudaMemsetAsync(stamp_.p, 0, stamp_.n * 4, cs_));
      fq_epoch_ = 1;
    }
  }
  RunCtr* slot = alloc_ctr(1);
  if (total > 0 && csr_deferred_ && !det_ && scan_pushes_ < 2 && total <= m_ / 64) {
    // a small frontier on a deferred push adjacency: enumerate its out-edges
    // from the resident CSC pages (a sweep over the sources) instead of
    // deriving the whole CSR for it
    ++scan_pushes_;
    PushArgs a{};
    a.list = list_.p;
    a.n_list = uint32_t(n_list);
    a.total_edges = total;
    a.values = values_.p;
    a.next = values_.p;
    a.changed = changed_.p;
    a.ctr = slot;
    a.census = census_.p;
    if (queue) {
      a.stamp = stamp_.p;
      a.epoch = fq_epoch_;
      a.q_list = list2_.p;
      a.outdeg = outdeg_.p;
      a.logstate = predictor_ == SR_PRED_WEAK ? logstate_.p : nullptr;
    }
    fbits_.reserve(size_t(n_) / 32 + 1);
    launch_push_scan(algo_, a, page_desc_.p, uint32_t(pages_.size()), fbits_.p, n_,
                     int(sm_count_) * blocks_per_sm_, cs_);
    SR_CUDA(cudaGetLastError());
    (void)st;
    return;
  }
  if (total > 0 && csr_deferred_) derive_csr_now();
  if (total > 0) {
    PushArgs a{};
    a.list = list_.p;
    a.pref = pref_.p;
    a.chunk_start = chunk_start_.p;
    a.n_list = uint32_t(n_list);
    a.chunk_shift = shift;
    a.total_edges = total;
    a.out_offsets = out_off_.p;
    a.out_neighbors = nbr_ptr();
    a.out_weights = w_ptr();
    a.values = values_.p;
    a.next = det_ ? next_.p : values_.p;
    a.changed = changed_.p;
    a.ctr = slot;
    a.census = census_.p;
    a.peers = peer_list();
    a.n_peers = n_peers_;
    if (queue) {
      a.stamp = stamp_.p;
      a.epoch = fq_epoch_;
      a.q_list = list2_.p;
      a.outdeg = outdeg_.p;
      a.logstate = predictor_ == SR_PRED_WEAK ? logstate_.p : nullptr;
    }
    const uint64_t chunks = (total + (1ull << shift) - 1) >> shift;
    const int grid = int(std::max<uint64_t>(
        1, std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_, (chunks + kWarpsPerBlock - 1) / kWarpsPerBlock)));
    launch_push(algo_, det_, a, grid, cs_);
    SR_CUDA(cudaGetLastError());
    if (det_) launch_push_commit(values_.p, next_.p, changed_.p, n_, slot, census_.p, cs_);
  }
  (void)st;
}

void Engine::exchange_round(bool pagerank, uint32_t ctr_from) {
  agg_slot_ = -1;
  if (!attached()) return;  // attached to a world (any size, incl. 1): merge every round
  SR_CUDA(cudaSetDevice(dev_));
  // The round's counters travel as ONE aggregate entry (sum of this round's
  // slots): ranks may use different numbers of slots in a pass (per-block
  // probes, fallbacks), so the slot arrays do not line up across ranks.
  RunCtr* agg = alloc_ctr(1);
  agg_slot_ = int(agg - ctr_.p);
  launch_sum_ctr_slots(ctr_.p, ctr_from, uint32_t(agg_slot_), agg, cs_);
  const size_t agg_words = sizeof(RunCtr) / 8;
  if (n_peers_ && !pagerank) {
    // peer exchange: every improvement is already in every replica once all
    // ranks' kernels of the round have finished -- barrier, then only the
    // scalars (min_changed, counters) are reduced
    round_barrier();
    if (loop_) {
      loopback_allreduce(loop_, rank_, &census_.p->min_changed, 1, kLoopU32, kLoopMin, cs_);
      loopback_allreduce(loop_, rank_, agg, agg_words, kLoopU64, kLoopSum, cs_);
    } else {
      const NcclApi& nc = nccl();
      nc.GroupStart();
      ncclResult_t r = nc.AllReduce(&census_.p->min_changed, &census_.p->min_changed, 1,
                                    ncclUint32, ncclMin, comm_, cs_);
      if (r == ncclSuccess)
        r = nc.AllReduce(agg, agg, agg_words, ncclUint64, ncclSum, comm_, cs_);
      nc.GroupEnd();
      if (r != ncclSuccess)
        throw EngineError(SR_E_NCCL, std::string("nccl: ") + nc.GetErrorString(r));
    }
    launch_mark_changed(n_, values_.p, round_snap_.p, changed_.p, cs_);
    return;
  }
  if (loop_) {  // in-process loopback (tests): the same reductions through host memory
    if (pagerank) {
      loopback_allreduce(loop_, rank_, rank_b_.p, n_, kLoopF32, kLoopSum, cs_);
      loopback_allreduce(loop_, rank_, contrib_b_.p, n_, kLoopF32, kLoopSum, cs_);
    } else {
      loopback_allreduce(loop_, rank_, values_.p, n_, kLoopU32, kLoopMin, cs_);
      loopback_allreduce(loop_, rank_, &census_.p->min_changed, 1, kLoopU32, kLoopMin, cs_);
    }
    loopback_allreduce(loop_, rank_, agg, agg_words, kLoopU64, kLoopSum, cs_);
    if (!pagerank) launch_mark_changed(n_, values_.p, round_snap_.p, changed_.p, cs_);
    return;
  }
  ncclResult_t r = ncclSuccess;
  SR_CUDA(cudaSetDevice(dev_));
  const NcclApi& nc = nccl();
  nc.GroupStart();
  if (pagerank) {
    r = nc.AllReduce(rank_b_.p, rank_b_.p, n_, ncclFloat, ncclSum, comm_, cs_);
    if (r == ncclSuccess)
      r = nc.AllReduce(contrib_b_.p, contrib_b_.p, n_, ncclFloat, ncclSum, comm_, cs_);
  } else {
    r = nc.AllReduce(values_.p, values_.p, n_, ncclUint32, ncclMin, comm_, cs_);
    if (r == ncclSuccess)
      r = nc.AllReduce(&census_.p->min_changed, &census_.p->min_changed, 1, ncclUint32, ncclMin,
                       comm_, cs_);
  }
  if (r == ncclSuccess) r = nc.AllReduce(agg, agg, agg_words, ncclUint64, ncclSum, comm_, cs_);
  nc.GroupEnd();
  if (r != ncclSuccess) throw EngineError(SR_E_NCCL, std::string("nccl: ") + nc.GetErrorString(r));
  if (!pagerank) launch_mark_changed(n_, values_.p, round_snap_.p, changed_.p, cs_);
}

// ---------------------------------------------------------------------------
// The pass loop (reference Runner::run, engine.cpp:371-416)
// ---------------------------------------------------------------------------
void Engine::run(const sr_run_config& cfg, uint32_t* values_out, float* ranks_out,
                 sr_metrics& m, std::vector<sr_pass_stats>& passes) {
  SR_CUDA(cudaSetDevice(dev_));
  // a deferred push adjacency is derived once the page set is run again
  // (it then pays for itself) or for the deterministic passes
  if (csr_deferred_ && cfg.algo != SR_ALGO_PAGERANK &&
      (runs_since_pages_ > 0 || cfg.clock == SR_CLOCK_VIRTUAL))
    derive_csr_now();
  if (cfg.algo != SR_ALGO_PAGERANK) maybe_derive_csr();  // PageRank reads out-degrees only
  validate(cfg);
  scan_pushes_ = 0;
  ++runs_since_pages_;
  algo_ = cfg.algo;
  source_ = cfg.source;
  predictor_ = cfg.algo == SR_ALGO_PAGERANK ? SR_PRED_OFF : cfg.predictor;
  det_ = cfg.clock == SR_CLOCK_VIRTUAL && cfg.algo != SR_ALGO_PAGERANK;
  record_trace_ = cfg.record_trace != 0;
  pr_damp_ = cfg.pr_damping;
  profile_kernels_ = cfg.profile_kernels != 0;
  relax_ev_used_ = 0;
  gathers_total_ = 0;
  streamed_total_ = 0;
  visits_total_ = 0;
  wtrace_.clear();
  wtrace_pool_used_ = 0;
  trace.clear();
  std::memset(&m, 0, sizeof(m));
  passes.clear();
  h2d_bytes_ = 0;
  first_touch_done_ = false;
  vwin_.reset(cfg.window_capacity);
  vclock_ = VClock{};
  vmodel_.bytes_per_unit = cfg.bytes_per_time_unit;
  vmodel_.edges_per_unit_per_worker = cfg.edges_per_time_unit_per_worker;
  vmodel_.workers = cfg.worker_count;
  alloc_run_state(cfg);
  if (cfg.algo != SR_ALGO_PAGERANK) setup_peers();  // every rank runs the same program
  else n_peers_ = 0;
  const uint64_t launches0 = kernel_launch_count();
  if (cfg.algo == SR_ALGO_PAGERANK) run_pagerank(cfg, ranks_out, m, passes);
  else run_traversal(cfg, values_out, m, passes);
  m.kernel_launches = kernel_launch_count() - launches0;  // every kernel of the run
  m.h2d_bytes = h2d_bytes_;
  m.gathers = gathers_total_;
  m.edges_streamed = streamed_total_;
  m.dest_visits = visits_total_;
  finish_wall_trace();
  if (profile_kernels_) {
    m.relax_seconds = collect_relax_seconds();
    m.relax_launches = relax_ev_used_;
  }
}

void Engine::run_traversal(const sr_run_config& cfg, uint32_t* values_out, sr_metrics& m,
                           std::vector<sr_pass_stats>& passes) {
  const bool weak = predictor_ == SR_PRED_WEAK;
  const bool strong = predictor_ == SR_PRED_STRONG;
  const size_t npad = values_.n;

  const auto wall0 = std::chrono::steady_clock::now();
  SR_CUDA(cudaEventRecord(ev_start_, cs_));
  // ---- initial state (VertexValues ctor programs.hpp:61-64; Runner ctor
  //      engine.cpp:225-245; initial_frontier engine.cpp:260-263) ----
  launch_init_values(algo_, source_, n_, values_.p, cs_);
  if (det_) SR_CUDA(cudaMemcpyAsync(next_.p, values_.p, size_t(n_) * 4, cudaMemcpyDeviceToDevice, cs_));
  SR_CUDA(cudaMemsetAsync(changed_.p, 0, npad, cs_));
  if (weak) {
    SR_CUDA(cudaMemsetAsync(status_.p, 0, npad, cs_));
    SR_CUDA(cudaMemsetAsync(logstate_.p, 0, npad, cs_));
  }
  SR_CUDA(cudaMemsetAsync(census_.p, 0, sizeof(Census), cs_));
  SR_CUDA(cudaMemsetAsync(&census_.p->min_changed, 0xff, 4, cs_));
  k_bfs_ = 0;
  s_cc_ = 0;
  l_sssp_ = 0;
  floor_sssp_ = 0;
  last_gather_frac_ = 1.0;  // the first dense pass gathers
  dense_gather_frac_ = 1.0;
  last_block_gather_frac_ = 1.0;
  sb_last_slot_ = -1;
  fallback_frac_ = -1;
  ctr_used_ = 0;
  if (algo_ != SR_ALGO_CC && queue_mode() && has_csr_ && !weak) {  // weak: census seeds the DFA histogram
    // the initial frontier {source} directly as a queue
    SR_CUDA(cudaMemsetAsync(census_.p, 0, kCensusResetBytes, cs_));
    launch_seed_queue(source_, outdeg_.p, list_.p, census_.p, cs_);
    read_census();
    fq_ready_ = true;
  } else {
    if (algo_ == SR_ALGO_CC) SR_CUDA(cudaMemsetAsync(changed_.p, 1, n_, cs_));
    else SR_CUDA(cudaMemsetAsync(changed_.p + source_, 1, 1, cs_));
    census(kPassInit);
    read_census();
    fq_ready_ = false;  // the initial frontier is in the changed flags
  }

  uint64_t f_count = census_h_.p->changed;
  uint64_t f_out = census_h_.p->out_edges;
  std::array<uint64_t, 6> hist{};
  for (int s = 0; s < 6; ++s) hist[s] = census_h_.p->status_hist[s];
  bool prev_dense = false;
  uint32_t pass_index = 0;

  auto account = [&](sr_pass_stats& st) {
    m.passes += 1;
    m.update_attempts += st.attempts;
    m.valid_updates += st.valid_updates;
    m.skipped_vertices += st.skipped;
    m.edges_read += st.edges_read;
    passes.push_back(st);
  };
  auto sum_ctr = [&](sr_pass_stats& st) {
    // the pass's reference counters: this rank's slots, or in a world the
    // round's all-reduced aggregate (exchange_round); the work counters
    // (gathers, streamed edges, destination scans) stay this rank's own
    uint64_t gathers = 0;
    for (size_t i = 0; i < size_t(ctr_used_); ++i) {
      if (int(i) == agg_slot_) continue;
      gathers += ctr_h_.p[i].gathers;
      streamed_total_ += ctr_h_.p[i].streamed;
      visits_total_ += ctr_h_.p[i].visits;
      if (agg_slot_ >= 0) continue;
      st.attempts += ctr_h_.p[i].attempts;
      st.valid_updates += ctr_h_.p[i].valid;
      st.skipped += ctr_h_.p[i].skipped;
      st.edges_read += ctr_h_.p[i].edges;
    }
    if (agg_slot_ >= 0 && size_t(agg_slot_) < size_t(ctr_used_)) {
      const RunCtr& ag = ctr_h_.p[agg_slot_];
      st.attempts += ag.attempts;
      st.valid_updates += ag.valid;
      st.skipped += ag.skipped;
      st.edges_read += ag.edges;
    }
    agg_slot_ = -1;
    gathers_total_ += gathers;
    last_gather_frac_ = st.edges_read ? double(gathers) / double(st.edges_read) : 0.0;
    last_block_gather_frac_ = 1.0;
    if (sb_last_slot_ >= 0 && size_t(sb_last_slot_) < size_t(ctr_used_)) {
      const RunCtr& lc = ctr_h_.p[sb_last_slot_];
      if (lc.edges) last_block_gather_frac_ = double(lc.gathers) / double(lc.edges);
    }
    if (fallback_frac_ >= 0) {  // the pass finished unblocked after a rare-gathers probe
      last_block_gather_frac_ = fallback_frac_;
      fallback_frac_ = -1;
    }
    sb_last_slot_ = -1;
  };
  auto begin_pass = [&]() {
    ctr_used_ = 0;
    SR_CUDA(cudaMemsetAsync(ctr_.p, 0, ctr_.n * sizeof(RunCtr), cs_));
    if (attached())
      SR_CUDA(cudaMemcpyAsync(round_snap_.p, values_.p, size_t(n_) * 4, cudaMemcpyDeviceToDevice, cs_));
    if (n_peers_) round_barrier();  // no rank writes into a replica before its owner's snapshot
  };
  auto after_census = [&]() {
    f_count = census_h_.p->changed;
    f_out = census_h_.p->out_edges;
    for (int s = 0; s < 6; ++s) hist[s] = census_h_.p->status_hist[s];
  };

  auto do_recovery = [&]() {
    // recovery_scan (engine.cpp:179-205): all-pull sweep, gate ignored,
    // scheduled as a baseline pass; changed vertices reset to status 0.
    begin_pass();
    fq_ready_ = false;
    SR_CUDA(cudaMemsetAsync(changed_.p, 0, npad, cs_));
    PassOut po = det_ ? dense_pass_virtual(cfg, kGateOff, true, pass_index)
                      : dense_pass_wall(cfg, kGateOff, true, pass_index, false);
    exchange_round(false);
    census(kPassRecovery);
    read_census();
    after_census();
    sr_pass_stats st{};
    st.pass_index = pass_index;
    st.kind = SR_PASS_RECOVERY;
    if (det_) {
      st.attempts = po.totals.attempts;
      st.valid_updates = po.totals.valid;
      st.skipped = po.totals.skipped;
      st.edges_read = po.totals.edges;
    } else {
      sum_ctr(st);
      if (last_pass_blocked_) st.valid_updates = f_count;  // destinations changed
    }
    st.changed_vertices = f_count;
    m.pages_transferred += po.pages_transferred;
    m.bytes_transferred += po.bytes_transferred;
    m.kernel_runs += po.kernel_runs;
    account(st);
    m.recovery_passes += 1;
    ++pass_index;
  };

  // A small queued frontier: the consecutive sparse passes run inside one
  // single-block launch (tail_loop_kernel) with the host loop's decisions;
  // the passes are accounted from the per-pass records afterwards.
  auto do_sparse_tail = [&]() -> bool {
    if (!queue_mode() || !fq_ready_ || csr_deferred_ || std::getenv("SERAPH_NO_TAIL")) return false;
    const uint64_t q = census_h_.p->own_push, e = census_h_.p->own_edges;
    if (q == 0 || q > kTailMaxQueue || e > kTailMaxEdges || f_count == 0) return false;
    if (uint64_t(fq_epoch_) + kTailMaxPasses + 2 >= 0xffffffffull) return false;
    tail_rec_.reserve(kTailMaxPasses);
    tail_res_.reserve(1);
    TailArgs t{};
    t.values = values_.p;
    t.out_offsets = out_off_.p;
    t.out_neighbors = nbr_ptr();
    t.out_weights = w_ptr();
    t.outdeg = outdeg_.p;
    t.stamp = stamp_.p;
    t.epoch0 = fq_epoch_ + 1;
    t.list = list_.p;
    t.list2 = list2_.p;
    t.q0 = uint32_t(q);
    t.max_passes = kTailMaxPasses;
    t.dense_threshold = cfg.density_threshold_fraction * double(m_);
    t.force_sparse = cfg.execution == SR_EXEC_FORCE_SPARSE ? 1 : 0;
    t.census = census_.p;
    t.logstate = predictor_ == SR_PRED_WEAK ? logstate_.p : nullptr;
    t.rec = tail_rec_.p;
    t.res = tail_res_.p;
    *reinterpret_cast<volatile uint32_t*>(&tail_res_.p->passes) = kTailPending;
    launch_tail_loop(algo_, t, cs_);
    wait_word(&tail_res_.p->passes, kTailPending);
    const uint32_t np_run = tail_res_.p->passes;
    fq_epoch_ += np_run;
    for (uint32_t k = 0; k < np_run; ++k) {
      const TailRecord& r = tail_rec_.p[k];
      sr_pass_stats st{};
      st.pass_index = pass_index;
      st.kind = SR_PASS_SPARSE_PUSH;
      st.attempts = r.edges;  // push: attempts and edges_read count edges (engine.cpp:77-78)
      st.edges_read = r.edges;
      st.valid_updates = r.valid;
      st.changed_vertices = r.changed;
      account(st);
      m.sparse_passes += 1;
      ++pass_index;
      f_count = r.changed;
      f_out = r.out_edges;
      census_h_.p->own_push = census_h_.p->push_count = r.queued;
      census_h_.p->own_edges = census_h_.p->out_edges = r.out_edges;
      census_h_.p->changed = r.changed;
    }
    return np_run > 0;
  };

  auto do_sparse = [&]() {
    // sparse_push_pass (engine.cpp:63-93) on the device frontier
    begin_pass();
    RunStats dummy;
    push_pass(cfg, dummy);
    exchange_round(false);
    if (queue_mode()) {  // the push built the next frontier queue and its census
      read_census();
      census_h_.p->own_push = census_h_.p->push_count;
      census_h_.p->own_edges = census_h_.p->out_edges;
      std::swap(list_, list2_);
      fq_ready_ = true;
    } else {
      census(kPassSparse);
      read_census();
    }
    after_census();
    sr_pass_stats st{};
    st.pass_index = pass_index;
    st.kind = SR_PASS_SPARSE_PUSH;
    sum_ctr(st);
    st.changed_vertices = f_count;
    account(st);
    m.sparse_passes += 1;
    ++pass_index;
  };


  auto do_dense = [&]() {
    // Runner::run_dense (engine.cpp:279-337)
    begin_pass();
    fq_ready_ = false;  // the frontier after a dense pass is in the changed flags
    sr_pass_stats st{};
    st.pass_index = pass_index;
    st.kind = SR_PASS_DENSE_PULL;
    if (weak) {
      for (int s = 0; s < 6; ++s) st.status_counts[s] = hist[s];
      st.has_status_counts = 1;
    }
    SR_CUDA(cudaMemsetAsync(changed_.p, 0, npad, cs_));
    const int gate = predictor_ == SR_PRED_STRONG ? kGateStrong
                     : predictor_ == SR_PRED_WEAK ? kGateWeak
                                                   : kGateOff;
    PassOut po = det_ ? dense_pass_virtual(cfg, gate, false, pass_index)
                      : dense_pass_wall(cfg, gate, false, pass_index, false);
    exchange_round(false);
    census(kPassDense);
    read_census();
    after_census();
    if (det_) {
      st.attempts = po.totals.attempts;
      st.valid_updates = po.totals.valid;
      st.skipped = po.totals.skipped;
      st.edges_read = po.totals.edges;
    } else {
      sum_ctr(st);
      if (last_pass_blocked_) st.valid_updates = f_count;  // destinations changed
      dense_gather_frac_ = last_gather_frac_;
    }
    st.changed_vertices = f_count;
    if (strong) {
      // refresh_thresholds (predictor.cpp:89-105).  SSSP l = min value
      // written since the last refresh.  CC s (LabelHistogram::refresh,
      // predictor.cpp:66-79: the smallest label whose population changed)
      // is the same quantity: labels only decrease, so the smallest label
      // written since the refresh gained a vertex and lost none (a vertex
      // leaving it would have written a smaller label), and every label
      // that changed population was either written (>= that minimum) or
      // left for a smaller written label.  No per-label histogram needed.
      k_bfs_ += 1;
      if (algo_ == SR_ALGO_SSSP || algo_ == SR_ALGO_CC) {
        (algo_ == SR_ALGO_SSSP ? l_sssp_ : s_cc_) = census_h_.p->min_changed;
        SR_CUDA(cudaMemsetAsync(&census_.p->min_changed, 0xff, 4, cs_));
      }
    }
    // K1's source floor (kernels.cu source_floor): the smallest value written
    // since the previous dense pass bounds every source that can still
    // improve a destination.  Not under the weak predictor, whose dormant
    // destinations miss relaxations until a recovery sweep.
    if (algo_ == SR_ALGO_SSSP && !weak && weights_ge1_) {
      if (strong) {
        floor_sssp_ = l_sssp_;
      } else {
        floor_sssp_ = census_h_.p->min_changed;
        SR_CUDA(cudaMemsetAsync(&census_.p->min_changed, 0xff, 4, cs_));
      }
    }
    m.pages_transferred += po.pages_transferred;
    m.bytes_transferred += po.bytes_transferred;
    m.kernel_runs += po.kernel_runs;
    account(st);
    m.dense_passes += 1;
    ++pass_index;
  };

  for (;;) {
    if (f_count == 0) {
      if (weak && prev_dense) {
        do_recovery();
        prev_dense = false;
        if (f_count == 0) break;
        continue;
      }
      break;
    }
    bool sparse;
    if (cfg.execution == SR_EXEC_FORCE_SPARSE) sparse = true;
    else if (cfg.execution == SR_EXEC_FORCE_DENSE) sparse = false;
    else  // density_switch (engine.cpp:56-61): dense iff out-edges > frac*|E|
      sparse = !(double(f_out) > cfg.density_threshold_fraction * double(m_));
    if (sparse && weak && prev_dense) {
      do_recovery();  // dense-to-sparse switch retrieves dormant actives
      prev_dense = false;
      if (f_count == 0) break;
      continue;
    }
    if (sparse) {
      if (!do_sparse_tail()) do_sparse();
      prev_dense = false;
    } else {
      do_dense();
      prev_dense = true;
    }
    if (pass_index > 100000) throw EngineError(SR_E_INTERNAL, "pass loop did not converge");
  }

  SR_CUDA(cudaEventRecord(ev_stop_, cs_));
  if (values_out)  // pageable destinations through the pinned chunks (stager)
    stager_.d2h_sync(values_out, values_.p, size_t(n_) * 4, cs_);
  if (weak)  // run-long prediction-log accumulators (also updated by the sparse loop)
    SR_CUDA(cudaMemcpyAsync(census_h_.p, census_.p, sizeof(Census), cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  const auto wall1 = std::chrono::steady_clock::now();
  float ms = 0;
  SR_CUDA(cudaEventElapsedTime(&ms, ev_start_, ev_stop_));
  m.device_seconds = ms * 1e-3;
  if (values_out) m.d2h_bytes = uint64_t(n_) * 4;
  m.virtual_makespan = vclock_.now;
  if (cfg.clock == SR_CLOCK_WALL)
    m.wall_seconds = std::chrono::duration<double>(wall1 - wall0).count();
  if (weak && census_h_.p->log_events > 0) {
    m.has_prediction_accuracy = 1;
    m.prediction_accuracy =
        double(census_h_.p->log_events - census_h_.p->log_incorrect) / double(census_h_.p->log_events);
  }
}

// ---------------------------------------------------------------------------
uint64_t Engine::verify_fixpoint(int algo, const uint32_t* values_host) {
  SR_CUDA(cudaSetDevice(dev_));
  if (csr_deferred_) derive_csr_now();
  if (!has_csr_edges_) throw EngineError(SR_E_CONFIG, "verify needs the csr adjacency");
  if (algo == SR_ALGO_SSSP && !csr_weighted_) throw EngineError(SR_E_CONFIG, "sssp needs weights");
  DBuf<unsigned long long> viol;
  viol.reserve(1);
  const size_t npad = size_t(n_) + 16;
  if (values_host) {
    values_.reserve(std::max(values_.n, npad));
    SR_CUDA(cudaMemcpyAsync(values_.p, values_host, size_t(n_) * 4, cudaMemcpyHostToDevice, cs_));
  } else if (!values_.p) {
    throw EngineError(SR_E_DATA, "verify: no values from a previous run");
  }
  SR_CUDA(cudaMemsetAsync(viol.p, 0, 8, cs_));
  launch_verify(algo, row_lo_, row_hi_, out_off_.p, nbr_ptr(), w_ptr(), values_.p, viol.p, cs_);
  unsigned long long h = 0;
  SR_CUDA(cudaMemcpyAsync(&h, viol.p, 8, cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  return h;
}

void Engine::bench_pull_sweep(int algo, uint32_t reps, double* ms, uint64_t* edges) {
  SR_CUDA(cudaSetDevice(dev_));
  if (streaming()) throw EngineError(SR_E_CONFIG, "sweep bench needs a resident page set");
  if (!values_.p) throw EngineError(SR_E_DATA, "sweep bench: run once first");
  algo_ = algo;
  const uint32_t np = uint32_t(pages_.size());
  std::vector<uint32_t> all(np);
  for (uint32_t p = 0; p < np; ++p) all[p] = p;
  ctr_used_ = 0;
  SR_CUDA(cudaMemsetAsync(ctr_.p, 0, sizeof(RunCtr), cs_));
  launch_pages(all, kGateOff, false, ctr_.p, nullptr, false, false);  // warm
  SR_CUDA(cudaMemsetAsync(ctr_.p, 0, sizeof(RunCtr), cs_));
  SR_CUDA(cudaEventRecord(ev_start_, cs_));
  for (uint32_t r = 0; r < reps; ++r) launch_pages(all, kGateOff, false, ctr_.p, nullptr, false, false);
  SR_CUDA(cudaEventRecord(ev_stop_, cs_));
  SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr_.p, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  float t = 0;
  SR_CUDA(cudaEventElapsedTime(&t, ev_start_, ev_stop_));
  *ms = reps ? t / reps : 0.0;
  *edges = reps ? ctr_h_.p[0].edges / reps : 0;
}

cudaEvent_t Engine::trace_event() {
  if (wtrace_pool_used_ == wtrace_pool_.size()) {
    cudaEvent_t e;
    SR_CUDA(cudaEventCreate(&e));
    wtrace_pool_.push_back(e);
  }
  return wtrace_pool_[wtrace_pool_used_++];
}

// Convert the recorded events to TraceEvents (milliseconds since the run's
// start event), sorted like VirtualClock::drain (scheduler.cpp:79-88).
void Engine::finish_wall_trace() {
  if (!record_trace_ || det_) return;
  std::vector<sr_trace_event> out;
  for (const WallTraceRec& r : wtrace_) {
    float ta = 0, tb = 0;
    SR_CUDA(cudaEventElapsedTime(&ta, ev_start_, r.a));
    SR_CUDA(cudaEventElapsedTime(&tb, ev_start_, r.b));
    const int end_kind = r.start_kind == SR_TRACE_XFER_START ? SR_TRACE_XFER_END : SR_TRACE_KERNEL_END;
    for (uint32_t p : r.pages) {
      out.push_back(sr_trace_event{double(ta), r.start_kind, p, r.pass, 0});
      out.push_back(sr_trace_event{double(tb), end_kind, p, r.pass, 0});
    }
  }
  std::stable_sort(out.begin(), out.end(), [](const sr_trace_event& a, const sr_trace_event& b) {
    if (a.time != b.time) return a.time < b.time;
    if (a.page_id != b.page_id) return a.page_id < b.page_id;
    return a.kind < b.kind;
  });
  trace.insert(trace.end(), out.begin(), out.end());
  wtrace_.clear();
  wtrace_pool_used_ = 0;
}

double Engine::collect_relax_seconds() {
  double total = 0;
  for (size_t i = 0; i < relax_ev_used_; ++i) {
    float ms = 0;
    SR_CUDA(cudaEventElapsedTime(&ms, relax_ev_[i].first, relax_ev_[i].second));
    total += ms * 1e-3;
  }
  return total;
}

void Engine::flush_l2(uint64_t bytes) {
  SR_CUDA(cudaSetDevice(dev_));
  l2_flush_.reserve(bytes);
  SR_CUDA(cudaMemsetAsync(l2_flush_.p, int(++flush_gen_ & 0xff), bytes, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
}

void Engine::attach_loopback(int rank, int world, const std::string& key, bool peer_exchange) {
  if (world < 1 || rank < 0 || rank >= world) throw EngineError(SR_E_CONFIG, "bad rank/world");
  if (pages_loaded_) throw EngineError(SR_E_CONFIG, "attach must precede load_pages");
  loop_ = loopback_group(key, world);
  rank_ = rank;
  world_ = world;
  peer_xchg_ = peer_exchange;
}

// Peer exchange: every rank learns the device addresses of the other ranks'
// value replicas (the loopback world shares one address space; an NCCL world
// would map them with CUDA IPC handles).  Re-run each run: values_ may move.
void Engine::setup_peers() {
  n_peers_ = 0;
  // (virtual-clock runs are single-device: validate() rejects them in a world)
  if (!peer_xchg_ || !attached() || world_ < 2 || det_) return;
  std::vector<uint32_t*> others;
  if (loop_) {
    const std::vector<void*> all = loopback_allgather_ptr(loop_, rank_, values_.p);
    for (int r = 0; r < world_; ++r)
      if (r != rank_) others.push_back(static_cast<uint32_t*>(all[size_t(r)]));
  } else {
    // NCCL world: all-gather the CUDA IPC handles of every rank's replica and
    // map the peers' (re-mapped only when a replica moved)
    const NcclApi& nc = nccl();
    cudaIpcMemHandle_t mine;
    SR_CUDA(cudaIpcGetMemHandle(&mine, values_.p));
    const size_t hs = sizeof(cudaIpcMemHandle_t);
    ipc_buf_.reserve(hs * size_t(world_ + 1));
    SR_CUDA(cudaMemcpyAsync(ipc_buf_.p + hs * world_, &mine, hs, cudaMemcpyHostToDevice, cs_));
    const ncclResult_t r = nc.AllGather(ipc_buf_.p + hs * world_, ipc_buf_.p, hs, ncclUint8,
                                        comm_, cs_);
    if (r != ncclSuccess) throw EngineError(SR_E_NCCL, std::string("nccl: ") + nc.GetErrorString(r));
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(world_));
    SR_CUDA(cudaMemcpyAsync(all.data(), ipc_buf_.p, hs * world_, cudaMemcpyDeviceToHost, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
    ipc_handles_.resize(size_t(world_));
    ipc_ptrs_.resize(size_t(world_), nullptr);
    uint32_t ok = 1;
    for (int q = 0; q < world_; ++q) {
      if (q == rank_) continue;
      if (!ipc_ptrs_[q] || std::memcmp(&ipc_handles_[q], &all[q], hs) != 0) {
        if (ipc_ptrs_[q]) cudaIpcCloseMemHandle(ipc_ptrs_[q]);
        ipc_ptrs_[q] = nullptr;
        if (cudaIpcOpenMemHandle(&ipc_ptrs_[q], all[q], cudaIpcMemLazyEnablePeerAccess) !=
            cudaSuccess) {
          (void)cudaGetLastError();
          ipc_ptrs_[q] = nullptr;
          ok = 0;
          continue;
        }
        ipc_handles_[q] = all[q];
      }
      others.push_back(static_cast<uint32_t*>(ipc_ptrs_[q]));
    }
    // every rank must take the same exchange: any rank that cannot map a
    // peer (no P2P path) turns the world back to the all-reduce exchange
    barrier_word_.reserve(2);
    SR_CUDA(cudaMemcpyAsync(barrier_word_.p + 1, &ok, 4, cudaMemcpyHostToDevice, cs_));
    const ncclResult_t r2 =
        nc.AllReduce(barrier_word_.p + 1, barrier_word_.p + 1, 1, ncclUint32, ncclMin, comm_, cs_);
    if (r2 != ncclSuccess)
      throw EngineError(SR_E_NCCL, std::string("nccl: ") + nc.GetErrorString(r2));
    SR_CUDA(cudaMemcpyAsync(&ok, barrier_word_.p + 1, 4, cudaMemcpyDeviceToHost, cs_));
    SR_CUDA(cudaStreamSynchronize(cs_));
    if (!ok) {
      for (void*& ptr : ipc_ptrs_)
        if (ptr) {
          cudaIpcCloseMemHandle(ptr);
          ptr = nullptr;
        }
      if (rank_ == 0)
        std::fprintf(stderr, "seraph: peer exchange unavailable (CUDA IPC over P2P failed); "
                             "using the all-reduce exchange\n");
      return;
    }
  }
  peers_dev_.reserve(others.size());
  SR_CUDA(cudaMemcpy(peers_dev_.p, others.data(), others.size() * sizeof(uint32_t*),
                     cudaMemcpyHostToDevice));
  n_peers_ = uint32_t(others.size());
}

// Every rank's work enqueued so far has finished (loopback: host barrier
// after a stream sync; NCCL: a one-word all-reduce on the compute stream,
// which also fences this rank's earlier peer stores before later kernels).
void Engine::round_barrier() {
  if (loop_) {
    SR_CUDA(cudaStreamSynchronize(cs_));
    loopback_barrier(loop_);
    return;
  }
  barrier_word_.reserve(1);
  const NcclApi& nc = nccl();
  const ncclResult_t r =
      nc.AllReduce(barrier_word_.p, barrier_word_.p, 1, ncclUint32, ncclMax, comm_, cs_);
  if (r != ncclSuccess) throw EngineError(SR_E_NCCL, std::string("nccl: ") + nc.GetErrorString(r));
}

void Engine::attach_world(int rank, int world, const uint8_t id[128]) {
  SR_CUDA(cudaSetDevice(dev_));
  if (world < 1 || rank < 0 || rank >= world) throw EngineError(SR_E_CONFIG, "bad rank/world");
  if (pages_loaded_) throw EngineError(SR_E_CONFIG, "attach_world must precede load_pages");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  const NcclApi& nc = nccl();
  if (comm_) nc.CommDestroy(comm_);
  comm_ = nullptr;
  const ncclResult_t r = nc.CommInitRank(&comm_, world, uid, rank);
  if (r != ncclSuccess) throw EngineError(SR_E_NCCL, std::string("nccl init: ") + nc.GetErrorString(r));
  rank_ = rank;
  world_ = world;
}

}  // namespace seraph
