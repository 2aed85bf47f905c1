// Host engine of libseraph: graph residency, the density-switched pass loop
// and the transfer scheduler.  The loop follows the reference Runner
// (proj/src/engine.cpp:225-416) decision for decision; all per-vertex work
// runs in the sm_100a kernels of kernels.cu.
#include "engine.h"
#include "devgraph.h"
#include "loopback.h"

#include <algorithm>
#include <chrono>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <thread>

#include "kernels.h"
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
}

Engine::~Engine() {
  cudaSetDevice(dev_);
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
  SR_CUDA(cudaMemcpyAsync(out_off_.p, off, (size_t(n) + 1) * 8, cudaMemcpyHostToDevice, xs_));
  uint64_t bytes = (uint64_t(n) + 1) * 8;
  has_csr_edges_ = nbr != nullptr;
  csr_weighted_ = false;
  if (nbr && m) {
    out_nbr_.reserve(m);
    SR_CUDA(cudaMemcpyAsync(out_nbr_.p, nbr, m * 4, cudaMemcpyDefault, xs_));
    bytes += m * 4;
    if (w) {
      out_w_.reserve(m);
      SR_CUDA(cudaMemcpyAsync(out_w_.p, w, m * 4, cudaMemcpyDefault, xs_));
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

// ---------------------------------------------------------------------------
// Device-side graph build (devgraph.cu): the
// reference's build_csr + build_csc_pages (graph.cpp:30-94) as stable radix
// sorts on the GPU, then the normal residency path (tiles, arena, push
// adjacency) with the page arrays copied device to device.
// ---------------------------------------------------------------------------
void Engine::build_graph_dev(uint32_t n, uint64_t m, DBuf<uint32_t>& src, DBuf<uint32_t>& dst,
                             DBuf<uint32_t>& w, bool weighted, uint32_t cap, bool csr_edges) {
  if (cap < 1) throw EngineError(SR_E_CONFIG, "page vertex capacity must be >= 1");
  if (n == 0) throw EngineError(SR_E_INPUT, "graph has no vertices");
  if (!dg_ids_valid(n, m, src.p, dst.p, cs_))
    throw EngineError(SR_E_INPUT, "edge endpoint out of range (graph.cpp:9-22)");
  const auto t0 = std::chrono::steady_clock::now();
  const uint32_t np = uint32_t((uint64_t(n) + cap - 1) / cap);
  DBuf<unsigned long long> in_off;
  DBuf<uint32_t> in_src, in_w, local;
  in_off.reserve(size_t(n) + 1);
  in_src.reserve(std::max<uint64_t>(m, 1));
  if (weighted) in_w.reserve(std::max<uint64_t>(m, 1));
  dg_stable_adjacency(n, m, dst.p, src.p, weighted ? w.p : nullptr, in_off.p, in_src.p,
                      weighted ? in_w.p : nullptr, cs_);
  out_off_.reserve(size_t(n) + 1);
  if (csr_edges) {
    out_nbr_.reserve(std::max<uint64_t>(m, 1));
    if (weighted) out_w_.reserve(std::max<uint64_t>(m, 1));
  }
  dg_stable_adjacency(n, m, src.p, csr_edges ? dst.p : nullptr, csr_edges && weighted ? w.p : nullptr,
                      out_off_.p, csr_edges ? out_nbr_.p : nullptr,
                      csr_edges && weighted ? out_w_.p : nullptr, cs_);
  local.reserve(size_t(n) + np);
  dg_page_offsets(n, cap, in_off.p, local.p, cs_);
  SR_CUDA(cudaStreamSynchronize(cs_));
  src.release();
  dst.release();
  w.release();
  n_ = n;
  m_ = m;
  has_csr_edges_ = csr_edges;
  csr_weighted_ = csr_edges && weighted;
  finish_csr();
  PinBuf<uint32_t> local_h;
  PinBuf<unsigned long long> in_off_h;
  local_h.reserve(size_t(n) + np);
  in_off_h.reserve(size_t(n) + 1);
  SR_CUDA(cudaMemcpy(local_h.p, local.p, (size_t(n) + np) * 4, cudaMemcpyDeviceToHost));
  SR_CUDA(cudaMemcpy(in_off_h.p, in_off.p, (size_t(n) + 1) * 8, cudaMemcpyDeviceToHost));
  std::vector<sr_page_view> views(np);
  for (uint32_t p = 0; p < np; ++p) {
    const uint64_t vb = uint64_t(p) * cap, ve = std::min<uint64_t>(vb + cap, n);
    const uint64_t e0 = in_off_h.p[vb], e1 = in_off_h.p[ve];
    views[p] = sr_page_view{uint32_t(vb), uint32_t(ve), local_h.p + vb + p, in_src.p + e0,
                            weighted ? in_w.p + e0 : nullptr, e1 - e0};
  }
  last_upload_seconds = 0;
  last_upload_bytes = 0;
  load_pages(n, cap, weighted, views.data(), np);  // device-to-device into the arena
  SR_CUDA(cudaDeviceSynchronize());
  last_upload_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

void Engine::build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                         const uint32_t* w, uint32_t cap, bool csr_edges) {
  SR_CUDA(cudaSetDevice(dev_));
  if (m && (!src || !dst)) throw EngineError(SR_E_INPUT, "edge list: null endpoints");
  DBuf<uint32_t> ds, dd, dw;
  ds.reserve(std::max<uint64_t>(m, 1));
  dd.reserve(std::max<uint64_t>(m, 1));
  if (m) {
    SR_CUDA(cudaMemcpyAsync(ds.p, src, m * 4, cudaMemcpyDefault, cs_));
    SR_CUDA(cudaMemcpyAsync(dd.p, dst, m * 4, cudaMemcpyDefault, cs_));
  }
  if (w) {
    dw.reserve(std::max<uint64_t>(m, 1));
    if (m) SR_CUDA(cudaMemcpyAsync(dw.p, w, m * 4, cudaMemcpyDefault, cs_));
  }
  build_graph_dev(n, m, ds, dd, dw, w != nullptr, cap, csr_edges);
}

void Engine::generate_graph(const sr_graph_spec& g, bool csr_edges) {
  SR_CUDA(cudaSetDevice(dev_));
  if (g.scale < 1 || g.scale > 31 || g.edge_factor < 1)
    throw EngineError(SR_E_CONFIG, "rmat: scale must be in [1, 31], edge factor >= 1");
  const double sum = g.a + g.b + g.c + g.d;
  if (g.a < 0 || g.b < 0 || g.c < 0 || g.d < 0 || sum < 1 - 1e-9 || sum > 1 + 1e-9)
    throw EngineError(SR_E_CONFIG, "rmat quadrant probabilities must be >= 0 and sum to 1");
  const bool weighted = g.weight_hi != 0;
  if (weighted && (g.weight_lo < 1 || g.weight_lo > g.weight_hi))
    throw EngineError(SR_E_CONFIG, "weights: need 1 <= lo <= hi");
  const uint32_t n = uint32_t(uint64_t(1) << g.scale);
  const uint64_t m0 = uint64_t(n) * g.edge_factor;
  DBuf<uint32_t> s0, d0, w0;
  s0.reserve(m0);
  d0.reserve(m0);
  dg_rmat(g.scale, m0, g.a, g.b, g.c, g.seed, s0.p, d0.p, cs_);
  if (weighted) {
    w0.reserve(m0);
    dg_weights(m0, g.weight_seed, g.weight_lo, g.weight_hi, w0.p, cs_);
  }
  if (!g.symmetrize) {
    build_graph_dev(n, m0, s0, d0, w0, weighted, g.page_vertex_capacity, csr_edges);
    return;
  }
  DBuf<uint32_t> s1, d1, w1;
  s1.reserve(2 * m0);
  d1.reserve(2 * m0);
  if (weighted) w1.reserve(2 * m0);
  dg_symmetrize(m0, s0.p, d0.p, weighted ? w0.p : nullptr, s1.p, d1.p, weighted ? w1.p : nullptr,
                cs_);
  SR_CUDA(cudaStreamSynchronize(cs_));
  s0.release();
  d0.release();
  w0.release();
  build_graph_dev(n, 2 * m0, s1, d1, w1, weighted, g.page_vertex_capacity, csr_edges);
}

// load_binary (ingest.cpp:176-218) straight into the device build: the file's
// edge records stream through two pinned staging buffers onto the GPU (copy
// stream, double-buffered against the reads), are split into src/dst/w and
// validated there.  Same checks and exception classes as the reference:
// FormatError for a bad header/size, FormatError wrapping the edge-list
// validation (ids < num_vertices, weights >= 1).
void Engine::load_srph(const char* path, uint32_t cap, bool csr_edges) {
  SR_CUDA(cudaSetDevice(dev_));
  const std::string p = path ? path : "";
  const int fd = ::open(p.c_str(), O_RDONLY);
  if (fd < 0) throw EngineError(SR_E_FORMAT, "cannot open '" + p + "'");
  struct FdGuard {
    int fd;
    ~FdGuard() { ::close(fd); }
  } guard{fd};
  struct stat stt {};
  if (fstat(fd, &stt) != 0) throw EngineError(SR_E_FORMAT, "cannot stat '" + p + "'");
  const uint64_t size = uint64_t(stt.st_size);
  if (size < 24)
    throw EngineError(SR_E_FORMAT, "'" + p + "': header needs 24 bytes, file has " +
                                       std::to_string(size));
  unsigned char hdr[24];
  if (::pread(fd, hdr, 24, 0) != 24) throw EngineError(SR_E_FORMAT, "'" + p + "': short read");
  if (std::memcmp(hdr, "SRPH", 4) != 0) throw EngineError(SR_E_FORMAT, "'" + p + "': bad magic");
  if (hdr[4] != 1)
    throw EngineError(SR_E_FORMAT, "'" + p + "': unsupported version " + std::to_string(hdr[4]));
  const bool weighted = (hdr[5] & 1) != 0;
  uint64_t nv = 0, m = 0;
  for (int k = 7; k >= 0; --k) {
    nv = (nv << 8) | hdr[8 + k];
    m = (m << 8) | hdr[16 + k];
  }
  if (nv > 0xffffffffull)
    throw EngineError(SR_E_FORMAT, "'" + p + "': vertex count exceeds 32-bit id range");
  const uint64_t rec = weighted ? 12 : 8;
  if (m > (size - 24) / rec || size != 24 + m * rec)
    throw EngineError(SR_E_FORMAT, "'" + p + "': expected " + std::to_string(24 + m * rec) +
                                       " bytes, file has " + std::to_string(size));
  const uint64_t bytes = m * rec;
  DBuf<uint32_t> raw;
  raw.reserve(std::max<uint64_t>(bytes / 4, 1));
  constexpr uint64_t kStage = 64ull << 20;
  PinBuf<uint8_t> stage[2];
  cudaEvent_t done[2];
  for (int b = 0; b < 2; ++b) {
    stage[b].reserve(kStage);
    SR_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
  }
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      cudaEventDestroy(e[0]);
      cudaEventDestroy(e[1]);
    }
  } evg{done};
  int k = 0;
  for (uint64_t at = 0; at < bytes; at += kStage, k ^= 1) {
    const uint64_t len = std::min(kStage, bytes - at);
    SR_CUDA(cudaEventSynchronize(done[k]));  // the buffer's previous copy has landed
    uint64_t got = 0;
    while (got < len) {
      const ssize_t r = ::pread(fd, stage[k].p + got, len - got, off_t(24 + at + got));
      if (r <= 0) throw EngineError(SR_E_FORMAT, "'" + p + "': short read");
      got += uint64_t(r);
    }
    SR_CUDA(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(raw.p) + at, stage[k].p, len,
                            cudaMemcpyHostToDevice, xs_));
    SR_CUDA(cudaEventRecord(done[k], xs_));
  }
  SR_CUDA(cudaStreamSynchronize(xs_));
  DBuf<uint32_t> src, dst, w;
  src.reserve(std::max<uint64_t>(m, 1));
  dst.reserve(std::max<uint64_t>(m, 1));
  if (weighted) w.reserve(std::max<uint64_t>(m, 1));
  dg_deinterleave(m, raw.p, weighted, src.p, dst.p, weighted ? w.p : nullptr, cs_);
  raw.release();
  if (!dg_ids_valid(uint32_t(nv), m, src.p, dst.p, cs_))
    throw EngineError(SR_E_FORMAT, "'" + p + "': edge has id >= num_vertices " + std::to_string(nv));
  if (weighted && !dg_weights_valid(m, w.p, cs_))
    throw EngineError(SR_E_FORMAT, "'" + p + "': edge has weight < 1");
  build_graph_dev(uint32_t(nv), m, src, dst, w, weighted, cap, csr_edges);
}

void Engine::graph_info(sr_graph_info& gi) const {
  gi = sr_graph_info{};
  gi.num_vertices = n_;
  gi.num_edges = m_;
  gi.num_pages = uint32_t(pages_.size());
  gi.page_vertex_capacity = cap_;
  gi.weighted = weighted_ ? 1 : 0;
  gi.has_csr_edges = has_csr_edges_ ? 1 : 0;
  gi.csr_weighted = csr_weighted_ ? 1 : 0;
  gi.csr_derived = csr_derived_ ? 1 : 0;
}

void Engine::export_graph(uint64_t* out_off, uint32_t* out_nbr, uint32_t* out_w, uint64_t* in_off,
                          uint32_t* in_src, uint32_t* in_w) {
  SR_CUDA(cudaSetDevice(dev_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  if ((out_off || out_nbr || out_w) && !has_csr_) throw EngineError(SR_E_DATA, "no csr loaded");
  if (out_off) SR_CUDA(cudaMemcpy(out_off, out_off_.p, (size_t(n_) + 1) * 8, cudaMemcpyDeviceToHost));
  if (out_nbr) {
    if (!has_csr_edges_) throw EngineError(SR_E_DATA, "csr adjacency not on the device");
    if (m_) SR_CUDA(cudaMemcpy(out_nbr, out_nbr_.p, m_ * 4, cudaMemcpyDeviceToHost));
  }
  if (out_w) {
    if (!csr_weighted_) throw EngineError(SR_E_DATA, "csr has no weights");
    if (m_) SR_CUDA(cudaMemcpy(out_w, out_w_.p, m_ * 4, cudaMemcpyDeviceToHost));
  }
  if (!(in_off || in_src || in_w)) return;
  if (!pages_loaded_) throw EngineError(SR_E_DATA, "no pages loaded");
  if (in_w && !weighted_) throw EngineError(SR_E_DATA, "pages have no weights");
  uint64_t at = 0;
  std::vector<uint32_t> loc;
  for (uint32_t p = 0; p < pages_.size(); ++p) {
    const PageMeta& pm = pages_[p];
    const uint32_t range = pm.ve - pm.vb;
    const bool dev = pm.h_offs == nullptr;  // resident: arena; out-of-core: pinned stage
    const PageDesc& d = page_desc_h_[p];
    const uint32_t* offs = dev ? d.offs : pm.h_offs;
    const uint32_t* srcp = dev ? d.src : pm.h_src;
    const uint32_t* wp = dev ? d.w : pm.h_w;
    if (!offs) throw EngineError(SR_E_DATA, "page " + std::to_string(p) + " is not held");
    if (in_off) {
      loc.resize(size_t(range) + 1);
      SR_CUDA(cudaMemcpy(loc.data(), offs, loc.size() * 4, cudaMemcpyDefault));
      for (uint32_t i = 0; i <= range; ++i) in_off[pm.vb + i] = at + loc[i];
    }
    if (pm.edges) {
      if (in_src) SR_CUDA(cudaMemcpy(in_src + at, srcp, pm.edges * 4, cudaMemcpyDefault));
      if (in_w) SR_CUDA(cudaMemcpy(in_w + at, wp, pm.edges * 4, cudaMemcpyDefault));
    }
    at += pm.edges;
  }
}

void Engine::maybe_derive_csr() {
  // sr_load_csr without out_neighbors + a resident page set: build the push
  // adjacency on the device instead of shipping it over the host link.
  if (!has_csr_ || has_csr_edges_ || !pages_loaded_ || !all_resident_ || world_ > 1) return;
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
  SR_CUDA(cudaMemsetAsync(csr_cursor_.p, 0, size_t(n_) * 4, cs_));
  for (const PageMeta& pm : pages_)
    launch_csr_from_pages(tiles_.p, tile_page_.p, page_desc_.p, pm.tile_begin, pm.tile_end,
                          out_off_.p, csr_cursor_.p, out_nbr_.p, weighted_ ? out_w_.p : nullptr,
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

void Engine::load_pages(uint32_t n, uint32_t cap, bool weighted, const sr_page_view* views,
                        uint32_t np) {
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
  // ---- residency: the whole (owned) page set in HBM when it fits ----
  uint64_t used_bytes = 0;
  std::vector<char> used(np, 0);
  for (uint32_t p = 0; p < np; ++p) {
    used[p] = pages_[p].vb < own_hi_ && pages_[p].ve > own_lo_;
    if (used[p]) used_bytes += pages_[p].bytes;
  }
  all_resident_ = budget_ == 0 || used_bytes <= budget_;
  ring_reset();
  plan_window_ = 0;
  plan_cached_ = size_t(-1);
  sb_.built = false;
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
      SR_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(d.offs), pm.h_offs, (size_t(d.range) + 1) * 4,
                              cudaMemcpyHostToDevice, xs_));
      if (pm.edges) {  // host (pinned/pageable) or device (sr_build_graph) sources
        SR_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(d.src), pm.h_src, pm.edges * 4,
                                cudaMemcpyDefault, xs_));
        if (weighted)
          SR_CUDA(cudaMemcpyAsync(const_cast<uint32_t*>(d.w), pm.h_w, pm.edges * 4,
                                  cudaMemcpyDefault, xs_));
      }
      SR_CUDA(cudaEventRecord(page_events_[p], xs_));
      pm.on_device = true;
      upload += pm.bytes;
    };
    uint32_t first = np;
    for (uint32_t p = 0; p < np && first == np; ++p)
      if (used[p]) first = p;
    if (first < np) copy_page(first);
    // 2) cut tiles on the host while that DMA runs, then the small uploads
    build_tiles(own_lo_, own_hi_, xs_);
    page_desc_.reserve(std::max<uint32_t>(np, 1));
    desc_stage_.reserve(std::max<uint32_t>(np, 1));
    std::memcpy(desc_stage_.p, page_desc_h_.data(), np * sizeof(PageDesc));
    SR_CUDA(cudaMemcpyAsync(page_desc_.p, desc_stage_.p, np * sizeof(PageDesc),
                            cudaMemcpyHostToDevice, xs_));
    SR_CUDA(cudaEventRecord(ev_tiles_, xs_));
    for (uint32_t p = first + 1; p < np; ++p)
      if (used[p]) copy_page(p);
    // 3) device-side push adjacency, page by page as each copy lands
    if (csr_derived_) {
      has_csr_edges_ = false;
      csr_derived_ = false;
    }
    const bool derive = has_csr_ && !has_csr_edges_ && world_ == 1 && n_ == n &&
                        m_ == page_edges_total_;
    SR_CUDA(cudaStreamWaitEvent(cs_, ev_tiles_, 0));
    if (derive && m_) {
      out_nbr_.reserve(m_);
      if (weighted) out_w_.reserve(m_);
      csr_cursor_.reserve(n_);
      SR_CUDA(cudaMemsetAsync(csr_cursor_.p, 0, size_t(n_) * 4, cs_));
      for (uint32_t p = 0; p < np; ++p) {
        if (!used[p]) continue;
        SR_CUDA(cudaStreamWaitEvent(cs_, page_events_[p], 0));
        launch_csr_from_pages(tiles_.p, tile_page_.p, page_desc_.p, pages_[p].tile_begin,
                              pages_[p].tile_end, out_off_.p, csr_cursor_.p, out_nbr_.p,
                              weighted ? out_w_.p : nullptr, sm_count_ * 8, cs_);
      }
      SR_CUDA(cudaGetLastError());
    }
    if (derive) {
      has_csr_edges_ = true;
      csr_weighted_ = weighted;
      csr_derived_ = true;
    }
    // compute work on the pages is ordered after every copy
    for (uint32_t p = 0; p < np; ++p)
      if (used[p]) SR_CUDA(cudaStreamWaitEvent(cs_, page_events_[p], 0));
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
        return;
      }
      std::memcpy(base + so, pm.h_src, pm.edges * 4);
      if (weighted) std::memcpy(base + wo, pm.h_w, pm.edges * 4);
    });
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
  if (c.algo != SR_ALGO_PAGERANK && !has_csr_edges_ && m_ > 0)
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
    chunk_start_.reserve(m_ / kPushChunk + 2);
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
      a.k_bfs = k_bfs_;
      a.s_cc = s_cc_;
      a.l_sssp = l_sssp_;
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

// ---------------------------------------------------------------------------
// Streaming window (out-of-core path)
// ---------------------------------------------------------------------------
void Engine::ensure_slots(uint32_t window, PassOut& po) {
  // Budget plan for the out-of-core path: a ring of `window` slots sized for
  // the largest streamed page, and the heaviest pages cached permanently --
  // the largest K for which the K biggest pages plus `window` slots of the
  // (K+1)-th biggest fit (RMAT page sizes follow the popcount of the page
  // index, so "heaviest" is not an id prefix).
  std::vector<uint32_t> used;
  for (uint32_t p = 0; p < pages_.size(); ++p)
    if (pages_[p].h_offs) used.push_back(p);
  std::stable_sort(used.begin(), used.end(),
                   [&](uint32_t x, uint32_t y) { return pages_[x].bytes > pages_[y].bytes; });
  const uint32_t want = std::max<uint32_t>(window, 2);
  const size_t U = used.size();
  // slot = the largest streamed page image (stream_image_words)
  std::vector<uint64_t> suf_words(U + 1, 0);
  for (size_t k = U; k-- > 0;)
    suf_words[k] = std::max(suf_words[k + 1], stream_image_words(pages_[used[k]], weighted_));
  size_t K = 0;
  bool fits = false;
  uint64_t prefix = 0;
  for (size_t k = 0; k < U; ++k) {
    const uint64_t slot_bytes = suf_words[k] * 4;
    if (prefix + want * slot_bytes <= budget_) {
      K = k;
      fits = true;
    }
    prefix += pages_[used[k]].bytes;
  }
  if (!fits)
    throw EngineError(SR_E_CONFIG, "hbm budget " + std::to_string(budget_) +
                                       " B cannot hold a window of " + std::to_string(want) +
                                       " page slots of " + std::to_string(suf_words[0] * 4) + " B");
  const bool same_plan = plan_window_ == want && plan_cached_ == K && ring_words_ > 0;
  if (same_plan) return;
  // (re)build the cache arena for pages used[0..K)
  SR_CUDA(cudaStreamSynchronize(cs_));
  for (auto& pm : pages_) {
    pm.on_device = false;
    pm.slot = -1;
  }
  uint64_t off_total = 0, edge_total = 0;
  for (size_t k = 0; k < K; ++k) {
    PageMeta& pm = pages_[used[k]];
    pm.off_base = off_total;
    pm.edge_base = edge_total;
    off_total += pm.ve - pm.vb + 1;
    edge_total += (pm.edges + 7) & ~7ull;
  }
  edge_total += 8;
  arena_offs_.release();
  arena_src_.release();
  arena_w_.release();
  if (K) {
    arena_offs_.reserve(off_total);
    arena_src_.reserve(std::max<uint64_t>(edge_total, 1));
    if (weighted_) arena_w_.reserve(std::max<uint64_t>(edge_total, 1));
  }
  for (size_t k = 0; k < K; ++k) {
    const uint32_t p = used[k];
    PageMeta& pm = pages_[p];
    uint32_t* o = arena_offs_.p + pm.off_base;
    uint32_t* sp = arena_src_.p + pm.edge_base;
    uint32_t* wp = weighted_ ? arena_w_.p + pm.edge_base : nullptr;
    SR_CUDA(cudaMemcpyAsync(o, pm.h_offs, (size_t(pm.ve - pm.vb) + 1) * 4, cudaMemcpyHostToDevice, xs_));
    if (pm.edges) {
      SR_CUDA(cudaMemcpyAsync(sp, pm.h_src, pm.edges * 4, cudaMemcpyHostToDevice, xs_));
      if (wp) SR_CUDA(cudaMemcpyAsync(wp, pm.h_w, pm.edges * 4, cudaMemcpyHostToDevice, xs_));
    }
    launch_set_page_desc(page_desc_.p, p, o, sp, wp, xs_);
    pm.on_device = true;
    po.pages_transferred += 1;
    po.bytes_transferred += pm.bytes;
    h2d_bytes_ += pm.bytes;
  }
  // the streaming ring: `window` images of the largest streamed page
  ring_reset();
  ring_words_ = std::max<uint64_t>(suf_words[K], 1) * want;
  ring_.release();
  ring_.reserve(ring_words_);
  SR_CUDA(cudaEventRecord(ev_step_, xs_));
  SR_CUDA(cudaStreamWaitEvent(cs_, ev_step_, 0));
  plan_window_ = want;
  plan_cached_ = K;
}

void Engine::ring_reset() {
  for (int e : ring_fifo_) {
    if (slots_[e].page >= 0 && size_t(slots_[e].page) < pages_.size())
      pages_[slots_[e].page].slot = -1;
    slots_[e].page = -1;
    slot_free_.push_back(e);
  }
  ring_fifo_.clear();
  ring_head_ = 0;
}

// Drop the oldest image from the ring unless a step that is about to run
// still needs it; the next copy into its space waits for its last reader.
bool Engine::ring_evict_oldest(const std::vector<char>& protect) {
  if (ring_fifo_.empty()) return false;
  const int e = ring_fifo_.front();
  StreamSlot& sl = slots_[e];
  if (sl.page >= 0 && protect[sl.page]) return false;
  SR_CUDA(cudaStreamWaitEvent(xs_, sl.freed, 0));
  if (sl.page >= 0) pages_[sl.page].slot = -1;
  sl.page = -1;
  ring_fifo_.pop_front();
  slot_free_.push_back(e);
  if (ring_fifo_.empty()) ring_head_ = 0;
  return true;
}

// Admit a page into the ring (one DMA of its staged image on the copy
// stream).  Returns false when it cannot be placed without evicting an image
// that `protect` marks as still needed.
bool Engine::make_resident(uint32_t page, long long step, const std::vector<char>& protect,
                           PassOut& po) {
  PageMeta& pm = pages_[page];
  if (pm.on_device || pm.slot >= 0) return true;
  const uint64_t need = stream_image_words(pm, weighted_);
  if (need > ring_words_) throw EngineError(SR_E_CONTRACT, "page larger than the streaming ring");
  uint64_t pos = 0;
  for (;;) {
    if (ring_fifo_.empty()) {
      pos = 0;
      break;
    }
    const uint64_t tail = slots_[ring_fifo_.front()].start;
    if (ring_head_ > tail) {
      // live region [tail, head): free space at [head, end) and [0, tail)
      if (ring_head_ + need <= ring_words_) {
        pos = ring_head_;
        break;
      }
      if (need <= tail) {
        pos = 0;
        break;
      }
    } else if (ring_head_ + need <= tail) {
      // wrapped: free space [head, tail)
      pos = ring_head_;
      break;
    }
    if (!ring_evict_oldest(protect)) return false;
  }
  int e;
  if (!slot_free_.empty()) {
    e = slot_free_.back();
    slot_free_.pop_back();
  } else {
    e = int(slots_.size());
    slots_.emplace_back();
    SR_CUDA(cudaEventCreateWithFlags(&slots_[e].ready, cudaEventDisableTiming));
    SR_CUDA(cudaEventCreateWithFlags(&slots_[e].freed, cudaEventDisableTiming));
    SR_CUDA(cudaEventRecord(slots_[e].freed, cs_));
  }
  StreamSlot& sl = slots_[e];
  sl.start = pos;
  sl.words = need;
  WallTraceRec* tr = nullptr;
  if (record_trace_) {
    wtrace_.push_back(WallTraceRec{trace_event(), trace_event(), {page}, SR_TRACE_XFER_START,
                                   cur_pass_});
    tr = &wtrace_.back();
    SR_CUDA(cudaEventRecord(tr->a, xs_));
  }
  // the staged page image (offsets | sources | weights, 32 B aligned) in ONE DMA
  uint32_t* base = ring_.p + pos;
  const size_t r1 = size_t(pm.ve - pm.vb) + 1, so = pad8(r1), wo = so + pad8(pm.edges);
  SR_CUDA(cudaMemcpyAsync(base, pm.h_offs, need * 4, cudaMemcpyHostToDevice, xs_));
  launch_set_page_desc(page_desc_.p, page, base, base + so, weighted_ ? base + wo : nullptr, xs_);
  if (tr) SR_CUDA(cudaEventRecord(tr->b, xs_));
  SR_CUDA(cudaEventRecord(sl.ready, xs_));
  sl.page = int(page);
  sl.last_use = step;
  pm.slot = e;
  ring_fifo_.push_back(e);
  ring_head_ = pos + need;
  po.pages_transferred += 1;
  po.bytes_transferred += pm.bytes;
  h2d_bytes_ += pm.bytes;
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
  if (mode == SR_SCHED_BASELINE && !stream && !pagerank && last_gather_frac_ >= 0.05 &&
      pull_block_verts()) {
    if (pull_blocked_pass(gate, alloc_ctr(1))) {
      last_pass_blocked_ = true;
      po.kernel_runs += order.size();
      return po;
    }
    --ctr_used_;  // the (zeroed) probe slot is the first one the unblocked steps take
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
  launch_census(n_, changed_.p, predictor_ == SR_PRED_WEAK ? status_.p : nullptr,
                predictor_ == SR_PRED_WEAK ? logstate_.p : nullptr,
                has_csr_ ? outdeg_.p : nullptr, pass_kind, own_lo_, own_hi_, blk_cnt_.p,
                blk_edges_.p, census_part_.p, census_.p, cs_);
}

void Engine::read_census() {
  if (ctr_used_ <= 64 && !std::getenv("SERAPH_NO_PUBLISH")) {
    // one kernel writes both into the mapped pinned buffers (UVA): no D2H DMAs
    launch_publish(census_.p, census_h_.p, ctr_.p, ctr_h_.p, ctr_used_, cs_);
  } else {
    SR_CUDA(cudaMemcpyAsync(census_h_.p, census_.p, sizeof(Census), cudaMemcpyDeviceToHost, cs_));
    if (ctr_used_)
      SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr_.p, size_t(ctr_used_) * sizeof(RunCtr),
                              cudaMemcpyDeviceToHost, cs_));
  }
  SR_CUDA(cudaStreamSynchronize(cs_));
}

void Engine::build_push_list() {
  const uint32_t nb = (n_ + kCensusBlockVerts - 1) / kCensusBlockVerts;
  launch_scan_blocks(nb, blk_cnt_.p, blk_edges_.p, cs_);
  launch_compact(n_, own_lo_, own_hi_, changed_.p, outdeg_.p, blk_cnt_.p, blk_edges_.p,
                 list_.p, pref_.p, chunk_start_.p, cs_);
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
  if (queue && fq_ready_) {
    launch_queue_prep(list_.p, uint32_t(n_list), outdeg_.p, pref_.p, chunk_start_.p, scan_tmp_.p,
                      scan_tmp_.n, cs_);
  } else {
    build_push_list();
  }
  if (queue) {
    SR_CUDA(cudaMemsetAsync(census_.p, 0, kCensusResetBytes, cs_));
    if (++fq_epoch_ == 0xffffffffu) {  // epochs exhausted: restart the stamps
      SR_CUDA(cudaMemsetAsync(stamp_.p, 0, stamp_.n * 4, cs_));
      fq_epoch_ = 1;
    }
  }
  RunCtr* slot = alloc_ctr(1);
  if (total > 0) {
    PushArgs a{};
    a.list = list_.p;
    a.pref = pref_.p;
    a.chunk_start = chunk_start_.p;
    a.n_list = uint32_t(n_list);
    a.total_edges = total;
    a.out_offsets = out_off_.p;
    a.out_neighbors = out_nbr_.p;
    a.out_weights = csr_weighted_ ? out_w_.p : nullptr;
    a.values = values_.p;
    a.next = det_ ? next_.p : values_.p;
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
    const uint64_t chunks = (total + kPushChunk - 1) / kPushChunk;
    const int grid = int(std::max<uint64_t>(
        1, std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_, (chunks + kWarpsPerBlock - 1) / kWarpsPerBlock)));
    launch_push(algo_, det_, a, grid, cs_);
    SR_CUDA(cudaGetLastError());
    if (det_) launch_push_commit(values_.p, next_.p, changed_.p, n_, slot, census_.p, cs_);
  }
  (void)st;
}

void Engine::exchange_round(bool pagerank) {
  if (!attached()) return;  // attached to a world (any size, incl. 1): merge every round
  SR_CUDA(cudaSetDevice(dev_));
  if (loop_) {  // in-process loopback (tests): the same reductions through host memory
    if (pagerank) {
      loopback_allreduce(loop_, rank_, rank_b_.p, n_, kLoopF32, kLoopSum, cs_);
      loopback_allreduce(loop_, rank_, contrib_b_.p, n_, kLoopF32, kLoopSum, cs_);
    } else {
      loopback_allreduce(loop_, rank_, values_.p, n_, kLoopU32, kLoopMin, cs_);
      loopback_allreduce(loop_, rank_, &census_.p->min_changed, 1, kLoopU32, kLoopMin, cs_);
    }
    // every rank reduces the same number of counter entries (same schedule)
    loopback_allreduce(loop_, rank_, ctr_.p, size_t(ctr_used_) * (sizeof(RunCtr) / 8), kLoopU64,
                       kLoopSum, cs_);
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
  if (r == ncclSuccess && ctr_used_)
    r = nc.AllReduce(ctr_.p, ctr_.p, size_t(ctr_used_) * (sizeof(RunCtr) / 8), ncclUint64,
                     ncclSum, comm_, cs_);
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
  maybe_derive_csr();
  validate(cfg);
  algo_ = cfg.algo;
  source_ = cfg.source;
  predictor_ = cfg.algo == SR_ALGO_PAGERANK ? SR_PRED_OFF : cfg.predictor;
  det_ = cfg.clock == SR_CLOCK_VIRTUAL && cfg.algo != SR_ALGO_PAGERANK;
  record_trace_ = cfg.record_trace != 0;
  pr_damp_ = cfg.pr_damping;
  profile_kernels_ = cfg.profile_kernels != 0;
  relax_ev_used_ = 0;
  gathers_total_ = 0;
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
  const uint64_t launches0 = kernel_launch_count();
  if (cfg.algo == SR_ALGO_PAGERANK) run_pagerank(cfg, ranks_out, m, passes);
  else run_traversal(cfg, values_out, m, passes);
  m.kernel_launches = kernel_launch_count() - launches0;  // every kernel of the run
  m.h2d_bytes = h2d_bytes_;
  m.gathers = gathers_total_;
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
  last_gather_frac_ = 1.0;  // the first dense pass gathers
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
    uint64_t gathers = 0;
    for (size_t i = 0; i < size_t(ctr_used_); ++i) {
      gathers += ctr_h_.p[i].gathers;
      st.attempts += ctr_h_.p[i].attempts;
      st.valid_updates += ctr_h_.p[i].valid;
      st.skipped += ctr_h_.p[i].skipped;
      st.edges_read += ctr_h_.p[i].edges;
    }
    gathers_total_ += gathers;
    last_gather_frac_ = st.edges_read ? double(gathers) / double(st.edges_read) : 0.0;
  };
  auto begin_pass = [&]() {
    ctr_used_ = 0;
    SR_CUDA(cudaMemsetAsync(ctr_.p, 0, ctr_.n * sizeof(RunCtr), cs_));
    if (attached())
      SR_CUDA(cudaMemcpyAsync(round_snap_.p, values_.p, size_t(n_) * 4, cudaMemcpyDeviceToDevice, cs_));
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
    if (!queue_mode() || !fq_ready_ || std::getenv("SERAPH_NO_TAIL")) return false;
    const uint64_t q = census_h_.p->own_push, e = census_h_.p->own_edges;
    if (q == 0 || q > kTailMaxQueue || e > kTailMaxEdges || f_count == 0) return false;
    if (uint64_t(fq_epoch_) + kTailMaxPasses + 2 >= 0xffffffffull) return false;
    tail_rec_.reserve(kTailMaxPasses);
    tail_res_.reserve(1);
    TailArgs t{};
    t.values = values_.p;
    t.out_offsets = out_off_.p;
    t.out_neighbors = out_nbr_.p;
    t.out_weights = csr_weighted_ ? out_w_.p : nullptr;
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
    launch_tail_loop(algo_, t, cs_);
    SR_CUDA(cudaStreamSynchronize(cs_));
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
  if (values_out)
    SR_CUDA(cudaMemcpyAsync(values_out, values_.p, size_t(n_) * 4, cudaMemcpyDeviceToHost, cs_));
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
// Source-blocked sub-pages for PageRank: when the contrib array outgrows the
// L2, every iteration sweeps the sub-pages block by block so the gathers of
// one sweep stay inside a blk_verts slice (SERAPH_PR_BLOCK_VERTS, default
// 16 Mi vertices = 64 MB of f32; 0 disables).
// ---------------------------------------------------------------------------
bool Engine::build_src_blocks(uint64_t blk) {
  if (sb_.built && sb_.blk_verts == blk) return true;
  if (!all_resident_) return false;  // sharded ranks block their own destinations
  if (blk == 0 || n_ <= blk) return false;
  sb_.built = false;
  const uint32_t np = uint32_t(pages_.size());
  for (uint32_t p = 0; p < np; ++p)
    if (pages_[p].vb != uint64_t(p) * cap_) return false;  // uniform cut (graph.cpp:75-92)
  const uint32_t nb = uint32_t((n_ + blk - 1) / blk);
  uint32_t n_tiles = 0;  // a sharded rank holds tiles for its own pages only
  for (const PageMeta& pm : pages_) n_tiles = std::max(n_tiles, pm.tile_end);
  const bool timing = std::getenv("SERAPH_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!timing) return;
    SR_CUDA(cudaStreamSynchronize(cs_));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[seraph] src blocks %s: %.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // 1) counts per (block, destination)
  DBuf<uint32_t> cnt;
  cnt.reserve(size_t(nb) * n_);
  SR_CUDA(cudaMemsetAsync(cnt.p, 0, size_t(nb) * n_ * 4, cs_));
  launch_src_block(0, tiles_.p, tile_page_.p, page_desc_.p, 0, n_tiles, n_, uint32_t(blk), np,
                   cnt.p, nullptr, nullptr, nullptr, nullptr, sm_count_ * 8, cs_);
  // 2) page-local offsets per sub-page, sub-page sizes
  DBuf<unsigned long long> goff, bp_edges, bp_base;
  goff.reserve(size_t(nb) * n_);
  bp_edges.reserve(size_t(nb) * np);
  bp_base.reserve(size_t(nb) * np);
  stage("count");
  launch_src_block_scan(cnt.p, goff.p, page_desc_.p, np, nb, n_, bp_edges.p, cs_);
  stage("scan");
  std::vector<unsigned long long> edges_h(size_t(nb) * np), base_h(size_t(nb) * np);
  SR_CUDA(cudaMemcpyAsync(edges_h.data(), bp_edges.p, edges_h.size() * 8, cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  unsigned long long at = 0;
  for (size_t k = 0; k < edges_h.size(); ++k) {  // block-major, 32 B aligned sub-pages
    base_h[k] = at;
    at += (edges_h[k] + 7) & ~7ull;
    if (edges_h[k] > 0xffffffffull) return false;
  }
  sb_.src.reserve(at + 8);
  if (weighted_) sb_.w.reserve(at + 8);
  else sb_.w.release();
  SR_CUDA(cudaMemcpyAsync(bp_base.p, base_h.data(), base_h.size() * 8, cudaMemcpyHostToDevice, cs_));
  // 3) scatter the sources (cnt reused as cursors)
  SR_CUDA(cudaMemsetAsync(cnt.p, 0, size_t(nb) * n_ * 4, cs_));
  launch_src_block(1, tiles_.p, tile_page_.p, page_desc_.p, 0, n_tiles, n_, uint32_t(blk), np,
                   cnt.p, goff.p, sb_.src.p, weighted_ ? sb_.w.p : nullptr, bp_base.p,
                   sm_count_ * 8, cs_);
  stage("scatter");
  // 4) u32 local offsets of every sub-page, then the tile cut on the device
  const size_t per_block = size_t(n_) + np;
  sb_.offs.reserve(size_t(nb) * per_block);
  launch_src_block_offs(n_, cap_, np, nb, goff.p, bp_edges.p, sb_.offs.p, cs_);
  const size_t K = sub_tile_windows(cap_, np, nb);
  const size_t K_blk = K / nb;  // windows per block
  DBuf<uint32_t> tcnt, tat;
  tcnt.reserve(K + 1);
  tat.reserve(K + 1);
  SR_CUDA(cudaMemsetAsync(tcnt.p + K, 0, 4, cs_));
  launch_sub_tiles(0, n_, cap_, np, nb, own_lo_, own_hi_, sb_.offs.p, tcnt.p, nullptr, nullptr,
                   nullptr, cs_);
  launch_exclusive_scan_u32(tcnt.p, tat.p, K + 1, cs_);
  sb_.block_tile_begin.assign(nb + 1, 0);
  for (uint32_t b = 0; b <= nb; ++b)
    SR_CUDA(cudaMemcpyAsync(&sb_.block_tile_begin[b], tat.p + size_t(b) * K_blk, 4,
                            cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  const uint32_t n_sub_tiles = sb_.block_tile_begin[nb];
  sb_.tiles.reserve(std::max<size_t>(n_sub_tiles, 1));
  sb_.tile_page.reserve(std::max<size_t>(n_sub_tiles, 1));
  launch_sub_tiles(1, n_, cap_, np, nb, own_lo_, own_hi_, sb_.offs.p, nullptr, tat.p, sb_.tiles.p,
                   sb_.tile_page.p, cs_);
  SR_CUDA(cudaGetLastError());
  stage("offsets + tile cut");
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
  SR_CUDA(cudaStreamSynchronize(cs_));
  sb_.acc.reserve(n_);
  SR_CUDA(cudaMemset(sb_.acc.p, 0, size_t(n_) * 4));
  sb_.blk_verts = uint32_t(blk);
  sb_.n_blocks = nb;
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

bool Engine::pull_blocked_pass(int gate, RunCtr* ctr) {
  const uint64_t blk = pull_block_verts();
  if (!blk || !build_src_blocks(blk)) return false;
  const uint32_t run_id = ++run_id_;
  for (uint32_t b = 0; b < sb_.n_blocks; ++b) {
    const uint32_t t0 = sb_.block_tile_begin[b], t1 = sb_.block_tile_begin[b + 1];
    if (t1 <= t0) continue;
    l2_window(values_.p + uint64_t(b) * blk, std::min<uint64_t>(blk, n_ - uint64_t(b) * blk) * 4);
    PullArgs a{};
    a.work = next_work_counter();
    a.tiles = sb_.tiles.p;
    a.tile_page = sb_.tile_page.p;
    a.pages = sb_.desc.p;
    a.seg.n = 1;
    a.seg.tile_begin[0] = t0;
    a.seg.task_prefix[0] = 0;
    a.seg.task_prefix[1] = t1 - t0;
    a.values = values_.p;
    a.next = values_.p;
    a.changed = changed_.p;
    a.status = status_.p;
    a.hub_stamp = hub_stamp_.p;
    a.run_id = run_id;
    a.ctr = ctr;
    a.census = census_.p;
    a.count_dest = b == 0 ? 1u : 0u;
    a.count_valid = 0;
    a.k_bfs = k_bfs_;
    a.s_cc = s_cc_;
    a.l_sssp = l_sssp_;
    const int grid = int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                            (uint64_t(t1 - t0) + kWarpsPerBlock - 1) / kWarpsPerBlock));
    auto* evp = relax_begin();
    launch_pull(algo_, gate, false, a, std::max(grid, 1), cs_);
    SR_CUDA(cudaGetLastError());
    if (evp) SR_CUDA(cudaEventRecord(evp->second, cs_));
    if (b == 0 && sb_.n_blocks > 1) {
      // Probe: blocking pays for gathers only.  If block 0 gathered for < 5 %
      // of its edges (converged labels/levels skip theirs), finish the pass
      // with one unblocked sweep instead of n_blocks - 1 more destination
      // passes (its relaxations are idempotent; the counters restart).
      SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr, sizeof(RunCtr), cudaMemcpyDeviceToHost, cs_));
      SR_CUDA(cudaStreamSynchronize(cs_));
      const RunCtr& c0 = ctr_h_.p[0];
      if (c0.edges > 0 && double(c0.gathers) < 0.05 * double(c0.edges)) {
        SR_CUDA(cudaMemsetAsync(ctr, 0, sizeof(RunCtr), cs_));
        l2_window(nullptr, 0);
        return false;
      }
    }
  }
  l2_window(nullptr, 0);
  return true;
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
    const int grid = int(std::min<uint64_t>(uint64_t(sm_count_) * blocks_per_sm_,
                                            (uint64_t(t1 - t0) + kWarpsPerBlock - 1) / kWarpsPerBlock));
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
// PageRank (new algorithm; conventions pinned in DESIGN.md §2)
// ---------------------------------------------------------------------------
void Engine::run_pagerank(const sr_run_config& cfg, float* ranks_out, sr_metrics& m,
                          std::vector<sr_pass_stats>& passes) {
  uint64_t pr_blk = 32ull << 20;  // tools/pr_blocks.py: 32 Mi best on RMAT-26, smaller lose
  if (const char* e = std::getenv("SERAPH_PR_BLOCK_VERTS")) pr_blk = std::strtoull(e, nullptr, 10);
  const bool blocked = build_src_blocks(pr_blk);
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
  for (uint32_t it = 0; it < cfg.pr_iterations; ++it) {
    ctr_begin.push_back(ctr_used_);
    if (attached()) {
      SR_CUDA(cudaMemsetAsync(rank_b_.p, 0, size_t(n_) * 4, cs_));
      SR_CUDA(cudaMemsetAsync(contrib_b_.p, 0, size_t(n_) * 4, cs_));
    }
    PassOut po;
    const float base = float((1.0 - cfg.pr_damping) / double(n_));
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
    exchange_round(true);
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
  if (ranks_out)
    SR_CUDA(cudaMemcpyAsync(ranks_out, rank_a_.p, size_t(n_) * 4, cudaMemcpyDeviceToHost, cs_));
  if (ctr_used_)
    SR_CUDA(cudaMemcpyAsync(ctr_h_.p, ctr_.p, size_t(ctr_used_) * sizeof(RunCtr),
                            cudaMemcpyDeviceToHost, cs_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  ctr_begin.push_back(ctr_used_);
  for (size_t it = 0; it + 1 < ctr_begin.size(); ++it) {
    if (blocked) continue;  // counted analytically above
    sr_pass_stats& st = passes[passes.size() - (ctr_begin.size() - 1) + it];
    for (uint32_t i = ctr_begin[it]; i < ctr_begin[it + 1]; ++i) {
      gathers_total_ += ctr_h_.p[i].gathers;
      st.attempts += ctr_h_.p[i].attempts;
      st.edges_read += ctr_h_.p[i].edges;
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

// ---------------------------------------------------------------------------
uint64_t Engine::verify_fixpoint(int algo, const uint32_t* values_host) {
  SR_CUDA(cudaSetDevice(dev_));
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
  launch_verify(algo, n_, out_off_.p, out_nbr_.p, csr_weighted_ ? out_w_.p : nullptr, values_.p,
                viol.p, cs_);
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

void Engine::attach_loopback(int rank, int world, const std::string& key) {
  if (world < 1 || rank < 0 || rank >= world) throw EngineError(SR_E_CONFIG, "bad rank/world");
  if (pages_loaded_) throw EngineError(SR_E_CONFIG, "attach must precede load_pages");
  loop_ = loopback_group(key, world);
  rank_ = rank;
  world_ = world;
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
