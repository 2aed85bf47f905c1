// Device-side graph construction of the engine:
// build from an edge list, generate, load SRPH files, export in the
// reference layouts.  Kernels in devgraph.cu.
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "devgraph.h"

namespace seraph {

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
  if (weighted && !dg_weights_valid(m, w.p, cs_))
    throw EngineError(SR_E_INPUT, "edge has weight < 1 (graph.cpp:9-22)");
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
  adj_host_ = false;  // built in HBM; load_pages moves it out if it breaks a budget
  row_lo_ = 0;
  row_hi_ = n;
  nbr_base_ = 0;
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
  const bool timing = std::getenv("SERAPH_TIMING") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto stage = [&](const char* what) {
    if (!timing) return;
    SR_CUDA(cudaStreamSynchronize(cs_));
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[seraph] generate_graph %s: %.3f s\n", what,
                 std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  DBuf<uint32_t> s0, d0, w0;
  s0.reserve(m0);
  d0.reserve(m0);
  dg_rmat(g.scale, m0, g.a, g.b, g.c, g.seed, s0.p, d0.p, cs_);
  stage("rmat");
  if (weighted) {
    w0.reserve(m0);
    dg_weights(m0, g.weight_seed, g.weight_lo, g.weight_hi, w0.p, cs_);
    stage("weights");
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
  stage("symmetrize");
  s0.release();
  d0.release();
  w0.release();
  build_graph_dev(n, 2 * m0, s1, d1, w1, weighted, g.page_vertex_capacity, csr_edges);
  stage("build");
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
  gi.adjacency_on_host = adj_host_ ? 1 : 0;
}

void Engine::export_graph(uint64_t* out_off, uint32_t* out_nbr, uint32_t* out_w, uint64_t* in_off,
                          uint32_t* in_src, uint32_t* in_w) {
  SR_CUDA(cudaSetDevice(dev_));
  SR_CUDA(cudaStreamSynchronize(cs_));
  if ((out_off || out_nbr || out_w) && !has_csr_) throw EngineError(SR_E_DATA, "no csr loaded");
  if (out_off) SR_CUDA(cudaMemcpy(out_off, out_off_.p, (size_t(n_) + 1) * 8, cudaMemcpyDeviceToHost));
  if (out_nbr) {
    if (csr_deferred_) {
      derive_csr_now();
      SR_CUDA(cudaStreamSynchronize(cs_));
    }
    if (!has_csr_edges_) throw EngineError(SR_E_DATA, "csr adjacency not on the device");
    if (row_lo_ != 0 || row_hi_ != n_)
      throw EngineError(SR_E_DATA, "a sharded rank holds only its own csr rows");
    if (m_) SR_CUDA(cudaMemcpy(out_nbr, nbr_ptr(), m_ * 4, cudaMemcpyDefault));
  }
  if (out_w) {
    if (!csr_weighted_) throw EngineError(SR_E_DATA, "csr has no weights");
    if (m_) SR_CUDA(cudaMemcpy(out_w, w_ptr(), m_ * 4, cudaMemcpyDefault));
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

}  // namespace seraph
