// pagestream_seraph.hpp -- C++ drop-in for the reference's hot path.
//
// Header-only bridge from the reference's own types
// (proj/include/pagestream/{graph,programs,engine,metrics}.hpp) to the C-ABI
// of libseraph.so (include/seraph.h).  A reference build replaces the body of
// pagestream::run (proj/src/engine.cpp:421-433) with
//     return pagestream::seraph::run(csr, pages, program, config);
// and links libseraph.so.  Errors come back as the
// reference's exception classes (proj/include/pagestream/errors.hpp:8-28).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "pagestream/engine.hpp"
#include "pagestream/errors.hpp"
#include "seraph.h"

namespace pagestream::seraph {

// Map an SR_E_* code onto the reference's exception taxonomy.
[[noreturn]] inline void rethrow(int rc, const char* msg) {
  const std::string m = msg ? msg : "libseraph error";
  switch (rc) {
    case SR_E_CONFIG: throw ConfigError(m);
    case SR_E_INPUT: throw InputError(m);
    case SR_E_CONTRACT: throw ContractError(m);
    case SR_E_DATA: throw DataError(m);
    case SR_E_FORMAT: throw FormatError(m);
    case SR_E_PARSE: throw ParseError(m);
    default: throw Error(m);
  }
}

// Options of a drop-in call beyond the reference's signature.
//  devices:    GPUs of this process to shard the run over (empty: the
//              SERAPH_DEVICES environment variable, e.g. "0,1,2,3", else GPU 0).
//              More than one device runs the sharded world (sr_group_*);
//              ClockMode::Virtual (the reference's deterministic schedule)
//              always runs on the first device alone.
//  generation: residency cache.  0 (default): every call uploads its graph,
//              exactly like the reference's run() reads its arguments.  g != 0:
//              the caller promises that the CsrGraph/PageSet objects at these
//              addresses are unchanged since the last call with the same g, so
//              a repeated run (run_matrix cells and repetitions,
//              bench.cpp:169-275) reuses the graph resident in HBM.
struct RunOptions {
  std::vector<int> devices;
  uint64_t generation = 0;
};

inline std::vector<int> env_devices() {
  std::vector<int> d;
  if (const char* e = std::getenv("SERAPH_DEVICES")) {
    std::string s(e);
    size_t at = 0;
    while (at < s.size()) {
      size_t comma = s.find(',', at);
      if (comma == std::string::npos) comma = s.size();
      if (comma > at) d.push_back(std::atoi(s.substr(at, comma - at).c_str()));
      at = comma + 1;
    }
  }
  if (d.empty()) d.push_back(0);
  return d;
}

// Identity of the graph a context holds (residency cache).
struct GraphKey {
  const void* csr = nullptr;
  const void* pages = nullptr;
  uint64_t generation = 0, n = 0, m = 0, np = 0;
  bool lean = false;  // loaded for PageRank (no push adjacency)
  bool operator==(const GraphKey& o) const {
    return generation != 0 && csr == o.csr && pages == o.pages && generation == o.generation &&
           n == o.n && m == o.m && np == o.np && lean == o.lean;
  }
};

// One context per device, reused across calls; run() is serialised per
// device (the reference allows concurrent run() calls, bench.cpp:254-259).
struct DeviceContext {
  sr_ctx* ctx = nullptr;
  std::mutex mu;
  GraphKey held;
  ~DeviceContext() {
    if (ctx) sr_close(ctx);
  }
};

inline DeviceContext& device_context(int device = 0) {
  static DeviceContext dc[16];
  DeviceContext& d = dc[device & 15];
  std::lock_guard<std::mutex> lk(d.mu);
  if (!d.ctx) {
    const int rc = sr_open(device, 0, &d.ctx);
    if (rc != SR_OK) rethrow(rc, sr_global_error());
  }
  return d;
}

// One multi-GPU world per device list.
struct GroupContext {
  sr_group* g = nullptr;
  std::mutex mu;
  GraphKey held;
  ~GroupContext() {
    if (g) sr_group_close(g);
  }
};

inline GroupContext& group_context(const std::vector<int>& devices) {
  static std::mutex reg_mu;
  static std::vector<std::pair<std::vector<int>, std::unique_ptr<GroupContext>>> reg;
  std::lock_guard<std::mutex> lk(reg_mu);
  for (auto& [k, gc] : reg)
    if (k == devices) return *gc;
  auto gc = std::make_unique<GroupContext>();
  const int rc = sr_group_open(devices.data(), int(devices.size()), 0, SR_EXCHANGE_PEER, &gc->g);
  if (rc != SR_OK) rethrow(rc, sr_group_last_error(nullptr));
  reg.emplace_back(devices, std::move(gc));
  return *reg.back().second;
}

inline sr_run_config to_c(const VertexProgram& program, const EngineConfig& config) {
  sr_run_config c;
  sr_default_config(&c);
  c.algo = int32_t(program.kind);  // AlgoKind: Bfs=0, Cc=1, Sssp=2 (types.hpp:20)
  c.source = program.source;
  c.predictor = int32_t(config.predictor);
  c.schedule = int32_t(config.schedule.kind);
  c.max_reentry_times = config.schedule.max_reentry_times;
  c.buffer_repetitions = config.schedule.buffer_repetitions;
  c.window_capacity = config.window_capacity;
  c.density_threshold_fraction = config.density_threshold_fraction;
  c.bytes_per_time_unit = config.transfer.bytes_per_time_unit;
  c.edges_per_time_unit_per_worker = config.transfer.edges_per_time_unit_per_worker;
  c.worker_count = config.transfer.worker_count;
  c.clock = config.clock == ClockMode::Wall ? SR_CLOCK_WALL : SR_CLOCK_VIRTUAL;
  c.execution = int32_t(config.execution);
  c.record_trace = config.record_trace ? 1 : 0;
  c.seed = config.seed;
  return c;
}

// pagestream::run (engine.hpp:125-126) executed by libseraph (options above).
inline RunResult run(const CsrGraph& csr, const PageSet& pages, const VertexProgram& program,
                     const EngineConfig& config, const RunOptions& opt) {
  config.validate();  // engine.cpp:422 (ConfigError on the host, as before)
  if (csr.num_vertices != pages.num_vertices)
    throw ConfigError("csr and page set disagree on vertex count");
  if (program.uses_weights() && (!csr.weighted() || !pages.weighted))
    throw ConfigError("sssp requires weighted graph structures");
  if (program.kind != AlgoKind::Cc && program.source >= csr.num_vertices)
    throw ConfigError("source vertex out of range");

  std::vector<sr_page_view> views(pages.pages.size());
  for (size_t i = 0; i < views.size(); ++i) {
    const CscPage& p = pages.pages[i];
    views[i] = sr_page_view{p.vertex_begin, p.vertex_end, p.in_offsets.data(),
                            p.in_sources.data(),
                            pages.weighted ? p.in_weights.data() : nullptr, p.edge_count()};
  }
  const sr_run_config c = to_c(program, config);
  RunResult r;
  r.values.resize(csr.num_vertices);
  sr_metrics m{};
  std::vector<sr_pass_stats> passes(256);
  uint32_t npass = 0;
  const std::vector<int> devices = opt.devices.empty() ? env_devices() : opt.devices;
  GraphKey key{&csr, &pages, opt.generation, csr.num_vertices, csr.num_edges(),
               pages.pages.size(), false};
  const uint64_t* off = csr.out_offsets.data();
  const uint32_t* nbr = csr.out_neighbors.data();
  const uint32_t* wts = csr.weighted() ? csr.out_weights.data() : nullptr;
  const int wp = pages.weighted ? 1 : 0;
  const uint32_t np = uint32_t(views.size());
  sr_ctx* trace_ctx = nullptr;
  if (devices.size() > 1 && config.clock == ClockMode::Wall) {  // sharded over the devices
    GroupContext& gc = group_context(devices);
    std::lock_guard<std::mutex> lk(gc.mu);
    for (;;) {
      int rc;
      if (gc.held == key) {
        rc = sr_group_run(gc.g, &c, r.values.data(), nullptr, &m, passes.data(),
                          uint32_t(passes.size()), &npass);
      } else {
        gc.held = GraphKey{};
        rc = sr_group_load_graph(gc.g, csr.num_vertices, csr.num_edges(), off, nbr, wts,
                                 pages.page_vertex_capacity, wp, views.data(), np, -1);
        if (rc == SR_OK) {
          gc.held = key;
          rc = sr_group_run(gc.g, &c, r.values.data(), nullptr, &m, passes.data(),
                            uint32_t(passes.size()), &npass);
        }
      }
      if (rc != SR_OK) rethrow(rc, sr_group_last_error(gc.g));
      if (npass <= passes.size()) break;
      passes.resize(npass);
    }
  } else {
    DeviceContext& dc = device_context(devices[0]);
    std::lock_guard<std::mutex> lk(dc.mu);
    for (;;) {
      int rc;
      if (dc.held == key) {
        rc = sr_run(dc.ctx, &c, r.values.data(), nullptr, &m, passes.data(),
                    uint32_t(passes.size()), &npass);
      } else {
        dc.held = GraphKey{};
        rc = sr_run_graph(dc.ctx, csr.num_vertices, csr.num_edges(), off, nbr, wts,
                          pages.page_vertex_capacity, wp, views.data(), np, &c, r.values.data(),
                          nullptr, &m, passes.data(), uint32_t(passes.size()), &npass);
        if (rc == SR_OK) dc.held = key;
      }
      if (rc != SR_OK) rethrow(rc, sr_last_error(dc.ctx));
      if (npass <= passes.size()) break;
      passes.resize(npass);  // rerun with room for every pass record
    }
    trace_ctx = dc.ctx;
  }
  MetricsReport& mr = r.metrics;
  mr.passes = m.passes;
  mr.sparse_passes = m.sparse_passes;
  mr.dense_passes = m.dense_passes;
  mr.recovery_passes = m.recovery_passes;
  mr.pages_transferred = m.pages_transferred;
  mr.bytes_transferred = m.bytes_transferred;
  mr.update_attempts = m.update_attempts;
  mr.valid_updates = m.valid_updates;
  mr.skipped_vertices = m.skipped_vertices;
  mr.edges_read = m.edges_read;
  mr.virtual_makespan = m.virtual_makespan;
  mr.wall_seconds = m.wall_seconds;
  if (m.has_prediction_accuracy) mr.prediction_accuracy = m.prediction_accuracy;
  for (uint32_t i = 0; i < npass; ++i) {
    const sr_pass_stats& s = passes[i];
    PassStats ps;
    ps.pass_index = s.pass_index;
    ps.kind = PassKind(s.kind);
    ps.attempts = s.attempts;
    ps.valid_updates = s.valid_updates;
    ps.skipped = s.skipped;
    ps.edges_read = s.edges_read;
    ps.changed_vertices = s.changed_vertices;
    for (int k = 0; k < 6; ++k) ps.status_counts[k] = s.status_counts[k];
    ps.has_status_counts = s.has_status_counts != 0;
    mr.per_pass.push_back(ps);
  }
  if (config.record_trace && trace_ctx) {
    uint64_t n = 0;
    sr_get_trace(trace_ctx, nullptr, 0, &n);
    std::vector<sr_trace_event> ev(n);
    sr_get_trace(trace_ctx, ev.data(), n, &n);
    for (const auto& e : ev)
      r.trace.push_back(TraceEvent{e.time, TraceEventKind(e.kind), e.page_id, e.pass_index});
  }
  return r;
}

// The reference's signature: the drop-in body of pagestream::run.
inline RunResult run(const CsrGraph& csr, const PageSet& pages, const VertexProgram& program,
                     const EngineConfig& config) {
  return run(csr, pages, program, config, RunOptions{});
}

// build_csr + build_csc_pages (graph.cpp:30-94) on the GPU (sr_build_graph:
// stable radix sorts, bit-identical arrays), returned as the reference's own
// types.  Same validation and exception classes as EdgeList::validate.
inline std::pair<CsrGraph, PageSet> build_graph(const EdgeList& el,
                                                VertexId page_vertex_capacity, int device = 0) {
  if (page_vertex_capacity < 1) throw ConfigError("page_vertex_capacity must be >= 1");
  el.validate();  // InputError on the host, as the reference builders do
  const uint64_t m = el.num_edges();
  std::vector<uint32_t> src(m), dst(m);
  for (uint64_t i = 0; i < m; ++i) {
    src[i] = el.edges[i].src;
    dst[i] = el.edges[i].dst;
  }
  const bool weighted = el.weighted();
  DeviceContext& dc = device_context(device);
  std::lock_guard<std::mutex> lk(dc.mu);
  dc.held = GraphKey{};  // the context's graph is replaced
  int rc = sr_build_graph(dc.ctx, el.num_vertices, m, src.data(), dst.data(),
                          weighted ? el.weights.data() : nullptr, page_vertex_capacity,
                          SR_BUILD_CSR_EDGES);
  if (rc != SR_OK) rethrow(rc, sr_last_error(dc.ctx));
  std::pair<CsrGraph, PageSet> out;
  CsrGraph& csr = out.first;
  PageSet& ps = out.second;
  const uint32_t n = el.num_vertices;
  csr.num_vertices = n;
  csr.out_offsets.resize(size_t(n) + 1);
  csr.out_neighbors.resize(m);
  if (weighted) csr.out_weights.resize(m);
  std::vector<uint64_t> in_off(size_t(n) + 1);
  std::vector<uint32_t> in_src(m), in_w(weighted ? m : 0);
  rc = sr_export_graph(dc.ctx, csr.out_offsets.data(), csr.out_neighbors.data(),
                       weighted ? csr.out_weights.data() : nullptr, in_off.data(), in_src.data(),
                       weighted ? in_w.data() : nullptr);
  if (rc != SR_OK) rethrow(rc, sr_last_error(dc.ctx));
  ps.num_vertices = n;
  ps.page_vertex_capacity = page_vertex_capacity;
  ps.weighted = weighted;
  for (uint64_t vb = 0; vb < n; vb += page_vertex_capacity) {
    const uint64_t ve = std::min<uint64_t>(vb + page_vertex_capacity, n);
    CscPage pg;
    pg.vertex_begin = VertexId(vb);
    pg.vertex_end = VertexId(ve);
    pg.in_offsets.resize(ve - vb + 1);
    for (uint64_t v = vb; v <= ve; ++v) pg.in_offsets[v - vb] = uint32_t(in_off[v] - in_off[vb]);
    pg.in_sources.assign(in_src.begin() + in_off[vb], in_src.begin() + in_off[ve]);
    if (weighted) pg.in_weights.assign(in_w.begin() + in_off[vb], in_w.begin() + in_off[ve]);
    ps.pages.push_back(std::move(pg));
  }
  return out;
}

inline CsrGraph build_csr(const EdgeList& el, int device = 0) {
  return build_graph(el, std::max<VertexId>(el.num_vertices, 1), device).first;
}

inline PageSet build_csc_pages(const EdgeList& el, VertexId page_vertex_capacity, int device = 0) {
  return build_graph(el, page_vertex_capacity, device).second;
}

}  // namespace pagestream::seraph
