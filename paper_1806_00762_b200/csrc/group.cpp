// Single-process multi-GPU contexts (sr_group_*): the reference's
// pagestream::run is one call in one process (engine.hpp:125-126; run_matrix
// runs cells with std::async, bench.cpp:254-259), so the drop-in reaches N
// GPUs from one process.  A group is a world of N contexts, one per listed
// device, each driven by its own host thread:
//   * distinct GPUs: NCCL communicators (ncclCommInitRank from one thread per
//     rank) and, with SR_EXCHANGE_PEER, the fused peer-store exchange over
//     CUDA IPC mappings of the replicas (engine.cpp setup_peers);
//   * a device listed twice (one-GPU boxes, tests): the in-process loopback
//     transport (loopback.cpp) -- same round protocol, host all-reduces.
// Each rank uploads its own destination shard of the pages and only its own
// CSR rows (Engine::load_csr_shard): per-rank host->device bytes and HBM are
// O(|E|/N).  Values and ranks come from rank 0's replica (identical on every
// rank after the last exchange); per-pass counters are already global.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "nccl_dyn.h"
#include "seraph.h"

struct sr_group {
  std::vector<seraph::Engine*> ranks;
  std::vector<int> devices;
  std::string err;
  bool loaded = false;
};

namespace {

thread_local std::string g_group_err;

struct RankErr {
  int code = SR_OK;
  std::string msg;
};

template <typename F>
RankErr capture(F&& f) {
  RankErr e;
  try {
    f();
  } catch (const seraph::EngineError& x) {
    e.code = x.code;
    e.msg = x.what();
  } catch (const std::bad_alloc&) {
    e.code = SR_E_OOM;
    e.msg = "host allocation failed";
  } catch (const std::exception& x) {
    e.code = SR_E_INTERNAL;
    e.msg = x.what();
  }
  return e;
}

// Run f(rank) on one thread per rank; the first failing rank's error wins.
template <typename F>
int per_rank(sr_group* g, F&& f) {
  const int n = int(g->ranks.size());
  std::vector<RankErr> errs(n);
  std::vector<std::thread> th;
  for (int r = 1; r < n; ++r)
    th.emplace_back([&, r] { errs[r] = capture([&] { f(r); }); });
  errs[0] = capture([&] { f(0); });
  for (auto& t : th) t.join();
  for (int r = 0; r < n; ++r)
    if (errs[r].code != SR_OK) {
      g->err = "rank " + std::to_string(r) + ": " + errs[r].msg;
      return errs[r].code;
    }
  return SR_OK;
}

void merge_metrics(const std::vector<sr_metrics>& ms, sr_metrics* out) {
  if (!out) return;
  sr_metrics m = ms[0];  // global per-pass counters (all-reduced every round)
  for (size_t r = 1; r < ms.size(); ++r) {
    m.pages_transferred += ms[r].pages_transferred;
    m.bytes_transferred += ms[r].bytes_transferred;
    m.h2d_bytes += ms[r].h2d_bytes;
    m.kernel_launches += ms[r].kernel_launches;
    m.kernel_runs += ms[r].kernel_runs;
    m.relax_seconds = std::max(m.relax_seconds, ms[r].relax_seconds);
    m.relax_launches += ms[r].relax_launches;
    m.gathers += ms[r].gathers;
    m.device_seconds = std::max(m.device_seconds, ms[r].device_seconds);
    m.wall_seconds = std::max(m.wall_seconds, ms[r].wall_seconds);
    m.upload_seconds = std::max(m.upload_seconds, ms[r].upload_seconds);
  }
  *out = m;
}

}  // namespace

extern "C" {

int sr_group_open(const int* devices, int n, uint64_t budget, int flags, sr_group** out) {
  if (!out || !devices || n < 1) return SR_E_CONFIG;
  *out = nullptr;
  sr_group* g = new (std::nothrow) sr_group();
  if (!g) return SR_E_OOM;
  g->devices.assign(devices, devices + n);
  RankErr e = capture([&] {
    for (int r = 0; r < n; ++r) g->ranks.push_back(new seraph::Engine(devices[r], budget));
    if (n == 1) return;
    std::vector<int> sorted(g->devices);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    const bool peer = (flags & SR_EXCHANGE_PEER) != 0;
    if (distinct) {  // NCCL world inside this process
      const seraph::NcclApi& nc = seraph::nccl();
      ncclUniqueId uid;
      const ncclResult_t rc = nc.GetUniqueId(&uid);
      if (rc != ncclSuccess)
        throw seraph::EngineError(SR_E_NCCL, std::string("nccl id: ") + nc.GetErrorString(rc));
      uint8_t id[128];
      static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
      std::memcpy(id, &uid, 128);
      const int rcg = per_rank(g, [&](int r) {
        g->ranks[r]->attach_world(r, n, id);
        g->ranks[r]->set_exchange(peer);
      });
      if (rcg != SR_OK) throw seraph::EngineError(rcg, g->err);
    } else {  // a device listed more than once: in-process loopback transport
      static std::atomic<unsigned long long> seq{0};  // never reuse a (possibly abandoned) key
      char key[64];
      std::snprintf(key, sizeof(key), "sr_group:%llu", seq.fetch_add(1) + 1);
      for (int r = 0; r < n; ++r) g->ranks[r]->attach_loopback(r, n, key, peer);
    }
  });
  if (e.code != SR_OK) {
    g_group_err = e.msg;
    for (auto* r : g->ranks) delete r;
    delete g;
    return e.code;
  }
  *out = g;
  return SR_OK;
}

void sr_group_close(sr_group* g) {
  if (!g) return;
  for (auto* r : g->ranks) delete r;
  delete g;
}

const char* sr_group_last_error(const sr_group* g) { return g ? g->err.c_str() : g_group_err.c_str(); }

int sr_group_size(const sr_group* g) { return g ? int(g->ranks.size()) : 0; }

int sr_group_load_graph(sr_group* g, uint32_t n, uint64_t m, const uint64_t* off,
                        const uint32_t* nbr, const uint32_t* w, uint32_t cap, int weighted_pages,
                        const sr_page_view* pages, uint32_t np, int algo_hint) {
  if (!g) return SR_E_CONFIG;
  g->loaded = false;
  const bool world1 = g->ranks.size() == 1;
  const int rc = per_rank(g, [&](int r) {
    seraph::Engine* e = g->ranks[r];
    if (world1) {  // the one-context path of sr_run_graph (lean CSR, derived adjacency)
      e->drop_csr();
      uint64_t page_bytes = 0;
      for (uint32_t i = 0; i < np; ++i)
        page_bytes += (uint64_t(pages[i].vertex_end - pages[i].vertex_begin) + 1 +
                       pages[i].edge_count * (weighted_pages ? 2 : 1)) * 4;
      const bool lean = algo_hint == SR_ALGO_PAGERANK ||
                        e->fits_budget(page_bytes + m * 4 * (w ? 2 : 1));
      e->load_csr(n, m, off, lean ? nullptr : nbr, lean ? nullptr : w, false);
      e->set_load_algo(algo_hint);
      e->load_pages(n, cap, weighted_pages != 0, pages, np);
      return;
    }
    e->drop_csr();
    e->set_load_algo(algo_hint);
    e->load_pages(n, cap, weighted_pages != 0, pages, np);  // this rank's shard only
    const bool pagerank = algo_hint == SR_ALGO_PAGERANK;    // out-degrees only
    e->load_csr_shard(n, m, off, pagerank ? nullptr : nbr, pagerank ? nullptr : w);
  });
  if (rc == SR_OK) g->loaded = true;
  return rc;
}

int sr_group_run(sr_group* g, const sr_run_config* cfg, uint32_t* values_out, float* ranks_out,
                 sr_metrics* metrics_out, sr_pass_stats* per_pass, uint32_t cap,
                 uint32_t* n_pass) {
  if (!g || !cfg) return SR_E_CONFIG;
  if (!g->loaded) {
    g->err = "no graph loaded (sr_group_load_graph)";
    return SR_E_CONFIG;
  }
  const int n = int(g->ranks.size());
  std::vector<sr_metrics> ms(n);
  std::vector<std::vector<sr_pass_stats>> passes(n);
  const int rc = per_rank(g, [&](int r) {
    ms[r] = sr_metrics{};
    g->ranks[r]->run(*cfg, r == 0 ? values_out : nullptr, r == 0 ? ranks_out : nullptr, ms[r],
                     passes[r]);
  });
  if (rc != SR_OK) return rc;
  merge_metrics(ms, metrics_out);
  if (n_pass) *n_pass = uint32_t(passes[0].size());
  if (per_pass)
    for (uint32_t i = 0; i < cap && i < passes[0].size(); ++i) per_pass[i] = passes[0][i];
  return SR_OK;
}

int sr_group_run_graph(sr_group* g, uint32_t n, uint64_t m, const uint64_t* off,
                       const uint32_t* nbr, const uint32_t* w, uint32_t cap, int weighted_pages,
                       const sr_page_view* pages, uint32_t np, const sr_run_config* cfg,
                       uint32_t* values_out, float* ranks_out, sr_metrics* metrics_out,
                       sr_pass_stats* per_pass, uint32_t pcap, uint32_t* n_pass) {
  if (!g || !cfg) return SR_E_CONFIG;
  const auto t0 = std::chrono::steady_clock::now();
  for (auto* e : g->ranks) {
    e->last_upload_seconds = 0;
    e->last_upload_bytes = 0;
  }
  int rc = sr_group_load_graph(g, n, m, off, nbr, w, cap, weighted_pages, pages, np, cfg->algo);
  if (rc != SR_OK) return rc;
  const double up = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  sr_metrics mm{};
  rc = sr_group_run(g, cfg, values_out, ranks_out, &mm, per_pass, pcap, n_pass);
  if (rc != SR_OK) return rc;
  mm.upload_seconds = up;
  for (auto* e : g->ranks) mm.h2d_bytes += e->last_upload_bytes;
  if (metrics_out) *metrics_out = mm;
  return SR_OK;
}

int sr_group_graph_info(const sr_group* g, int rank, sr_graph_info* out) {
  if (!g || !out || rank < 0 || rank >= int(g->ranks.size())) return SR_E_CONFIG;
  g->ranks[rank]->graph_info(*out);
  return SR_OK;
}

}  // extern "C"
