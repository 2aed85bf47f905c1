// extern "C" boundary of libseraph (include/seraph.h).  Every entry point
// catches, records the message and returns the SR_E_* code that the C++
// drop-in rethrows as the matching pagestream exception (errors.hpp:8-28).
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "devgraph.h"
#include "engine.h"
#include "nccl_dyn.h"
#include "seraph.h"

struct sr_ctx {
  seraph::Engine* eng = nullptr;
  std::string err;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guard(sr_ctx* ctx, F&& f) {
  try {
    f();
    return SR_OK;
  } catch (const seraph::EngineError& e) {
    (ctx ? ctx->err : g_err) = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    (ctx ? ctx->err : g_err) = "host allocation failed";
    return SR_E_OOM;
  } catch (const std::exception& e) {
    (ctx ? ctx->err : g_err) = e.what();
    return SR_E_INTERNAL;
  }
}

void copy_passes(const std::vector<sr_pass_stats>& passes, sr_pass_stats* out, uint32_t cap,
                 uint32_t* n_out) {
  if (n_out) *n_out = uint32_t(passes.size());
  if (out)
    for (uint32_t i = 0; i < cap && i < passes.size(); ++i) out[i] = passes[i];
}

}  // namespace

extern "C" {

int sr_abi_version(void) { return SERAPH_ABI_VERSION; }

const char* sr_global_error(void) { return g_err.c_str(); }

void sr_default_config(sr_run_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->algo = SR_ALGO_BFS;
  c->predictor = SR_PRED_OFF;
  c->schedule = SR_SCHED_BASELINE;
  c->max_reentry_times = 2;
  c->buffer_repetitions = 3;
  c->window_capacity = 8;
  c->density_threshold_fraction = 0.05;
  c->bytes_per_time_unit = 11.0;
  c->edges_per_time_unit_per_worker = 1.75;
  c->worker_count = 4;
  c->clock = SR_CLOCK_VIRTUAL;
  c->execution = SR_EXEC_DENSITY_SWITCHED;
  c->pr_iterations = 20;
  c->pr_damping = 0.85;
}

int sr_open(int device, uint64_t budget, sr_ctx** out) {
  if (!out) return SR_E_CONFIG;
  *out = nullptr;
  sr_ctx* ctx = new (std::nothrow) sr_ctx();
  if (!ctx) return SR_E_OOM;
  const int rc = guard(nullptr, [&] { ctx->eng = new seraph::Engine(device, budget); });
  if (rc != SR_OK) {
    delete ctx;
    return rc;
  }
  *out = ctx;
  return SR_OK;
}

void sr_close(sr_ctx* ctx) {
  if (!ctx) return;
  delete ctx->eng;
  delete ctx;
}

const char* sr_last_error(const sr_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int sr_device_query(int device, sr_device_info* out) {
  return guard(nullptr, [&] {
    if (!out) throw seraph::EngineError(SR_E_CONFIG, "null output");
    cudaDeviceProp prop{};
    SR_CUDA(cudaGetDeviceProperties(&prop, device));
    SR_CUDA(cudaSetDevice(device));
    size_t fr = 0, tot = 0;
    SR_CUDA(cudaMemGetInfo(&fr, &tot));
    std::memset(out, 0, sizeof(*out));
    out->device = device;
    out->sm_count = prop.multiProcessorCount;
    out->l2_bytes = prop.l2CacheSize;
    out->cc_major = prop.major;
    out->cc_minor = prop.minor;
    out->total_mem = tot;
    out->free_mem = fr;
    const size_t len = strnlen(prop.name, sizeof(out->name) - 1);  // name stays NUL-terminated
    std::memcpy(out->name, prop.name, len);
  });
}

int sr_load_csr(sr_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                const uint32_t* w) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->load_csr(n, m, off, nbr, w); });
}

int sr_load_pages(sr_ctx* ctx, uint32_t n, uint32_t cap, int weighted, const sr_page_view* pages,
                  uint32_t np) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->load_pages(n, cap, weighted != 0, pages, np); });
}

int sr_build_graph(sr_ctx* ctx, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const uint32_t* w, uint32_t cap, int flags) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->build_graph(n, m, src, dst, w, cap, flags & SR_BUILD_CSR_EDGES); });
}

int sr_generate_graph(sr_ctx* ctx, const sr_graph_spec* spec, int flags) {
  if (!ctx || !spec) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->generate_graph(*spec, flags & SR_BUILD_CSR_EDGES); });
}

int sr_load_srph(sr_ctx* ctx, const char* path, uint32_t cap, int flags) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->load_srph(path, cap, flags & SR_BUILD_CSR_EDGES); });
}

int sr_attach_loopback(sr_ctx* ctx, int rank, int world, const char* group, int flags) {
  if (!ctx || !group) return SR_E_CONFIG;
  return guard(ctx, [&] {
    ctx->eng->attach_loopback(rank, world, group, (flags & SR_EXCHANGE_PEER) != 0);
  });
}

int sr_set_exchange(sr_ctx* ctx, int flags) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->set_exchange((flags & SR_EXCHANGE_PEER) != 0); });
}

int sr_graph_info_get(const sr_ctx* ctx, sr_graph_info* out) {
  if (!ctx || !out) return SR_E_CONFIG;
  ctx->eng->graph_info(*out);
  return SR_OK;
}

int sr_export_graph(sr_ctx* ctx, uint64_t* out_offsets, uint32_t* out_neighbors,
                    uint32_t* out_weights, uint64_t* in_offsets, uint32_t* in_sources,
                    uint32_t* in_weights) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] {
    ctx->eng->export_graph(out_offsets, out_neighbors, out_weights, in_offsets, in_sources,
                           in_weights);
  });
}

int sr_rmat_generate_device(int device, int scale, uint64_t edge_factor, double a, double b,
                            double c, double d, uint64_t seed, uint32_t* src, uint32_t* dst,
                            uint64_t weight_seed, uint32_t weight_lo, uint32_t weight_hi,
                            uint32_t* w) {
  (void)d;  // implied: a + b + c + d = 1 (the generator compares against a, a+b, a+b+c)
  if (scale < 1 || scale > 31 || edge_factor < 1 || !src || !dst) return SR_E_CONFIG;
  if (w && (weight_lo < 1 || weight_lo > weight_hi)) return SR_E_CONFIG;
  return guard(nullptr, [&] {
    SR_CUDA(cudaSetDevice(device));
    const uint64_t m = (uint64_t(1) << scale) * edge_factor;
    uint32_t *ds = nullptr, *dd = nullptr, *dw = nullptr;
    SR_CUDA(cudaMalloc(&ds, m * 4));
    SR_CUDA(cudaMalloc(&dd, m * 4));
    if (w) SR_CUDA(cudaMalloc(&dw, m * 4));
    seraph::dg_rmat(scale, m, a, b, c, seed, ds, dd, nullptr);
    if (w) seraph::dg_weights(m, weight_seed, weight_lo, weight_hi, dw, nullptr);
    cudaError_t e = cudaMemcpy(src, ds, m * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(dst, dd, m * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && w) e = cudaMemcpy(w, dw, m * 4, cudaMemcpyDeviceToHost);
    cudaFree(ds);
    cudaFree(dd);
    if (dw) cudaFree(dw);
    SR_CUDA(e);
  });
}

uint64_t sr_loaded_page_bytes(const sr_ctx* ctx) {
  return ctx && ctx->eng ? ctx->eng->page_bytes_total() : 0;
}

int sr_run(sr_ctx* ctx, const sr_run_config* cfg, uint32_t* values_out, float* ranks_out,
           sr_metrics* metrics_out, sr_pass_stats* per_pass, uint32_t cap, uint32_t* n_pass) {
  if (!ctx || !cfg) return SR_E_CONFIG;
  return guard(ctx, [&] {
    sr_metrics m{};
    std::vector<sr_pass_stats> passes;
    ctx->eng->run(*cfg, values_out, ranks_out, m, passes);
    if (metrics_out) *metrics_out = m;
    copy_passes(passes, per_pass, cap, n_pass);
  });
}

int sr_run_graph(sr_ctx* ctx, uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                 const uint32_t* w, uint32_t cap, int weighted_pages, const sr_page_view* pages,
                 uint32_t np,
                 const sr_run_config* cfg, uint32_t* values_out, float* ranks_out,
                 sr_metrics* metrics_out, sr_pass_stats* per_pass, uint32_t pcap,
                 uint32_t* n_pass) {
  if (!ctx || !cfg) return SR_E_CONFIG;
  return guard(ctx, [&] {
    const auto t0 = std::chrono::steady_clock::now();
    ctx->eng->last_upload_seconds = 0;
    ctx->eng->last_upload_bytes = 0;
    const bool weighted = weighted_pages != 0;
    // Resident page set on one device: upload only the CSR offsets and derive
    // the push adjacency on the device (half the bytes over the host link).
    uint64_t page_bytes = 0;
    for (uint32_t i = 0; i < np; ++i)
      page_bytes += (uint64_t(pages[i].vertex_end - pages[i].vertex_begin) + 1 +
                     pages[i].edge_count * (weighted ? 2 : 1)) * 4;
    // A forced budget covers pages + adjacency: derive on the device only when
    // both fit, else hand the adjacency over (load_pages keeps it in pinned
    // host memory when it does not fit).  PageRank needs only the offsets.
    const uint64_t adj_bytes = m * 4 * (w ? 2 : 1);
    const bool pagerank = cfg->algo == SR_ALGO_PAGERANK;
    if (ctx->eng->world() > 1) {  // sharded rank: its pages, then only its own CSR rows
      ctx->eng->drop_csr();
      ctx->eng->set_load_algo(cfg->algo);
      ctx->eng->load_pages(n, cap, weighted, pages, np);
      ctx->eng->load_csr_shard(n, m, off, pagerank ? nullptr : nbr, pagerank ? nullptr : w);
      const double up =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      sr_metrics mm{};
      std::vector<sr_pass_stats> passes;
      ctx->eng->run(*cfg, values_out, ranks_out, mm, passes);
      mm.upload_seconds = up;
      mm.h2d_bytes += ctx->eng->last_upload_bytes;
      if (metrics_out) *metrics_out = mm;
      copy_passes(passes, per_pass, pcap, n_pass);
      return;
    }
    const bool derive = pagerank ||
                        (ctx->eng->world() == 1 && ctx->eng->fits_budget(page_bytes + adj_bytes));
    // the offsets DMA stays queued ahead of the page DMAs on the copy stream
    // (load_pages synchronises it before the host buffers are released)
    ctx->eng->load_csr(n, m, off, derive ? nullptr : nbr, derive ? nullptr : w, /*sync=*/false);
    ctx->eng->set_load_algo(cfg->algo);
    ctx->eng->load_pages(n, cap, weighted, pages, np);
    const double up = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    sr_metrics mm{};
    std::vector<sr_pass_stats> passes;
    ctx->eng->run(*cfg, values_out, ranks_out, mm, passes);
    mm.upload_seconds = up;
    mm.h2d_bytes += ctx->eng->last_upload_bytes;
    if (metrics_out) *metrics_out = mm;
    copy_passes(passes, per_pass, pcap, n_pass);
  });
}

int sr_get_trace(const sr_ctx* ctx, sr_trace_event* out, uint64_t cap, uint64_t* n_out) {
  if (!ctx) return SR_E_CONFIG;
  const auto& t = ctx->eng->trace;
  if (n_out) *n_out = t.size();
  if (out)
    for (uint64_t i = 0; i < cap && i < t.size(); ++i) out[i] = t[i];
  return SR_OK;
}

int sr_verify_fixpoint(sr_ctx* ctx, int algo, const uint32_t* values_host, uint64_t* viol) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] {
    const uint64_t v = ctx->eng->verify_fixpoint(algo, values_host);
    if (viol) *viol = v;
  });
}

int sr_bench_pull_sweep(sr_ctx* ctx, int algo, uint32_t reps, double* ms, uint64_t* edges) {
  if (!ctx || !ms || !edges) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->bench_pull_sweep(algo, reps, ms, edges); });
}

int sr_nccl_unique_id(uint8_t out[128]) {
  return guard(nullptr, [&] {
    const seraph::NcclApi& nc = seraph::nccl();
    ncclUniqueId id;
    const ncclResult_t r = nc.GetUniqueId(&id);
    if (r != ncclSuccess)
      throw seraph::EngineError(SR_E_NCCL, std::string("ncclGetUniqueId: ") + nc.GetErrorString(r));
    static_assert(sizeof(id) == 128, "nccl unique id size");
    std::memcpy(out, &id, 128);
  });
}

int sr_host_alloc(uint64_t bytes, void** out) {
  return guard(nullptr, [&] {
    if (!out) throw seraph::EngineError(SR_E_CONFIG, "null output");
    *out = nullptr;
    if (bytes) SR_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  });
}

void sr_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int sr_device_sync(int device) {
  return guard(nullptr, [&] {
    SR_CUDA(cudaSetDevice(device));
    SR_CUDA(cudaDeviceSynchronize());
  });
}

int sr_bench_h2d(int device, uint64_t bytes, uint32_t reps, double* gbps) {
  return guard(nullptr, [&] {
    if (!gbps || !bytes) throw seraph::EngineError(SR_E_CONFIG, "bad arguments");
    SR_CUDA(cudaSetDevice(device));
    seraph::PinBuf<uint8_t> h;
    seraph::DBuf<uint8_t> d;
    h.reserve(bytes);
    d.reserve(bytes);
    std::memset(h.p, 1, bytes);
    cudaStream_t st;
    cudaEvent_t a, b;
    SR_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    SR_CUDA(cudaEventCreate(&a));
    SR_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (uint32_t r = 0; r < reps + 1; ++r) {
      SR_CUDA(cudaEventRecord(a, st));
      SR_CUDA(cudaMemcpyAsync(d.p, h.p, bytes, cudaMemcpyHostToDevice, st));
      SR_CUDA(cudaEventRecord(b, st));
      SR_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      SR_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (r > 0 && ms < best) best = ms;  // first copy warms the path
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(st);
    *gbps = double(bytes) / (double(best) * 1e-3) / 1e9;
  });
}

int sr_flush_l2(sr_ctx* ctx, uint64_t bytes) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->flush_l2(bytes); });
}

int sr_attach_world(sr_ctx* ctx, int rank, int world, const uint8_t id[128]) {
  if (!ctx) return SR_E_CONFIG;
  return guard(ctx, [&] { ctx->eng->attach_world(rank, world, id); });
}

}  // extern "C"
