/*
 * seraph.h — C-ABI of the B200-native subgraph-iteration engine.
 *
 * This is the drop-in boundary for the reference's hot path
 *   pagestream::run(const CsrGraph&, const PageSet&, const VertexProgram&,
 *                   const EngineConfig&) -> RunResult
 * (/root/reference/proj/include/pagestream/engine.hpp:125-126, implemented at
 *  proj/src/engine.cpp:421-433).  Everything below that call in the reference
 * (Runner::run engine.cpp:371-416, schedule_dense_pass scheduler.cpp:420-435,
 * dense_pull_page engine.cpp:132-177, sparse_push_pass engine.cpp:63-93,
 * recovery_scan engine.cpp:179-205, the predictor bookkeeping in
 * predictor.cpp) executes inside libseraph.so on the GPU.
 *
 * Plain C types only: pointers, sizes, PODs.  No torch, no STL.
 * Every entry point returns 0 on success or a negative SR_E_* code that maps
 * 1:1 onto the reference's exception taxonomy (errors.hpp:8-28); the message
 * is available from sr_last_error().
 */
#ifndef SERAPH_H_
#define SERAPH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SERAPH_ABI_VERSION 1

/* ---- error codes (reference errors.hpp:8-28) --------------------------- */
#define SR_OK 0
#define SR_E_CONFIG (-1)   /* pagestream::ConfigError   */
#define SR_E_INPUT (-2)    /* pagestream::InputError    */
#define SR_E_CONTRACT (-3) /* pagestream::ContractError */
#define SR_E_DATA (-4)     /* pagestream::DataError     */
#define SR_E_FORMAT (-5)   /* pagestream::FormatError   */
#define SR_E_PARSE (-6)    /* pagestream::ParseError    */
#define SR_E_CUDA (-7)     /* pagestream::Error (device failure)     */
#define SR_E_NCCL (-8)     /* pagestream::Error (collective failure) */
#define SR_E_OOM (-9)      /* pagestream::Error (device memory)      */
#define SR_E_INTERNAL (-10)

/* ---- enums (reference types.hpp:20, predictor.hpp:12, scheduler.hpp:31-37,
 *      engine.hpp:15-17, scheduler.hpp:55) ------------------------------- */
enum { SR_ALGO_BFS = 0, SR_ALGO_CC = 1, SR_ALGO_SSSP = 2, SR_ALGO_PAGERANK = 3 };
enum { SR_PRED_OFF = 0, SR_PRED_STRONG = 1, SR_PRED_WEAK = 2 };
enum {
  SR_SCHED_BASELINE = 0,
  SR_SCHED_REENTRY = 1,
  SR_SCHED_DOUBLE_BUFFER = 2,
  SR_SCHED_PIPELINED = 3,
  SR_SCHED_PIPELINED_FINE = 4
};
enum { SR_CLOCK_VIRTUAL = 0, SR_CLOCK_WALL = 1 };
enum { SR_EXEC_DENSITY_SWITCHED = 0, SR_EXEC_FORCE_SPARSE = 1, SR_EXEC_FORCE_DENSE = 2 };
enum { SR_PASS_SPARSE_PUSH = 0, SR_PASS_DENSE_PULL = 1, SR_PASS_RECOVERY = 2 };
enum {
  SR_TRACE_XFER_START = 0,
  SR_TRACE_XFER_END = 1,
  SR_TRACE_KERNEL_START = 2,
  SR_TRACE_KERNEL_END = 3,
  SR_TRACE_REENTRY = 4
};

#define SR_UNREACHED 0xffffffffu /* types.hpp:14 kUnreached */

typedef struct sr_ctx sr_ctx;

/* One CSC page (graph.hpp:46-55): contiguous destination range
 * [vertex_begin, vertex_end) with page-local u32 in_offsets (range+1
 * entries), in_sources and optional in_weights (edge_count entries). */
typedef struct {
  uint32_t vertex_begin;
  uint32_t vertex_end;
  const uint32_t* in_offsets;
  const uint32_t* in_sources;
  const uint32_t* in_weights; /* NULL when unweighted */
  uint64_t edge_count;
} sr_page_view;

/* EngineConfig (engine.hpp:39-52) + VertexProgram (programs.hpp:14-50)
 * + TransferModel (scheduler.hpp:19-29) + ScheduleMode (scheduler.hpp:38-47),
 * flattened.  Initialise with sr_default_config(). */
typedef struct {
  int32_t algo;     /* SR_ALGO_* */
  uint32_t source;  /* BFS/SSSP source; ignored for CC/PageRank */
  int32_t predictor;
  int32_t schedule;
  int32_t max_reentry_times;  /* MRT, default 2 */
  int32_t buffer_repetitions; /* double-buffer reps, default 3 */
  uint32_t window_capacity;   /* B, default 8 */
  double density_threshold_fraction; /* default 0.05 */
  double bytes_per_time_unit;        /* TransferModel, default 11.0 */
  double edges_per_time_unit_per_worker; /* default 1.75 */
  int32_t worker_count;              /* default 4 */
  int32_t clock;                     /* SR_CLOCK_* */
  int32_t execution;                 /* SR_EXEC_* */
  int32_t record_trace;
  uint64_t seed;
  /* PageRank (new algorithm, no reference counterpart) */
  uint32_t pr_iterations; /* default 20 */
  double pr_damping;      /* default 0.85 */
  /* Time every relax-kernel launch (K1 pull / K8 PageRank) with CUDA events
   * on the compute stream; totals land in sr_metrics.relax_seconds. */
  int32_t profile_kernels;
  int32_t pad_;
} sr_run_config;

/* PassStats (metrics.hpp:17-29). */
typedef struct {
  uint32_t pass_index;
  int32_t kind; /* SR_PASS_* */
  uint64_t attempts;
  uint64_t valid_updates;
  uint64_t skipped;
  uint64_t edges_read;
  uint64_t changed_vertices;
  uint64_t status_counts[6];
  int32_t has_status_counts;
  int32_t pad_;
} sr_pass_stats;

/* MetricsReport (metrics.hpp:31-57) plus device-side timing. */
typedef struct {
  uint64_t passes;
  uint64_t sparse_passes;
  uint64_t dense_passes;
  uint64_t recovery_passes;
  uint64_t pages_transferred;
  uint64_t bytes_transferred;
  uint64_t update_attempts;
  uint64_t valid_updates;
  uint64_t skipped_vertices;
  uint64_t edges_read;
  double virtual_makespan;
  double wall_seconds;
  int32_t has_prediction_accuracy;
  int32_t pad_;
  double prediction_accuracy;
  /* B200 extras */
  double device_seconds;   /* CUDA-event time of the run on the compute stream */
  double upload_seconds;   /* host->device graph upload inside sr_run_graph */
  uint64_t kernel_launches;
  uint64_t h2d_bytes;      /* bytes actually moved host->device during the run */
  uint64_t d2h_bytes;
  uint64_t kernel_runs;    /* page-runs (DensePassOutcome::kernel_runs) */
  double relax_seconds;    /* sum of timed K1/K8 launch durations (profile_kernels) */
  uint64_t relax_launches;
  uint64_t gathers;        /* source values K1/K8 actually loaded (skips excluded) */
  /* edges whose source (+ weight) K1 streamed in: edges of destinations that
   * cannot improve are counted in edges_read (the reference's definition)
   * but never loaded */
  uint64_t edges_streamed;
  /* destinations K1's phase A scanned (value + in_offsets read), every
   * launch: a source-blocked pass scans each destination once per block */
  uint64_t dest_visits;
} sr_metrics;

typedef struct {
  double time;
  int32_t kind; /* SR_TRACE_* */
  uint32_t page_id;
  uint32_t pass_index;
  uint32_t pad_;
} sr_trace_event;

/* Device properties the bench reports. */
typedef struct {
  int32_t device;
  int32_t sm_count;
  int32_t l2_bytes;
  int32_t cc_major;
  int32_t cc_minor;
  int32_t pad_;
  uint64_t total_mem;
  uint64_t free_mem;
  char name[64];
} sr_device_info;

/* ---- library --------------------------------------------------------- */
int sr_abi_version(void);
void sr_default_config(sr_run_config* cfg);
/* Thread-local message of the last failing call made without a context. */
const char* sr_global_error(void);

/* ---- context lifecycle ------------------------------------------------ */
/* hbm_budget_bytes: device bytes the engine may use for graph pages
 * (0 = no forced budget: use what the device has).  When the page set does
 * not fit the budget, pages stream from pinned host memory through a ring of
 * window_capacity device slots (the out-of-core path). */
int sr_open(int device, uint64_t hbm_budget_bytes, sr_ctx** out);
void sr_close(sr_ctx* ctx);
const char* sr_last_error(const sr_ctx* ctx);
int sr_device_query(int device, sr_device_info* out);

/* ---- graph upload (replaces the host-side residency of CsrGraph/PageSet,
 *      graph.hpp:30-65).  Host arrays are borrowed for the call only. -------- */
int sr_load_csr(sr_ctx* ctx, uint32_t num_vertices, uint64_t num_edges,
                const uint64_t* out_offsets, const uint32_t* out_neighbors,
                const uint32_t* out_weights /* nullable */);
int sr_load_pages(sr_ctx* ctx, uint32_t num_vertices, uint32_t page_vertex_capacity,
                  int weighted, const sr_page_view* pages, uint32_t n_pages);
/* Bytes of CSC pages under the reference layout rule (page_bytes,
 * graph.cpp:96-100) summed over the loaded page set. */
uint64_t sr_loaded_page_bytes(const sr_ctx* ctx);

/* ---- the hot path ------------------------------------------------------ */
/* Run one algorithm on the loaded graph.  values_out: |V| u32 (BFS levels,
 * SSSP distances, CC labels; may be NULL); ranks_out: |V| f32 for PageRank
 * (may be NULL).  per_pass may be NULL; *n_pass_out receives the pass count
 * even when it exceeds per_pass_cap. */
int sr_run(sr_ctx* ctx, const sr_run_config* cfg, uint32_t* values_out, float* ranks_out,
           sr_metrics* metrics_out, sr_pass_stats* per_pass, uint32_t per_pass_cap,
           uint32_t* n_pass_out);

/* One-shot equivalent of pagestream::run(csr, pages, program, config):
 * upload CSR + pages from host memory, run, copy values back. */
int sr_run_graph(sr_ctx* ctx, uint32_t num_vertices, uint64_t num_edges,
                 const uint64_t* out_offsets, const uint32_t* out_neighbors,
                 const uint32_t* out_weights, uint32_t page_vertex_capacity, int weighted,
                 const sr_page_view* pages, uint32_t n_pages, const sr_run_config* cfg,
                 uint32_t* values_out, float* ranks_out, sr_metrics* metrics_out,
                 sr_pass_stats* per_pass, uint32_t per_pass_cap, uint32_t* n_pass_out);

/* Trace of the last sr_run (TraceEvent, scheduler.hpp:57-68). */
int sr_get_trace(const sr_ctx* ctx, sr_trace_event* out, uint64_t cap, uint64_t* n_out);

/* Device fixpoint-law verifier (test_engine.cpp:152-168 law; reference.cpp
 * verify :101-116): counts edges (u,v,w) of the loaded CSR with
 * combine(values[u],w) < values[v].  values_host may be NULL to check the
 * values left by the last run. */
int sr_verify_fixpoint(sr_ctx* ctx, int algo, const uint32_t* values_host,
                       uint64_t* violations_out);

/* Kernel-only timing hook for the bench: runs `reps` full dense pull sweeps
 * (K1, every page, predictor off) over the resident page set on the current
 * values and returns the mean per-sweep device milliseconds and edges. */
int sr_bench_pull_sweep(sr_ctx* ctx, int algo, uint32_t reps, double* ms_per_sweep,
                        uint64_t* edges_per_sweep);

/* ---- device-side graph build ----------------------
 * The reference's build_csr + build_csc_pages (graph.cpp:30-94) on the GPU:
 * stable radix sorts, so the CSR/CSC arrays are bit-identical to the host
 * builders (within a source/destination the input edge order is kept).  The
 * result is loaded as if by sr_load_csr + sr_load_pages with pages of
 * page_vertex_capacity vertices.  With SR_BUILD_CSR_EDGES the push adjacency
 * is built in the reference's order (else only out_offsets; the adjacency is
 * then derived from the resident pages). */
#define SR_BUILD_CSR_EDGES 1

/* Synthetic graph recipe: generate_rmat (ingest.cpp:112-141 quadrant law,
 * counter-based stream of sr_rmat_generate), optional assign_weights range
 * (weight_hi == 0: unweighted), optional symmetrize (graph.cpp:102-118). */
typedef struct {
  int32_t scale;
  uint32_t edge_factor;
  double a, b, c, d;
  uint64_t seed;
  uint32_t weight_lo, weight_hi;
  uint64_t weight_seed;
  int32_t symmetrize;
  uint32_t page_vertex_capacity;
} sr_graph_spec;

typedef struct {
  uint32_t num_vertices;
  uint32_t num_pages;
  uint64_t num_edges;
  uint32_t page_vertex_capacity;
  int32_t weighted;      /* pages carry in_weights */
  int32_t has_csr_edges; /* push adjacency on the device */
  int32_t csr_weighted;
  int32_t csr_derived;   /* adjacency derived from the pages (order within a source arbitrary) */
  /* the push adjacency lives in pinned host memory, read zero-copy by the
   * sparse passes: pages + adjacency exceed the context's hbm budget */
  int32_t adjacency_on_host;
} sr_graph_info;

/* Edge list in host or device memory (src/dst/w: num_edges entries, w NULL
 * when unweighted). */
int sr_build_graph(sr_ctx* ctx, uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                   const uint32_t* dst, const uint32_t* w, uint32_t page_vertex_capacity,
                   int flags);
/* Generate + build entirely on the device (no host edge list). */
int sr_generate_graph(sr_ctx* ctx, const sr_graph_spec* spec, int flags);
/* load_binary (ingest.cpp:176-218): an SRPH edge-list file (header "SRPH",
 * version 1, flags bit0 = weighted, u64 |V|, u64 |E|; records u32 src, dst
 * [, w]) streamed onto the device and built as sr_build_graph does.  Errors:
 * SR_E_FORMAT for the header/size checks and invalid edges, as the reference. */
int sr_load_srph(sr_ctx* ctx, const char* path, uint32_t page_vertex_capacity, int flags);
int sr_graph_info_get(const sr_ctx* ctx, sr_graph_info* out);
/* Copy the loaded graph back in the reference layouts (any pointer may be
 * NULL): CSR out_offsets (|V|+1) / out_neighbors / out_weights (|E|), global
 * CSC in_offsets (|V|+1, u64) / in_sources / in_weights (|E|). */
int sr_export_graph(sr_ctx* ctx, uint64_t* out_offsets, uint32_t* out_neighbors,
                    uint32_t* out_weights, uint64_t* in_offsets, uint32_t* in_sources,
                    uint32_t* in_weights);
/* The device generator alone, copied to host arrays (parity with
 * sr_rmat_generate / sr_weights_generate). w may be NULL. */
int sr_rmat_generate_device(int device, int scale, uint64_t edge_factor, double a, double b,
                            double c, double d, uint64_t seed, uint32_t* src, uint32_t* dst,
                            uint64_t weight_seed, uint32_t weight_lo, uint32_t weight_hi,
                            uint32_t* w);

/* ---- host plumbing ------------------------------------------------------ */
/* Page-locked host buffers (cudaHostAlloc): inputs in pinned memory upload at
 * full link speed and are what the out-of-core path streams from. */
int sr_host_alloc(uint64_t bytes, void** out);
void sr_host_free(void* p);
/* cudaDeviceSynchronize on `device` (bench bracketing without torch). */
int sr_device_sync(int device);
/* Host-link roofline denominator: pinned host -> device cudaMemcpyAsync of
 * `bytes`, best of `reps`, timed with CUDA events (GB/s = 1e9 B/s). */
int sr_bench_h2d(int device, uint64_t bytes, uint32_t reps, double* gbps);
/* Evict the L2 between timed steps: write a device buffer of `bytes`
 * (> L2 size) on the context's compute stream. */
int sr_flush_l2(sr_ctx* ctx, uint64_t bytes);

/* ---- multi-GPU (one process per GPU) ----------------------------------- */
/* 128-byte NCCL unique id, created on rank 0 and broadcast by the host. */
int sr_nccl_unique_id(uint8_t out[128]);
/* Make ctx a shard of a world: destination ranges of the loaded pages are
 * cut into `world` edge-balanced shards (sr_shard_plan) and this rank relaxes
 * only its own; vertex arrays are merged once per global round with an NCCL
 * min (sum for PageRank) all-reduce over NVLink. */
int sr_attach_world(sr_ctx* ctx, int rank, int world, const uint8_t unique_id[128]);

/* Test/dev transport: make ctx rank `rank` of `world` contexts of THIS process
 * (any devices, including one shared GPU) whose exchange all-reduces go
 * through host memory instead of NCCL; `group` names the world.  Each rank's
 * sr_run must be driven from its own thread.  Exercises the sharded round
 * protocol of sr_attach_world where NCCL cannot (two ranks on one GPU).
 * flags & SR_EXCHANGE_PEER: the relax kernels store every improvement
 * straight into the other ranks' value replicas (peer memory) and a round
 * ends with a barrier instead of the |V|-sized MIN all-reduce. */
#define SR_EXCHANGE_PEER 1
int sr_attach_loopback(sr_ctx* ctx, int rank, int world, const char* group, int flags);
/* Exchange of an attached world (either transport): 0 = |V|-sized MIN
 * all-reduce per round (default), SR_EXCHANGE_PEER = peer stores + barrier
 * (NCCL worlds map the peers' replicas with CUDA IPC; all GPUs of one node
 * must have peer access over NVLink). */
int sr_set_exchange(sr_ctx* ctx, int flags);

/* ---- multi-GPU from ONE process (the reference's run() is one call in one
 *      process: engine.hpp:125-126, bench.cpp:254-259) ---------------------
 * A group is a world of n contexts, rank r on devices[r], each driven by its
 * own host thread inside the calls below.  Distinct devices: NCCL
 * communicators created in this process (+ the peer exchange when flags &
 * SR_EXCHANGE_PEER); a device listed more than once: the in-process loopback
 * transport (one-GPU boxes, tests).  Every rank uploads only its destination
 * shard of the pages and only its own CSR adjacency rows (per-rank bytes
 * O(|E|/n)); values/ranks come from rank 0's replica; per-pass counters are
 * global; transfer counters are summed and times are the max over ranks. */
typedef struct sr_group sr_group;
int sr_group_open(const int* devices, int n, uint64_t hbm_budget_bytes, int flags,
                  sr_group** out);
void sr_group_close(sr_group* g);
const char* sr_group_last_error(const sr_group* g);
int sr_group_size(const sr_group* g);
/* Upload (each rank its shard) and keep the graph resident for sr_group_run.
 * algo_hint: the algorithm the graph is loaded for (SR_ALGO_PAGERANK skips the
 * adjacency), or -1. */
int sr_group_load_graph(sr_group* g, uint32_t num_vertices, uint64_t num_edges,
                        const uint64_t* out_offsets, const uint32_t* out_neighbors,
                        const uint32_t* out_weights, uint32_t page_vertex_capacity, int weighted,
                        const sr_page_view* pages, uint32_t n_pages, int algo_hint);
int sr_group_run(sr_group* g, const sr_run_config* cfg, uint32_t* values_out, float* ranks_out,
                 sr_metrics* metrics_out, sr_pass_stats* per_pass, uint32_t per_pass_cap,
                 uint32_t* n_pass_out);
/* sr_run_graph over the group: load + run in one call. */
int sr_group_run_graph(sr_group* g, uint32_t num_vertices, uint64_t num_edges,
                       const uint64_t* out_offsets, const uint32_t* out_neighbors,
                       const uint32_t* out_weights, uint32_t page_vertex_capacity, int weighted,
                       const sr_page_view* pages, uint32_t n_pages, const sr_run_config* cfg,
                       uint32_t* values_out, float* ranks_out, sr_metrics* metrics_out,
                       sr_pass_stats* per_pass, uint32_t per_pass_cap, uint32_t* n_pass_out);
/* Graph placement of one rank (its shard). */
int sr_group_graph_info(const sr_group* g, int rank, sr_graph_info* out);

/* ---- host-side graph utilities (no GPU needed) ------------------------- */
/* Edge-balanced contiguous cut of the destination space into `parts`
 * ranges: cuts[0]=0 ... cuts[parts]=num_vertices, chosen so that every range
 * holds ~1/parts of the in-edges (offsets = global CSC row offsets). */
int sr_shard_plan(uint32_t num_vertices, const uint64_t* in_offsets_global, uint32_t parts,
                  uint32_t* cuts);
/* Counter-based (splitmix64) parallel RMAT generator: same quadrant law as
 * generate_rmat (ingest.cpp:112-141) but a different random stream, so it
 * scales to RMAT-29.  src/dst: num_vertices*edge_factor entries. */
int sr_rmat_generate(int scale, uint64_t edge_factor, double a, double b, double c, double d,
                     uint64_t seed, uint32_t* src, uint32_t* dst, int threads);
/* Uniform [lo,hi] weights, counter-based and parallel. */
int sr_weights_generate(uint64_t num_edges, uint64_t seed, uint32_t lo, uint32_t hi,
                        uint32_t* weights, int threads);
/* Parallel counting-sort builders with the reference's layouts:
 * build_csr (graph.cpp:30-48) and build_csc_pages (graph.cpp:50-94).
 * sr_build_csc writes global in_offsets (u64, |V|+1) and the transposed
 * sources/weights; sr_page_offsets derives the page-local u32 offsets
 * (|V| + n_pages entries, page p at p_begin + p). */
int sr_build_csr(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                 const uint32_t* dst, const uint32_t* w, uint64_t* out_offsets,
                 uint32_t* out_neighbors, uint32_t* out_weights, int threads);
int sr_build_csc(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                 const uint32_t* dst, const uint32_t* w, uint64_t* in_offsets,
                 uint32_t* in_sources, uint32_t* in_weights, int threads);
int sr_page_offsets(uint32_t num_vertices, uint32_t page_vertex_capacity,
                    const uint64_t* in_offsets_global, uint32_t* local_offsets);
/* Out-degree prefix (CSR out_offsets) without the adjacency: enough for
 * sr_load_csr(..., NULL, NULL) when the pages are resident. */
int sr_out_offsets(uint32_t num_vertices, uint64_t num_edges, const uint32_t* src,
                   uint64_t* out_offsets, int threads);
/* symmetrize (graph.cpp:102-118), parallel: 2*num_edges outputs. */
int sr_symmetrize(uint64_t num_edges, const uint32_t* src, const uint32_t* dst,
                  const uint32_t* w, uint32_t* out_src, uint32_t* out_dst, uint32_t* out_w,
                  int threads);

#ifdef __cplusplus
}
#endif

#endif /* SERAPH_H_ */
