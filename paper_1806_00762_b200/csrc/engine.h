// Host engine: owns the device state of one context and runs the
// density-switched push/pull loop of the reference's Runner
// (proj/src/engine.cpp:225-416) on the GPU.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <deque>
#include <string>
#include <vector>

#include "device_types.h"
#include "errors.h"
#include "seraph.h"
#include "stager.h"
#include "vsched.h"

namespace seraph {

uint32_t k1_grab(uint64_t tiles, int grid, const char* env, uint32_t cap = 8);

struct LoopbackGroup;

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void reserve(size_t count) {
    if (count <= n && p) return;
    release();
    if (count) {
      SR_CUDA(cudaMalloc(&p, count * sizeof(T)));
      n = count;
    }
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

template <typename T>
struct PinBuf {
  T* p = nullptr;
  size_t n = 0;
  PinBuf() = default;
  PinBuf(const PinBuf&) = delete;
  PinBuf& operator=(const PinBuf&) = delete;
  ~PinBuf() { release(); }
  void reserve(size_t count) {
    if (count <= n && p) return;
    release();
    if (count) {
      SR_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&p), count * sizeof(T), cudaHostAllocDefault));
      n = count;
    }
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

struct PageMeta {
  uint32_t vb = 0, ve = 0;
  uint64_t edges = 0;
  uint64_t bytes = 0;        // page_bytes (graph.cpp:96-100)
  uint32_t tile_begin = 0, tile_end = 0;
  bool on_device = false;    // permanently resident (arena)
  uint64_t off_base = 0, edge_base = 0;  // arena placement
  // host copy used for streaming (pinned)
  const uint32_t* h_offs = nullptr;
  const uint32_t* h_src = nullptr;
  const uint32_t* h_w = nullptr;
  int slot = -1;             // streaming slot holding the page
};

// One streamed page image placed in the byte ring (offsets | sources |
// weights, 32 B aligned): entries are allocated contiguously and evicted
// oldest first, so many small pages can be in flight at once.
struct StreamSlot {
  uint64_t start = 0, words = 0;  // position in the ring (words)
  int page = -1;
  long long last_use = -1;   // step index of the last launch that read it
  cudaEvent_t ready = nullptr;  // copy finished (copy stream)
  cudaEvent_t freed = nullptr;  // last reader finished (compute stream)
};

inline uint64_t pad8(uint64_t words) { return (words + 7) & ~uint64_t(7); }
// Words of a page's streaming image: offsets, sources and weights, each
// starting 32 B aligned (K1's vector runs), + 8 words of read slack.
inline uint64_t stream_image_words(const PageMeta& pm, bool weighted) {
  const uint64_t e = pad8(pm.edges);
  return pad8(uint64_t(pm.ve - pm.vb) + 1) + e * (weighted ? 2 : 1) + 8;
}

struct PassOut {
  RunStats totals;
  uint64_t kernel_runs = 0;
  uint64_t pages_transferred = 0;
  uint64_t bytes_transferred = 0;
};

class Engine {
 public:
  Engine(int device, uint64_t budget);
  ~Engine();

  void load_csr(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                const uint32_t* w, bool sync = true);
  void load_pages(uint32_t n, uint32_t cap, bool weighted, const sr_page_view* pages,
                  uint32_t np);
  // Sharded rank of a world (after load_pages, which cuts the owned
  // destination range): the full out_offsets (vertex state) and only the
  // adjacency rows of the owned vertices -- the only rows this rank's pushes
  // read (the push list is compacted over [own_lo, own_hi)).  O(|E|/N).
  void load_csr_shard(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                      const uint32_t* w);
  // Forget the CSR of a previous graph (before a load_pages of a new one).
  void drop_csr();
  uint64_t page_bytes_total() const { return page_bytes_total_; }
  // True when a page set of `bytes` would be held resident (no streaming).
  bool fits_budget(uint64_t bytes) const { return budget_ == 0 || bytes <= budget_; }
  // the push adjacency lives in pinned host memory (read zero-copy by the
  // sparse passes) because pages + adjacency exceed the HBM budget
  bool adjacency_on_host() const { return adj_host_; }
  int world() const { return world_; }
  void run(const sr_run_config& cfg, uint32_t* values_out, float* ranks_out, sr_metrics& m,
           std::vector<sr_pass_stats>& passes);
  uint64_t verify_fixpoint(int algo, const uint32_t* values_host);
  // device-side graph build (devgraph.cu): edge list (host or device
  // pointers) or the on-device RMAT generator -> stable CSR/CSC -> resident
  void build_graph(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                   const uint32_t* w, uint32_t cap, bool csr_edges);
  void generate_graph(const sr_graph_spec& spec, bool csr_edges);
  void load_srph(const char* path, uint32_t cap, bool csr_edges);
  void graph_info(sr_graph_info& gi) const;
  void export_graph(uint64_t* out_off, uint32_t* out_nbr, uint32_t* out_w, uint64_t* in_off,
                    uint32_t* in_src, uint32_t* in_w);
  void bench_pull_sweep(int algo, uint32_t reps, double* ms, uint64_t* edges);
  void attach_world(int rank, int world, const uint8_t id[128]);
  void attach_loopback(int rank, int world, const std::string& key, bool peer_exchange);
  void flush_l2(uint64_t bytes);
  DBuf<uint8_t> l2_flush_;
  unsigned flush_gen_ = 0;

  std::string err;
  std::vector<sr_trace_event> trace;
  double last_upload_seconds = 0;
  uint64_t last_upload_bytes = 0;

 private:
  // ---- configuration of the current run ----
  struct RunState;
  void validate(const sr_run_config& cfg) const;
  void alloc_run_state(const sr_run_config& cfg);
  void run_traversal(const sr_run_config& cfg, uint32_t* values_out, sr_metrics& m,
                     std::vector<sr_pass_stats>& passes);
  void run_pagerank(const sr_run_config& cfg, float* ranks_out, sr_metrics& m,
                    std::vector<sr_pass_stats>& passes);

  // dense-pass drivers
  PassOut dense_pass_wall(const sr_run_config& cfg, int gate, bool recovery, uint32_t pass_index,
                          bool pagerank);
  PassOut dense_pass_virtual(const sr_run_config& cfg, int gate, bool recovery,
                             uint32_t pass_index);
  RunStats launch_pages(const std::vector<uint32_t>& pages, int gate, bool det, RunCtr* ctr,
                        const RunCtr* prev, bool per_page, bool pagerank);
  void push_pass(const sr_run_config& cfg, RunStats& st);
  bool reentry_on_device(const std::vector<uint32_t>& pages, int gate, int runs, bool per_page);
  DBuf<uint32_t> runs_done_;  // K2: runs the last cooperative reentry launch executed
  void census(int pass_kind);
  void build_push_list(uint32_t shift);
  // Deferred push adjacency (big lean graphs, one run per load: the CSR
  // neighbours derivation costs more than the rare pushes it serves).
  bool csr_deferred_ = false;
  uint32_t runs_since_pages_ = 0;
  uint32_t scan_pushes_ = 0;  // CSC-scan pushes in the current run
  DBuf<uint32_t> fbits_;      // frontier bitmap of a CSC-scan push
  bool defer_csr(uint64_t m, int algo) const;
  void derive_csr_now();

 public:
  // sr_run_graph: the algorithm the next load_pages is for (-1 = unknown)
  void set_load_algo(int algo) { load_algo_ = algo; }

 private:
  int load_algo_ = -1;
  uint32_t push_chunk_shift(uint64_t total) const;
  void read_census();
  bool published_ = false;  // the last census published itself (read_census only syncs)
  DBuf<unsigned> pub_done_;
  PinBuf<unsigned> pub_seq_h_;  // last publish sequence number (read_census spins on it)
  unsigned pub_seq_ = 0;
  void wait_published(unsigned seq);
  void wait_word(const uint32_t* word, uint32_t pending);
  static constexpr uint32_t kTailPending = 0xffffffffu;  // tail_res_.passes until the tail loop ends
  void exchange_round(bool pagerank, uint32_t ctr_from = 0);
  int agg_slot_ = -1;  // counter slot holding the round's all-reduced aggregate (worlds)

  // streaming
  bool streaming() const { return !all_resident_; }
  void ensure_slots(uint32_t window, PassOut& po);
  uint32_t plan_window_ = 0;
  size_t plan_cached_ = size_t(-1);
  bool make_resident(uint32_t page, long long step, const std::vector<char>& protect,
                     PassOut& po);
  void build_tiles(uint32_t lo, uint32_t hi, cudaStream_t st);
  std::vector<cudaEvent_t> page_events_;  // resident upload: copy done per page
  cudaEvent_t ev_tiles_ = nullptr;
  cudaEvent_t ev_csr_ = nullptr;  // load_csr's work on the copy stream (before the pages)
  PinBuf<uint4> tile_stage_;
  PinBuf<uint32_t> tile_page_stage_, hub_stage_;
  PinBuf<PageDesc> desc_stage_;
  DBuf<unsigned long long> csr_cursor_;  // CSR derivation: next free slot per source

  int dev_ = 0;
  uint64_t budget_ = 0;
  int sm_count_ = 148;
  cudaStream_t cs_ = nullptr;  // compute stream
  cudaStream_t xs_ = nullptr;  // copy stream
  cudaEvent_t ev_start_ = nullptr, ev_stop_ = nullptr, ev_step_ = nullptr;

  // CSR (push stage, out-degrees)
  uint32_t n_ = 0;
  uint64_t m_ = 0;
  bool has_csr_ = false, has_csr_edges_ = false, csr_weighted_ = false;
  DBuf<unsigned long long> out_off_;
  DBuf<uint32_t> out_nbr_, out_w_;
  DBuf<uint32_t> outdeg_;  // u32 out-degrees (census/compaction vector loads)
  void maybe_derive_csr();  // push adjacency = transpose of resident pages
  void finish_csr(bool sync = true);  // out-degrees + flags after the CSR arrays are in place
  void build_graph_dev(uint32_t n, uint64_t m, DBuf<uint32_t>& src, DBuf<uint32_t>& dst,
                       DBuf<uint32_t>& w, bool weighted, uint32_t cap, bool csr_edges);
  bool csr_derived_ = false;
  // Forced HBM budget = CSC pages + push adjacency.  The adjacency is staged
  // in pinned host memory at load_csr and placed by load_pages once the page
  // bytes are known: on the device when pages + adjacency fit, else it stays
  // on the host and the sparse passes (K3 push, tail loop) read the
  // frontier's rows zero-copy over the host link -- the pages keep the HBM.
  PinBuf<uint32_t> host_nbr_, host_w_;
  HostStager stager_;  // pageable host -> device uploads through pinned chunks
  bool adj_host_ = false;
  uint64_t page_budget_ = 0;  // HBM left for pages (budget_ - device adjacency)
  void place_adjacency(uint64_t used_page_bytes, PassOut* po);
  // Rows [row_lo_, row_hi_) of the adjacency are held; a sharded rank holds
  // only its own rows, stored from edge off[row_lo_] = nbr_base_ on (the
  // kernels index with absolute CSR offsets, so the base is subtracted here).
  uint32_t row_lo_ = 0, row_hi_ = 0;
  uint64_t nbr_base_ = 0;
  const uint32_t* nbr_ptr() const {
    return (adj_host_ ? host_nbr_.p : out_nbr_.p) - nbr_base_;
  }
  const uint32_t* w_ptr() const {
    return csr_weighted_ ? (adj_host_ ? host_w_.p : out_w_.p) - nbr_base_ : nullptr;
  }

  // pages
  bool pages_loaded_ = false;
  uint32_t page_n_ = 0, cap_ = 0;
  bool weighted_ = false;
  std::vector<PageMeta> pages_;
  std::vector<uint32_t> hub_vertex_h_;
  uint64_t page_bytes_total_ = 0;
  uint64_t page_edges_total_ = 0;
  bool all_resident_ = true;
  DBuf<uint32_t> arena_offs_, arena_src_, arena_w_;
  PinBuf<uint32_t> stage_;  // pinned host copy of streamed pages
  DBuf<uint4> tiles_;
  DBuf<uint32_t> tile_page_;
  DBuf<PageDesc> page_desc_;
  std::vector<PageDesc> page_desc_h_;
  DBuf<uint32_t> hub_vertex_, hub_stamp_;
  DBuf<float> hub_sum_;
  uint32_t n_hubs_ = 0;
  std::vector<StreamSlot> slots_;  // entry pool (events created once; index = PageMeta::slot)
  std::vector<int> slot_free_;     // unused pool entries
  std::deque<int> ring_fifo_;      // live entries, oldest first
  DBuf<uint32_t> ring_;            // the streaming ring (HBM budget minus the cached pages)
  uint64_t ring_words_ = 0, ring_head_ = 0;
  void ring_reset();
  bool ring_evict_oldest(const std::vector<char>& protect);
  long long step_counter_ = 0;
  bool first_touch_done_ = false;  // resident path: admission counted once per run

  // run state
  DBuf<uint32_t> values_, next_, round_snap_;
  DBuf<uint8_t> changed_, status_, logstate_;
  DBuf<uint32_t> list_, chunk_start_, blk_cnt_;
  // frontier queue of the sparse passes (queue_mode): next queue, per-vertex
  // epoch stamps that deduplicate appends, whether list_ holds a queue
  DBuf<uint32_t> list2_, stamp_;
  DBuf<uint8_t> scan_tmp_;  // cub scan temporaries of the queue prep (no per-pass malloc)
  PinBuf<TailRecord> tail_rec_;  // small-frontier tail: per-pass records (mapped)
  PinBuf<TailResult> tail_res_;
  uint32_t fq_epoch_ = 0;
  bool fq_ready_ = false;
  bool queue_mode() const;
  DBuf<unsigned long long> pref_, blk_edges_, census_part_;
  DBuf<Census> census_;
  PinBuf<Census> census_h_;
  DBuf<RunCtr> ctr_;
  PinBuf<RunCtr> ctr_h_;
  uint32_t ctr_used_ = 0;  // entries of ctr_ handed out in the current pass
  RunCtr* alloc_ctr(size_t entries);
  DBuf<unsigned> work_;     // K1 per-launch tile counters (ring, zeroed on wrap)
  size_t work_used_ = 0;
  unsigned* next_work_counter();
  DBuf<float> rank_a_, rank_b_, contrib_a_, contrib_b_, inv_outdeg_;
  uint32_t run_id_ = 0;
  uint64_t h2d_bytes_ = 0;
  uint64_t gathers_total_ = 0;
  uint64_t streamed_total_ = 0;  // edges K1 streamed in (RunCtr::streamed)
  uint64_t visits_total_ = 0;    // destinations K1 scanned (RunCtr::visits)
  int blocks_per_sm_ = 4;

  // algorithm state of the current run
  int algo_ = 0;
  uint32_t source_ = 0;
  int predictor_ = 0;
  bool det_ = false;
  unsigned long long k_bfs_ = 0;
  uint32_t s_cc_ = 0, l_sssp_ = 0;
  uint32_t floor_sssp_ = 0;  // K1's source floor (PullArgs::src_floor)
  // every loaded page weight >= 1 (EdgeList::validate, graph.cpp:9-22); the
  // SSSP source floor assumes it, so hand-built page sets with weight-0
  // edges run without it (the reference's run() accepts them)
  bool weights_ge1_ = true;
  DBuf<unsigned> wflag_;
  VWindow vwin_;
  VClock vclock_;
  VModel vmodel_;
  bool record_trace_ = false;
  // Wall-clock trace (record_trace in ClockMode::Wall): CUDA events around
  // every launch (compute stream) and page transfer (copy stream).
  struct WallTraceRec {
    cudaEvent_t a, b;
    std::vector<uint32_t> pages;
    int start_kind;  // SR_TRACE_KERNEL_START / SR_TRACE_REENTRY / SR_TRACE_XFER_START
    uint32_t pass;
  };
  std::vector<WallTraceRec> wtrace_;
  std::vector<cudaEvent_t> wtrace_pool_;
  size_t wtrace_pool_used_ = 0;
  cudaEvent_t trace_event();
  bool trace_reentry_ = false;
  uint32_t cur_pass_ = 0;
  void finish_wall_trace();
  double pr_damp_ = 0.85;
  bool profile_kernels_ = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> relax_ev_;  // pool
  size_t relax_ev_used_ = 0;
  double collect_relax_seconds();

  // Source-blocked copy of the resident pages for PageRank (K8 locality):
  // sub-page (p, b) holds page p's in-edges whose source lies in block b.
  struct SrcBlocks {
    bool built = false;
    uint32_t blk_verts = 0, n_blocks = 0;
    DBuf<uint32_t> offs, src, w;
    // build temporaries kept across builds (multi-GB for big graphs:
    // cudaMalloc/cudaFree of them cost more than the build kernels)
    DBuf<uint32_t> t_cnt, t_tcnt, t_tat;
    DBuf<unsigned char> t_scan;
    DBuf<unsigned long long> t_goff, bp_edges, bp_base, t_part;
    std::vector<unsigned long long> page_base;
    bool pending = false;  // sb_begin done, sb_finish not yet
    DBuf<uint4> tiles;
    DBuf<uint32_t> tile_page;
    DBuf<PageDesc> desc;
    DBuf<float> acc;
    std::vector<uint32_t> block_tile_begin;  // n_blocks + 1
    std::vector<uint32_t> sub_tile_begin;    // n_blocks * n_pages + 1 (first tile of (b, p))
  } sb_;
  bool build_src_blocks(uint64_t blk_verts);
  bool sb_begin(uint64_t blk_verts);  // layout + buffers (page-major sub-pages)
  void sb_page(uint32_t p);           // page p's sub-pages (enqueued on cs_)
  bool sb_finish();                   // tile cut + descriptors (syncs cs_)
  // K8 hot-source staging (pr_pull_kernel<true>): the highest out-degree
  // sources' contributions live in shared memory; K8 reads an encoded copy
  // of its source array (hot sources -> kHotBit | slot) through its own page
  // descriptors.  Built once per page set / source-block layout.
  struct PrHot {
    bool built = false;
    bool blocked = false;
    const uint32_t* key = nullptr;  // source array the encoding was made from
    uint32_t n_hot = 0;
    int blocks_per_sm = 1;
    DBuf<uint32_t> enc, hot_vertex, slot_of;
    DBuf<float> hot_contrib;
    DBuf<PageDesc> desc;
    DBuf<unsigned long long> cnt;
  } pr_hot_;
  bool prepare_pr_hot(bool blocked);
  uint64_t pull_block_verts();
  uint64_t pr_block_verts() const;  // K8 source-block size (0: unblocked)
  double hot_source_coverage(uint64_t k);
  double coverage_ = -1;
  uint64_t coverage_k_ = 0;
  bool pull_blocked_pass(int gate, RunCtr* ctr, bool count_valid = false);
  Segments diag_first_segments(uint32_t b, uint32_t t0, uint32_t t1) const;
  bool diag_range(uint32_t b, uint32_t t0, uint32_t t1, uint32_t& d0, uint32_t& d1) const;
  Segments range_segments(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) const;
  int diag_local_iterations() const;
  bool probe_every_block() const;
  bool list_ok() const;
  double list_frac() const;
  bool last_pass_blocked_ = false;  // valid updates of the pass = destinations changed
  double last_gather_frac_ = 1.0;  // gathers / edges read of the last pass
  double dense_gather_frac_ = 1.0;  // ... of the last dense pass (K1 LIST choice)
  // A blocked pass's last block launch counts into its own slot: when even
  // its gathers were rare (labels / levels at the floor), the next dense pass
  // sweeps unblocked without probing block 0 first.
  int sb_last_slot_ = -1;
  double last_block_gather_frac_ = 1.0;
  double fallback_frac_ = -1;  // gathers/edges of the probe that ended a blocked pass
  std::pair<cudaEvent_t, cudaEvent_t>* relax_begin();
  void l2_window(const void* base, size_t bytes);
  int l2_persist_max_ = -1;  // persisting-L2 carve-out (bytes; 0 = unavailable/disabled)
  bool l2_window_set_ = false;
  int l2_bytes_ = 0;
  // persistent sparse stage buffers
  void pr_blocked_pass(float base, float damp);

  // multi-GPU
  int rank_ = 0, world_ = 1;
  ncclComm_t comm_ = nullptr;
  LoopbackGroup* loop_ = nullptr;  // in-process loopback collective (tests)
  // peer exchange: improvements are stored straight into the other ranks'
  // value replicas; a round ends with a barrier instead of a MIN all-reduce
  bool peer_xchg_ = false;
  DBuf<uint32_t*> peers_dev_;
  uint32_t n_peers_ = 0;
  void setup_peers();
  void round_barrier();  // all ranks reached this point of the round (peer exchange)
  // NCCL worlds: the peers' replicas mapped through CUDA IPC (cached per handle)
  std::vector<cudaIpcMemHandle_t> ipc_handles_;
  std::vector<void*> ipc_ptrs_;
  DBuf<unsigned char> ipc_buf_;
  DBuf<uint32_t> barrier_word_;

 public:
  void set_exchange(bool peer) { peer_xchg_ = peer; }

 private:
  uint32_t* const* peer_list() const { return n_peers_ ? peers_dev_.p : nullptr; }
  bool attached() const { return comm_ != nullptr || loop_ != nullptr; }
  uint32_t own_lo_ = 0, own_hi_ = 0;  // owned destination range
};

}  // namespace seraph
