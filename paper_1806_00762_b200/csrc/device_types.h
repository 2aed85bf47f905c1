// Device-side data layout shared by the kernels (kernels.cu) and the host
// engine (engine.cpp).  See DESIGN.md §3 "Data layout in HBM".
#pragma once

#include <cstdint>

namespace seraph {

constexpr uint32_t kUnreached = 0xffffffffu;  // reference types.hpp:14

enum Algo : int { kBfs = 0, kCc = 1, kSssp = 2, kPageRank = 3 };
enum GateKind : int { kGateOff = 0, kGateStrong = 1, kGateWeak = 2 };
enum PassKindDev : int { kPassSparse = 0, kPassDense = 1, kPassRecovery = 2, kPassInit = 3 };

// K1 work decomposition.  A page's destinations are cut at load time into
// warp tiles: either a run of whole destinations (<= kTileMaxDests dests and
// ~kTileEdgeBudget edges) or one chunk of a hub destination's in-edges.
constexpr int kWarpsPerBlock = 8;
constexpr int kBlockThreads = kWarpsPerBlock * 32;
constexpr uint32_t kTileMaxDests = 128;  // 16 KB smem per block: 6 blocks/SM + L1 room
constexpr uint32_t kTileEdgeBudget = 1024;
constexpr uint32_t kHubChunk = 1024;      // edges per hub chunk tile
constexpr uint32_t kHubFlag = 0x80000000u;  // tile.w flag: w & ~flag = hub id
constexpr int kMaxSegments = 8;           // tile ranges per launch
constexpr int kDiagIters = 1;             // blocked K1: diagonal sweeps until locally quiet (cap)
constexpr int kRootDiagReps = 6;
constexpr double kListFrac = 0.3;        // gathers/edges of the previous launch below which K1 runs its LIST variant
// K8 hot-source staging (pr_pull_kernel<true, kHotWarps>): blocks of
// kHotWarps warps (1.5 KB of tile scratch each) + a shared-memory table of
// f32 contributions of the hottest sources, encoded kHotBit | slot.  Measured
// on RMAT-26 (tools/c3ab.sh): 8 warps x 2048 entries (5 blocks/SM, L1 keeps
// ~128 KB) is best, -4.5 %; bigger tables cost L1 capacity and occupancy
// (16 K entries: +28 %, 64 K: +250 %).
constexpr int kHotWarps = 8;
constexpr uint32_t kHotDefault = 2048;
constexpr uint32_t kHotSmemBytes = 232448;  // 227 KB opt-in per CTA
constexpr uint32_t kHotBit = 0x80000000u;

// Tile (uint4): x = edge_lo, y = edge_hi (page-local edge indices),
// z = dest_lo (page-local), w = dest_hi (exclusive) or kHubFlag|hub_id.

// One page as the kernels see it: page-local CSC arrays wherever the page
// currently lives (resident arena or a streaming slot).
struct PageDesc {
  uint32_t vertex_begin;
  uint32_t range;
  uint64_t edge_count;
  const uint32_t* offs;  // range+1 page-local offsets (graph.hpp:49)
  const uint32_t* src;   // in_sources
  const uint32_t* w;     // in_weights or nullptr
};

// Per page-run counters (KernelRunStats, scheduler.hpp:145-158).
struct RunCtr {
  unsigned long long attempts;
  unsigned long long valid;
  unsigned long long skipped;
  unsigned long long edges;
  unsigned long long gathers;  // source values actually loaded (roofline bytes)
  unsigned long long streamed;  // edges whose source (+ weight) K1 actually streamed in
  unsigned long long visits;    // destinations K1's phase A scanned (value + offsets read)
};

// Scalars produced by the per-pass census (K4/K5), read back once per pass.
struct Census {
  // --- reset before every census ---
  unsigned long long changed;      // changed vertices (next frontier size)
  unsigned long long push_count;   // changed vertices with out-degree > 0
  unsigned long long out_edges;    // sum of out-degree of changed vertices
  unsigned long long status_hist[6];
  unsigned long long valid;        // deterministic push: destinations improved
  unsigned long long own_push;     // push-list entries owned by this rank
  unsigned long long own_edges;    // their out-edge volume
  // --- run-long accumulators ---
  unsigned long long log_events;   // PredictionLog events (weak)
  unsigned long long log_incorrect;
  unsigned int min_changed;        // strong SSSP l / CC s accumulator (all kernels)
};
constexpr unsigned kCensusResetBytes = 12 * sizeof(unsigned long long);

struct Segments {
  uint32_t n;
  uint32_t tile_begin[kMaxSegments];
  uint32_t task_prefix[kMaxSegments + 1];
};

struct PullArgs {
  unsigned* work;          // per-launch tile counter (dynamic scheduling)
  const uint4* tiles;
  const uint32_t* tile_page;
  const PageDesc* pages;
  Segments seg;
  uint32_t* values;        // async: read+write; det: read-only snapshot
  uint32_t* next;          // det: write target (== values in async)
  uint8_t* changed;        // changed-this-pass flags (engine.cpp:312-315)
  const uint8_t* status;   // weak predictor DFA state (predictor.hpp:29)
  uint32_t* hub_stamp;     // last run id that counted a hub's valid update
  uint32_t run_id;
  RunCtr* ctr;             // counters of this run: [page] or [0]
  const RunCtr* prev_ctr;  // reentry: skip pages whose previous run was quiet
  uint32_t ctr_per_page;   // 1: ctr/prev_ctr indexed by page, 0: all in ctr[0]
  Census* census;          // min_changed accumulator
  uint32_t count_dest;     // 1: count attempts/skipped (0 on source blocks > 0)
  uint32_t count_valid;    // 1: count valid updates (0 in source-blocked passes)
  uint32_t* const* peers;  // peer exchange: the other ranks' value replicas (else null)
  uint32_t n_peers;
  unsigned long long k_bfs;  // strong thresholds (predictor.hpp:47-52)
  uint32_t s_cc;
  uint32_t l_sssp;
  uint32_t src_floor;  // SSSP: lower bound of every source that can still improve (0 = none)
  uint32_t floor_step; // SSSP: smallest edge weight bound (1; 0 when a page holds weight-0 edges)
  uint32_t grab;       // tiles per work-counter grab (0 = kGrab)
  uint32_t list;       // converging launch (few gathers expected): K1's LIST
                       // variant relaxes sparse live destinations in its scan
};

// K2 (pull_reentry_kernel): up to `runs` runs of one page set in one
// cooperative launch; run r uses work[r] and ctr[r * ctr_stride ...].
struct ReentryArgs {
  unsigned* work;
  RunCtr* ctr;
  uint32_t ctr_stride;  // counters per run (pages of the set, per-page gating)
  uint32_t runs;        // MRT
  uint32_t* runs_done;  // runs actually executed (device -> host)
  uint32_t dest_every_run;  // 1: attempts/skips counted by every run (reentry), 0: by run 0 only
};

struct PrArgs {
  unsigned* work;  // per-launch tile counter
  const uint4* tiles;
  const uint32_t* tile_page;
  const PageDesc* pages;
  Segments seg;
  const float* contrib_in;
  float* rank_out;
  float* contrib_out;
  const float* inv_outdeg;
  float* hub_sum;
  float* acc;   // source-blocked mode: partial sums accumulate here (else null)
  RunCtr* ctr;
  float base;   // (1-d)/N
  float damp;   // d
  const float* hot_contrib;  // hot-source contributions (null: no staging)
  uint32_t n_hot;
};

struct PushArgs {
  const uint32_t* list;              // frontier ids with out-degree > 0 (sorted)
  const unsigned long long* pref;    // exclusive prefix of out-degree
  const uint32_t* chunk_start;       // first list entry of every push chunk
  uint32_t n_list;
  uint32_t chunk_shift;  // log2 of the edges per warp task (kPushChunk max)
  unsigned long long total_edges;
  const unsigned long long* out_offsets;
  const uint32_t* out_neighbors;
  const uint32_t* out_weights;
  uint32_t* values;
  uint32_t* next;  // det mode target
  uint8_t* changed;
  RunCtr* ctr;
  Census* census;
  // Frontier-queue mode (O(frontier) sparse passes; null stamp = changed
  // flags + census/compaction): the first improvement of v in this pass
  // (stamp[v] < epoch) appends v to q_list when it has out-edges and feeds
  // census->changed / push_count / out_edges; push_count is the queue cursor.
  uint32_t* stamp;
  uint32_t epoch;
  uint32_t* q_list;
  const uint32_t* outdeg;
  uint8_t* logstate;  // weak predictor: PredictionLog of first-time changes (else null)
  uint32_t* const* peers;  // peer exchange: the other ranks' value replicas (else null)
  uint32_t n_peers;
};
constexpr uint32_t kPushChunk = 256;  // flattened edges per warp task

// Small-frontier tail (K3 in one CTA): consecutive sparse passes whose queue
// fits kTailMaxQueue vertices / kTailMaxEdges out-edges run inside ONE
// single-block launch (block barriers only, no grid sync, no host round
// trip); the loop leaves when the frontier is empty, dense enough for a
// pull, or too big for one block.
constexpr uint32_t kTailMaxQueue = 8192;
constexpr uint32_t kTailMaxEdges = 1u << 16;
constexpr uint32_t kTailMaxPasses = 64;
struct TailRecord {
  unsigned long long edges, valid, changed, out_edges, queued;
};
struct TailResult {
  uint32_t passes;   // sparse passes run
  uint32_t reason;   // 0 converged, 1 dense next, 2 frontier too big, 3 pass cap
};
struct TailArgs {
  uint32_t* values;
  const unsigned long long* out_offsets;
  const uint32_t* out_neighbors;
  const uint32_t* out_weights;
  const uint32_t* outdeg;
  uint32_t* stamp;
  uint32_t epoch0;      // pass k uses epoch0 + k
  uint32_t* list;       // in: the queue (q0 entries); out: the final queue
  uint32_t* list2;      // scratch queue
  uint32_t q0;
  uint32_t max_passes;
  double dense_threshold;  // density_switch: dense iff out-edges > this
  int force_sparse;
  Census* census;       // strong-predictor min_changed accumulator
  uint8_t* logstate;    // weak predictor: PredictionLog of first-time changes (else null)
  TailRecord* rec;      // [max_passes] (mapped host memory)
  TailResult* res;      // (mapped host memory)
};


}  // namespace seraph
