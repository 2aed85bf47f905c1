// sm_100a kernels of the subgraph-iteration engine.
//
//   K1  pull_relax      dense pull over CSC pages   (ref engine.cpp:103-177)
//   K3  push_relax      sparse push over frontier   (ref engine.cpp:63-93)
//   K4  census/compact  changed flags -> frontier   (ref engine.cpp:312-315, :12-19)
//   K5  weak DFA step   in the census               (ref engine.cpp:317-328, predictor.cpp:18-41)
//   K6  cc_refresh      strong CC threshold         (ref predictor.cpp:55-105)
//   K7  recovery sweep  = K1 with the gate off      (ref engine.cpp:179-205)
//   K8  pr_pull         PageRank pull-sum           (new; no reference counterpart)
//
// The path is sparse and irregular: no tensor cores.  Everything is sized
// for HBM/L2 bandwidth: warp-cooperative, coalesced edge streams, shuffle
// based segmented reductions, ballot/prefix-sum compaction, persistent grids.
#include <cooperative_groups.h>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device_types.h"
#include "errors.h"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace seraph {

// Kernels launched by this thread (sr_metrics.kernel_launches: every launch
// wrapper below counts its own launches).
thread_local uint64_t t_launches = 0;
inline void note_launch(uint64_t k = 1) { t_launches += k; }
uint64_t kernel_launch_count() { return t_launches; }

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kCensusParts = 13;  // per-block census partials
constexpr int kLaneEdges = 8;  // consecutive edges per lane per K1 phase-B round
constexpr uint32_t kBndWords = 33;  // K1 entry-start bitmap words (span <= 1031 positions)
// K1 phase A in-place relaxation (see pull_relax_body): at most
// kInplaceMax live destinations of a 32-destination chunk, each with at most
// kInplaceDeg in-edges (0 disables; -D overrides for A/B builds)
#ifndef SERAPH_INPLACE_MAX
#define SERAPH_INPLACE_MAX 8
#endif
#ifndef SERAPH_INPLACE_DEG
#define SERAPH_INPLACE_DEG 16
#endif
constexpr int kInplaceMax = SERAPH_INPLACE_MAX;
constexpr uint32_t kInplaceDeg = SERAPH_INPLACE_DEG;
#ifndef SERAPH_SCAN_U
#define SERAPH_SCAN_U 4
#endif
constexpr int kScanU = SERAPH_SCAN_U;  // 32-destination chunks per step of the grab-wide gate scan
#ifndef SERAPH_SCAN_LIST
#define SERAPH_SCAN_LIST 1
#endif
#ifndef SERAPH_LIST_DEG
#define SERAPH_LIST_DEG 64
#endif
constexpr bool kScanList = SERAPH_SCAN_LIST != 0;  // PullArgs::list launches use the LIST kernel
constexpr uint32_t kListDeg = SERAPH_LIST_DEG;       // ... of at most this in-degree
constexpr uint32_t kGrab = 4;   // tiles a warp takes per work-counter atomic
constexpr uint32_t kNone = 0xffffffffu;  // no entry (K8 segmented merge)

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T x, int lane) {
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    T y = __shfl_up_sync(kFull, x, off);
    if (lane >= off) x += y;
  }
  return x;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
  return x;
}

__device__ __forceinline__ uint32_t warp_min(uint32_t x) { return __reduce_min_sync(kFull, x); }

// Random 4-byte gathers of vertex values (K1 async) and contributions (K8)
// go through L1 (allocating loads).  Measured on C2/C3/C4: ld.global.cg is
// 1.1-1.5x slower and ld.global.nc.L1::no_allocate 1.05-1.7x slower -- the
// L1 serves the hub values that many tiles gather.
__device__ __forceinline__ uint32_t gather_rw(const uint32_t* p) { return *p; }
__device__ __forceinline__ float gather_ro(const float* p) { return __ldg(p); }

// Peer exchange (sr_attach_* with the peer transport): an improvement is
// written straight into every other rank's replica of the value array (P2P
// over NVLink between GPUs; same-device pointers in the loopback world), so
// the round ends with a barrier instead of a |V|-sized MIN all-reduce.  A
// pulled destination has one writer per round (its owner): plain stores;
// hub chunks and pushes may race: atomicMin.
__device__ __forceinline__ void peer_store(uint32_t* const* peers, uint32_t n, uint32_t v,
                                           uint32_t x) {
  for (uint32_t r = 0; r < n; ++r) __stcg(peers[r] + v, x);
}
__device__ __forceinline__ void peer_min(uint32_t* const* peers, uint32_t n, uint32_t v,
                                         uint32_t x) {
  for (uint32_t r = 0; r < n; ++r) atomicMin(peers[r] + v, x);
}

// VertexProgram::combine (programs.hpp:31-45): saturating at kUnreached.
template <int A>
__device__ __forceinline__ uint32_t combine(uint32_t a, uint32_t w) {
  if (A == kCc) return a;
  if (a == kUnreached) return kUnreached;
  if (A == kBfs) return a + 1u;
  const uint32_t s = a + w;
  return s < a ? kUnreached : s;
}

// PredictorGate::should_attempt (engine.hpp:86-98) with strong_converged
// (predictor.cpp:43-53) and weak_should_attempt (predictor.hpp:32-34).
template <int A, int G>
__device__ __forceinline__ bool gate_attempt(uint32_t v, uint32_t cur, const PullArgs& a) {
  if (G == kGateOff) return true;
  if (G == kGateWeak) {
    const uint8_t s = a.status[v];
    return s == 0 || s == 1 || s == 5;
  }
  if (A == kBfs) return !(cur != kUnreached && (unsigned long long)cur <= a.k_bfs);
  if (A == kCc) return !(cur < a.s_cc);
  return !(cur < a.l_sssp);
}

// Map a flat task index of this launch onto a tile index.
__device__ __forceinline__ uint32_t task_to_tile(const Segments& seg, uint32_t t) {
  uint32_t s = 0;
#pragma unroll 1
  while (s + 1 < seg.n && t >= seg.task_prefix[s + 1]) ++s;
  return seg.tile_begin[s] + (t - seg.task_prefix[s]);
}

struct ActEntry {
  uint32_t local;   // page-local destination
  uint32_t estart;  // page-local first in-edge
  uint32_t pref;    // exclusive prefix of active edges inside the tile
  uint32_t cur;     // destination value when the tile was gated
};

// Per-lane counters: 32-bit where a lane's share is bounded by the edges it
// processes itself (registers are the K1 bottleneck), 64-bit for the edges
// of attempted destinations (a lane counts whole hub in-degrees).
struct LaneCtr {
  uint32_t attempts, valid, skipped, gathers;
  unsigned long long edges;
  uint32_t runs;    // warp-uniform: 8-edge runs streamed in (x8 = RunCtr::streamed)
  uint32_t visits;  // warp-uniform: destinations scanned by phase A (RunCtr::visits)
  __device__ void clear() {
    attempts = valid = skipped = gathers = runs = visits = 0;
    edges = 0;
  }
};

__device__ __forceinline__ void flush_ctr(LaneCtr& c, RunCtr* dst, int lane) {
  unsigned long long at = warp_sum<unsigned long long>(c.attempts),
                     va = warp_sum<unsigned long long>(c.valid),
                     sk = warp_sum<unsigned long long>(c.skipped), ed = warp_sum(c.edges),
                     ga = warp_sum<unsigned long long>(c.gathers);
  if (lane == 0 && dst) {
    if (at) atomicAdd(&dst->attempts, at);
    if (va) atomicAdd(&dst->valid, va);
    if (sk) atomicAdd(&dst->skipped, sk);
    if (ed) atomicAdd(&dst->edges, ed);
    if (ga) atomicAdd(&dst->gathers, ga);
    if (c.runs) atomicAdd(&dst->streamed, 8ull * c.runs);
    if (c.visits) atomicAdd(&dst->visits, (unsigned long long)c.visits);
  }
  c.clear();
}

// Smallest candidate any in-edge can produce (values are >= 0):
// combine(0, w) = 1 for BFS, 0 for CC; SSSP bounds per edge by its weight.
// A destination whose value is <= this bound cannot improve: its sources
// are not gathered (it still counts as attempted with all its edges read,
// the reference's accounting, engine.cpp:103-128).
template <int A>
__device__ __forceinline__ uint32_t candidate_floor() {
  return A == kBfs ? 1u : 0u;
}

// SSSP source floor (PullArgs::src_floor, set by the host from the smallest
// value written since the previous dense pass -- under the strong predictor
// that is its l; 0 under the weak predictor).  Every pass relaxes every edge
// whose source changed in the previous pass (dense pulls see all in-edges of
// every gated-in destination, the strong gate only drops destinations below
// l, pushes cover the whole frontier), so a source that did not change is
// already folded into its destinations; the ones that did hold values >= the
// floor, and every value written later is >= floor + 1.  Hence a candidate is
// >= floor + w: destinations at <= floor + 1 cannot improve and an edge with
// w >= value - floor cannot improve its destination -- neither is gathered.
// Attempt/skip/edge counters and the values are unchanged (the reference's
// accounting); only `gathers` drops.
template <int A>
__device__ __forceinline__ uint32_t source_floor(const PullArgs& a) {
  return A == kSssp ? a.src_floor : 0u;
}
template <int A>
__device__ __forceinline__ uint32_t dest_floor(const PullArgs& a) {
  if (A != kSssp) return candidate_floor<A>();
  const uint32_t f = a.src_floor;
  // weights >= 1 (graph.cpp:9-22); pages loaded with weight-0 edges (the
  // reference's run() accepts hand-built PageSets) run with floor_step 0
  return f >= kUnreached - 1 ? kUnreached : f + a.floor_step;
}

// End-of-kernel flush: warp sums -> shared memory -> one atomic per counter
// per block (thousands of same-address atomics per launch would serialise).
// `scratch` reuses the caller's tile shared memory (>= 40 words): extra
// static shared memory would push 4 blocks/SM past a carveout step and
// shrink the L1 that serves the gathers.
template <int W = kWarpsPerBlock>
__device__ __forceinline__ void block_flush(LaneCtr& c, RunCtr* dst, uint32_t lane_min,
                                            Census* census, uint32_t* scratch) {
  constexpr int kCtr = 7;
  constexpr int kWarpsPerBlock = W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long* red = reinterpret_cast<unsigned long long*>(scratch);
  uint32_t* mins = scratch + 2 * kCtr * kWarpsPerBlock;
  const unsigned long long v[kCtr] = {warp_sum<unsigned long long>(c.attempts),
                                      warp_sum<unsigned long long>(c.valid),
                                      warp_sum<unsigned long long>(c.skipped), warp_sum(c.edges),
                                      warp_sum<unsigned long long>(c.gathers),
                                      8ull * c.runs,  // runs, visits: warp-uniform
                                      (unsigned long long)c.visits};
  lane_min = warp_min(lane_min);
  __syncthreads();  // every warp is done with its tile scratch
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kCtr; ++k) red[k * kWarpsPerBlock + warp] = v[k];
    mins[warp] = lane_min;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t m = lane < kWarpsPerBlock ? mins[lane] : kUnreached;
    m = warp_min(m);
    if (lane < kCtr && dst) {
      unsigned long long x = 0;
#pragma unroll
      for (int w = 0; w < kWarpsPerBlock; ++w) x += red[lane * kWarpsPerBlock + w];
      if (x) atomicAdd(&dst->attempts + lane, x);
    }
    if (lane == 0 && census && m != kUnreached) atomicMin(&census->min_changed, m);
  }
  c.clear();
}

// ---------------------------------------------------------------------------
// K1: dense pull relaxation.  One warp per tile; persistent grid; warps grab
// kGrab consecutive tiles at a time from a per-launch work counter, so a
// warp stuck on dense tiles does not leave the others idle at the tail.
//
// Range tile, phase A: lanes walk 32 destinations at a time, load value and
// offsets, apply the predictor gate and compact the attempted destinations
// with in-edges into a shared-memory list (ballot + scan), so the edges of
// skipped destinations are never read.  Phase B: the attempted destinations'
// in-edges form one gap-free stream; each lane takes kLaneEdges CONSECUTIVE
// positions (one shared-memory binary search per run), issues all source,
// weight and gather loads back to back (memory-level parallelism), folds the
// run per destination in registers and merges partial minima across lanes
// with a shared-memory atomicMin.  Phase C: one lane per destination
// compares the minimum with the gated value and stores it (the page owns its
// destinations: plain store, no global atomic).
// Hub tile: one kHubChunk slice of a high in-degree destination; warp
// min-reduce, global atomicMin, and a run-id stamp that counts the
// destination's valid update once per run.
// One lane relaxes its own destination v (BFS/CC: no weights): its deg
// in-edges 4 source loads at a time, then their gathers; stores the minimum
// if it improves the gated value cur (one writer per destination, as phase C).
template <int A, bool DET>
__device__ __forceinline__ void relax_own(const PullArgs& a, const uint32_t* __restrict__ es,
                                          uint32_t deg, uint32_t v, uint32_t cur, LaneCtr& c,
                                          uint32_t& lane_min) {
  uint32_t best = kUnreached;
#pragma unroll 1
  for (uint32_t e = 0; e < deg; e += 4) {
    uint32_t sx[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) sx[k] = e + k < deg ? __ldcs(es + e + k) : 0u;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e + k < deg)
        best = min(best, combine<A>(DET ? __ldg(a.values + sx[k]) : gather_rw(a.values + sx[k]), 0u));
  }
  c.gathers += deg;
  if (best < cur) {
    if (DET) {
      a.next[v] = best;
    } else {
      a.values[v] = best;
      if (a.n_peers) peer_store(a.peers, a.n_peers, v, best);
    }
    a.changed[v] = 1;
    c.valid += a.count_valid;
    lane_min = min(lane_min, best);
  }
}

// ---------------------------------------------------------------------------
// 6 blocks x 8 warps per SM at <= 40 registers (measured best: 5 blocks at 48
// registers and 7-8 blocks at 32 registers with spills are 3-20 % slower)
template <int A, int G, bool DET, bool LIST>
__device__ __forceinline__ void pull_relax_body(const PullArgs& a, unsigned* a_work, RunCtr* a_ctr,
                                                const RunCtr* a_prev_ctr, uint32_t a_run_id,
                                                uint32_t a_count_dest) {
  __shared__ __align__(16) uint32_t s_pref[kWarpsPerBlock][kTileMaxDests];
  __shared__ uint32_t s_loc[kWarpsPerBlock][kTileMaxDests];
  __shared__ uint32_t s_cur[kWarpsPerBlock][kTileMaxDests];
  __shared__ uint32_t s_best[kWarpsPerBlock][kTileMaxDests];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  uint32_t* best_of = s_best[warp];
  const uint32_t total = a.seg.task_prefix[a.seg.n];
  const uint32_t grab = a.grab ? a.grab : kGrab;

  LaneCtr c;
  c.clear();
  uint32_t lane_min = kUnreached;
  uint32_t cur_page = 0xffffffffu;
  PageDesc pd{};
  const uint32_t* __restrict__ values_ro = a.values;

  for (;;) {
    uint32_t t0 = 0;
    if (lane == 0) t0 = atomicAdd(a_work, grab);
    t0 = __shfl_sync(kFull, t0, 0);
    if (t0 >= total) break;
    const uint32_t t1 = min(t0 + grab, total);
    // Grab-wide gate scan: when the grab's tiles are consecutive range tiles
    // of one page (one contiguous destination range), gate that range with
    // coalesced loads first.  If no destination in it can still improve (the
    // later passes of a converging run; sub-pages after the root block
    // settled) the grab is counted here and none of its tiles is entered;
    // otherwise the scan stops at the first live chunk and the tiles run.
    if (A != kSssp && !a_prev_ctr && t1 - t0 > 1 && t1 - t0 <= 32) {
      const uint32_t n = t1 - t0;
      uint32_t tp = 0;
      uint4 tl = make_uint4(0, 0, 0, 0);
      if (lane < n) {
        const uint32_t ti = task_to_tile(a.seg, t0 + lane);
        tp = a.tile_page[ti];
        tl = a.tiles[ti];
      }
      const uint32_t p0 = __shfl_sync(kFull, tp, 0);
      const uint32_t prev_w = __shfl_up_sync(kFull, tl.w, 1);
      const bool ok = lane >= n || (tp == p0 && !(tl.w & kHubFlag) && (lane == 0 || tl.z == prev_w));
      if (__all_sync(kFull, ok)) {
        if (p0 != cur_page) {
          if (a.ctr_per_page && cur_page != 0xffffffffu) flush_ctr(c, a_ctr + cur_page, lane);
          cur_page = p0;
          pd = a.pages[p0];
        }
        const uint32_t dl = __shfl_sync(kFull, tl.z, 0), dh = __shfl_sync(kFull, tl.w, n - 1);
        const uint32_t vb = pd.vertex_begin;
        const uint32_t* __restrict__ offs = pd.offs;
        const uint32_t* __restrict__ gsrc = pd.src;
        uint32_t n_att = 0, n_skip = 0, n_edges = 0, n_list = 0;
        bool live = false;
        // kScanU chunks of 32 destinations per step, all loads issued
        // before the first use (one memory round trip per step)
#pragma unroll 1
        for (uint32_t base = dl; base < dh; base += 32 * kScanU) {
          uint32_t cu[kScanU], o0[kScanU];
#pragma unroll
          for (int u = 0; u < kScanU; ++u) {
            const uint32_t i = base + u * 32 + lane;
            cu[u] = kUnreached;
            o0[u] = 0;
            if (i <= dh) o0[u] = offs[i];
            if (i < dh) cu[u] = DET ? __ldg(values_ro + vb + i) : a.values[vb + i];
          }
#pragma unroll
          for (int u = 0; u < kScanU; ++u) {
            const uint32_t i = base + u * 32 + lane;
            // offs[i + 1]: the next lane's load (lane 31: the next chunk's lane 0)
            uint32_t o1 = __shfl_down_sync(kFull, o0[u], 1);
            const uint32_t nx = __shfl_sync(kFull, u + 1 < kScanU ? o0[u + 1 < kScanU ? u + 1 : u] : 0u, 0);
            if (lane == 31) o1 = (u + 1 < kScanU) ? nx : (i < dh ? offs[i + 1] : 0u);
            uint32_t deg = 0;
            bool lv = false;
            if (i < dh) {
              deg = o1 - o0[u];
              const bool att = gate_attempt<A, G>(vb + i, cu[u], a);
              n_att += att;
              n_skip += !att;
              n_edges += att ? deg : 0u;
              lv = att && deg > 0 && cu[u] > dest_floor<A>(a);
            }
            if (LIST) {
              // sparse live destinations of low in-degree are listed (shared
              // memory) and relaxed in place after the scan; a denser or
              // heavier chunk sends the whole grab to the tile path
              const unsigned lm = __ballot_sync(kFull, lv);
              if (lm) {
                const uint32_t k = __popc(lm);
                if (n_list + k <= kTileMaxDests && __all_sync(kFull, !lv || deg <= kListDeg)) {
                  if (lv) {
                    const uint32_t pos = n_list + __popc(lm & lanemask_lt());
                    s_loc[warp][pos] = vb + i;
                    s_pref[warp][pos] = o0[u];
                    s_cur[warp][pos] = cu[u];
                    best_of[pos] = deg;
                  }
                  n_list += k;
                } else {
                  live = true;
                }
              }
            } else {
              live = live || lv;
            }
          }
          if (__any_sync(kFull, live)) break;
        }
        if (!__any_sync(kFull, live)) {
          c.attempts += n_att & (0u - a_count_dest);
          c.skipped += n_skip & (0u - a_count_dest);
          c.edges += n_edges;
          c.visits += dh - dl;
          if (LIST && n_list) {
            __syncwarp();
            uint32_t runs_l = 0;
            for (uint32_t j = lane; j < n_list; j += 32) {
              const uint32_t deg = best_of[j];
              relax_own<A, DET>(a, gsrc + s_pref[warp][j], deg, s_loc[warp][j], s_cur[warp][j], c,
                                lane_min);
              runs_l += (deg + 7) >> 3;
            }
            c.runs += __reduce_add_sync(kFull, runs_l);
            __syncwarp();
          }
          continue;
        }
      }
    }
    for (uint32_t t = t0; t < t1; ++t) {
      const uint32_t ti = task_to_tile(a.seg, t);
      const uint32_t p = a.tile_page[ti];
      if (p != cur_page) {
        if (a.ctr_per_page && cur_page != 0xffffffffu) flush_ctr(c, a_ctr + cur_page, lane);
        cur_page = p;
        pd = a.pages[p];
      }
      // quiet page (L2 read: in the K2 loop the previous run's counters were
      // written by other SMs' atomics within this launch)
      if (a_prev_ctr && __ldcg(&a_prev_ctr[a.ctr_per_page ? p : 0].valid) == 0) continue;
      const uint4 tile = a.tiles[ti];
      const uint32_t vb = pd.vertex_begin;
      const uint32_t* __restrict__ offs = pd.offs;
      const uint32_t* __restrict__ src = pd.src;
      const uint32_t* __restrict__ wts = pd.w;

      if (tile.w & kHubFlag) {
        // ---- hub chunk -----------------------------------------------------
        const uint32_t d = tile.z;
        const uint32_t v = vb + d;
        const uint32_t cur = DET ? __ldg(values_ro + v) : *(volatile uint32_t*)(a.values + v);
        const bool att = gate_attempt<A, G>(v, cur, a);
        const uint32_t lo_d = offs[d];
        if (lane == 0 && tile.x == lo_d) {  // owner chunk counts the visit once
          c.attempts += att & a_count_dest;
          c.skipped += !att & a_count_dest;
          c.edges += att ? (unsigned long long)(offs[d + 1] - lo_d) : 0ull;
        }
        if (!att || cur <= dest_floor<A>(a)) continue;
        c.runs += (tile.y - (tile.x & ~7u) + 7) >> 3;
        c.visits += tile.x == lo_d;  // the hub's first chunk reads its value and offsets
        const uint32_t thr = cur - source_floor<A>(a);  // live edges: w < thr
        // lanes take aligned 8-edge runs (two uint4 loads of sources and
        // weights), drop edges that cannot improve, gather the rest back to
        // back (~47 % of RMAT in-edges are in hub chunks)
        uint32_t best = kUnreached;
        for (uint32_t p0 = (tile.x & ~7u) + lane * kLaneEdges; p0 < tile.y;
             p0 += 32 * kLaneEdges) {
          const uint4* sp = reinterpret_cast<const uint4*>(src + p0);
          const uint4 s0 = __ldcs(sp), s1 = __ldcs(sp + 1);
          uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
          if (A == kSssp) {
            const uint4* wp = reinterpret_cast<const uint4*>(wts + p0);
            w0 = __ldcs(wp);
            w1 = __ldcs(wp + 1);
          }
          const uint32_t si[kLaneEdges] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
          const uint32_t wv[kLaneEdges] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
          unsigned live = 0;
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t)
            if (p0 + t >= tile.x && p0 + t < tile.y && (A != kSssp || wv[t] < thr))
              live |= 1u << t;
          uint32_t sv[kLaneEdges];
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t)
            sv[t] = (live >> t & 1u) ? (DET ? __ldg(values_ro + si[t]) : gather_rw(a.values + si[t]))
                                     : kUnreached;
          c.gathers += __popc(live);
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t) best = min(best, combine<A>(sv[t], wv[t]));
        }
        best = warp_min(best);
        if (lane == 0 && best < cur) {
          bool improved;
          if (DET) {
            atomicMin(a.next + v, best);
            improved = true;
          } else {
            const uint32_t old = atomicMin(a.values + v, best);
            improved = best < old;
            if (improved && a.n_peers) peer_min(a.peers, a.n_peers, v, best);
          }
          if (improved) {
            a.changed[v] = 1;
            lane_min = min(lane_min, best);
            const uint32_t hub = tile.w & ~kHubFlag;
            if (a.count_valid && atomicMax(a.hub_stamp + hub, a_run_id) < a_run_id) c.valid += 1;
          }
        }
        continue;
      }

      // ---- range tile: phase A (gate + entry list) ---------------------------
      // Entries = destinations with in-edges, in edge order; bit 31 of
      // s_loc marks the attempted ones.  pref = first edge relative to ebase.
      const uint32_t dl = tile.z, dh = tile.w;
      const uint32_t ebase = tile.x & ~7u;  // 32-byte aligned run grid
      c.visits += dh - dl;
      uint32_t n_ent = 0;
      unsigned any_att = 0, any_dead = 0;
      // entry starts as a bitmap over the tile's edge positions (span <=
      // kTileEdgeBudget + 7 -> <= 33 words) + per-word prefix counts: a run's
      // first entry and its entry steps come from one word, no search
      uint32_t* bnd = s_pref[warp];        // words [0, kBndWords)
      uint32_t* wpre = s_pref[warp] + 64;  // words [64, 64 + kBndWords)
      // one-chunk tiles (<= 32 destinations: every tile of a graph of
      // average in-degree >= 32) clear the bitmap only once the gate found a
      // destination that can still improve -- a dead tile (later passes,
      // sub-pages after the root block settled) costs loads and ballots only.
      // Not for SSSP: the extra live range spills at the 40-register cap
      // (C4 CC 7.93 -> 7.76 ms; SSSP C2 +2 % with the spill).
      const bool lazy = A != kSssp && dh - dl <= 32;
      if (!lazy) {
        bnd[lane] = 0;
        if (lane < kBndWords - 32) bnd[32 + lane] = 0;
        __syncwarp();
      }
      for (uint32_t base = dl; base < dh; base += 32) {
        const uint32_t i = base + lane;
        const bool in = i < dh;
        uint32_t cur = 0, lo = 0, deg = 0;
        bool att = false;
        if (in) {
          const uint32_t v = vb + i;
          cur = DET ? __ldg(values_ro + v) : a.values[v];
          lo = __ldcs(offs + i);
          deg = __ldcs(offs + i + 1) - lo;
          att = gate_attempt<A, G>(v, cur, a);
        }
        c.attempts += att & a_count_dest;
        c.skipped += (in && !att) & a_count_dest;
        c.edges += att ? deg : 0u;
        bool need = att && cur > dest_floor<A>(a);  // can it still improve?
        const bool has = in && deg > 0;
        if (kInplaceMax && A != kSssp) {
          // Few live destinations in this chunk, each with few in-edges (a
          // converging pass: most destinations already sit at the floor):
          // each live lane relaxes its own destination right here -- its
          // in-edges 4 loads at a time, then their gathers -- and the
          // chunk's entries count as dead for the tile's bitmap / run
          // machinery (phases B and C), which is skipped when no chunk of the
          // tile still needs it.  One writer per destination (the lane), as
          // in phase C.  C4 7.34 -> 7.17 ms (the block launches after the
          // root block and the confirming pass); C1/C2 unchanged.  Not SSSP:
          // the 40-register cap.
          const unsigned lm = __ballot_sync(kFull, has && need);
          if (lm && __popc(lm) <= kInplaceMax &&
              __all_sync(kFull, !(has && need) || deg <= kInplaceDeg)) {
            if (has && need) relax_own<A, DET>(a, src + lo, deg, vb + i, cur, c, lane_min);
            c.runs += __reduce_add_sync(kFull, (has && need) ? (deg + 7) >> 3 : 0u);
            need = false;
          }
        }
        const unsigned m = __ballot_sync(kFull, has);
        any_att |= __ballot_sync(kFull, has && need);
        any_dead |= __ballot_sync(kFull, has && !need);
        if (lazy) {
          if (!any_att) break;
          bnd[lane] = 0;
          if (lane < kBndWords - 32) bnd[32 + lane] = 0;
          __syncwarp();
        }
        if (has) {
          const uint32_t pos = n_ent + __popc(m & lanemask_lt());
          const uint32_t p0 = lo - ebase;
          atomicOr(bnd + (p0 >> 5), 1u << (p0 & 31));
          s_loc[warp][pos] = i | (need ? 0x80000000u : 0u);
          s_cur[warp][pos] = cur;
          best_of[pos] = kUnreached;
        }
        n_ent += __popc(m);
      }
      __syncwarp();
      if (!any_att) {
        __syncwarp();
        continue;
      }
      const uint32_t* loc_of = s_loc[warp];
      const uint32_t lo_pos = tile.x - ebase;   // first valid position
      const uint32_t span = tile.y - ebase;     // one past the last position
      {
        const uint32_t c = __popc(bnd[lane]);
        const uint32_t inc = warp_incl_scan(c, lane);
        wpre[lane] = inc - c;
        if (lane == 31) wpre[32] = inc;
      }
      __syncwarp();

      // ---- phase B: aligned 8-edge runs, vector loads, masked gathers --------
      for (uint32_t r0 = 0; r0 < span; r0 += 32 * kLaneEdges) {
        const uint32_t pos0 = r0 + lane * kLaneEdges;
        bool loaded = false;  // this lane streams its run in (live positions)
        if (pos0 < span && pos0 + kLaneEdges > lo_pos) {
          const uint32_t q = max(pos0, lo_pos);
          // runs are 8-aligned, so the run's 8 positions sit in one bitmap word
          const uint32_t bw = bnd[pos0 >> 5];
          const uint32_t ent0 = wpre[pos0 >> 5] + __popc(bw & (0xffffffffu >> (31 - (q & 31)))) - 1;
          // adv bit t: an entry starts at position pos0 + t (after q)
          const unsigned adv = (bw >> (pos0 & 31)) & (0xffu << (q - pos0 + 1)) & 0xffu;
          const uint32_t hi_t = min(span - pos0, (uint32_t)kLaneEdges);
          // every entry of the tile can still improve (the common case of a
          // first dense pass): the live positions are the run's valid ones
          unsigned live = (0xffu >> (8 - hi_t)) & (0xffu << (q - pos0)) & 0xffu;
          if (any_dead) {
            live = 0;
            uint32_t e = ent0, from = q - pos0;
            unsigned rem = adv;
#pragma unroll 1
            for (;;) {
              const uint32_t upto = rem ? (uint32_t)__ffs(rem) - 1 : hi_t;
              if (loc_of[e] >> 31) live |= (0xffu >> (8 - upto)) & (0xffu << from);
              if (!rem) break;
              from = upto;
              rem &= rem - 1;
              ++e;
            }
          }
          loaded = live != 0;
          if (live) {
            const uint4* sp = reinterpret_cast<const uint4*>(src + ebase + pos0);
            const uint4 s0 = __ldcs(sp), s1 = __ldcs(sp + 1);
            uint4 w0 = make_uint4(0, 0, 0, 0), w1 = w0;
            if (A == kSssp) {
              const uint4* wp = reinterpret_cast<const uint4*>(wts + ebase + pos0);
              w0 = __ldcs(wp);
              w1 = __ldcs(wp + 1);
            }
            const uint32_t sv_idx[kLaneEdges] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
            const uint32_t wv[kLaneEdges] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            if (A == kSssp) {
              // sources are >= source_floor, so an edge with w >= value - floor
              // cannot improve its destination: no gather (the wavefront-bound
              // part of K1).  Live entries have value > floor + 1; the others'
              // bits are already clear, so their wrap-around is harmless.
              const uint32_t fl = source_floor<A>(a);
              uint32_t et = ent0, cur_t = s_cur[warp][ent0];
#pragma unroll
              for (int t = 0; t < kLaneEdges; ++t) {
                if (adv >> t & 1u) cur_t = s_cur[warp][++et];
                if (wv[t] >= cur_t - fl) live &= ~(1u << t);
              }
            }
            uint32_t sv[kLaneEdges];
#pragma unroll
            for (int t = 0; t < kLaneEdges; ++t)
              sv[t] = (live >> t & 1u) ? (DET ? __ldg(values_ro + sv_idx[t])
                                              : gather_rw(a.values + sv_idx[t]))
                                       : kUnreached;
            c.gathers += __popc(live);
            uint32_t run_ent = 0xffffffffu, run_best = kUnreached, et = ent0;
#pragma unroll
            for (int t = 0; t < kLaneEdges; ++t) {
              et += adv >> t & 1u;
              if (!(live >> t & 1u)) continue;
              if (et != run_ent) {
                if (run_ent != 0xffffffffu) atomicMin(best_of + run_ent, run_best);
                run_ent = et;
                run_best = kUnreached;
              }
              run_best = min(run_best, combine<A>(sv[t], wv[t]));
            }
            atomicMin(best_of + run_ent, run_best);
          }
        }
        c.runs += __popc(__ballot_sync(kFull, loaded));
      }
      __syncwarp();
      // ---- phase C: one lane per attempted destination stores its minimum ---
      for (uint32_t i = lane; i < n_ent; i += 32) {
        const uint32_t l = loc_of[i];
        const uint32_t b = best_of[i];
        if ((l >> 31) && b < s_cur[warp][i]) {
          const uint32_t v = vb + (l & 0x7fffffffu);
          if (DET) {
            a.next[v] = b;
          } else {
            a.values[v] = b;
            if (a.n_peers) peer_store(a.peers, a.n_peers, v, b);
          }
          a.changed[v] = 1;
          c.valid += a.count_valid;
          lane_min = min(lane_min, b);
        }
      }
      __syncwarp();
    }
  }
  if (a.ctr_per_page) {
    if (cur_page != 0xffffffffu) flush_ctr(c, a_ctr + cur_page, lane);
    block_flush(c, nullptr, lane_min, a.census, &s_pref[0][0]);
  } else {
    block_flush(c, a_ctr, lane_min, a.census, &s_pref[0][0]);
  }
}

// LIST: the converging-launch variant (PullArgs::list): its grab-wide scan
// also relaxes sparse live destinations itself.  A separate instantiation:
// the list state costs registers (spills) that the gather-heavy launches
// must not pay.
template <int A, int G, bool DET, bool LIST>
__global__ void __launch_bounds__(kBlockThreads, 6) pull_relax_kernel(PullArgs a) {
  pull_relax_body<A, G, DET, LIST>(a, a.work, a.ctr, a.prev_ctr, a.run_id, a.count_dest);
}

// ---------------------------------------------------------------------------
// K2: local convergence on the device (reentry, scheduler.cpp:272-291: re-run
// the resident set while it still changes, up to MRT runs).  ONE cooperative
// launch loops: run r relaxes every page whose run r-1 had valid updates
// (device quiet-page gate), a grid barrier, and the loop stops as soon as a
// whole run was quiet -- no host round trip and no launch per re-run.
// ---------------------------------------------------------------------------
template <int A, int G>
__global__ void __launch_bounds__(kBlockThreads, 5) pull_reentry_kernel(PullArgs a,
                                                                         ReentryArgs r) {
  cg::grid_group grid = cg::this_grid();
  for (uint32_t it = 0; it < r.runs; ++it) {
    RunCtr* ctr = r.ctr + size_t(it) * r.ctr_stride;
    pull_relax_body<A, G, false, false>(a, r.work + it, ctr,
                                 it ? r.ctr + size_t(it - 1) * r.ctr_stride : nullptr,
                                 a.run_id + it, (it == 0 || r.dest_every_run) ? a.count_dest : 0u);
    grid.sync();  // every page's counters of run `it` are final and visible
    unsigned long long v = 0;
    for (uint32_t p = 0; p < r.ctr_stride; ++p) v += __ldcg(&ctr[p].valid);
    if (v == 0 || it + 1 == r.runs) {
      if (blockIdx.x == 0 && threadIdx.x == 0) *r.runs_done = it + 1;
      break;
    }
  }
}

// ---------------------------------------------------------------------------
// Device-side CSR adjacency from the resident CSC pages (§8(f) row 1): every
// in-edge (src -> v, w) of every page is scattered to out_off[src] + a
// per-source cursor.  Same tile walk as K1 (aligned 8-edge runs per lane).
// Order inside an adjacency list is arbitrary; the push kernel and the
// fixpoint are order-independent (SURVEY §7 "Asynchronous semantics").
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlockThreads)
csr_from_pages_kernel(const uint4* __restrict__ tiles, const uint32_t* __restrict__ tile_page,
                      const PageDesc* __restrict__ pages, uint32_t tile_lo, uint32_t tile_hi,
                      unsigned long long* cursor, uint32_t* out_nbr, uint32_t* out_w) {
  __shared__ __align__(16) uint32_t s_pref[kWarpsPerBlock][kTileMaxDests];
  __shared__ uint32_t s_loc[kWarpsPerBlock][kTileMaxDests];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (uint32_t ti = tile_lo + blockIdx.x * kWarpsPerBlock + warp; ti < tile_hi;
       ti += gridDim.x * kWarpsPerBlock) {
    const PageDesc pd = pages[tile_page[ti]];
    const uint4 tile = tiles[ti];
    const uint32_t* __restrict__ src = pd.src;
    const uint32_t* __restrict__ wts = pd.w;
    if (tile.w & kHubFlag) {
      const uint32_t v = pd.vertex_begin + tile.z;
      for (uint32_t e = tile.x + lane; e < tile.y; e += 32) {
        const uint32_t s = src[e];
        const unsigned long long pos = atomicAdd(cursor + s, 1ull);
        out_nbr[pos] = v;
        if (out_w) out_w[pos] = wts[e];
      }
      continue;
    }
    const uint32_t dl = tile.z, dh = tile.w;
    const uint32_t ebase = tile.x & ~7u;
    uint32_t n_ent = 0;
    for (uint32_t base = dl; base < dh; base += 32) {
      const uint32_t i = base + lane;
      uint32_t lo = 0, deg = 0;
      if (i < dh) {
        lo = pd.offs[i];
        deg = pd.offs[i + 1] - lo;
      }
      const unsigned m = __ballot_sync(kFull, deg > 0);
      if (deg > 0) {
        const uint32_t pos = n_ent + __popc(m & lanemask_lt());
        s_pref[warp][pos] = lo - ebase;
        s_loc[warp][pos] = i;
      }
      n_ent += __popc(m);
    }
    __syncwarp();
    const uint32_t lo_pos = tile.x - ebase, span = tile.y - ebase;
    for (uint32_t r0 = 0; n_ent && r0 < span; r0 += 32 * kLaneEdges) {
      const uint32_t pos0 = r0 + lane * kLaneEdges;
      if (pos0 < span && pos0 + kLaneEdges > lo_pos) {
        const uint32_t q = max(pos0, lo_pos);
        uint32_t lo = 0, hi = n_ent - 1;
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (s_pref[warp][mid] <= q) lo = mid;
          else hi = mid - 1;
        }
        uint32_t ent = lo;
        uint32_t nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
#pragma unroll
        for (int t = 0; t < kLaneEdges; ++t) {
          const uint32_t pp = pos0 + t;
          if (pp >= span) break;
          if (pp >= nxt) {
            ++ent;
            nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
          }
          if (pp < lo_pos) continue;
          const uint32_t e = ebase + pp;
          const uint32_t s = src[e];
          const unsigned long long pos = atomicAdd(cursor + s, 1ull);
          out_nbr[pos] = pd.vertex_begin + s_loc[warp][ent];
          if (out_w) out_w[pos] = wts[e];
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Source-blocked page split (K8 locality): every in-edge
// (s -> v) of a resident page goes to sub-page (page, s / blk_verts), so one
// sweep over the sub-pages of a block gathers only a blk_verts-wide slice of
// the vertex array (L2-resident).  mode 0 counts per (block, destination),
// mode 1 scatters the sources using goff (exclusive scan of the counts) and
// cur (zeroed counts) as cursors.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlockThreads)
src_block_kernel(int mode, const uint4* __restrict__ tiles, const uint32_t* __restrict__ tile_page,
                 const PageDesc* __restrict__ pages, uint32_t tile_lo, uint32_t tile_hi,
                 uint32_t n, uint32_t blk_verts, uint32_t n_pages, uint32_t* cnt,
                 unsigned long long* goff, uint32_t* out_src, uint32_t* out_w) {
  __shared__ uint32_t s_pref[kWarpsPerBlock][kTileMaxDests];
  __shared__ uint32_t s_loc[kWarpsPerBlock][kTileMaxDests];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // mode 1: goff holds absolute cursors (src_block_page_fix_kernel)
  for (uint32_t ti = tile_lo + blockIdx.x * kWarpsPerBlock + warp; ti < tile_hi;
       ti += gridDim.x * kWarpsPerBlock) {
    const uint32_t pg = tile_page[ti];
    const PageDesc pd = pages[pg];
    const uint4 tile = tiles[ti];
    const uint32_t* __restrict__ src = pd.src;
    if (tile.w & kHubFlag) {
      // one destination, up to kHubChunk in-edges: lanes whose sources fall
      // in the same block share ONE atomic (match_any groups) -- RMAT hubs
      // would otherwise serialise thousands of atomics on one counter
      const uint32_t v = pd.vertex_begin + tile.z;
      for (uint32_t e0 = tile.x; e0 < tile.y; e0 += 32) {
        const uint32_t e = e0 + lane;
        const bool ok = e < tile.y;
        const uint32_t sv = ok ? src[e] : 0u;
        const uint32_t b = ok ? sv / blk_verts : kNone;
        const unsigned grp = __match_any_sync(kFull, b);
        const int leader = __ffs(grp) - 1;
        const uint32_t k_n = __popc(grp);
        const size_t k = size_t(b) * n + v;
        if (mode == 0) {
          if (ok && lane == leader) atomicAdd(cnt + k, k_n);
        } else {
          unsigned long long o = 0;
          if (ok && lane == leader) o = atomicAdd(goff + k, (unsigned long long)k_n);
          o = __shfl_sync(kFull, o, leader) + __popc(grp & lanemask_lt());
          if (ok) {
            out_src[o] = sv;
            if (out_w) out_w[o] = pd.w[e];
          }
        }
      }
      continue;
    }
    const uint32_t dl = tile.z, dh = tile.w;
    const uint32_t ebase = tile.x & ~7u;
    uint32_t n_ent = 0;
    for (uint32_t base = dl; base < dh; base += 32) {
      const uint32_t i = base + lane;
      uint32_t lo = 0, deg = 0;
      if (i < dh) {
        lo = pd.offs[i];
        deg = pd.offs[i + 1] - lo;
      }
      const unsigned m = __ballot_sync(kFull, deg > 0);
      if (deg > 0) {
        const uint32_t pos = n_ent + __popc(m & lanemask_lt());
        s_pref[warp][pos] = lo - ebase;
        s_loc[warp][pos] = i;
      }
      n_ent += __popc(m);
    }
    __syncwarp();
    const uint32_t lo_pos = tile.x - ebase, span = tile.y - ebase;
    for (uint32_t r0 = 0; n_ent && r0 < span; r0 += 32 * kLaneEdges) {
      const uint32_t pos0 = r0 + lane * kLaneEdges;
      if (pos0 < span && pos0 + kLaneEdges > lo_pos) {
        const uint32_t q = max(pos0, lo_pos);
        uint32_t lo = 0, hi = n_ent - 1;
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (s_pref[warp][mid] <= q) lo = mid;
          else hi = mid - 1;
        }
        uint32_t ent = lo;
        uint32_t nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
        for (int t = 0; t < kLaneEdges; ++t) {
          const uint32_t pp = pos0 + t;
          if (pp >= span) break;
          if (pp >= nxt) {
            ++ent;
            nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
          }
          if (pp < lo_pos) continue;
          const uint32_t sv = src[ebase + pp];
          const size_t k = size_t(sv / blk_verts) * n + pd.vertex_begin + s_loc[warp][ent];
          if (mode == 0) {
            atomicAdd(cnt + k, 1u);
          } else {
            const unsigned long long o = atomicAdd(goff + k, 1ull);
            out_src[o] = sv;
            if (out_w) out_w[o] = pd.w[ebase + pp];
          }
        }
      }
    }
    __syncwarp();
  }
}

__global__ void pr_block_finalize_kernel(uint32_t lo, uint32_t hi, float* acc, float* rank_out,
                                         float* contrib_out, const float* __restrict__ inv_outdeg,
                                         float base, float damp) {
  for (uint32_t v = lo + blockIdx.x * blockDim.x + threadIdx.x; v < hi;
       v += gridDim.x * blockDim.x) {
    const float r = base + damp * acc[v];
    rank_out[v] = r;
    contrib_out[v] = r * inv_outdeg[v];
    acc[v] = 0.f;
  }
}

__global__ void outdeg_kernel(const unsigned long long* __restrict__ off, uint32_t n,
                              uint32_t* deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    deg[v] = (uint32_t)(off[v + 1] - off[v]);
}

__global__ void commit_kernel(uint32_t* __restrict__ values, const uint32_t* __restrict__ next,
                              uint32_t lo, uint32_t hi) {
  for (uint32_t v = lo + blockIdx.x * blockDim.x + threadIdx.x; v < hi;
       v += gridDim.x * blockDim.x)
    values[v] = next[v];
}

// ---------------------------------------------------------------------------
// K8: PageRank pull-sum (Jacobi: contrib_in is read-only in the launch).
// Same tile walk as K1: entries per destination, aligned 8-edge lane runs
// with uint4 source loads, gathers of contrib[src], per-lane fold and a
// shared-memory float atomicAdd merge; hub chunks go through hub_sum.
// ---------------------------------------------------------------------------
//
// HOT (north_star "shared-memory staging of hot vertex values"): the n_hot
// highest out-degree sources have their contributions staged in shared memory
// once per launch (a.hot_contrib, compacted by pr_hot_gather_kernel), and the
// launch reads a source array in which those sources are encoded as
// kHotBit | slot (Engine::prepare_pr_hot).  A random 4-byte gather through
// L1 costs one L1TEX wavefront per lane (one 128 B line each); a shared-memory
// gather costs one bank cycle per conflicting lane, so every hot-source edge
// leaves the L1 gather queue.  One block of W warps per SM holds the table.
template <bool HOT, int W>
__global__ void __launch_bounds__(W * 32) pr_pull_kernel(PrArgs a) {
  __shared__ __align__(16) uint32_t s_pref[W][kTileMaxDests];
  __shared__ uint32_t s_loc[W][kTileMaxDests];
  __shared__ float s_sum[W][kTileMaxDests];
  extern __shared__ float s_hot[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  float* sum_of = s_sum[warp];
  const uint32_t total = a.seg.task_prefix[a.seg.n];
  LaneCtr c;
  c.clear();
  uint32_t cur_page = 0xffffffffu;
  PageDesc pd{};
  const float* __restrict__ contrib = a.contrib_in;
  if (HOT) {
    const float4* h4 = reinterpret_cast<const float4*>(a.hot_contrib);
    float4* s4 = reinterpret_cast<float4*>(s_hot);
    for (uint32_t i = threadIdx.x; i < (a.n_hot + 3) / 4; i += W * 32) s4[i] = __ldcg(h4 + i);
    __syncthreads();
  }
  auto gather = [&](uint32_t s) -> float {
    if (HOT && (s & kHotBit)) return s_hot[s & ~kHotBit];
    return gather_ro(contrib + s);
  };

  for (;;) {
    uint32_t t0 = 0;
    if (lane == 0) t0 = atomicAdd(a.work, kGrab);
    t0 = __shfl_sync(kFull, t0, 0);
    if (t0 >= total) break;
    const uint32_t t1 = min(t0 + kGrab, total);
    for (uint32_t t = t0; t < t1; ++t) {
      const uint32_t ti = task_to_tile(a.seg, t);
      const uint32_t p = a.tile_page[ti];
      if (p != cur_page) {
        cur_page = p;
        pd = a.pages[p];
      }
      const uint4 tile = a.tiles[ti];
      const uint32_t vb = pd.vertex_begin;
      const uint32_t* __restrict__ offs = pd.offs;
      const uint32_t* __restrict__ src = pd.src;
      if (tile.w & kHubFlag) {
        const uint32_t d = tile.z;
        const uint32_t lo_d = offs[d];
        if (lane == 0 && tile.x == lo_d) {
          c.attempts += 1;
          c.edges += offs[d + 1] - lo_d;
        }
        float sum = 0.f;
        if (lane == 0) c.gathers += tile.y - tile.x;
        for (uint32_t p0 = (tile.x & ~7u) + lane * kLaneEdges; p0 < tile.y;
             p0 += 32 * kLaneEdges) {
          const uint4* sp = reinterpret_cast<const uint4*>(src + p0);
          const uint4 s0 = __ldcs(sp), s1 = __ldcs(sp + 1);
          const uint32_t si[kLaneEdges] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
          float x[kLaneEdges];
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t)
            x[t] = (p0 + t >= tile.x && p0 + t < tile.y) ? gather(si[t]) : 0.f;
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t) sum += x[t];
        }
        sum = warp_sum(sum);
        if (lane == 0) {
          if (a.acc) atomicAdd(a.acc + vb + d, sum);  // source-blocked partial
          else atomicAdd(a.hub_sum + (tile.w & ~kHubFlag), sum);
        }
        continue;
      }
      const uint32_t dl = tile.z, dh = tile.w;
      const uint32_t ebase = tile.x & ~7u;
      uint32_t n_ent = 0;
      for (uint32_t base = dl; base < dh; base += 32) {
        const uint32_t i = base + lane;
        const bool in = i < dh;
        uint32_t lo = 0, deg = 0;
        if (in) {
          lo = __ldcs(offs + i);
          deg = __ldcs(offs + i + 1) - lo;
          if (deg == 0 && !a.acc) {  // no in-edges: teleport share only
            const uint32_t v = vb + i;
            a.rank_out[v] = a.base;
            a.contrib_out[v] = a.base * a.inv_outdeg[v];
          }
        }
        c.attempts += in;
        c.edges += deg;
        const unsigned m = __ballot_sync(kFull, deg > 0);
        if (deg > 0) {
          const uint32_t pos = n_ent + __popc(m & lanemask_lt());
          s_pref[warp][pos] = lo - ebase;
          s_loc[warp][pos] = i;
          sum_of[pos] = 0.f;
        }
        n_ent += __popc(m);
      }
      __syncwarp();
      if (n_ent == 0) {
        __syncwarp();
        continue;
      }
      const uint32_t lo_pos = tile.x - ebase, span = tile.y - ebase;
      // Per-destination merge without shared-memory atomics (a float
      // atomicAdd on shared memory is a CAS spin loop, ATOMS.CAST.SPIN): a
      // lane's runs strictly inside its 8 positions are complete destinations
      // (plain store); its first/last runs may continue across lanes, so
      // their partial sums are combined by a segmented warp scan and written
      // once, by the lane where the destination's run ends in this round.
      for (uint32_t r0 = 0; r0 < span; r0 += 32 * kLaneEdges) {
        const uint32_t pos0 = r0 + lane * kLaneEdges;
        uint32_t id_f = kNone, id_l = kNone;
        float s_f = 0.f, s_l = 0.f;
        bool multi = false;
        if (pos0 < span && pos0 + kLaneEdges > lo_pos) {
          const uint32_t q = max(pos0, lo_pos);
          uint32_t lo = 0, hi = n_ent - 1;
          while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            if (s_pref[warp][mid] <= q) lo = mid;
            else hi = mid - 1;
          }
          uint32_t ent = lo;
          uint32_t nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
          uint32_t eid[kLaneEdges];  // (K8 has registers to spare: measured faster than K1's adv mask)
          unsigned live = 0;
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t) {
            const uint32_t pp = pos0 + t;
            if (pp >= nxt && pp < span) {
              ++ent;
              nxt = (ent + 1 < n_ent) ? s_pref[warp][ent + 1] : span;
            }
            eid[t] = ent;
            if (pp >= lo_pos && pp < span) live |= 1u << t;
          }
          const uint4* sp = reinterpret_cast<const uint4*>(src + ebase + pos0);
          const uint4 s0 = __ldcs(sp), s1 = __ldcs(sp + 1);
          const uint32_t sidx[kLaneEdges] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
          float x[kLaneEdges];
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t)
            x[t] = (live >> t & 1u) ? gather(sidx[t]) : 0.f;
          c.gathers += __popc(live);
          uint32_t run_ent = kNone;
          float run = 0.f;
#pragma unroll
          for (int t = 0; t < kLaneEdges; ++t) {
            if (!(live >> t & 1u)) continue;
            if (eid[t] != run_ent) {
              if (run_ent != kNone) {
                if (!multi) {
                  id_f = run_ent;
                  s_f = run;
                } else {
                  sum_of[run_ent] = run;  // complete inside this lane
                }
                multi = true;
              }
              run_ent = eid[t];
              run = 0.f;
            }
            run += x[t];
          }
          id_l = run_ent;
          s_l = run;
          if (!multi) {
            id_f = run_ent;
            s_f = run;
          }
        }
        uint32_t prev_l = __shfl_up_sync(kFull, id_l, 1);
        uint32_t next_f = __shfl_down_sync(kFull, id_f, 1);
        if (lane == 0) prev_l = kNone;
        if (lane == 31) next_f = kNone;
        const bool cont = id_f != kNone && id_f == prev_l;
        // segmented inclusive scan of the last-run partials; a segment head
        // is every lane except a single-run lane continuing its predecessor
        const unsigned heads = __ballot_sync(kFull, multi || !cont);
        const int head = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
        float X = s_l;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float y = __shfl_up_sync(kFull, X, off);
          if (lane - off >= head) X += y;
        }
        const float x_prev = __shfl_up_sync(kFull, X, 1);
        if (multi) sum_of[id_f] += s_f + (cont ? x_prev : 0.f);
        if (id_l != kNone && next_f != id_l) sum_of[id_l] += X;
        __syncwarp();
      }
      __syncwarp();
      for (uint32_t i = lane; i < n_ent; i += 32) {
        const uint32_t v = vb + s_loc[warp][i];
        if (a.acc) {  // source-blocked: this block's partial sum
          atomicAdd(a.acc + v, sum_of[i]);
          continue;
        }
        const float r = a.base + a.damp * sum_of[i];
        a.rank_out[v] = r;
        a.contrib_out[v] = r * a.inv_outdeg[v];
      }
      __syncwarp();
    }
  }
  block_flush<W>(c, a.ctr, kUnreached, nullptr, &s_pref[0][0]);
}

// Hot-set staging for K8 (see pr_pull_kernel): compact the hot sources'
// contributions of this iteration (n_hot random gathers, once per launch).
__global__ void pr_hot_gather_kernel(const uint32_t* __restrict__ hot_vertex, uint32_t n_hot,
                                     const float* __restrict__ contrib, float* hot_contrib) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_hot) hot_contrib[i] = contrib[hot_vertex[i]];
}

// Round aggregate of a world's counters: out = sum of slots [from, to) (the
// exchange all-reduces this one fixed-size entry: ranks may use different
// numbers of counter slots in a pass -- probes, fallbacks -- so the slot
// arrays themselves do not line up across ranks).
__global__ void sum_ctr_slots_kernel(const RunCtr* slots, uint32_t from, uint32_t to,
                                     RunCtr* out) {
  constexpr uint32_t kWords = sizeof(RunCtr) / 8;
  const uint32_t f = threadIdx.x;
  if (f >= kWords) return;
  const unsigned long long* w = reinterpret_cast<const unsigned long long*>(slots);
  unsigned long long s = 0;
  for (uint32_t i = from; i < to; ++i) s += w[size_t(i) * kWords + f];
  reinterpret_cast<unsigned long long*>(out)[f] = s;
}

// Vertices with out-degree >= d (binary search of the hot threshold).
__global__ void count_deg_ge_kernel(const uint32_t* __restrict__ deg, uint32_t n, uint32_t d,
                                    unsigned long long* out) {
  uint32_t k = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    k += deg[v] >= d;
  k = __reduce_add_sync(kFull, k);
  if ((threadIdx.x & 31) == 0 && k) atomicAdd(out, (unsigned long long)k);
}

// Slots of the hot set: every vertex with out-degree >= d (at most cap of
// them by the threshold choice); slot_of[v] = slot (else kUnreached).
__global__ void hot_assign_kernel(const uint32_t* __restrict__ deg, uint32_t n, uint32_t d,
                                  uint32_t cap, unsigned* counter, uint32_t* slot_of,
                                  uint32_t* hot_vertex) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    uint32_t slot = kUnreached;
    if (deg[v] >= d) {
      const uint32_t k = atomicAdd(counter, 1u);
      if (k < cap) {
        slot = k;
        hot_vertex[k] = v;
      }
    }
    slot_of[v] = slot;
  }
}

// Encoded source stream: hot sources -> kHotBit | slot, others unchanged
// (words >= n are alignment padding and are copied as they are).
__global__ void hot_encode_kernel(const uint4* __restrict__ in, uint4* out, uint64_t n4,
                                  const uint32_t* __restrict__ slot_of, uint32_t n) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n4;
       i += uint64_t(gridDim.x) * blockDim.x) {
    uint4 v = __ldcs(in + i);
    uint32_t* e = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (e[k] < n) {
        const uint32_t sl = slot_of[e[k]];
        if (sl != kUnreached) e[k] = kHotBit | sl;
      }
    }
    __stcs(out + i, v);
  }
}

__global__ void pr_hub_finalize_kernel(const uint32_t* hub_vertex, uint32_t n_hubs,
                                       float* hub_sum, float* rank_out, float* contrib_out,
                                       const float* inv_outdeg, float base, float damp) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= n_hubs) return;
  const uint32_t v = hub_vertex[h];
  const float r = base + damp * hub_sum[h];
  rank_out[v] = r;
  contrib_out[v] = r * inv_outdeg[v];
  hub_sum[h] = 0.f;
}

__global__ void pr_init_kernel(float* rank, float* contrib, const float* inv_outdeg, uint32_t n,
                               float init) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    rank[v] = init;
    contrib[v] = init * inv_outdeg[v];
  }
}

__global__ void inv_outdeg_kernel(const unsigned long long* off, uint32_t n, float* inv) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const unsigned long long d = off[v + 1] - off[v];
    inv[v] = d ? 1.0f / (float)d : 0.0f;
  }
}

// ---------------------------------------------------------------------------
// K3: sparse push.  The frontier list (ids with out-degree > 0, ascending)
// and its exclusive out-degree prefix form one flat edge space; each warp
// task is kPushChunk consecutive edges whose first list entry was recorded
// by the compaction (chunk_start), so no search over the prefix is needed.
// ---------------------------------------------------------------------------
// Body shared by the standalone push launch and the persistent sparse loop:
// frontier list / prefix / chunk starts are read through L2 (__ldcg) because
// the persistent loop rewrites them every pass from other SMs.
struct QueueCtr {
  unsigned long long changed, out_edges, log_incorrect;
};

// PredictionLog::record_change (predictor.cpp:107-138) for a vertex that
// changed: a pending "converged" prediction on it was wrong.
__device__ __forceinline__ void log_first_change(uint8_t* logstate, uint32_t v,
                                                 unsigned long long& incorrect) {
  const uint8_t ls = logstate[v];
  if (ls & 8) ++incorrect;
  logstate[v] = 4;  // fails=0, armed, no pending
}

template <int A, bool DET>
__device__ __forceinline__ void push_body(const PushArgs& a, uint32_t gw, uint32_t nw, LaneCtr& c,
                                          uint32_t& lane_min, QueueCtr* qc = nullptr) {
  const int lane = threadIdx.x & 31;
  const unsigned long long cmask = (1ull << a.chunk_shift) - 1;
  const unsigned long long nchunks = (a.total_edges + cmask) >> a.chunk_shift;
  for (unsigned long long ch = gw; ch < nchunks; ch += nw) {
    const unsigned long long q_lo = ch << a.chunk_shift;
    const unsigned long long q_hi = min(q_lo + cmask + 1, a.total_edges);
    uint32_t ad = __ldcg(a.chunk_start + ch);
    for (unsigned long long q0 = q_lo; q0 < q_hi; q0 += 32) {
      // window of up to 32 consecutive frontier entries starting at ad
      const uint32_t wi = ad + lane;
      long long rel = 1ll << 40;  // entry start relative to q0
      uint32_t u = 0, uval = kUnreached;
      unsigned long long ebase = 0;
      if (wi < a.n_list) {
        rel = (long long)__ldcg(a.pref + wi) - (long long)q0;
        u = __ldcg(a.list + wi);
        ebase = a.out_offsets[u];
        uval = DET ? __ldg(a.values + u) : __ldcg(a.values + u);
      }
      const int relc = rel > 64 ? 64 : (int)rel;  // entries before q0 are negative
      const unsigned long long q = q0 + lane;
      const bool qv = q < q_hi;
      uint32_t k = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int b = __shfl_sync(kFull, relc, k + step);
        if (b <= lane) k += step;
      }
      const int my_rel = __shfl_sync(kFull, relc, k);
      const unsigned long long my_base_lo = __shfl_sync(kFull, (unsigned)ebase, k);
      const unsigned long long my_base_hi = __shfl_sync(kFull, (unsigned)(ebase >> 32), k);
      const uint32_t my_val = __shfl_sync(kFull, uval, k);
      uint32_t app_v = 0;
      bool app = false;
      if (qv) {
        const unsigned long long eidx =
            ((my_base_hi << 32) | my_base_lo) + (unsigned long long)((long long)lane - my_rel);
        const uint32_t v = a.out_neighbors[eidx];
        const uint32_t w = (A == kSssp) ? a.out_weights[eidx] : 0u;
        const uint32_t cand = combine<A>(my_val, w);
        c.attempts += 1;
        c.edges += 1;
        if (DET) {
          if (cand < __ldg(a.values + v)) {
            atomicMin(a.next + v, cand);
            a.changed[v] = 1;
          }
        } else if (cand < *(volatile uint32_t*)(a.values + v)) {
          const uint32_t old = atomicMin(a.values + v, cand);
          if (cand < old) {
            c.valid += 1;
            lane_min = min(lane_min, cand);
            if (a.n_peers) peer_min(a.peers, a.n_peers, v, cand);
            if (a.stamp) {
              if (atomicMax(a.stamp + v, a.epoch) < a.epoch) {  // first change this pass
                const uint32_t d = __ldg(a.outdeg + v);
                if (a.logstate) log_first_change(a.logstate, v, qc->log_incorrect);
                qc->changed += 1;
                qc->out_edges += d;
                app = d > 0;
                app_v = v;
              }
            } else {
              a.changed[v] = 1;
            }
          }
        }
      }
      if (!DET && a.stamp) {  // warp-aggregated append to the next frontier queue
        const unsigned m = __ballot_sync(kFull, app);
        if (m) {
          const int leader = __ffs(m) - 1;
          unsigned long long base = 0;
          if (lane == leader) base = atomicAdd(&a.census->push_count, (unsigned long long)__popc(m));
          base = __shfl_sync(kFull, base, leader);
          if (app) a.q_list[base + __popc(m & lanemask_lt())] = app_v;
        }
      }
      // advance the window start to the entry that contains q0 + 32
      int end_rel = __shfl_sync(kFull, relc, (k + 1) & 31);
      if (k == 31) {
        end_rel = 64;
        if (ad + 32 < a.n_list) {
          const long long r = (long long)__ldcg(a.pref + ad + 32) - (long long)q0;
          end_rel = r > 64 ? 64 : (int)r;
        }
      }
      const uint32_t k_last = __shfl_sync(kFull, k, 31);
      const int e_last = __shfl_sync(kFull, end_rel, 31);
      ad += k_last + (e_last <= 32 ? 1u : 0u);
    }
  }
}

__device__ __forceinline__ void push_flush(const PushArgs& a, LaneCtr& c, QueueCtr& qc,
                                           uint32_t lane_min);

template <int A, bool DET>
__global__ void __launch_bounds__(kBlockThreads) push_relax_kernel(PushArgs a) {
  LaneCtr c;
  c.clear();
  QueueCtr qc{0, 0, 0};
  uint32_t lane_min = kUnreached;
  push_body<A, DET>(a, blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5),
                    gridDim.x * kWarpsPerBlock, c, lane_min, &qc);
  push_flush(a, c, qc, lane_min);
}

// Push epilogue shared by the CSR push and the CSC-scan push: queue totals
// and run counters, one atomic per counter per block.
__device__ __forceinline__ void push_flush(const PushArgs& a, LaneCtr& c, QueueCtr& qc,
                                           uint32_t lane_min) {
  __shared__ __align__(16) uint32_t s_scratch[2 * 5 * kWarpsPerBlock + kWarpsPerBlock];
  __shared__ unsigned long long s_q[3][kWarpsPerBlock];
  if (a.stamp) {  // next-frontier size and out-edge volume: one atomic per block
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned long long ch = warp_sum(qc.changed), oe = warp_sum(qc.out_edges),
                             li = warp_sum(qc.log_incorrect);
    if (lane == 0) {
      s_q[0][w] = ch;
      s_q[1][w] = oe;
      s_q[2][w] = li;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      unsigned long long t = 0;
      for (int k = 0; k < kWarpsPerBlock; ++k) t += s_q[threadIdx.x][k];
      unsigned long long* dst = threadIdx.x == 0 ? &a.census->changed
                                : threadIdx.x == 1 ? &a.census->out_edges
                                                   : &a.census->log_incorrect;
      if (t) atomicAdd(dst, t);
    }
  }
  block_flush(c, a.ctr, lane_min, a.census, s_scratch);
}

// ---------------------------------------------------------------------------
// Sparse push over the CSC (the push adjacency not derived yet, DESIGN §4
// "deferred push adjacency"): every in-edge (s -> v) of the resident pages
// whose source is in the frontier bitmap is relaxed exactly as the CSR push
// relaxes s's out-edge (same candidate, same first-change bookkeeping and
// counters); one warp per destination, lanes over its in-edges.
// ---------------------------------------------------------------------------
constexpr uint32_t kScanFilterWords = 4096;     // 16 KB: 131072 hashed bits
constexpr uint32_t kScanFilterMaxList = 16384;  // larger frontiers: global bitmap only

template <int A>
__global__ void __launch_bounds__(kBlockThreads) push_scan_kernel(PushArgs a,
                                                                  const PageDesc* __restrict__ pages,
                                                                  uint32_t n_pages,
                                                                  const uint32_t* __restrict__ fbits) {
  // shared-memory prefilter of the frontier (hashed bitmap): almost every
  // source is rejected without touching the global bitmap
  __shared__ uint32_t s_filt[kScanFilterWords];
  const bool filt = a.n_list <= kScanFilterMaxList;
  for (uint32_t i = threadIdx.x; i < kScanFilterWords; i += blockDim.x) s_filt[i] = filt ? 0u : ~0u;
  __syncthreads();
  if (filt)
    for (uint32_t i = threadIdx.x; i < a.n_list; i += blockDim.x) {
      const uint32_t h = a.list[i] & (kScanFilterWords * 32 - 1);
      atomicOr(s_filt + (h >> 5), 1u << (h & 31));
    }
  __syncthreads();
  LaneCtr c;
  c.clear();
  QueueCtr qc{0, 0, 0};
  uint32_t lane_min = kUnreached;
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  for (uint32_t p = 0; p < n_pages; ++p) {
    const PageDesc pd = pages[p];
    // flat sweep over the page's in-edges, 32 per warp step (streaming
    // loads); the destination of the rare frontier edge is found by a
    // binary search of the page offsets
    for (uint64_t e0 = gw * 128; e0 < pd.edge_count; e0 += nw * 128) {
      // 4 consecutive edges per lane (one 16-byte load; page arrays are
      // padded to 8 edges), then one edge per inner step
      const uint64_t eb = e0 + uint64_t(lane) * 4;
      uint4 s4 = make_uint4(0, 0, 0, 0);
      if (eb < pd.edge_count) s4 = __ldcs(reinterpret_cast<const uint4*>(pd.src + eb));
      const uint32_t sv4[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
      const uint64_t e = eb + k;
      uint32_t app_v = 0;
      bool app = false;
      if (e < pd.edge_count) {
        const uint32_t s = sv4[k];
        const uint32_t h = s & (kScanFilterWords * 32 - 1);
        if ((s_filt[h >> 5] >> (h & 31) & 1u) && (fbits[s >> 5] >> (s & 31) & 1u)) {
          uint32_t lo = 0, hi = pd.range;  // last i with offs[i] <= e
          while (lo + 1 < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (pd.offs[mid] <= e) lo = mid;
            else hi = mid;
          }
          const uint32_t v = pd.vertex_begin + lo;
          const uint32_t w = (A == kSssp) ? pd.w[e] : 0u;
          const uint32_t cand = combine<A>(__ldcg(a.values + s), w);
          c.attempts += 1;
          c.edges += 1;
          if (cand < *(volatile uint32_t*)(a.values + v)) {
            const uint32_t old = atomicMin(a.values + v, cand);
            if (cand < old) {
              c.valid += 1;
              lane_min = min(lane_min, cand);
              if (a.stamp) {
                if (atomicMax(a.stamp + v, a.epoch) < a.epoch) {
                  const uint32_t d = __ldg(a.outdeg + v);
                  if (a.logstate) log_first_change(a.logstate, v, qc.log_incorrect);
                  qc.changed += 1;
                  qc.out_edges += d;
                  app = d > 0;
                  app_v = v;
                }
              } else {
                a.changed[v] = 1;
              }
            }
          }
        }
      }
      if (a.stamp) {
        const unsigned m = __ballot_sync(kFull, app);
        if (m) {
          const int leader = __ffs(m) - 1;
          unsigned long long base = 0;
          if (lane == leader) base = atomicAdd(&a.census->push_count, (unsigned long long)__popc(m));
          base = __shfl_sync(kFull, base, leader);
          if (app) a.q_list[base + __popc(m & lanemask_lt())] = app_v;
        }
      }
      }
    }
  }
  push_flush(a, c, qc, lane_min);
}

__global__ void set_bits_kernel(const uint32_t* __restrict__ list, uint32_t q, uint32_t* bits) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < q; i += gridDim.x * blockDim.x)
    atomicOr(bits + (list[i] >> 5), 1u << (list[i] & 31));
}

// Frontier queue -> push inputs: exclusive out-degree prefix of the queue
// and the first queue entry of every kPushChunk-edge chunk.
__global__ void queue_degrees_kernel(const uint32_t* __restrict__ list, uint32_t q,
                                     const uint32_t* __restrict__ outdeg, unsigned long long* deg) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= q; i += gridDim.x * blockDim.x)
    deg[i] = i < q ? outdeg[list[i]] : 0ull;
}

// One thread per queue entry, or (`per_warp`: few entries with many chunks,
// e.g. a hub source) one warp per entry with the lanes striding its chunks.
__global__ void queue_chunks_kernel(const unsigned long long* __restrict__ pref, uint32_t q,
                                    uint32_t shift, int per_warp, uint32_t* chunk_start) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t nt = uint64_t(gridDim.x) * blockDim.x;
  const uint32_t step = per_warp ? 32u : 1u;
  const uint32_t sub = per_warp ? uint32_t(tid & 31) : 0u;
  const unsigned long long cm = (1ull << shift) - 1;
  for (uint64_t i = per_warp ? tid >> 5 : tid; i < q; i += per_warp ? nt >> 5 : nt) {
    const unsigned long long lo = pref[i], hi = pref[i + 1];
    for (unsigned long long ch = ((lo + cm) >> shift) + sub; ch < ((hi + cm) >> shift); ch += step)
      chunk_start[ch] = uint32_t(i);
  }
}

__global__ void push_commit_kernel(uint32_t* __restrict__ values, const uint32_t* __restrict__ next,
                                   const uint8_t* __restrict__ changed, uint32_t n, RunCtr* ctr,
                                   Census* c) {
  unsigned long long cnt = 0;
  uint32_t mn = kUnreached;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (changed[v]) {
      const uint32_t nv = next[v];
      if (nv < values[v]) {
        values[v] = nv;
        ++cnt;
        mn = min(mn, nv);
      }
    }
  }
  cnt = warp_sum(cnt);
  mn = warp_min(mn);
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(&ctr->valid, cnt);
    if (mn != kUnreached) atomicMin(&c->min_changed, mn);
  }
}

// ---------------------------------------------------------------------------
// K4/K5 census: one pass over the per-vertex byte arrays.  Weak DFA step
// (predictor.cpp:18-41) for dense passes, status reset for recovery
// (engine.cpp:197-202), PredictionLog bookkeeping (predictor.cpp:107-138)
// folded into one byte per vertex, status histogram of the NEXT pass,
// frontier size and out-edge volume (density_switch input, engine.cpp:56-61).
// logstate byte: bits0-1 consecutive fails (saturated at 3), bit2 armed,
// bit3 one pending (not yet falsified) converged-prediction event.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint8_t log_change(uint8_t ls, unsigned long long& incorrect) {
  if (ls & 8) ++incorrect;
  return 4;  // fails=0, armed, no pending
}
__device__ __forceinline__ uint8_t log_attempt(uint8_t ls, bool changed,
                                               unsigned long long& events,
                                               unsigned long long& incorrect) {
  if (changed) return log_change(ls, incorrect);
  uint8_t fails = ls & 3;
  if (fails < 3) ++fails;
  uint8_t out = (ls & ~3) | fails;
  if ((ls & 4) && fails == 2) {
    ++events;
    out = (out & ~4) | 8;
  }
  return out;
}

// Census body (grid-stride over 4096-vertex chunks, 256 threads); per-pass
// totals go to cz_pass, run-long accumulators (prediction log) to cz_run.
// ST: the weak predictor's status/log bytes are present (13 partials);
// otherwise only the frontier counts (5 partials, fewer live registers).
template <bool ST>
__device__ __forceinline__ void census_body(uint32_t n, const uint8_t* changed, uint8_t* status,
                                            uint8_t* logstate, const uint32_t* __restrict__ outdeg,
                                            int pass_kind, uint32_t own_lo, uint32_t own_hi,
                                            uint32_t* blk_cnt, unsigned long long* blk_edges,
                                            Census* cz_pass, Census* cz_run, uint32_t bid,
                                            uint32_t nblk) {
  // grid-stride over 4096-vertex chunks; per-chunk (count, edges) for the
  // compaction scan, run totals reduced once per block (few global atomics)
  __shared__ unsigned long long s_chunk[2][8];
  constexpr int kParts = ST ? kCensusParts : 5;
  __shared__ unsigned long long s_tot[kParts][8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t nchunks = (n + kCensusBlockVerts - 1) / kCensusBlockVerts;
  unsigned long long tot[kCensusParts];
#pragma unroll
  for (int k = 0; k < kCensusParts; ++k) tot[k] = 0;
  if (!ST) status = logstate = nullptr;
  for (uint32_t ch = bid; ch < nchunks; ch += nblk) {
    const uint32_t v0 = ch * kCensusBlockVerts + threadIdx.x * 16;
    unsigned long long own_push = 0, own_edges = 0;
    if (v0 < n) {
      const uint4 cw = __ldcg(reinterpret_cast<const uint4*>(changed + v0));
      const uint8_t* cb = reinterpret_cast<const uint8_t*>(&cw);
      const uint32_t cwv[4] = {cw.x, cw.y, cw.z, cw.w};
      uint4 sw{}, lw{};
      if (status) sw = __ldcg(reinterpret_cast<const uint4*>(status + v0));
      if (logstate) lw = __ldcg(reinterpret_cast<const uint4*>(logstate + v0));
      uint8_t* sb = reinterpret_cast<uint8_t*>(&sw);
      uint8_t* lb = reinterpret_cast<uint8_t*>(&lw);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // out-degrees only of 4-vertex groups holding a changed vertex
        uint4 d4 = make_uint4(0, 0, 0, 0);
        if (outdeg && cwv[k]) d4 = reinterpret_cast<const uint4*>(outdeg + v0)[k];
        const uint32_t dk[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = 4 * k + jj;
          const uint32_t v = v0 + j;
          if (v >= n) break;
          const bool ch_ = cb[j] != 0;
          if (ch_) {
            const unsigned long long d = dk[jj];
            tot[0] += 1;
            tot[1] += d > 0;
            tot[2] += d;
            if (v >= own_lo && v < own_hi) {
              own_edges += d;
              own_push += d > 0;
            }
          }
          if (status) {
            uint8_t st = sb[j];
            if (pass_kind == kPassDense) {
              const bool attempt_state = (st == 0 || st == 1 || st == 5);
              if (attempt_state) {
                if (logstate) lb[j] = log_attempt(lb[j], ch_, tot[5], tot[6]);
                st = ch_ ? 0 : (st == 0 ? 5 : (st == 5 ? 3 : 4));
              } else {
                st = (st == 3) ? 2 : (st == 2 ? 1 : 3);
              }
            } else if (ch_ && pass_kind != kPassInit) {
              if (pass_kind == kPassRecovery) st = 0;
              if (logstate) lb[j] = log_change(lb[j], tot[6]);
            }
            sb[j] = st;
            switch (st) {
              case 0: tot[7]++; break;
              case 1: tot[8]++; break;
              case 2: tot[9]++; break;
              case 3: tot[10]++; break;
              case 4: tot[11]++; break;
              default: tot[12]++; break;
            }
          }
        }
      }
      if (status) *reinterpret_cast<uint4*>(status + v0) = sw;
      if (logstate) *reinterpret_cast<uint4*>(logstate + v0) = lw;
    }
    tot[3] += own_push;
    tot[4] += own_edges;
    own_push = warp_sum(own_push);
    own_edges = warp_sum(own_edges);
    if (lane == 0) {
      s_chunk[0][w] = own_push;
      s_chunk[1][w] = own_edges;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long a = 0, b = 0;
      for (int i = 0; i < 8; ++i) {
        a += s_chunk[0][i];
        b += s_chunk[1][i];
      }
      blk_cnt[ch] = (uint32_t)a;
      blk_edges[ch] = b;
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < kParts; ++k) {
    const unsigned long long x = warp_sum(tot[k]);
    if (lane == 0) s_tot[k][w] = x;
  }
  __syncthreads();
  if (threadIdx.x < kParts) {
    unsigned long long a = 0;
    for (int i = 0; i < 8; ++i) a += s_tot[threadIdx.x][i];
    if (a) {
      unsigned long long* dst;
      switch (threadIdx.x) {
        case 0: dst = &cz_pass->changed; break;
        case 1: dst = &cz_pass->push_count; break;
        case 2: dst = &cz_pass->out_edges; break;
        case 3: dst = &cz_pass->own_push; break;
        case 4: dst = &cz_pass->own_edges; break;
        case 5: dst = &cz_run->log_events; break;
        case 6: dst = &cz_run->log_incorrect; break;
        default: dst = &cz_pass->status_hist[threadIdx.x - 7]; break;
      }
      atomicAdd(dst, a);
    }
  }
  __syncthreads();  // s_tot is reused by the next call in a persistent loop
}

template <bool ST>
__global__ void __launch_bounds__(256, ST ? 1 : 8) census_kernel(uint32_t n, const uint8_t* __restrict__ changed,
                                                     uint8_t* status, uint8_t* logstate,
                                                     const uint32_t* __restrict__ outdeg,
                                                     int pass_kind, uint32_t own_lo, uint32_t own_hi,
                                                     uint32_t* blk_cnt,
                                                     unsigned long long* blk_edges, Census* cz,
                                                     Publish pub) {
  census_body<ST>(n, changed, status, logstate, outdeg, pass_kind, own_lo, own_hi, blk_cnt,
                  blk_edges, cz, cz, blockIdx.x, gridDim.x);
  if (!pub.done) return;
  // the last block to finish publishes the pass's census and run counters
  // into the mapped pinned buffers (no separate publish launch per pass)
  __shared__ bool s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(pub.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const uint32_t words = sizeof(Census) / 4;
  const uint32_t cwords = pub.n_ctr * uint32_t(sizeof(RunCtr) / 8);
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
    reinterpret_cast<uint32_t*>(pub.cz_host)[i] = __ldcg(reinterpret_cast<const uint32_t*>(cz) + i);
  for (uint32_t i = threadIdx.x; i < cwords; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(pub.ctr_host)[i] =
        __ldcg(reinterpret_cast<const unsigned long long*>(pub.ctr) + i);
  if (pub.seq_host) {  // the host spins on this word instead of a stream sync
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(pub.seq_host) = pub.seq;
  }
  if (threadIdx.x == 0) *pub.done = 0;  // ready for the next pass
}

// Exclusive scan of the per-chunk (count, edges) pairs by ONE block (any
// blockDim that is a multiple of 32).
__device__ __forceinline__ void scan_body(uint32_t nb, uint32_t* cnt, unsigned long long* edges) {
  __shared__ uint32_t s_c[32];
  __shared__ unsigned long long s_e[32];
  __shared__ uint32_t carry_c;
  __shared__ unsigned long long carry_e;
  if (threadIdx.x == 0) {
    carry_c = 0;
    carry_e = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (uint32_t base = 0; base < nb; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t xc = i < nb ? __ldcg(cnt + i) : 0u;
    const unsigned long long xe = i < nb ? __ldcg(edges + i) : 0ull;
    uint32_t ic = warp_incl_scan(xc, lane);
    unsigned long long ie = warp_incl_scan(xe, lane);
    if (lane == 31) {
      s_c[w] = ic;
      s_e[w] = ie;
    }
    __syncthreads();
    if (w == 0) {
      uint32_t tc = lane < nwarps ? s_c[lane] : 0u;
      unsigned long long te = lane < nwarps ? s_e[lane] : 0ull;
      uint32_t sc = warp_incl_scan(tc, lane);
      unsigned long long se = warp_incl_scan(te, lane);
      s_c[lane] = sc - tc;
      s_e[lane] = se - te;
    }
    __syncthreads();
    const uint32_t oc = carry_c + s_c[w] + ic - xc;
    const unsigned long long oe = carry_e + s_e[w] + ie - xe;
    __syncthreads();
    if (i < nb) {
      cnt[i] = oc;
      edges[i] = oe;
    }
    if (threadIdx.x == blockDim.x - 1) {
      carry_c = oc + xc;
      carry_e = oe + xe;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) scan_blocks_kernel(uint32_t nb, uint32_t* cnt,
                                                           unsigned long long* edges) {
  scan_body(nb, cnt, edges);
}

// Ordered compaction of changed vertices with out-degree > 0 into the push
// list, with their exclusive out-degree prefix and push-chunk starts; clears
// the changed flags for the next pass.
__device__ __forceinline__ void compact_chunk(uint32_t chunk, uint32_t n, uint32_t own_lo,
                                              uint32_t own_hi, uint8_t* changed,
                                              const uint32_t* __restrict__ outdeg,
                                              const uint32_t* blk_off,
                                              const unsigned long long* blk_eoff, uint32_t* list,
                                              unsigned long long* pref, uint32_t* chunk_start,
                                              uint32_t shift) {
  __shared__ uint32_t s_c[8];
  __shared__ unsigned long long s_e[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t v0 = chunk * kCensusBlockVerts + threadIdx.x * 16;
  uint4 cw = make_uint4(0, 0, 0, 0);
  if (v0 < n) cw = __ldcg(reinterpret_cast<const uint4*>(changed + v0));
  const uint8_t* cb = reinterpret_cast<const uint8_t*>(&cw);
  uint32_t cnt = 0;
  unsigned long long edges = 0;
  uint32_t deg[16];
  const uint32_t cwv[4] = {cw.x, cw.y, cw.z, cw.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    // out-degrees only of 4-vertex groups holding a changed vertex
    uint4 d4 = make_uint4(0, 0, 0, 0);
    if (cwv[k]) d4 = reinterpret_cast<const uint4*>(outdeg + v0)[k];
    const uint32_t dk[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      const int j = 4 * k + jj;
      const uint32_t v = v0 + j;
      deg[j] = (v < n && cb[j] && v >= own_lo && v < own_hi) ? dk[jj] : 0u;
      cnt += deg[j] > 0;
      edges += deg[j];
    }
  }
  const uint32_t ic = warp_incl_scan(cnt, lane);
  const unsigned long long ie = warp_incl_scan(edges, lane);
  if (lane == 31) {
    s_c[w] = ic;
    s_e[w] = ie;
  }
  __syncthreads();
  uint32_t wc = 0;
  unsigned long long we = 0;
  for (int i = 0; i < w; ++i) {
    wc += s_c[i];
    we += s_e[i];
  }
  uint32_t pos = __ldcg(blk_off + chunk) + wc + ic - cnt;
  unsigned long long ep = __ldcg(blk_eoff + chunk) + we + ie - edges;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (deg[j] > 0) {
      list[pos] = v0 + j;
      pref[pos] = ep;
      const unsigned long long cm = (1ull << shift) - 1;
      const unsigned long long c_lo = (ep + cm) >> shift;
      const unsigned long long c_hi = (ep + deg[j] + cm) >> shift;
      for (unsigned long long ch = c_lo; ch < c_hi; ++ch) chunk_start[ch] = pos;
      ++pos;
      ep += deg[j];
    }
  }
  if (v0 < n && (cw.x | cw.y | cw.z | cw.w))
    *reinterpret_cast<uint4*>(changed + v0) = make_uint4(0, 0, 0, 0);
  __syncthreads();  // s_c/s_e reused by the next chunk
}

__global__ void __launch_bounds__(256) compact_kernel(uint32_t n, uint32_t own_lo, uint32_t own_hi,
                                                      uint8_t* changed,
                                                      const uint32_t* __restrict__ outdeg,
                                                      const uint32_t* __restrict__ blk_off,
                                                      const unsigned long long* __restrict__ blk_eoff,
                                                      uint32_t* list, unsigned long long* pref,
                                                      uint32_t* chunk_start, uint32_t shift) {
  compact_chunk(blockIdx.x, n, own_lo, own_hi, changed, outdeg, blk_off, blk_eoff, list, pref,
                chunk_start, shift);
}


// ---------------------------------------------------------------------------
// K6: strong CC threshold.  The reference keeps exact per-label counts and
// diffs them against the previous refresh (predictor.cpp:55-87).  The net
// change of label L since the refresh is  #{v: cur_v = L} - #{v: snap_v = L},
// so it is computed from (snapshot, current) pairs of moved vertices, with
// match_any aggregation of the hot label, and the minimum label with a
// nonzero net change is s.
// ---------------------------------------------------------------------------
__global__ void init_values_kernel(int algo, uint32_t source, uint32_t n, uint32_t* values) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    values[v] = (algo == kCc) ? v : (v == source ? 0u : kUnreached);
}

__global__ void fill_u32_kernel(uint32_t* p, uint32_t n, uint32_t x) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = x;
}

template <int A>
__global__ void verify_kernel(uint32_t lo, uint32_t n, const unsigned long long* __restrict__ off,
                              const uint32_t* __restrict__ nbr, const uint32_t* __restrict__ w,
                              const uint32_t* __restrict__ values, unsigned long long* viol) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long bad = 0;
  for (uint32_t u = lo + gw; u < n; u += nw) {
    const uint32_t vu = values[u];
    for (unsigned long long e = off[u] + lane; e < off[u + 1]; e += 32) {
      const uint32_t cand = combine<A>(vu, A == kSssp ? w[e] : 0u);
      if (cand < values[nbr[e]]) ++bad;
    }
  }
  bad = warp_sum(bad);
  if (lane == 0 && bad) atomicAdd(viol, bad);
}

inline int grid_for(unsigned long long work, int block, int cap = 148 * 16) {
  unsigned long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (unsigned long long)cap) g = cap;
  return (int)g;
}

__global__ void mark_changed_kernel(uint32_t n, const uint32_t* __restrict__ values,
                                    const uint32_t* __restrict__ snap, uint8_t* changed) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (values[v] < snap[v]) changed[v] = 1;
}

__global__ void set_page_desc_kernel(PageDesc* d, uint32_t page, const uint32_t* offs,
                                     const uint32_t* src, const uint32_t* w) {
  d[page].offs = offs;
  d[page].src = src;
  d[page].w = w;
}

}  // namespace

void launch_mark_changed(uint32_t n, const uint32_t* values, const uint32_t* snap,
                         uint8_t* changed, cudaStream_t s) {
  if (!n) return;
  note_launch();
  mark_changed_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, values, snap, changed);
}

void launch_set_page_desc(PageDesc* d, uint32_t page, const uint32_t* offs, const uint32_t* src,
                          const uint32_t* w, cudaStream_t s) {
  note_launch();
  set_page_desc_kernel<<<1, 1, 0, s>>>(d, page, offs, src, w);
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <int A, int G, bool D>
static void pull_dispatch3(const PullArgs& a, int grid, cudaStream_t s) {
  note_launch();
  if (A != kSssp && !D && kScanList && a.list)
    pull_relax_kernel<A, G, D, A != kSssp && !D><<<grid, kBlockThreads, 0, s>>>(a);
  else
    pull_relax_kernel<A, G, D, false><<<grid, kBlockThreads, 0, s>>>(a);
}
template <int A, int G>
static void pull_dispatch2(bool det, const PullArgs& a, int grid, cudaStream_t s) {
  if (det) pull_dispatch3<A, G, true>(a, grid, s);
  else pull_dispatch3<A, G, false>(a, grid, s);
}
template <int A>
static void pull_dispatch1(int gate, bool det, const PullArgs& a, int grid, cudaStream_t s) {
  switch (gate) {
    case kGateStrong: pull_dispatch2<A, kGateStrong>(det, a, grid, s); break;
    case kGateWeak: pull_dispatch2<A, kGateWeak>(det, a, grid, s); break;
    default: pull_dispatch2<A, kGateOff>(det, a, grid, s); break;
  }
}

void launch_pull(int algo, int gate, bool det, const PullArgs& a, int grid, cudaStream_t s) {
  switch (algo) {
    case kBfs: pull_dispatch1<kBfs>(gate, det, a, grid, s); break;
    case kCc: pull_dispatch1<kCc>(gate, det, a, grid, s); break;
    default: pull_dispatch1<kSssp>(gate, det, a, grid, s); break;
  }
}

template <int A, int G>
static bool reentry_launch(const PullArgs& a, const ReentryArgs& r, int grid, cudaStream_t s) {
  static int max_grid = -1;
  if (max_grid < 0) {
    int nb = 0, dev = 0, sms = 0;
    SR_CUDA(cudaGetDevice(&dev));
    SR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    SR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pull_reentry_kernel<A, G>,
                                                          kBlockThreads, 0));
    max_grid = nb * sms;
  }
  if (max_grid < 1) return false;
  grid = std::min(grid, max_grid);  // persistent warps: any grid works, all co-resident
  PullArgs aa = a;
  ReentryArgs rr = r;
  void* args[] = {&aa, &rr};
  SR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(pull_reentry_kernel<A, G>),
                                      dim3(grid), dim3(kBlockThreads), args, 0, s));
  note_launch();
  return true;
}

template <int A>
static bool reentry_dispatch(int gate, const PullArgs& a, const ReentryArgs& r, int grid,
                             cudaStream_t s) {
  switch (gate) {
    case kGateStrong: return reentry_launch<A, kGateStrong>(a, r, grid, s);
    case kGateWeak: return reentry_launch<A, kGateWeak>(a, r, grid, s);
    default: return reentry_launch<A, kGateOff>(a, r, grid, s);
  }
}

bool launch_pull_reentry(int algo, int gate, const PullArgs& a, const ReentryArgs& r, int grid,
                         cudaStream_t s) {
  switch (algo) {
    case kBfs: return reentry_dispatch<kBfs>(gate, a, r, grid, s);
    case kCc: return reentry_dispatch<kCc>(gate, a, r, grid, s);
    default: return reentry_dispatch<kSssp>(gate, a, r, grid, s);
  }
}

int pull_blocks_per_sm(int algo, int gate, bool det) {
  int nb = 0;
  (void)gate;
  (void)det;
  if (algo == kSssp)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pull_relax_kernel<kSssp, kGateOff, false, false>,
                                                  kBlockThreads, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pull_relax_kernel<kBfs, kGateOff, false, false>,
                                                  kBlockThreads, 0);
  return nb > 0 ? nb : 1;
}

void launch_commit(uint32_t* values, const uint32_t* next, uint32_t lo, uint32_t hi,
                   cudaStream_t s) {
  if (hi <= lo) return;
  note_launch();
  commit_kernel<<<grid_for(hi - lo, 256), 256, 0, s>>>(values, next, lo, hi);
}

// Hot-staged K8: warps per block (SERAPH_PR_HOT_WARPS = 8 | 16 | 32; A/B knob)
int pr_hot_warps() {
  static int w = [] {
    const char* e = std::getenv("SERAPH_PR_HOT_WARPS");
    const int v = e ? std::atoi(e) : kHotWarps;
    return (v == 8 || v == 16 || v == 32) ? v : kHotWarps;
  }();
  return w;
}

template <int W>
static void set_hot_attr() {
  static bool attr = false;
  if (!attr) {
    SR_CUDA(cudaFuncSetAttribute(pr_pull_kernel<true, W>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kHotSmemBytes - W * 1536)));
    attr = true;
  }
}

template <int W>
static int hot_occupancy(size_t dyn) {
  set_hot_attr<W>();
  int b = 0;
  SR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, pr_pull_kernel<true, W>, W * 32, dyn));
  return b;
}

// Resident blocks per SM of the hot-staged K8 with an n_hot-entry table.
int pr_hot_blocks_per_sm(uint32_t n_hot) {
  const size_t dyn = size_t((n_hot + 3) & ~3u) * 4;
  int b = 1;
  switch (pr_hot_warps()) {
    case 8: b = hot_occupancy<8>(dyn); break;
    case 32: b = hot_occupancy<32>(dyn); break;
    default: b = hot_occupancy<16>(dyn);
  }
  return std::max(b, 1);
}

// Largest table the selected block shape can hold.
uint32_t pr_hot_table_max() {
  return uint32_t((kHotSmemBytes - pr_hot_warps() * 1536) / 4) & ~255u;
}

template <int W>
static void launch_pr_hot_w(const PrArgs& a, int grid, size_t dyn, cudaStream_t s) {
  set_hot_attr<W>();
  pr_pull_kernel<true, W><<<grid, W * 32, dyn, s>>>(a);
}

void launch_pr_pull(const PrArgs& a, int grid, cudaStream_t s) {
  note_launch();
  if (a.hot_contrib) {
    const size_t dyn = size_t((a.n_hot + 3) & ~3u) * 4;
    switch (pr_hot_warps()) {
      case 8: launch_pr_hot_w<8>(a, grid, dyn, s); break;
      case 32: launch_pr_hot_w<32>(a, grid, dyn, s); break;
      default: launch_pr_hot_w<16>(a, grid, dyn, s);
    }
    return;
  }
  pr_pull_kernel<false, kWarpsPerBlock><<<grid, kBlockThreads, 0, s>>>(a);
}

void launch_pr_hot_gather(const uint32_t* hot_vertex, uint32_t n_hot, const float* contrib,
                          float* hot_contrib, cudaStream_t s) {
  if (!n_hot) return;
  note_launch();
  pr_hot_gather_kernel<<<(n_hot + 255) / 256, 256, 0, s>>>(hot_vertex, n_hot, contrib,
                                                           hot_contrib);
}

void launch_sum_ctr_slots(const RunCtr* slots, uint32_t from, uint32_t to, RunCtr* out,
                          cudaStream_t s) {
  note_launch();
  sum_ctr_slots_kernel<<<1, 32, 0, s>>>(slots, from, to, out);
}

void launch_count_deg_ge(const uint32_t* deg, uint32_t n, uint32_t d, unsigned long long* out,
                         cudaStream_t s) {
  note_launch();
  count_deg_ge_kernel<<<grid_for(n, 256), 256, 0, s>>>(deg, n, d, out);
}

void launch_hot_assign(const uint32_t* deg, uint32_t n, uint32_t d, uint32_t cap,
                       unsigned* counter, uint32_t* slot_of, uint32_t* hot_vertex, cudaStream_t s) {
  note_launch();
  hot_assign_kernel<<<grid_for(n, 256), 256, 0, s>>>(deg, n, d, cap, counter, slot_of, hot_vertex);
}

void launch_hot_encode(const uint32_t* in, uint32_t* out, uint64_t words, const uint32_t* slot_of,
                       uint32_t n, cudaStream_t s) {
  if (!words) return;
  note_launch();
  const uint64_t n4 = (words + 3) / 4;
  hot_encode_kernel<<<grid_for(n4, 256), 256, 0, s>>>(
      reinterpret_cast<const uint4*>(in), reinterpret_cast<uint4*>(out), n4, slot_of, n);
}

void launch_pr_hub_finalize(const uint32_t* hub_vertex, uint32_t n_hubs, float* hub_sum,
                            float* rank_out, float* contrib_out, const float* inv_outdeg,
                            float base, float damp, cudaStream_t s) {
  if (!n_hubs) return;
  note_launch();
  pr_hub_finalize_kernel<<<(n_hubs + 255) / 256, 256, 0, s>>>(hub_vertex, n_hubs, hub_sum,
                                                              rank_out, contrib_out, inv_outdeg,
                                                              base, damp);
}

void launch_pr_init(float* rank, float* contrib, const float* inv_outdeg, uint32_t n, float init,
                    cudaStream_t s) {
  note_launch();
  pr_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(rank, contrib, inv_outdeg, n, init);
}

void launch_inv_outdeg(const unsigned long long* out_offsets, uint32_t n, float* inv,
                       cudaStream_t s) {
  note_launch();
  inv_outdeg_kernel<<<grid_for(n, 256), 256, 0, s>>>(out_offsets, n, inv);
}

size_t queue_prep_temp_bytes(uint32_t max_q) {
  size_t tb = 0;
  SR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (unsigned long long*)nullptr,
                                        (unsigned long long*)nullptr, uint64_t(max_q) + 1));
  return tb;
}

// ---------------------------------------------------------------------------
// Small-frontier tail: consecutive sparse passes (sparse_push_pass,
// engine.cpp:63-93) in ONE block.  Per pass: block scan of the queue's
// out-degrees into shared memory, edges strided over the 1024 threads (entry
// by binary search over the prefix), asynchronous atomicMin relaxations, and
// the next queue built from first-time improvements (epoch stamps) with a
// shared cursor.  Same decisions as the host loop: stop when nothing
// changed, when the next frontier's out-edges exceed the density threshold
// (the host runs the dense pass), or when it outgrows one block.
// ---------------------------------------------------------------------------
template <int A>
__global__ void __launch_bounds__(1024) tail_loop_kernel(TailArgs t) {
  __shared__ uint32_t s_pref[kTailMaxQueue + 1];
  __shared__ uint32_t s_wsum[32];
  __shared__ unsigned long long s_red[5][32];
  __shared__ uint32_t s_qn;
  __shared__ unsigned s_stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* cur = t.list;
  uint32_t* nxt = t.list2;
  uint32_t q = t.q0;
  uint32_t lane_min = kUnreached;
  uint32_t pass = 0;
  unsigned reason = 3;
  for (; pass < t.max_passes; ++pass) {
    // exclusive out-degree prefix of the queue (q <= kTailMaxQueue: 8 per thread)
    constexpr int kPer = kTailMaxQueue / 1024;
    uint32_t d[kPer], loc = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t i = tid * kPer + k;
      d[k] = i < q ? __ldg(t.outdeg + cur[i]) : 0u;
      loc += d[k];
    }
    const uint32_t incl = warp_incl_scan(loc, lane);
    if (lane == 31) s_wsum[warp] = incl;
    if (tid == 0) s_qn = 0;
    __syncthreads();
    if (warp == 0) {
      const uint32_t x = s_wsum[lane];
      s_wsum[lane] = warp_incl_scan(x, lane) - x;
    }
    __syncthreads();
    uint32_t run = s_wsum[warp] + incl - loc;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t i = tid * kPer + k;
      if (i <= q) s_pref[i] = run;
      run += d[k];
    }
    if (tid == int(blockDim.x) - 1 && q == kTailMaxQueue) s_pref[kTailMaxQueue] = run;
    __syncthreads();
    const uint32_t total = s_pref[q];
    // relax every out-edge of the queue
    unsigned long long valid = 0, changed = 0, out_next = 0, log_inc = 0;
    const uint32_t epoch = t.epoch0 + pass;
    for (uint32_t e = tid; e < total; e += blockDim.x) {
      uint32_t lo = 0, hi = q - 1;  // last entry with s_pref <= e
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_pref[mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      const uint32_t u = cur[lo];
      const unsigned long long ei = t.out_offsets[u] + (e - s_pref[lo]);
      const uint32_t v = t.out_neighbors[ei];
      const uint32_t w = (A == kSssp) ? t.out_weights[ei] : 0u;
      const uint32_t cand = combine<A>(__ldcg(t.values + u), w);
      if (cand < *(volatile uint32_t*)(t.values + v)) {
        const uint32_t old = atomicMin(t.values + v, cand);
        if (cand < old) {
          valid += 1;
          lane_min = min(lane_min, cand);
          if (atomicMax(t.stamp + v, epoch) < epoch) {
            const uint32_t dv = __ldg(t.outdeg + v);
            if (t.logstate) log_first_change(t.logstate, v, log_inc);
            changed += 1;
            out_next += dv;
            if (dv) nxt[atomicAdd(&s_qn, 1u)] = v;  // the scratch queue holds |V|
          }
        }
      }
    }
    const unsigned long long vals[4] = {warp_sum(valid), warp_sum(changed), warp_sum(out_next),
                                        warp_sum(log_inc)};
    if (lane == 0)
      for (int k = 0; k < 4; ++k) s_red[k][warp] = vals[k];
    __syncthreads();
    if (tid == 0) {
      unsigned long long tot[4] = {0, 0, 0, 0};
      for (int w = 0; w < int(blockDim.x >> 5); ++w)
        for (int k = 0; k < 4; ++k) tot[k] += s_red[k][w];
      if (tot[3]) atomicAdd(&t.census->log_incorrect, tot[3]);
      TailRecord r;
      r.edges = total;
      r.valid = tot[0];
      r.changed = tot[1];
      r.out_edges = tot[2];
      r.queued = s_qn;
      t.rec[pass] = r;
      unsigned stop = 0xffffffffu;
      if (tot[1] == 0) stop = 0;
      else if (!t.force_sparse && double(tot[2]) > t.dense_threshold) stop = 1;
      else if (s_qn > kTailMaxQueue || tot[2] > kTailMaxEdges) stop = 2;
      s_stop = stop;
    }
    __syncthreads();
    const unsigned stop = s_stop;
    q = s_qn;
    uint32_t* tmp = cur;
    cur = nxt;
    nxt = tmp;
    __syncthreads();  // s_pref / s_qn reuse
    if (stop != 0xffffffffu) {
      reason = stop;
      ++pass;
      break;
    }
  }
  // the final queue (the next frontier) back in t.list for the host path
  if (cur != t.list)
    for (uint32_t i = tid; i < q; i += blockDim.x) t.list[i] = cur[i];
  lane_min = warp_min(lane_min);
  if (lane == 0 && lane_min != kUnreached) atomicMin(&t.census->min_changed, lane_min);
  // pinned results: the per-pass records and the reason first, `passes` last
  // behind a system fence (the host spins on it, Engine::do_sparse_tail)
  __threadfence_system();
  __syncthreads();
  if (tid == 0) {
    t.res->reason = reason;
    __threadfence_system();
    *reinterpret_cast<volatile uint32_t*>(&t.res->passes) = pass;
  }
}

void launch_tail_loop(int algo, const TailArgs& a, cudaStream_t s) {
  note_launch();
  switch (algo) {
    case kBfs: tail_loop_kernel<kBfs><<<1, 1024, 0, s>>>(a); break;
    case kCc: tail_loop_kernel<kCc><<<1, 1024, 0, s>>>(a); break;
    default: tail_loop_kernel<kSssp><<<1, 1024, 0, s>>>(a); break;
  }
}

// Pass results to the host: the census and the run counters are written
// straight into mapped pinned memory by one tiny kernel (no D2H copies).
__global__ void publish_kernel(const Census* __restrict__ cz, Census* cz_host,
                               const RunCtr* __restrict__ ctr, RunCtr* ctr_host, uint32_t n_ctr,
                               unsigned* seq_host, unsigned seq) {
  const uint32_t words = sizeof(Census) / 4;
  const uint32_t cwords = n_ctr * uint32_t(sizeof(RunCtr) / 8);
  for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
    reinterpret_cast<uint32_t*>(cz_host)[i] = reinterpret_cast<const uint32_t*>(cz)[i];
  for (uint32_t i = threadIdx.x; i < cwords; i += blockDim.x)
    reinterpret_cast<unsigned long long*>(ctr_host)[i] =
        reinterpret_cast<const unsigned long long*>(ctr)[i];
  if (seq_host) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned*>(seq_host) = seq;
  }
}

void launch_publish(const Census* cz, Census* cz_host, const RunCtr* ctr, RunCtr* ctr_host,
                    uint32_t n_ctr, unsigned* seq_host, unsigned seq, cudaStream_t s) {
  note_launch();
  publish_kernel<<<1, 256, 0, s>>>(cz, cz_host, ctr, ctr_host, n_ctr, seq_host, seq);
}

// Initial BFS/SSSP frontier {source} as a queue (initial_frontier,
// engine.cpp:260-263) without the |V|-sized census and compaction.
__global__ void seed_queue_kernel(uint32_t source, const uint32_t* __restrict__ outdeg,
                                  uint32_t* list, Census* cz) {
  const uint32_t d = outdeg[source];
  cz->changed = 1;
  cz->push_count = d > 0;
  cz->out_edges = d;
  cz->own_push = d > 0;
  cz->own_edges = d;
  if (d) list[0] = source;
}

void launch_seed_queue(uint32_t source, const uint32_t* outdeg, uint32_t* list, Census* cz,
                       cudaStream_t s) {
  note_launch();
  seed_queue_kernel<<<1, 1, 0, s>>>(source, outdeg, list, cz);
}

void launch_queue_prep(const uint32_t* list, uint32_t q, const uint32_t* outdeg,
                       unsigned long long* pref, uint32_t* chunk_start, uint32_t shift,
                       uint64_t total_edges, void* tmp, size_t tmp_bytes, cudaStream_t s) {
  if (!q) return;
  note_launch();
  queue_degrees_kernel<<<grid_for(uint64_t(q) + 1, 256), 256, 0, s>>>(list, q, outdeg, pref);
  SR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, pref, pref, uint64_t(q) + 1, s));
  note_launch(2);  // cub: tile-state init + scan
  note_launch();
  const uint64_t chunks = (total_edges >> shift) + 1;
  const int per_warp = chunks > 8ull * q ? 1 : 0;
  queue_chunks_kernel<<<grid_for(per_warp ? uint64_t(q) * 32 : q, 256), 256, 0, s>>>(
      pref, q, shift, per_warp, chunk_start);
}

void launch_push(int algo, bool det, const PushArgs& a, int grid, cudaStream_t s) {
  note_launch();
  switch (algo) {
    case kBfs:
      if (det) push_relax_kernel<kBfs, true><<<grid, kBlockThreads, 0, s>>>(a);
      else push_relax_kernel<kBfs, false><<<grid, kBlockThreads, 0, s>>>(a);
      break;
    case kCc:
      if (det) push_relax_kernel<kCc, true><<<grid, kBlockThreads, 0, s>>>(a);
      else push_relax_kernel<kCc, false><<<grid, kBlockThreads, 0, s>>>(a);
      break;
    default:
      if (det) push_relax_kernel<kSssp, true><<<grid, kBlockThreads, 0, s>>>(a);
      else push_relax_kernel<kSssp, false><<<grid, kBlockThreads, 0, s>>>(a);
      break;
  }
}


void launch_push_scan(int algo, const PushArgs& a, const PageDesc* pages, uint32_t n_pages,
                      uint32_t* fbits, uint32_t n, int grid, cudaStream_t s) {
  SR_CUDA(cudaMemsetAsync(fbits, 0, (size_t(n) / 32 + 1) * 4, s));
  if (a.n_list) {
    note_launch();
    set_bits_kernel<<<grid_for(a.n_list, 256), 256, 0, s>>>(a.list, a.n_list, fbits);
  }
  note_launch();
  switch (algo) {
    case kBfs: push_scan_kernel<kBfs><<<grid, kBlockThreads, 0, s>>>(a, pages, n_pages, fbits); break;
    case kCc: push_scan_kernel<kCc><<<grid, kBlockThreads, 0, s>>>(a, pages, n_pages, fbits); break;
    default: push_scan_kernel<kSssp><<<grid, kBlockThreads, 0, s>>>(a, pages, n_pages, fbits); break;
  }
}

void launch_push_commit(uint32_t* values, const uint32_t* next, const uint8_t* changed,
                        uint32_t n, RunCtr* ctr, Census* c, cudaStream_t s) {
  note_launch();
  push_commit_kernel<<<grid_for(n, 256), 256, 0, s>>>(values, next, changed, n, ctr, c);
}

void launch_census(uint32_t n, const uint8_t* changed, uint8_t* status, uint8_t* logstate,
                   const uint32_t* out_offsets, int pass_kind, uint32_t own_lo,
                   uint32_t own_hi, uint32_t* blk_cnt, unsigned long long* blk_edges,
                   unsigned long long* part, Census* c, const Publish& pub, cudaStream_t s) {
  const uint32_t nb = (n + kCensusBlockVerts - 1) / kCensusBlockVerts;
  if (!nb) return;
  (void)part;
  const uint32_t cap = 148u * 8u;  // measured: 592 / 1184 / 2368 / nb blocks -> 1184 best
  const int grid = int(nb < cap ? nb : cap);
  note_launch();
  if (status || logstate)
    census_kernel<true><<<grid, 256, 0, s>>>(n, changed, status, logstate, out_offsets, pass_kind,
                                             own_lo, own_hi, blk_cnt, blk_edges, c, pub);
  else
    census_kernel<false><<<grid, 256, 0, s>>>(n, changed, status, logstate, out_offsets, pass_kind,
                                              own_lo, own_hi, blk_cnt, blk_edges, c, pub);
}

void launch_scan_blocks(uint32_t nblocks, uint32_t* blk_cnt, unsigned long long* blk_edges,
                        cudaStream_t s) {
  if (!nblocks) return;
  note_launch();
  scan_blocks_kernel<<<1, 1024, 0, s>>>(nblocks, blk_cnt, blk_edges);
}

void launch_compact(uint32_t n, uint32_t own_lo, uint32_t own_hi, uint8_t* changed,
                    const uint32_t* out_offsets, const uint32_t* blk_off,
                    const unsigned long long* blk_eoff, uint32_t* list, unsigned long long* pref,
                    uint32_t* chunk_start, uint32_t shift, cudaStream_t s) {
  const uint32_t nb = (n + kCensusBlockVerts - 1) / kCensusBlockVerts;
  if (!nb) return;
  note_launch();
  compact_kernel<<<nb, 256, 0, s>>>(n, own_lo, own_hi, changed, out_offsets, blk_off, blk_eoff,
                                    list, pref, chunk_start, shift);
}

void launch_csr_from_pages(const uint4* tiles, const uint32_t* tile_page, const PageDesc* pages,
                           uint32_t tile_lo, uint32_t tile_hi, unsigned long long* cursor,
                           uint32_t* out_nbr, uint32_t* out_w, int grid, cudaStream_t s) {
  if (tile_hi <= tile_lo) return;
  const uint32_t need = (tile_hi - tile_lo + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (uint32_t(grid) > need) grid = int(need);
  note_launch();
  csr_from_pages_kernel<<<grid, kBlockThreads, 0, s>>>(tiles, tile_page, pages, tile_lo, tile_hi,
                                                       cursor, out_nbr, out_w);
}

void launch_src_block(int mode, const uint4* tiles, const uint32_t* tile_page,
                      const PageDesc* pages, uint32_t tile_lo, uint32_t tile_hi, uint32_t n,
                      uint32_t blk_verts, uint32_t n_pages, uint32_t* cnt,
                      unsigned long long* goff, uint32_t* out_src, uint32_t* out_w, int grid,
                      cudaStream_t s) {
  if (tile_hi <= tile_lo) return;
  const uint32_t need = (tile_hi - tile_lo + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (uint32_t(grid) > need) grid = int(need);
  note_launch();
  src_block_kernel<<<grid, kBlockThreads, 0, s>>>(mode, tiles, tile_page, pages, tile_lo, tile_hi,
                                                  n, blk_verts, n_pages, cnt, goff, out_src, out_w);
}

// ---------------------------------------------------------------------------
// Device tile cut of the source-blocked sub-pages (replaces the host cut for
// them: no |V| x blocks offsets round trip).  The cut_tiles rule of the
// resident pages (engine.cpp) applied per 128-destination window, one thread
// per window: a hub (> kHubChunk in-edges) becomes one tile per chunk, other
// destinations are packed greedily into tiles of <= kTileMaxDests
// destinations and <= kTileEdgeBudget edges.
// ---------------------------------------------------------------------------
struct SubCut {
  uint32_t n, cap, n_pages, wpp;  // wpp: 128-destination windows per page
  uint32_t own_lo, own_hi;        // this rank's destinations (global ids)
  const uint32_t* offs;  // [n_blocks][n + n_pages] sub-page local offsets
};

// mode 0: tile count of every window into cnt; mode 1: write the tiles at the
// exclusive scan `at` of those counts
__global__ void sub_tiles_kernel(int mode, SubCut c, uint32_t n_blocks, uint32_t* cnt,
                                 const uint32_t* __restrict__ at, uint4* tiles,
                                 uint32_t* tile_page) {
  const uint64_t total = uint64_t(n_blocks) * c.n_pages * c.wpp;
  for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < total;
       k += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t bp = uint32_t(k / c.wpp), w = uint32_t(k % c.wpp);
    const uint32_t b = bp / c.n_pages, p = bp % c.n_pages;
    const uint32_t vb = p * c.cap, range = min(c.cap, c.n - vb);
    // the window, clipped to this rank's destination range
    const uint32_t lo = max(w * kTileMaxDests, c.own_lo > vb ? min(c.own_lo - vb, range) : 0u);
    const uint32_t hi = min(min(w * kTileMaxDests + kTileMaxDests, range),
                            c.own_hi > vb ? min(c.own_hi - vb, range) : 0u);
    const uint32_t* o = c.offs + size_t(b) * (size_t(c.n) + c.n_pages) + size_t(p) * c.cap + p;
    uint32_t t = mode ? at[k] : 0u;
    uint32_t i = lo;
    while (i < hi) {
      const uint32_t e0 = o[i], deg = o[i + 1] - e0;
      if (deg > kHubChunk) {
        for (uint32_t e = e0; e < e0 + deg; e += kHubChunk, ++t)
          if (mode) {
            tiles[t] = make_uint4(e, min(e + kHubChunk, e0 + deg), i, kHubFlag);
            tile_page[t] = bp;
          }
        ++i;
        continue;
      }
      uint32_t j = i + 1, e = o[j];
      while (j < hi) {
        const uint32_t e2 = o[j + 1];
        if (e2 - e > kHubChunk || e2 - e0 > kTileEdgeBudget) break;
        e = e2;
        ++j;
      }
      if (mode) {
        tiles[t] = make_uint4(e0, e, i, j);
        tile_page[t] = bp;
      }
      ++t;
      i = j;
    }
    if (!mode) cnt[k] = t;
  }
}

void launch_sub_tiles(int mode, uint32_t n, uint32_t cap, uint32_t n_pages, uint32_t n_blocks,
                      uint32_t own_lo, uint32_t own_hi, const uint32_t* offs, uint32_t* cnt,
                      const uint32_t* at, uint4* tiles, uint32_t* tile_page, cudaStream_t s) {
  if (!n || !n_blocks) return;
  const uint32_t wpp = (cap + kTileMaxDests - 1) / kTileMaxDests;
  const SubCut c{n, cap, n_pages, wpp, own_lo, own_hi, offs};
  note_launch();
  sub_tiles_kernel<<<grid_for(uint64_t(n_blocks) * n_pages * wpp, 256), 256, 0, s>>>(
      mode, c, n_blocks, cnt, at, tiles, tile_page);
}

uint64_t sub_tile_windows(uint32_t cap, uint32_t n_pages, uint32_t n_blocks) {
  return uint64_t(n_blocks) * n_pages * ((cap + kTileMaxDests - 1) / kTileMaxDests);
}

// Out-degree histogram (vertices and edges per degree, degrees >= kDegHistCap
// pooled in the last bucket): block-level shared-memory counts, one global
// atomic per non-empty bucket per block.
__global__ void __launch_bounds__(256) degree_hist_kernel(const uint32_t* __restrict__ outdeg,
                                                          uint32_t n, unsigned long long* hist_v,
                                                          unsigned long long* hist_e) {
  __shared__ uint32_t s_v[kDegHistCap + 1];
  __shared__ unsigned long long s_e[kDegHistCap + 1];
  for (uint32_t i = threadIdx.x; i <= kDegHistCap; i += blockDim.x) {
    s_v[i] = 0;
    s_e[i] = 0;
  }
  __syncthreads();
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint32_t d = outdeg[v];
    const uint32_t b = min(d, kDegHistCap);
    atomicAdd(s_v + b, 1u);
    atomicAdd(s_e + b, (unsigned long long)d);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i <= kDegHistCap; i += blockDim.x)
    if (s_v[i]) {
      atomicAdd(hist_v + i, (unsigned long long)s_v[i]);
      atomicAdd(hist_e + i, s_e[i]);
    }
}

void launch_degree_hist(const uint32_t* outdeg, uint32_t n, unsigned long long* hist_v,
                        unsigned long long* hist_e, cudaStream_t s) {
  if (!n) return;
  note_launch();
  degree_hist_kernel<<<grid_for(n, 256, 148 * 4), 256, 0, s>>>(outdeg, n, hist_v, hist_e);
}

size_t exclusive_scan_u32_temp_bytes(size_t count) {
  size_t tb = 0;
  SR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, static_cast<const uint32_t*>(nullptr),
                                        static_cast<uint32_t*>(nullptr), count));
  return tb;
}

// The caller owns the temporary storage (stream-ordered allocations inside
// a build showed multi-100 ms stalls next to multi-GB buffers).
void launch_exclusive_scan_u32(const uint32_t* in, uint32_t* out, size_t count, void* tmp,
                               size_t tmp_bytes, cudaStream_t s) {
  if (!count) return;
  SR_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, count, s));
  note_launch(2);
}

// ---- per-page exclusive scan of the (block, destination) counts of page p:
// nb segments of `range` u32 counts -> u64 page-local offsets, in parallel
// chunks (a segment scanned by one thread block took ~8 ms per page) ----
constexpr uint32_t kSegChunk = 4096;  // 1024 threads x 4

__global__ void __launch_bounds__(1024) seg_chunk_sum_kernel(const uint32_t* __restrict__ cnt,
                                                             size_t n, uint32_t vb, uint32_t range,
                                                             uint32_t chunks,
                                                             unsigned long long* part) {
  __shared__ unsigned long long s_w[32];
  const uint32_t b = blockIdx.x / chunks, c = blockIdx.x % chunks;
  const uint32_t* seg = cnt + size_t(b) * n + vb;
  unsigned long long x = 0;
  for (uint32_t i = c * kSegChunk + threadIdx.x; i < min(range, (c + 1) * kSegChunk); i += 1024)
    x += seg[i];
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    x = warp_sum(s_w[threadIdx.x]);
    if (threadIdx.x == 0) part[blockIdx.x] = x;
  }
}

// per block b: exclusive scan of its chunk sums in place; the total -> bp_edges
__global__ void __launch_bounds__(1024) seg_part_scan_kernel(unsigned long long* part,
                                                             uint32_t chunks, uint32_t p,
                                                             uint32_t n_pages,
                                                             unsigned long long* bp_edges) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const uint32_t b = blockIdx.x;
  unsigned long long* q = part + size_t(b) * chunks;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t c0 = 0; c0 < chunks; c0 += 1024) {
    const uint32_t i = c0 + threadIdx.x;
    const unsigned long long x = i < chunks ? q[i] : 0ull;
    const unsigned long long incl = warp_incl_scan(x, lane);
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
      const unsigned long long t = s_w[lane];
      s_w[lane] = warp_incl_scan(t, lane) - t;
    }
    __syncthreads();
    const unsigned long long ex = s_carry + s_w[w] + incl - x;
    if (i < chunks) q[i] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex + x;
    __syncthreads();
  }
  if (threadIdx.x == 0) bp_edges[size_t(b) * n_pages + p] = s_carry;
}

__global__ void __launch_bounds__(1024) seg_chunk_scan_kernel(const uint32_t* __restrict__ cnt,
                                                              size_t n, uint32_t vb,
                                                              uint32_t range, uint32_t chunks,
                                                              const unsigned long long* part,
                                                              unsigned long long* goff) {
  __shared__ unsigned long long s_w[32];
  __shared__ unsigned long long s_carry;
  const uint32_t b = blockIdx.x / chunks, c = blockIdx.x % chunks;
  const uint32_t* seg = cnt + size_t(b) * n + vb;
  unsigned long long* out = goff + size_t(b) * n + vb;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = part[blockIdx.x];
  __syncthreads();
  const uint32_t end = min(range, (c + 1) * kSegChunk);
  for (uint32_t c0 = c * kSegChunk; c0 < end; c0 += 1024) {
    const uint32_t i = c0 + threadIdx.x;
    const unsigned long long x = i < end ? seg[i] : 0ull;
    const unsigned long long incl = warp_incl_scan(x, lane);
    if (lane == 31) s_w[w] = incl;
    __syncthreads();
    if (w == 0) {
      const unsigned long long t = s_w[lane];
      s_w[lane] = warp_incl_scan(t, lane) - t;
    }
    __syncthreads();
    const unsigned long long ex = s_carry + s_w[w] + incl - x;
    if (i < end) out[i] = ex;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = ex + x;
    __syncthreads();
  }
}

uint32_t src_block_scan_parts(uint32_t cap, uint32_t n_blocks) {
  return n_blocks * ((cap + kSegChunk - 1) / kSegChunk);
}

// ---- page-major per-page build (Engine::sb_page): sub-page (p, b) lives at
// page_base + sum_{b' < b} pad8(edges(p, b')), so page p's sub-pages are
// built from page p alone, as soon as its DMA has landed ----
__global__ void src_block_page_base_kernel(uint32_t p, uint32_t n_pages, uint32_t n_blocks,
                                           unsigned long long page_base,
                                           const unsigned long long* __restrict__ bp_edges,
                                           unsigned long long* bp_base) {
  if (threadIdx.x != 0) return;
  unsigned long long at = page_base;
  for (uint32_t b = 0; b < n_blocks; ++b) {
    bp_base[size_t(b) * n_pages + p] = at;
    at += (bp_edges[size_t(b) * n_pages + p] + 7) & ~7ull;
  }
}

// page p: u32 sub-page local offsets from the page-local goff, then goff +=
// the sub-page base (absolute scatter cursors)
__global__ void src_block_page_fix_kernel(uint32_t p, uint32_t vb, uint32_t range, uint32_t n,
                                          uint32_t cap, uint32_t n_pages, uint32_t n_blocks,
                                          unsigned long long* goff,
                                          const unsigned long long* __restrict__ bp_edges,
                                          const unsigned long long* __restrict__ bp_base,
                                          uint32_t* offs) {
  const size_t per = size_t(range) + 1;
  const size_t total = size_t(n_blocks) * per;
  for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < total;
       k += size_t(gridDim.x) * blockDim.x) {
    const uint32_t b = uint32_t(k / per), i = uint32_t(k % per);
    uint32_t* o = offs + size_t(b) * (size_t(n) + n_pages) + size_t(p) * cap + p;
    if (i < range) {
      const size_t g = size_t(b) * n + vb + i;
      const unsigned long long x = goff[g];
      o[i] = uint32_t(x);
      goff[g] = x + bp_base[size_t(b) * n_pages + p];
    } else {
      o[range] = uint32_t(bp_edges[size_t(b) * n_pages + p]);
    }
  }
}

void launch_src_block_page(const uint32_t* cnt, unsigned long long* goff, const PageDesc* pages,
                           uint32_t p, uint32_t vb, uint32_t range, uint32_t n, uint32_t cap,
                           uint32_t n_pages, uint32_t n_blocks, unsigned long long page_base,
                           unsigned long long* bp_edges, unsigned long long* bp_base,
                           uint32_t* offs, unsigned long long* part, cudaStream_t s) {
  if (!n_blocks) return;
  (void)pages;
  note_launch(5);
  const uint32_t chunks = std::max<uint32_t>(1, (range + kSegChunk - 1) / kSegChunk);
  seg_chunk_sum_kernel<<<n_blocks * chunks, 1024, 0, s>>>(cnt, n, vb, range, chunks, part);
  seg_part_scan_kernel<<<n_blocks, 1024, 0, s>>>(part, chunks, p, n_pages, bp_edges);
  seg_chunk_scan_kernel<<<n_blocks * chunks, 1024, 0, s>>>(cnt, n, vb, range, chunks, part, goff);
  src_block_page_base_kernel<<<1, 32, 0, s>>>(p, n_pages, n_blocks, page_base, bp_edges, bp_base);
  src_block_page_fix_kernel<<<grid_for(uint64_t(n_blocks) * (range + 1), 256), 256, 0, s>>>(
      p, vb, range, n, cap, n_pages, n_blocks, goff, bp_edges, bp_base, offs);
}

void launch_pr_block_finalize(uint32_t lo, uint32_t hi, float* acc, float* rank_out,
                              float* contrib_out, const float* inv_outdeg, float base, float damp,
                              cudaStream_t s) {
  if (hi <= lo) return;
  note_launch();
  pr_block_finalize_kernel<<<grid_for(hi - lo, 256), 256, 0, s>>>(lo, hi, acc, rank_out,
                                                                   contrib_out, inv_outdeg, base,
                                                                   damp);
}

void launch_outdeg(const unsigned long long* off, uint32_t n, uint32_t* deg, cudaStream_t s) {
  if (!n) return;
  note_launch();
  outdeg_kernel<<<grid_for(n, 256), 256, 0, s>>>(off, n, deg);
}

void launch_init_values(int algo, uint32_t source, uint32_t n, uint32_t* values, cudaStream_t s) {
  if (!n) return;
  note_launch();
  init_values_kernel<<<grid_for(n, 256), 256, 0, s>>>(algo, source, n, values);
}

void launch_init_hub_stamp(uint32_t* stamp, uint32_t n, cudaStream_t s) {
  if (!n) return;
  note_launch();
  fill_u32_kernel<<<grid_for(n, 256), 256, 0, s>>>(stamp, n, 0u);
}

void launch_verify(int algo, uint32_t lo, uint32_t hi, const unsigned long long* out_offsets,
                   const uint32_t* nbr, const uint32_t* w, const uint32_t* values,
                   unsigned long long* violations, cudaStream_t s) {
  if (hi <= lo) return;
  const int g = grid_for((unsigned long long)(hi - lo) * 32, 256);
  note_launch();
  switch (algo) {
    case kBfs: verify_kernel<kBfs><<<g, 256, 0, s>>>(lo, hi, out_offsets, nbr, w, values, violations); break;
    case kCc: verify_kernel<kCc><<<g, 256, 0, s>>>(lo, hi, out_offsets, nbr, w, values, violations); break;
    default: verify_kernel<kSssp><<<g, 256, 0, s>>>(lo, hi, out_offsets, nbr, w, values, violations); break;
  }
}

}  // namespace seraph
