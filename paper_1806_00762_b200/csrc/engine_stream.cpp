// Out-of-core transfer scheduling of the engine: the HBM budget plan
// (permanently cached heavy pages + a streaming byte ring) and page
// admission on the copy stream.  The pass schedules that drive it are in
// engine.cpp (dense_pass_wall).
#include "engine.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace seraph {

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
    if (prefix + want * slot_bytes <= page_budget_) {
      K = k;
      fits = true;
    }
    prefix += pages_[used[k]].bytes;
  }
  if (!fits)
    throw EngineError(SR_E_CONFIG, "hbm budget " + std::to_string(page_budget_) +
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

}  // namespace seraph
