// Deterministic virtual-clock pass scheduler used by SR_CLOCK_VIRTUAL runs.
//
// Behaviour follows the reference's schedule_dense_pass / PassRunner
// (proj/src/scheduler.cpp:188-435): resident-first page order (:211-228),
// FIFO slot eviction with the victim Q-position t-B (:241-247), one transfer
// channel (:249), baseline/reentry (:272-291), double-buffer (:293-330),
// pipelined(-fine) super-subgraph sets with idle-slot re-entry (:332-390),
// work-conserving finish times (:166-186).  The kernel callback runs one
// page on the GPU and returns its counters; it is invoked in exactly the
// reference's admission order, so counters and trace are reproducible.
//
// One deliberate difference: the pipelined-fine idle loop stops re-entering
// a page whose run reads no edges (it cannot advance compute time).  The
// reference livelocks there (scheduler.cpp:348-360).
#pragma once

#include <cstdint>
#include <functional>
#include <optional>
#include <vector>

#include "seraph.h"

namespace seraph {

struct RunStats {
  uint64_t attempts = 0, valid = 0, skipped = 0, edges = 0;
  RunStats& operator+=(const RunStats& o) {
    attempts += o.attempts;
    valid += o.valid;
    skipped += o.skipped;
    edges += o.edges;
    return *this;
  }
};

struct VModel {  // TransferModel (scheduler.hpp:19-29)
  double bytes_per_unit = 11.0;
  double edges_per_unit_per_worker = 1.75;
  int workers = 4;
  double xfer_time(uint64_t bytes) const { return double(bytes) / bytes_per_unit; }
  double kernel_time(uint64_t edges) const {
    return double(edges) / (edges_per_unit_per_worker * double(workers));
  }
};

// Resident page slots carried across passes (Window, scheduler.hpp:96-123).
class VWindow {
 public:
  explicit VWindow(uint32_t cap = 8) : cap_(cap) {}
  uint32_t capacity() const { return cap_; }
  std::vector<uint32_t> resident_sorted() const;
  uint32_t resident_count() const { return uint32_t(pages_.size()); }
  void admit(uint32_t page);
  void evict(uint32_t page);
  void reset(uint32_t cap) {
    cap_ = cap;
    pages_.clear();
  }

 private:
  uint32_t cap_;
  std::vector<uint32_t> pages_;
};

struct VPassResult {
  RunStats totals;
  uint64_t kernel_runs = 0;
  uint64_t pages_transferred = 0;
  uint64_t bytes_transferred = 0;
  double start = 0, end = 0;
};

using VKernel = std::function<RunStats(uint32_t page)>;

struct VClock {
  double now = 0;
  std::vector<sr_trace_event> pending;
};

// Runs every page at least once under `mode`; appends trace events (sorted
// by (time, page, kind) per pass, scheduler.cpp:79-88) when trace != null.
VPassResult vschedule_pass(const std::vector<uint64_t>& page_bytes, int mode, int mrt, int reps,
                           VWindow& window, VClock& clock, const VModel& tm,
                           const VKernel& kernel, uint32_t pass_index,
                           std::vector<sr_trace_event>* trace);

}  // namespace seraph
