// Virtual-clock pass scheduler (deterministic mode).  See vsched.h.
#include "vsched.h"

#include <algorithm>
#include <numeric>
#include <stdexcept>
#include <string>

#include "errors.h"

namespace seraph {

std::vector<uint32_t> VWindow::resident_sorted() const {
  std::vector<uint32_t> r = pages_;
  std::sort(r.begin(), r.end());
  return r;
}

void VWindow::admit(uint32_t page) {
  if (std::find(pages_.begin(), pages_.end(), page) != pages_.end())
    throw EngineError(SR_E_CONTRACT, "page " + std::to_string(page) + " already resident");
  if (pages_.size() >= cap_)
    throw EngineError(SR_E_CONTRACT, "window full admitting page " + std::to_string(page));
  pages_.push_back(page);
}

void VWindow::evict(uint32_t page) {
  auto it = std::find(pages_.begin(), pages_.end(), page);
  if (it == pages_.end())
    throw EngineError(SR_E_CONTRACT, "evicting non-resident page " + std::to_string(page));
  pages_.erase(it);
}

namespace {

// Kernels launched together at t0 share the worker pool evenly among the
// ones still running (reference scheduler.cpp:166-186).
std::vector<double> pool_finish_times(const std::vector<uint64_t>& work, double t0,
                                      const VModel& tm) {
  const size_t n = work.size();
  std::vector<size_t> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return work[a] < work[b]; });
  const double rate = tm.edges_per_unit_per_worker * double(tm.workers);
  std::vector<double> end(n, t0);
  double t = t0;
  uint64_t done = 0;
  for (size_t k = 0; k < n; ++k) {
    const size_t i = idx[k];
    t += double(work[i] - done) * double(n - k) / rate;
    done = work[i];
    end[i] = t;
  }
  return end;
}

struct Pass {
  const std::vector<uint64_t>& bytes;
  VWindow& win;
  VClock& clock;
  const VModel& tm;
  const VKernel& kernel;
  uint32_t pass_index;
  bool tracing;

  VPassResult out;
  std::vector<uint32_t> q;       // admission order: resident first, then by id
  std::vector<double> arrival;   // per q position
  std::vector<double> done_at;   // per q position; < 0 while kernel work is pending
  size_t cursor = 0;
  uint32_t free_slots = 0;
  double channel = 0, compute = 0;

  void emit(double t, int kind, uint32_t page) {
    if (tracing) clock.pending.push_back(sr_trace_event{t, kind, page, pass_index, 0});
  }

  void prepare() {
    const uint32_t n = uint32_t(bytes.size());
    std::vector<uint32_t> res = win.resident_sorted();
    std::vector<char> is_res(n, 0);
    for (uint32_t p : res)
      if (p < n) {
        is_res[p] = 1;
        q.push_back(p);
      }
    for (uint32_t p = 0; p < n; ++p)
      if (!is_res[p]) q.push_back(p);
    arrival.assign(n, clock.now);
    done_at.assign(n, -1.0);
    free_slots = win.capacity() - win.resident_count();
    channel = compute = clock.now;
    cursor = res.size();
  }

  void stream_through(size_t limit, double not_before) {
    while (cursor <= limit) {
      const size_t t = cursor++;
      const uint32_t page = q[t];
      double ready = clock.now;
      if (free_slots > 0) {
        --free_slots;
      } else {
        if (t < win.capacity())
          throw EngineError(SR_E_CONTRACT, "transfer scheduled with no slot available");
        const size_t victim = t - win.capacity();
        if (done_at[victim] < 0)
          throw EngineError(SR_E_CONTRACT, "eviction victim still has pending kernel work");
        ready = done_at[victim];
        win.evict(q[victim]);
      }
      const double start = std::max({channel, ready, not_before});
      const double end = start + tm.xfer_time(bytes[page]);
      win.admit(page);
      arrival[t] = end;
      channel = end;
      emit(start, SR_TRACE_XFER_START, page);
      emit(end, SR_TRACE_XFER_END, page);
      out.pages_transferred += 1;
      out.bytes_transferred += bytes[page];
    }
  }

  RunStats run_at(uint32_t page, double start, bool reentry, double& end) {
    RunStats st = kernel(page);
    end = start + tm.kernel_time(st.edges);
    emit(start, reentry ? SR_TRACE_REENTRY : SR_TRACE_KERNEL_START, page);
    emit(end, SR_TRACE_KERNEL_END, page);
    out.totals += st;
    out.kernel_runs += 1;
    return st;
  }

  // Kernels of one set start together; counters accumulate in call order.
  std::vector<double> run_set(size_t lo, size_t hi, double t0, bool reentry) {
    std::vector<uint64_t> work;
    work.reserve(hi - lo);
    for (size_t i = lo; i < hi; ++i) {
      RunStats st = kernel(q[i]);
      work.push_back(st.edges);
      out.totals += st;
      out.kernel_runs += 1;
      emit(t0, reentry ? SR_TRACE_REENTRY : SR_TRACE_KERNEL_START, q[i]);
    }
    std::vector<double> ends = pool_finish_times(work, t0, tm);
    for (size_t k = 0; k < ends.size(); ++k) emit(ends[k], SR_TRACE_KERNEL_END, q[lo + k]);
    return ends;
  }

  void baseline(bool reentry, int mrt) {
    for (size_t i = 0; i < q.size(); ++i) {
      stream_through(i, 0.0);
      double start = std::max(compute, arrival[i]);
      double end = start;
      for (int runs = 1;; ++runs) {
        RunStats st = run_at(q[i], start, runs > 1, end);
        if (!reentry || runs >= mrt || st.valid == 0) break;
        start = end;
      }
      done_at[i] = end;
      compute = end;
    }
  }

  void double_buffer(int reps) {
    const size_t n = q.size();
    const size_t half = std::max<size_t>(1, win.capacity() / 2);
    for (size_t lo = 0; lo < n; lo += half) {
      const size_t hi = std::min(lo + half, n);
      stream_through(hi - 1, 0.0);
      double t0 = compute;
      for (size_t i = lo; i < hi; ++i) t0 = std::max(t0, arrival[i]);
      std::vector<double> ends;
      for (int r = 1; r <= reps; ++r) {
        ends = run_set(lo, hi, t0, r > 1);
        for (double e : ends) t0 = std::max(t0, e);
      }
      for (size_t i = lo; i < hi; ++i) done_at[i] = ends[i - lo];
      compute = t0;
    }
  }

  void pipelined(bool fine) {
    const size_t n = q.size();
    const size_t slots = std::min<size_t>(win.capacity() - 1, n);
    const size_t sets = n - slots + 1;
    stream_through(slots - 1, 0.0);
    for (size_t j = 0; j < sets; ++j) {
      double needed = arrival[j + slots - 1];
      if (j == 0)
        for (size_t i = 0; i < slots; ++i) needed = std::max(needed, arrival[i]);
      if (fine && j > 0) {
        // compute idles while the stream is still in flight: re-run the
        // lowest-id page of the previous set (fill_idle_slot -> ReentryOne)
        while (needed > compute) {
          size_t victim = j - 1;
          for (size_t i = j - 1; i < j - 1 + slots; ++i)
            if (q[i] < q[victim]) victim = i;
          double end;
          run_at(q[victim], compute, true, end);
          done_at[victim] = end;
          if (!(end > compute)) break;  // zero-edge run: no progress possible
          compute = end;
        }
      }
      const double t0 = std::max(compute, needed);
      std::vector<double> ends = run_set(j, j + slots, t0, false);
      double last = t0;
      for (size_t k = 0; k < ends.size(); ++k) {
        done_at[j + k] = ends[k];
        last = std::max(last, ends[k]);
      }
      compute = last;
      if (j + slots < n) stream_through(j + slots, fine ? 0.0 : t0);
    }
  }
};

}  // namespace

VPassResult vschedule_pass(const std::vector<uint64_t>& page_bytes, int mode, int mrt, int reps,
                           VWindow& window, VClock& clock, const VModel& tm,
                           const VKernel& kernel, uint32_t pass_index,
                           std::vector<sr_trace_event>* trace) {
  Pass p{page_bytes, window, clock, tm, kernel, pass_index, trace != nullptr, {}, {}, {}, {}};
  p.out.start = clock.now;
  if (!page_bytes.empty()) {
    p.prepare();
    switch (mode) {
      case SR_SCHED_REENTRY: p.baseline(true, mrt); break;
      case SR_SCHED_DOUBLE_BUFFER: p.double_buffer(reps); break;
      case SR_SCHED_PIPELINED: p.pipelined(false); break;
      case SR_SCHED_PIPELINED_FINE: p.pipelined(true); break;
      default: p.baseline(false, 1); break;
    }
    p.out.end = std::max(p.compute, p.channel);
  } else {
    p.out.end = clock.now;
  }
  if (p.out.end > clock.now) clock.now = p.out.end;
  if (trace) {
    std::stable_sort(clock.pending.begin(), clock.pending.end(),
                     [](const sr_trace_event& a, const sr_trace_event& b) {
                       if (a.time != b.time) return a.time < b.time;
                       if (a.page_id != b.page_id) return a.page_id < b.page_id;
                       return a.kind < b.kind;
                     });
    trace->insert(trace->end(), clock.pending.begin(), clock.pending.end());
    clock.pending.clear();
  }
  return p.out;
}

}  // namespace seraph
