// Host -> device uploads from pageable memory at link speed.
//
// The reference's callers hand pagestream::run plain std::vector arrays
// (graph.hpp:30-65): pageable memory.  A cudaMemcpyAsync from pageable memory
// is staged by the driver through its own pinned buffers on one host thread
// (well below the host link).  The stager pipelines instead: sources are
// copied by `threads` host threads into a pinned byte ring (bump allocation,
// pieces of at most kPiece bytes), and each piece's DMA is queued at once, so
// host copies of later pieces overlap the copy engine and many small arrays
// (page offsets, small pages) can be in flight together.  The upload runs at
// min(host memcpy bandwidth, link bandwidth).  Pinned and device sources are
// passed straight to cudaMemcpyAsync.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace seraph {

class HostStager {
 public:
  HostStager() = default;
  HostStager(const HostStager&) = delete;
  HostStager& operator=(const HostStager&) = delete;
  ~HostStager();

  // True when `p` is ordinary pageable host memory (not pinned, not device).
  static bool pageable(const void* p);
  // Enqueue dst[0, bytes) <- src on `s`.  Pageable sources go through the
  // pinned ring (this call returns once the last piece is queued: src may be
  // released on return).  Other sources: cudaMemcpyAsync.
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
  // Wait until every queued piece has left the ring.
  void sync();
  // dst <- src (device -> pageable host) through the ring, synchronously
  // (the DMA of a piece overlaps the host copy of the previous one).
  void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s);
  uint64_t staged_bytes() const { return staged_; }

 private:
  static constexpr size_t kPiece = 32ull << 20;
  size_t ring_bytes_ = 128ull << 20;  // SERAPH_STAGE_RING_MB
  void ensure();
  // [offset, offset + len) of the ring, free for reuse (waits for old DMAs)
  size_t reserve(size_t len);
  void retire_oldest();
  cudaEvent_t take_event();
  void copy_parallel(void* dst, const void* src, size_t bytes);
  void worker(int k);

  char* ring_ = nullptr;
  size_t head_ = 0;
  struct Inflight {
    size_t start, end;
    cudaEvent_t ev;
  };
  std::deque<Inflight> fifo_;
  std::vector<cudaEvent_t> free_events_;
  uint64_t staged_ = 0;

  // copy thread pool (threads_ - 1 workers + the calling thread)
  int threads_ = 1;
  std::vector<std::thread> pool_;
  std::mutex mu_;
  std::condition_variable cv_job_, cv_done_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  int job_threads_ = 0;
  bool stop_ = false;
  char* job_dst_ = nullptr;
  const char* job_src_ = nullptr;
  size_t job_bytes_ = 0;
};

}  // namespace seraph
