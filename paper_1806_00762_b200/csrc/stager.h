// Host -> device uploads from pageable memory at link speed.
//
// The reference's callers hand pagestream::run plain std::vector arrays
// (graph.hpp:30-65): pageable memory.  A cudaMemcpyAsync from pageable memory
// is staged by the driver through its own pinned buffers on one host thread
// (well below the host link).  The stager pipelines instead: the source is
// cut into chunks, `threads` host threads copy chunk i into one of `nbuf`
// pinned buffers while the copy engine moves chunk i-1, so the upload runs at
// min(host memcpy bandwidth, link bandwidth).  Pinned and device sources are
// passed straight to cudaMemcpyAsync.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
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
  // pinned chunk ring (this call returns once the last chunk is enqueued;
  // src may be released only after sync()).  Other sources: cudaMemcpyAsync.
  void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
  // Wait until every staged chunk has left its pinned buffer.
  void sync();
  // Enqueue dst <- src (device -> pageable host) through the pinned chunks
  // and wait for it (DMA of chunk i+1 overlaps the host copy of chunk i).
  void d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s);
  uint64_t staged_bytes() const { return staged_; }

 private:
  size_t chunk_ = 32ull << 20;  // SERAPH_STAGE_CHUNK_MB
  static constexpr int kBufs = 4;
  void ensure();
  void copy_parallel(void* dst, const void* src, size_t bytes);
  void worker(int k);

  std::vector<void*> buf_;
  std::vector<cudaEvent_t> ev_;
  std::vector<bool> ev_live_;
  int next_ = 0;
  uint64_t staged_ = 0;
  int device_ = -1;

  // copy thread pool (threads_ - 1 workers + the calling thread)
  int threads_ = 1;
  std::vector<std::thread> pool_;
  std::mutex mu_;
  std::condition_variable cv_job_, cv_done_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  char* job_dst_ = nullptr;
  const char* job_src_ = nullptr;
  size_t job_bytes_ = 0;
};

}  // namespace seraph
