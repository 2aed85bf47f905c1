#include "stager.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "errors.h"

namespace seraph {

HostStager::~HostStager() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_job_.notify_all();
  for (auto& t : pool_) t.join();
  for (auto& f : fifo_) {
    cudaEventSynchronize(f.ev);
    cudaEventDestroy(f.ev);
  }
  for (cudaEvent_t e : free_events_) cudaEventDestroy(e);
  if (ring_) cudaFreeHost(ring_);
}

bool HostStager::pageable(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

void HostStager::ensure() {
  if (ring_) return;
  if (const char* e = std::getenv("SERAPH_STAGE_RING_MB"))
    ring_bytes_ = std::max<size_t>(size_t(std::max(1, std::atoi(e))) << 20, kPiece);
  void* r = nullptr;
  SR_CUDA(cudaHostAlloc(&r, ring_bytes_, cudaHostAllocPortable));
  ring_ = static_cast<char*>(r);
  unsigned h = std::thread::hardware_concurrency();
  int t = h ? int(std::min<unsigned>(h, 16)) : 4;  // 16-core box: 8 -> 16 threads 0.44 -> 0.43 s for C4
  if (const char* e = std::getenv("SERAPH_STAGE_THREADS")) t = std::max(1, std::atoi(e));
  threads_ = t;
  for (int k = 1; k < threads_; ++k) pool_.emplace_back(&HostStager::worker, this, k);
}

cudaEvent_t HostStager::take_event() {
  if (!free_events_.empty()) {
    cudaEvent_t e = free_events_.back();
    free_events_.pop_back();
    return e;
  }
  cudaEvent_t e;
  SR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return e;
}

void HostStager::retire_oldest() {
  Inflight f = fifo_.front();
  fifo_.pop_front();
  SR_CUDA(cudaEventSynchronize(f.ev));
  free_events_.push_back(f.ev);
}

// Bump allocation in the ring: the region must not overlap a piece whose DMA
// may still be reading it (the in-flight pieces are the FIFO, oldest first).
size_t HostStager::reserve(size_t len) {
  len = (len + 255) & ~size_t(255);
  if (head_ + len > ring_bytes_) head_ = 0;  // wrap: the tail end is skipped
  for (;;) {
    bool clash = false;
    for (const Inflight& f : fifo_)
      if (f.start < head_ + len && head_ < f.end) {
        clash = true;
        break;
      }
    if (!clash) break;
    retire_oldest();
  }
  const size_t at = head_;
  head_ += len;
  return at;
}

void HostStager::worker(int k) {
  uint64_t seen = 0;
  for (;;) {
    char* dst;
    const char* src;
    size_t bytes;
    int parts;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_job_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      dst = job_dst_;
      src = job_src_;
      bytes = job_bytes_;
      parts = job_threads_;
    }
    if (k < parts) {
      const size_t a = bytes * k / parts, b = bytes * (k + 1) / parts;
      std::memcpy(dst + a, src + a, b - a);
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) cv_done_.notify_one();
    }
  }
}

// memcpy on up to `threads_` threads, >= 1 MB per thread
void HostStager::copy_parallel(void* dst, const void* src, size_t bytes) {
  const int parts = int(std::min<size_t>(size_t(threads_), bytes >> 20));
  if (parts <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  {
    std::lock_guard<std::mutex> lk(mu_);
    job_dst_ = static_cast<char*>(dst);
    job_src_ = static_cast<const char*>(src);
    job_bytes_ = bytes;
    job_threads_ = parts;
    pending_ = threads_ - 1;
    ++gen_;
  }
  cv_job_.notify_all();
  std::memcpy(dst, src, bytes / parts);  // part 0 on the calling thread
  std::unique_lock<std::mutex> lk(mu_);
  cv_done_.wait(lk, [&] { return pending_ == 0; });
}

void HostStager::h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return;
  if (!pageable(src)) {
    SR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    return;
  }
  ensure();
  for (size_t off = 0; off < bytes; off += kPiece) {
    const size_t len = std::min(kPiece, bytes - off);
    const size_t at = reserve(len);
    copy_parallel(ring_ + at, static_cast<const char*>(src) + off, len);
    SR_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, ring_ + at, len,
                            cudaMemcpyHostToDevice, s));
    const cudaEvent_t ev = take_event();
    SR_CUDA(cudaEventRecord(ev, s));
    fifo_.push_back(Inflight{at, at + ((len + 255) & ~size_t(255)), ev});
    staged_ += len;
  }
}

void HostStager::d2h_sync(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  if (!bytes) return;
  if (!pageable(dst)) {
    SR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    SR_CUDA(cudaStreamSynchronize(s));
    return;
  }
  ensure();
  sync();  // the whole ring is free: pieces alternate between its halves
  const size_t half = ring_bytes_ / 2, piece = std::min(kPiece, half);
  const size_t nch = (bytes + piece - 1) / piece;
  cudaEvent_t ev[2] = {take_event(), take_event()};
  auto issue = [&](size_t k) {
    const size_t off = k * piece, len = std::min(piece, bytes - off);
    SR_CUDA(cudaMemcpyAsync(ring_ + (k & 1) * half, static_cast<const char*>(src) + off, len,
                            cudaMemcpyDeviceToHost, s));
    SR_CUDA(cudaEventRecord(ev[k & 1], s));
  };
  issue(0);
  if (nch > 1) issue(1);
  for (size_t k = 0; k < nch; ++k) {
    const size_t off = k * piece, len = std::min(piece, bytes - off);
    SR_CUDA(cudaEventSynchronize(ev[k & 1]));
    copy_parallel(static_cast<char*>(dst) + off, ring_ + (k & 1) * half, len);
    if (k + 2 < nch) issue(k + 2);
  }
  free_events_.push_back(ev[0]);
  free_events_.push_back(ev[1]);
}

void HostStager::sync() {
  while (!fifo_.empty()) retire_oldest();
}

}  // namespace seraph
