// In-process loopback collective (see loopback.h).
#include "loopback.h"

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "errors.h"

namespace seraph {

struct LoopbackGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<unsigned char>> slots;
  std::vector<void*> ptrs;

  // generation barrier over the `world` ranks; a rank that never arrives
  // (it failed before the collective) turns into an error here instead of a
  // hang (SERAPH_LOOPBACK_TIMEOUT_S, default 600 s)
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      long secs = 600;
      if (const char* e = std::getenv("SERAPH_LOOPBACK_TIMEOUT_S")) secs = std::max(1L, std::atol(e));
      if (!cv.wait_for(lk, std::chrono::seconds(secs), [&] { return generation != gen; })) {
        --arrived;
        throw EngineError(SR_E_INTERNAL, "loopback world: a rank did not reach the collective");
      }
    }
  }
};

namespace {

std::mutex g_registry_mu;
std::map<std::string, std::unique_ptr<LoopbackGroup>> g_registry;

// element-wise reduction over the ranks' slots; a rank that contributed
// fewer elements counts as the identity for the missing ones
template <typename T>
void reduce_into(std::vector<std::vector<unsigned char>>& slots, size_t count, LoopOp op, T* out) {
  for (size_t i = 0; i < count; ++i) {
    bool have = false;
    T acc{};
    for (size_t r = 0; r < slots.size(); ++r) {
      if ((i + 1) * sizeof(T) > slots[r].size()) continue;
      T x;
      std::memcpy(&x, slots[r].data() + i * sizeof(T), sizeof(T));
      acc = !have ? x : (op == kLoopMin ? std::min(acc, x) : T(acc + x));
      have = true;
    }
    out[i] = acc;
  }
}

}  // namespace

LoopbackGroup* loopback_group(const std::string& key, int world) {
  std::lock_guard<std::mutex> lk(g_registry_mu);
  auto& g = g_registry[key];
  if (!g || g->world != world) {
    g = std::make_unique<LoopbackGroup>();
    g->world = world;
    g->slots.resize(size_t(world));
    g->ptrs.resize(size_t(world));
  }
  return g.get();
}

void loopback_barrier(LoopbackGroup* g) { g->barrier(); }

std::vector<void*> loopback_allgather_ptr(LoopbackGroup* g, int rank, void* mine) {
  g->ptrs[size_t(rank)] = mine;
  g->barrier();
  std::vector<void*> all = g->ptrs;
  g->barrier();  // everyone has copied before the next allgather overwrites
  return all;
}

void loopback_allreduce(LoopbackGroup* g, int rank, void* buf, size_t count, LoopType t, LoopOp op,
                        cudaStream_t s) {
  const size_t esz = t == kLoopU64 ? 8 : 4;
  SR_CUDA(cudaStreamSynchronize(s));
  auto& mine = g->slots[size_t(rank)];
  mine.resize(count * esz);
  if (count) SR_CUDA(cudaMemcpy(mine.data(), buf, count * esz, cudaMemcpyDeviceToHost));
  g->barrier();  // every rank's contribution is in
  std::vector<unsigned char> out(count * esz);
  if (t == kLoopU32) reduce_into(g->slots, count, op, reinterpret_cast<uint32_t*>(out.data()));
  else if (t == kLoopU64)
    reduce_into(g->slots, count, op, reinterpret_cast<unsigned long long*>(out.data()));
  else reduce_into(g->slots, count, op, reinterpret_cast<float*>(out.data()));
  g->barrier();  // everyone has read the slots before they are reused
  if (count) SR_CUDA(cudaMemcpy(buf, out.data(), count * esz, cudaMemcpyHostToDevice));
}

}  // namespace seraph
