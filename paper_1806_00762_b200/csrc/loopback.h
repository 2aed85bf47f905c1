// In-process loopback collective: the all-reduces of the multi-GPU exchange
// (engine.cpp exchange_round) between contexts of ONE process, through host
// memory.  Lets the sharded round protocol run on a single GPU (two ranks =
// two contexts on the same device, driven from two threads) in tests, where
// NCCL refuses two ranks on one device.  Not a transport for production.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>
#include <vector>

namespace seraph {

struct LoopbackGroup;

enum LoopType { kLoopU32 = 0, kLoopU64 = 1, kLoopF32 = 2 };
enum LoopOp { kLoopMin = 0, kLoopSum = 1 };

// The group `key` of `world` ranks (created by the first caller).
LoopbackGroup* loopback_group(const std::string& key, int world);
// Blocking all-reduce of `count` elements of device buffer `buf` (stream `s`
// is synchronised first); every rank of the group must call it in the same order.
void loopback_allreduce(LoopbackGroup* g, int rank, void* buf, size_t count, LoopType t, LoopOp op,
                        cudaStream_t s);
// Host barrier over the group's ranks.
void loopback_barrier(LoopbackGroup* g);
// Every rank's pointer, indexed by rank (peer exchange: the value replicas).
std::vector<void*> loopback_allgather_ptr(LoopbackGroup* g, int rank, void* mine);

}  // namespace seraph
