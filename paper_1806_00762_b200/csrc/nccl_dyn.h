// NCCL entry points resolved at run time (dlopen), so libseraph neither pins
// an NCCL version at link time nor shadows the one the host process (e.g.
// torch.distributed) already loaded: dlopen("libnccl.so.2") returns the
// resident copy when there is one.
#pragma once

#include <nccl.h>

namespace seraph {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Throws EngineError(SR_E_NCCL) when libnccl cannot be loaded.
const NcclApi& nccl();

}  // namespace seraph
