// Engine exception carrying the C-ABI error code (include/seraph.h), which
// the C++ drop-in maps back onto the reference's exception classes
// (proj/include/pagestream/errors.hpp:8-28).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "seraph.h"

namespace seraph {

struct EngineError : std::runtime_error {
  int code;
  EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e == cudaSuccess) return;
  const int code = (e == cudaErrorMemoryAllocation) ? SR_E_OOM : SR_E_CUDA;
  throw EngineError(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                              std::to_string(line) + ")");
}

}  // namespace seraph

#define SR_CUDA(x) ::seraph::cuda_check((x), #x, __FILE__, __LINE__)
