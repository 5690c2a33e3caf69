// Host-side error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "../../include/bnmc_gpu.h"

namespace bnmc_host {

struct Status {
  int code;
  std::string msg;
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Status{code, msg}; }

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(BNMC_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace bnmc_host

#define CK(x) ::bnmc_host::cuda_check((x), #x)
