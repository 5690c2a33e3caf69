// NCCL entry points resolved at first use (dlopen of libnccl.so.2): the
// library needs NCCL only for multi-GPU tables and communicators, so a
// single-GPU process never depends on it. Types come from the NCCL header;
// a missing library or symbol is status BNMC_NCCL.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

#include "host_util.hpp"

namespace bnmc_host {

struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string error;
  bool ok = false;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("BNMC_NCCL_LIB");
    void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.error = std::string("cannot load NCCL: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && api.error.empty()) api.error = std::string("NCCL symbol missing: ") + name;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommInitAll, "ncclCommInitAll");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.AllGather, "ncclAllGather");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.GetVersion, "ncclGetVersion");
    api.ok = api.error.empty();
  });
  if (!api.ok) raise(BNMC_NCCL, api.error);
  return api;
}

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    raise(BNMC_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace bnmc_host

#define NK(x) ::bnmc_host::nccl_check((x), #x)
