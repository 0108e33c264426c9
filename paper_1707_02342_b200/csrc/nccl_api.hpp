// nccl_api.hpp — NCCL resolved at run time (dlopen), so the library loads on
// hosts without NCCL; only the multi-GPU path needs it.  Whichever
// libnccl.so.2 the process already mapped (e.g. torch's) is reused.
#pragma once

#include <dlfcn.h>
#include <nccl.h>

#include <string>

#include "errors.hpp"

namespace mppi_host {

struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline NcclApi& nccl() {
  static NcclApi api;
  if (!api.lib) {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (!api.lib) throw Error(MPPI_ERR_NCCL, "cannot dlopen libnccl.so.2");
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(api.lib, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(api.lib, "ncclCommInitRank"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(api.lib, "ncclAllGather"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(api.lib, "ncclCommDestroy"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(api.lib, "ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.CommDestroy) {
      api.lib = nullptr;
      throw Error(MPPI_ERR_NCCL, "libnccl is missing required symbols");
    }
  }
  return api;
}

}  // namespace mppi_host

#define NCCL_TRY(expr)                                                                         \
  do {                                                                                         \
    ncclResult_t r__ = (expr);                                                                 \
    if (r__ != ncclSuccess)                                                                    \
      throw ::mppi_host::Error(MPPI_ERR_NCCL,                                                  \
                               std::string(#expr) + ": " +                                     \
                                   (::mppi_host::nccl().GetErrorString                         \
                                        ? ::mppi_host::nccl().GetErrorString(r__)              \
                                        : "?"));                                               \
  } while (0)
