// sma_host.h -- host-side internals shared by libsma's translation units:
// error reporting (thread-local message behind sma_last_error), the dlopen'ed
// NCCL entry points, and the host bookkeeping helpers.  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>

#include "../../include/sma.h"

namespace sma {

// Record a printf-style message for sma_last_error() and return `st`.
sma_status fail(sma_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

// libsma does not link NCCL: it binds the few entry points it needs from the
// process's libnccl.so.2 (the one torch already loaded, else the system one),
// so a single-GPU process never needs NCCL and there is one NCCL per process.
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // optional (user-buffer registration; absent in old NCCLs)
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommRegister)(const ncclComm_t, void*, size_t, void**) = nullptr;
  ncclResult_t (*CommDeregister)(const ncclComm_t, void*) = nullptr;
};
extern NcclApi g_nccl;
bool nccl_load();  // thread-safe, once per process; false (g_nccl.why) if unavailable

// Fisher-Yates permutation of [0, N) for `epoch` (reading R10), int32 output.
void plan_epoch_permutation(int64_t N, uint64_t seed, int64_t epoch, int32_t* perm);

}  // namespace sma
