// ndgx_nccl.h -- NCCL, loaded at run time.
//
// libndgx.so does not link NCCL: a single-GPU user never needs it, and in a
// PyTorch process dlopen("libnccl.so.2") returns the NCCL torch already
// loaded (same soname), so both share one library.  Types and enums come
// from the system nccl.h (2.27); the entry points used here are stable.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

namespace ndgx {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// The loaded library, or nullptr with *why set.
const Nccl* nccl(std::string* why);

}  // namespace ndgx
