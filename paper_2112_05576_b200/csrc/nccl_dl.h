// nccl_dl.h -- NCCL, loaded at run time (dlopen) for the theta-sharded
// multi-GPU path.
//
// The library does not link NCCL: a process that imports torch already has
// torch's libnccl.so.2 mapped, and dlopen("libnccl.so.2") then returns that
// very copy (same soname), so the library and torch.distributed share one
// NCCL.  A C++ host without torch gets the system libnccl.so.2.
// EAB_NCCL_LIB overrides the path.  nccl.h is used for its types only.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

namespace eab {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*CommAbort)(ncclComm_t);
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*GetVersion)(int*);
    const char* (*GetErrorString)(ncclResult_t);
};

// The loaded API; throws Failure(EA_ERR_NCCL) when libnccl cannot be loaded.
const NcclApi& nccl();
// Failure(EA_ERR_NCCL, "<what>: <ncclGetErrorString>") unless r == ncclSuccess.
void nccl_check(ncclResult_t r, const char* what);

}  // namespace eab

#define EAB_NCCL(x) ::eab::nccl_check((x), #x)
