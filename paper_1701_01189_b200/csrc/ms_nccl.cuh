// ms_nccl.cuh -- NCCL for the sharded multisplit, bound at run time with dlopen
// so that libms loads (and every single-GPU call works) without NCCL.  The
// process's NCCL is used when one is already loaded (PyTorch's copy: dlopen
// of the soname returns it), else the loader's search path decides.  Types
// come from the NCCL 2.28 header; only the handful of calls below are used.
#pragma once
#include <dlfcn.h>

#include <mutex>

#include <nccl.h>

namespace ms {

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  // failure detection (optional symbols: checked where used)
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

inline const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define MS_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
    MS_NCCL_SYM(GetUniqueId);
    MS_NCCL_SYM(CommInitRank);
    MS_NCCL_SYM(CommDestroy);
    MS_NCCL_SYM(AllGather);
    MS_NCCL_SYM(AllReduce);
    MS_NCCL_SYM(Send);
    MS_NCCL_SYM(Recv);
    MS_NCCL_SYM(GroupStart);
    MS_NCCL_SYM(GroupEnd);
    MS_NCCL_SYM(CommGetAsyncError);
    MS_NCCL_SYM(CommAbort);
#undef MS_NCCL_SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.AllReduce && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  return api;
}

}  // namespace ms
