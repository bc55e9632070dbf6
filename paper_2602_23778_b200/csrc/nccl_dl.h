// nccl_dl.h -- NCCL entry points resolved at run time (dlopen), so librefine.so has no link-time
// dependency on NCCL and world == 1 never touches it.  The process's already-loaded libnccl
// (torch's bundled NCCL 2.28) is found by its soname; REFINE_NCCL_PATH overrides the lookup.
#pragma once
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>

namespace rf {

typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclChar = 0, ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclInt = 2, ncclUint32 = 3, ncclInt64 = 4,
               ncclUint64 = 5, ncclFloat16 = 6, ncclHalf = 6, ncclFloat32 = 7, ncclFloat = 7, ncclFloat64 = 8,
               ncclDouble = 8 } ncclDataType_t;

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline Nccl& nccl() {
  static Nccl n;
  static bool tried = false;
  if (tried) return n;
  tried = true;
  // REFINE_NCCL_PATH (a full path to libnccl.so.2) is tried first; otherwise the soname, which
  // finds the copy the process already loaded (torch's) or the loader's search path.
  const char* env = getenv("REFINE_NCCL_PATH");
  const char* names[] = {env && env[0] ? env : "libnccl.so.2", "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    fprintf(stderr, "[refine] NCCL not found (dlopen libnccl.so.2 failed)\n");
    return n;
  }
#define RF_SYM(field, sym) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, sym))
  RF_SYM(GetUniqueId, "ncclGetUniqueId");
  RF_SYM(CommInitRank, "ncclCommInitRank");
  RF_SYM(CommDestroy, "ncclCommDestroy");
  RF_SYM(AllGather, "ncclAllGather");
  RF_SYM(Broadcast, "ncclBroadcast");
  RF_SYM(Send, "ncclSend");
  RF_SYM(Recv, "ncclRecv");
  RF_SYM(GroupStart, "ncclGroupStart");
  RF_SYM(GroupEnd, "ncclGroupEnd");
  RF_SYM(GetErrorString, "ncclGetErrorString");
#undef RF_SYM
  n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.AllGather && n.Broadcast && n.Send && n.Recv &&
         n.GroupStart && n.GroupEnd;
  return n;
}

}  // namespace rf
