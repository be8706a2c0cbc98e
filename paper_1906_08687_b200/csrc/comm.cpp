// comm.cpp — NCCL over NVLink/NVSwitch for combining per-GPU partial aggregates
// (domain parallelism: partition the largest relation, merge partials).
// NCCL is loaded with dlopen so the process shares the libnccl.so.2 that torch
// already mapped (one NCCL per process).
#include <dlfcn.h>

#include <cstdio>

#include "comm.h"

namespace lmfao {

struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};

static NcclApi& api() {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (a.h) {
      a.GetUniqueId = (int (*)(void*))dlsym(a.h, "ncclGetUniqueId");
      a.CommInitRank = (int (*)(void**, int, NcclUniqueId, int))dlsym(a.h, "ncclCommInitRank");
      a.CommDestroy = (int (*)(void*))dlsym(a.h, "ncclCommDestroy");
      a.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(a.h, "ncclAllReduce");
      a.GetErrorString = (const char* (*)(int))dlsym(a.h, "ncclGetErrorString");
      a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce;
    }
  }
  return a;
}

bool nccl_available() { return api().ok; }

int nccl_unique_id(void* out) {
  if (!api().ok) return -1;
  return api().GetUniqueId(out);
}

int nccl_init(void** comm, int world, const void* id, int rank) {
  if (!api().ok) return -1;
  NcclUniqueId u;
  std::memcpy(u.internal, id, sizeof(u.internal));
  return api().CommInitRank(comm, world, u, rank);
}

int nccl_destroy(void* comm) { return api().ok && comm ? api().CommDestroy(comm) : 0; }

// ncclDataType_t: ncclUint64 = 5, ncclFloat64 = 9; ncclRedOp_t: ncclSum = 0
int nccl_allreduce_f64(void* comm, double* buf, size_t n, cudaStream_t st) {
  return api().AllReduce(buf, buf, n, 9, 0, comm, st);
}
int nccl_allreduce_u64(void* comm, unsigned long long* buf, size_t n, cudaStream_t st) {
  return api().AllReduce(buf, buf, n, 5, 0, comm, st);
}

const char* nccl_error(int e) {
  if (api().GetErrorString) return api().GetErrorString(e);
  return "NCCL unavailable";
}

}  // namespace lmfao
