#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstring>

namespace lmfao {
struct NcclUniqueId {
  char internal[128];
};
bool nccl_available();
int nccl_unique_id(void* out);
int nccl_init(void** comm, int world, const void* id, int rank);
int nccl_destroy(void* comm);
int nccl_allreduce_f64(void* comm, double* buf, size_t n, cudaStream_t st);
int nccl_allreduce_u64(void* comm, unsigned long long* buf, size_t n, cudaStream_t st);
const char* nccl_error(int e);
}  // namespace lmfao
