// comm.h — the cross-GPU data path of lmfao_run (private).
//
// Domain parallelism (partition the largest relation, merge the partial
// results): one process per GPU, each holding a contiguous shard of the sorted root.  A
// Comm moves partial aggregates between the ranks of one run:
//   * all-reduce (sum)       small outputs (the covariance batch's 780 values, small tables),
//                            complete on every rank;
//   * reduce-scatter (sum)   large dense group-by tables: each rank keeps the sums of its own
//                            contiguous range of cells;
//   * peer memory            every rank maps the others' exchange buffers, so a kernel writes
//                            the groups of a sparse cuboid straight into their owner's buffer
//                            (device-side counts: no host round trip inside lmfao_run);
//   * send / recv            lmfao_gather_result (a synchronising call) assembles a distributed
//                            output on one rank.
// Two implementations: NCCL over NVLink / NVSwitch (one process per GPU, peer memory by CUDA
// IPC handles), and a loopback group of contexts of one process on one device, driven by one
// host thread per rank, which runs the same kernels with host barriers between the phases
// (tests of the multi-GPU path on one GPU; no kernel ever waits for another rank's kernel).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace lmfao {

struct NcclUniqueId {
  char internal[128];
};
bool nccl_available();
int nccl_unique_id(void* out);

enum CommType { COMM_F64 = 0, COMM_U64 = 1, COMM_U8 = 2 };

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() {}
  // sum over ranks, in place (identical on every rank)
  virtual int allreduce_sum(void* buf, size_t n, CommType t, cudaStream_t st) = 0;
  // buf holds world * chunk elements; afterwards [rank * chunk, (rank + 1) * chunk) holds the sums
  virtual int reduce_scatter_sum(void* buf, size_t chunk, CommType t, cudaStream_t st) = 0;
  // recv[r * bytes .. (r + 1) * bytes) = rank r's send
  virtual int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) = 0;
  // point-to-point, host-known sizes, grouped (start, sends / recvs, end)
  virtual int group_start() = 0;
  virtual int group_end(cudaStream_t st) = 0;
  virtual int send(const void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  virtual int recv(void* buf, size_t bytes, int peer, cudaStream_t st) = 0;
  // collective, plan time: every rank's device buffer `mine` (same size on every rank) mapped
  // into this process; peers[rank] = mine
  virtual int map_peers(void* mine, std::vector<void*>& peers, cudaStream_t st) = 0;
  virtual void unmap_peers(std::vector<void*>& peers) = 0;
  // CUDA Graph capture of a run is allowed (NCCL: yes; loopback: no, it synchronises the host)
  virtual bool capturable() const = 0;
  // loopback: a host barrier between the phases of a run (the kernels of a phase that read
  // another rank's data start after every rank finished the previous phase)
  virtual int phase(cudaStream_t st) { return 0; }
  // NCCL: ncclCommGetAsyncError
  virtual int async_error() { return 0; }
  virtual std::string error_string(int e) const = 0;
  virtual const char* backend() const = 0;
};

// world > 1, one process per GPU; unique_id from lmfao_unique_id on rank 0.  err: NCCL status
Comm* make_nccl_comm(int rank, int world, const void* unique_id, int& err);
// an in-process group named `group`; every member must be created before the first collective
Comm* make_loopback_comm(const char* group, int rank, int world, int device);

// host-only helpers of the partition (also exported through the C ABI for the CPU tests)
inline void shard_range(int64_t n, int part, int nparts, int64_t& lo, int64_t& hi) {
  lo = n * part / nparts;
  hi = n * (part + 1) / nparts;
}
// cells [lo, hi) of an output with ncells cells owned by `rank` (reduce-scatter chunks: equal
// chunks of ceil(ncells / world) cells, the last ranks' possibly short or empty)
inline void owner_range(int64_t ncells, int rank, int world, int64_t& lo, int64_t& hi) {
  const int64_t chunk = (ncells + world - 1) / world;
  lo = std::min<int64_t>(ncells, chunk * rank);
  hi = std::min<int64_t>(ncells, chunk * (rank + 1));
}
inline int owner_of(int64_t cell, int64_t ncells, int world) {
  const int64_t chunk = (ncells + world - 1) / world;
  return (int)(cell / chunk);
}

}  // namespace lmfao
