// comm.cpp — the two Comm implementations (see comm.h).
//
// NCCL is loaded with dlopen so the process shares the libnccl.so.2 that torch already
// mapped (one NCCL per process); the enum values below are nccl.h 2.28's.  Peer memory of
// the NCCL ranks is mapped with CUDA IPC handles exchanged by an NCCL all-gather.
#include "comm.h"

#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>

#include "internal.h"

namespace lmfao {

namespace {
// nccl.h 2.28: ncclDataType_t ncclUint8 = 1, ncclUint64 = 5, ncclFloat64 = 8; ncclRedOp_t ncclSum = 0
constexpr int NCCL_U8 = 1, NCCL_U64 = 5, NCCL_F64 = 8, NCCL_SUM = 0;
int nccl_type(CommType t) { return t == COMM_F64 ? NCCL_F64 : (t == COMM_U64 ? NCCL_U64 : NCCL_U8); }
size_t type_bytes(CommType t) { return t == COMM_U8 ? 1 : 8; }

struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*ReduceScatter)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*CommGetAsyncError)(void*, int*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool ok = false;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (a.h) break;
    }
    if (!a.h) return;
    auto sym = [](const char* s) { return dlsym(a.h, s); };
    a.GetUniqueId = (int (*)(void*))sym("ncclGetUniqueId");
    a.CommInitRank = (int (*)(void**, int, NcclUniqueId, int))sym("ncclCommInitRank");
    a.CommDestroy = (int (*)(void*))sym("ncclCommDestroy");
    a.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))sym("ncclAllReduce");
    a.ReduceScatter = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))sym("ncclReduceScatter");
    a.AllGather = (int (*)(const void*, void*, size_t, int, void*, cudaStream_t))sym("ncclAllGather");
    a.Send = (int (*)(const void*, size_t, int, int, void*, cudaStream_t))sym("ncclSend");
    a.Recv = (int (*)(void*, size_t, int, int, void*, cudaStream_t))sym("ncclRecv");
    a.GroupStart = (int (*)())sym("ncclGroupStart");
    a.GroupEnd = (int (*)())sym("ncclGroupEnd");
    a.CommGetAsyncError = (int (*)(void*, int*))sym("ncclCommGetAsyncError");
    a.GetErrorString = (const char* (*)(int))sym("ncclGetErrorString");
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.ReduceScatter && a.AllGather &&
           a.Send && a.Recv && a.GroupStart && a.GroupEnd;
  });
  return a;
}

// ---------------------------------------------------------------------------------- NCCL
struct NcclComm : Comm {
  void* comm = nullptr;
  ~NcclComm() override {
    if (comm) api().CommDestroy(comm);
  }
  int allreduce_sum(void* buf, size_t n, CommType t, cudaStream_t st) override {
    return n ? api().AllReduce(buf, buf, n, nccl_type(t), NCCL_SUM, comm, st) : 0;
  }
  int reduce_scatter_sum(void* buf, size_t chunk, CommType t, cudaStream_t st) override {
    if (!chunk) return 0;
    char* own = (char*)buf + (size_t)rank * chunk * type_bytes(t);  // in place (NCCL: recv = send + rank * count)
    return api().ReduceScatter(buf, own, chunk, nccl_type(t), NCCL_SUM, comm, st);
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    return api().AllGather(send, recv, bytes, NCCL_U8, comm, st);
  }
  int group_start() override { return api().GroupStart(); }
  int group_end(cudaStream_t) override { return api().GroupEnd(); }
  int send(const void* buf, size_t bytes, int peer, cudaStream_t st) override {
    return bytes ? api().Send(buf, bytes, NCCL_U8, peer, comm, st) : 0;
  }
  int recv(void* buf, size_t bytes, int peer, cudaStream_t st) override {
    return bytes ? api().Recv(buf, bytes, NCCL_U8, peer, comm, st) : 0;
  }
  int map_peers(void* mine, std::vector<void*>& peers, cudaStream_t st) override {
    // CUDA IPC handles of every rank's buffer, all-gathered over NCCL
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, mine) != cudaSuccess) return -1;
    const size_t hb = sizeof(h);
    DevBuf d;
    if (d.alloc(hb * (world + 1))) return -1;
    if (cudaMemcpyAsync(d.as<char>() + hb * world, &h, hb, cudaMemcpyHostToDevice, st)) return -1;
    if (int e = allgather(d.as<char>() + hb * world, d.p, hb, st)) return e;
    std::vector<cudaIpcMemHandle_t> all(world);
    if (cudaMemcpyAsync(all.data(), d.p, hb * world, cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st)) return -1;
    peers.assign(world, nullptr);
    for (int r = 0; r < world; r++) {
      if (r == rank) {
        peers[r] = mine;
        continue;
      }
      if (cudaIpcOpenMemHandle(&peers[r], all[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return -1;
    }
    return 0;
  }
  void unmap_peers(std::vector<void*>& peers) override {
    for (int r = 0; r < (int)peers.size(); r++)
      if (r != rank && peers[r]) cudaIpcCloseMemHandle(peers[r]);
    peers.clear();
  }
  bool capturable() const override { return true; }
  int async_error() override {
    int e = 0;
    if (api().CommGetAsyncError && api().CommGetAsyncError(comm, &e) != 0) return -1;
    return e == 7 ? 0 : e;  // ncclInProgress: not an error
  }
  std::string error_string(int e) const override {
    if (e == -1) return "CUDA IPC / NCCL setup failed";
    return api().GetErrorString ? api().GetErrorString(e) : "NCCL unavailable";
  }
  const char* backend() const override { return "nccl"; }
};

// ---------------------------------------------------------------------------------- loopback
// An in-process group: every member publishes a pointer, waits for the others, reads theirs.
struct Group {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<const void*> slot;            // published pointer per rank
  // [src][dst] send buffers of the current group call, in order (matched with the receives in
  // order, as NCCL matches the sends and receives between two ranks)
  std::vector<std::vector<std::vector<std::pair<const void*, size_t>>>> p2p;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
std::mutex g_groups_mu;
std::map<std::string, std::weak_ptr<Group>> g_groups;

__global__ void k_sum_ranks_f64(const double* const* src, int world, size_t n, double* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < world; r++) s += src[r][i];  // rank order: identical on every rank
    out[i] = s;
  }
}
__global__ void k_sum_ranks_u64(const unsigned long long* const* src, int world, size_t n, unsigned long long* out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (int r = 0; r < world; r++) s += src[r][i];
    out[i] = s;
  }
}

struct LoopbackComm : Comm {
  std::shared_ptr<Group> g;
  DevBuf scratch, ptrs;
  ~LoopbackComm() override {}
  int publish_and_wait(const void* p, std::vector<const void*>& all) {
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->slot[rank] = p;
    }
    g->barrier();
    {
      std::lock_guard<std::mutex> lk(g->mu);
      all = g->slot;
    }
    return 0;
  }
  // out[i] = Σ_r buf_r[i + off] over i < n (rank order)
  int sum(const void* buf, size_t off, size_t n, CommType t, void* out, cudaStream_t st) {
    std::vector<const void*> all;
    if (cudaStreamSynchronize(st)) return -1;
    publish_and_wait(buf, all);
    std::vector<const void*> src(world);
    for (int r = 0; r < world; r++) src[r] = (const char*)all[r] + off * type_bytes(t);
    if (ptrs.bytes < world * sizeof(void*) + 256 && ptrs.alloc(world * sizeof(void*))) return -1;
    if (cudaMemcpyAsync(ptrs.p, src.data(), world * sizeof(void*), cudaMemcpyHostToDevice, st)) return -1;
    const unsigned grid = (unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 148 * 8));
    if (n) {
      if (t == COMM_F64) k_sum_ranks_f64<<<grid, 256, 0, st>>>((const double* const*)ptrs.p, world, n, (double*)out);
      else k_sum_ranks_u64<<<grid, 256, 0, st>>>((const unsigned long long* const*)ptrs.p, world, n,
                                                  (unsigned long long*)out);
    }
    if (cudaStreamSynchronize(st)) return -1;
    g->barrier();  // every rank has read every buffer
    return 0;
  }
  int allreduce_sum(void* buf, size_t n, CommType t, cudaStream_t st) override {
    if (t == COMM_U8) return -1;
    if (scratch.bytes < n * 8 + 256 && scratch.alloc(n * 8)) return -1;
    if (int e = sum(buf, 0, n, t, scratch.p, st)) return e;
    if (n && cudaMemcpyAsync(buf, scratch.p, n * 8, cudaMemcpyDeviceToDevice, st)) return -1;
    return cudaStreamSynchronize(st) ? -1 : 0;
  }
  int reduce_scatter_sum(void* buf, size_t chunk, CommType t, cudaStream_t st) override {
    if (t == COMM_U8) return -1;
    if (scratch.bytes < chunk * 8 + 256 && scratch.alloc(chunk * 8)) return -1;
    if (int e = sum(buf, (size_t)rank * chunk, chunk, t, scratch.p, st)) return e;
    if (chunk && cudaMemcpyAsync((char*)buf + (size_t)rank * chunk * 8, scratch.p, chunk * 8,
                                 cudaMemcpyDeviceToDevice, st))
      return -1;
    return cudaStreamSynchronize(st) ? -1 : 0;
  }
  int allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) override {
    std::vector<const void*> all;
    if (cudaStreamSynchronize(st)) return -1;
    publish_and_wait(send, all);
    for (int r = 0; r < world; r++)
      if (bytes && cudaMemcpyAsync((char*)recv + r * bytes, all[r], bytes, cudaMemcpyDeviceToDevice, st)) return -1;
    if (cudaStreamSynchronize(st)) return -1;
    g->barrier();
    return 0;
  }
  std::vector<std::pair<void*, std::pair<size_t, int>>> pending_recv;
  int group_start() override {
    pending_recv.clear();
    std::lock_guard<std::mutex> lk(g->mu);
    for (int d = 0; d < world; d++) g->p2p[rank][d].clear();
    return 0;
  }
  int send(const void* buf, size_t bytes, int peer, cudaStream_t) override {
    std::lock_guard<std::mutex> lk(g->mu);
    g->p2p[rank][peer].push_back({buf, bytes});
    return 0;
  }
  int recv(void* buf, size_t bytes, int peer, cudaStream_t) override {
    pending_recv.push_back({buf, {bytes, peer}});
    return 0;
  }
  int group_end(cudaStream_t st) override {
    if (cudaStreamSynchronize(st)) return -1;
    g->barrier();  // every rank's sends are registered
    std::vector<size_t> next(world, 0);  // per source: the next of its sends to this rank
    for (auto& pr : pending_recv) {
      const int src_rank = pr.second.second;
      const void* src = nullptr;
      size_t n = (size_t)-1;
      {
        std::lock_guard<std::mutex> lk(g->mu);
        auto& q = g->p2p[src_rank][rank];
        if (next[src_rank] < q.size()) {
          src = q[next[src_rank]].first;
          n = q[next[src_rank]].second;
        }
        next[src_rank]++;
      }
      if (n != pr.second.first) return -2;  // mismatched sizes (NCCL would hang)
      if (n && cudaMemcpyAsync(pr.first, src, n, cudaMemcpyDeviceToDevice, st)) return -1;
    }
    if (cudaStreamSynchronize(st)) return -1;
    g->barrier();  // every copy done: the senders may reuse their buffers
    pending_recv.clear();
    return 0;
  }
  int map_peers(void* mine, std::vector<void*>& peers, cudaStream_t st) override {
    std::vector<const void*> all;
    if (cudaStreamSynchronize(st)) return -1;
    publish_and_wait(mine, all);
    peers.assign(world, nullptr);
    for (int r = 0; r < world; r++) peers[r] = const_cast<void*>(all[r]);
    g->barrier();
    return 0;
  }
  void unmap_peers(std::vector<void*>& peers) override { peers.clear(); }
  bool capturable() const override { return false; }
  int phase(cudaStream_t st) override {
    if (cudaStreamSynchronize(st)) return -1;
    g->barrier();
    return 0;
  }
  std::string error_string(int e) const override {
    return e == -2 ? "loopback send/recv size mismatch" : "loopback collective failed (CUDA error)";
  }
  const char* backend() const override { return "loopback"; }
};
}  // namespace

bool nccl_available() { return api().ok; }

int nccl_unique_id(void* out) {
  if (!api().ok) return -1;
  return api().GetUniqueId(out);
}

Comm* make_nccl_comm(int rank, int world, const void* unique_id, int& err) {
  err = -1;
  if (!api().ok) return nullptr;
  NcclUniqueId u;
  std::memcpy(u.internal, unique_id, sizeof(u.internal));
  auto* c = new NcclComm();
  c->rank = rank;
  c->world = world;
  err = api().CommInitRank(&c->comm, world, u, rank);
  if (err != 0) {
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

Comm* make_loopback_comm(const char* group, int rank, int world, int device) {
  std::shared_ptr<Group> g;
  {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto& w = g_groups[group];
    g = w.lock();
    if (!g) {
      g = std::make_shared<Group>();
      g->world = world;
      g->slot.assign(world, nullptr);
      g->p2p.assign(world, std::vector<std::vector<std::pair<const void*, size_t>>>(world));
      w = g;
    }
  }
  if (g->world != world) return nullptr;
  auto* c = new LoopbackComm();
  c->rank = rank;
  c->world = world;
  c->g = g;
  return c;
}

}  // namespace lmfao
