// internal.h — private declarations of liblmfao_gpu (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/lmfao_gpu.h"

#define CUDA_TRY(x)                          \
  do {                                       \
    cudaError_t e__ = (x);                   \
    if (e__ != cudaSuccess) return e__;      \
  } while (0)

namespace lmfao {

#ifdef __CUDACC__
// Reductions without a return value on a known state space.  Pointers that come from
// kernel-argument structs or shared-memory descriptors are generic to the compiler, which
// then emits a generic ATOM that waits for its result (to branch to a shared-memory CAS
// loop); these emit RED, which the SM issues and forgets.
__device__ __forceinline__ void gred_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void gred_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void gred_add(unsigned* p, unsigned v) {
  asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void sred_add(double* p, double v) {
  asm volatile("red.shared.add.f64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "d"(v) : "memory");
}
#endif

// LMFAO_TRACE=1: wall-clock checkpoints of the host-side phases on stderr (tools/e2e_phases.py).
struct PhaseTrace {
  bool on;
  const char* name;
  std::chrono::steady_clock::time_point t;
  explicit PhaseTrace(const char* n) : name(n), t(std::chrono::steady_clock::now()) {
    const char* e = std::getenv("LMFAO_TRACE");
    on = e && e[0] == '1';
  }
  void mark(const char* what, cudaStream_t st = nullptr) {
    if (!on) return;
    if (st) cudaStreamSynchronize(st);
    auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lmfao] %s/%s %.3f ms\n", name, what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Stream the owning buffers below are ordered on.  Every ABI entry point sets it to its
// context's stream (StreamScope); allocations then come from the device's stream-ordered
// memory pool (cudaMallocAsync / cudaFreeAsync, release threshold raised in lmfao_create),
// which keeps freed memory cached instead of handing it back to the driver with an implicit
// device-wide synchronisation on every cudaFree.  Outside a scope (pooled == false) the
// buffers use plain cudaMalloc / cudaFree.
struct AllocScope {
  cudaStream_t st = nullptr;
  bool pooled = false;
};
inline AllocScope& alloc_scope() {
  static thread_local AllocScope s;
  return s;
}
struct StreamScope {
  AllocScope prev;
  StreamScope(cudaStream_t st, bool pooled = true) : prev(alloc_scope()) {
    static const bool off = [] {  // LMFAO_NO_POOL=1: plain cudaMalloc / cudaFree (A/B measurements)
      const char* e = std::getenv("LMFAO_NO_POOL");
      return e && e[0] == '1';
    }();
    alloc_scope() = AllocScope{st, pooled && !off};
  }
  ~StreamScope() { alloc_scope() = prev; }
  StreamScope(const StreamScope&) = delete;
  StreamScope& operator=(const StreamScope&) = delete;
};

// Owning device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t st = nullptr;  // stream it was allocated on (pooled buffers are freed there)
  bool pooled = false;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), st(o.st), pooled(o.pooled) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      reset();
      p = o.p; bytes = o.bytes; st = o.st; pooled = o.pooled;
      o.p = nullptr; o.bytes = 0;
    }
    return *this;
  }
  ~DevBuf() { reset(); }
  void reset() {
    if (p) {
      if (pooled) cudaFreeAsync(p, st);
      else cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  cudaError_t alloc(size_t b) {
    reset();
    // 256 B of slack: TMA bulk copies round tail sizes up to 16 B
    b += 256;
    const AllocScope& sc = alloc_scope();
    pooled = sc.pooled;
    st = sc.st;
    cudaError_t e = pooled ? cudaMallocAsync(&p, b, st) : cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    else p = nullptr;
    return e;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};

// The dynamic shared-memory opt-in of a kernel (cudaFuncAttributeMaxDynamicSharedMemorySize) is
// per device: raise it on the current device when a launch needs more than set there so far.
cudaError_t ensure_smem_attr(const void* func, size_t smem);

// ---- device primitives (prims.cu), all on stream st ----
cudaError_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t st);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t st);
cudaError_t radix_sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n, int key_bits, cudaStream_t st,
                             const unsigned long long* n_dev = nullptr);
cudaError_t iota_u32(uint32_t* a, int64_t n, cudaStream_t st);
cudaError_t gather_bytes(const void* in, const uint32_t* perm, void* out, int64_t n, int elem_bytes, cudaStream_t st);
cudaError_t dict_encode_i32(const int32_t* col, int64_t n, DevBuf& dict, int64_t& ndict, DevBuf* codes,
                            cudaStream_t st);
cudaError_t lookup_dense(const int32_t* vals, int64_t n, const int32_t* dict, int64_t nd, int32_t* out,
                         cudaStream_t st);
// two-attribute join keys: dictionary over the distinct (a, b) pairs (order-preserving u64 images)
cudaError_t dict_encode_pair(const int32_t* a, const int32_t* b, int64_t n, DevBuf& dict, int64_t& ndict, DevBuf* codes,
                             cudaStream_t st);
cudaError_t lookup_dense_pair(const int32_t* a, const int32_t* b, int64_t n, const uint64_t* dict, int64_t nd,
                              int32_t* out, cudaStream_t st);
cudaError_t keep_rows(const std::vector<const int32_t*>& fks, int64_t n, DevBuf& idx, int64_t& nkeep,
                      cudaStream_t st);
cudaError_t sort_perm_by_dense(const int32_t* dense, int64_t n, int64_t nkeys, DevBuf& perm, cudaStream_t st);
cudaError_t sort_perm_composite(const std::vector<const int32_t*>& keys, const std::vector<int64_t>& nkeys, int64_t n,
                                DevBuf& perm, cudaStream_t st);
cudaError_t segment_offsets(const int32_t* dkey, int64_t n, int64_t nkeys, DevBuf& off, cudaStream_t st);

// ---- generic evaluation (generic.cu) ----
constexpr int MAX_COLS = 48;
constexpr int MAX_CHILD = 8;

// A node's evaluation context: its columns, and per child the dense FK column
// and the child's view V_c [nkeys_c x W_c] (row-major FP64).
struct NodeArgs {
  int64_t nrows;
  const void* cols[MAX_COLS];
  int32_t col_is_int[MAX_COLS];
  int32_t nchild;
  const int32_t* fk[MAX_CHILD];
  const double* V[MAX_CHILD];
  int32_t W[MAX_CHILD];
};

// Program encoding (int32 stream + double stream), interpreted per row:
//   term   := n_own, (kind, col)*n_own, then one slot id per child (nchild ints); coef in dbl stream,
//             followed by n_own params in dbl stream.
//   output := n_terms, term*   (value = Σ terms)
// Views: one output per slot; root: one output per (query, udaf).
struct Program {
  std::vector<int32_t> ip;
  std::vector<double> dp;
  std::vector<int32_t> out_ioff, out_doff;  // start offsets per output
};

// A leaf child whose slots are products of <= 2 identity factors on its own columns
// (ca/cb null: factor 1).
struct ViewLinArgs {
  int64_t nrows;
  int nslots;
  const void* ca[64];
  const void* cb[64];
  unsigned char ia[64], ib[64];
};
cudaError_t launch_view_lin(const ViewLinArgs& a, const int32_t* dense_key, double* V, cudaStream_t st);

cudaError_t launch_view_build(const NodeArgs& a, const int32_t* dense_key, const int32_t* prog_i, const double* prog_d,
                              const int32_t* ioff, const int32_t* doff, int nslots, double* V, cudaStream_t st);

// No-group-by outputs: per-block partial sums (deterministic fixed-order combine).
cudaError_t launch_root_scalar(const NodeArgs& a, const int32_t* prog_i, const double* prog_d, const int32_t* ioff,
                               const int32_t* doff, int nout, double* partials, unsigned long long* count_partials,
                               int grid, cudaStream_t st);
cudaError_t launch_combine_partials(const double* partials, const unsigned long long* cpart, int grid, int nout,
                                    double* out, unsigned long long* count_out, cudaStream_t st);

// Group-by outputs: dense cell table, FP64 atomics; counts u64.
struct GroupArgs {
  int32_t ngb;
  const int32_t* code[8];   // per group attr: code column (root rows) or per-child-key code table
  int32_t code_child[8];    // -1: code[] indexed by root row; else child index (code[] indexed by fk)
  int64_t stride[8];        // mixed radix
};
cudaError_t launch_root_group(const NodeArgs& a, const GroupArgs& g, const int32_t* prog_i, const double* prog_d,
                              const int32_t* ioff, const int32_t* doff, int nudaf, double* table,
                              unsigned long long* counts, cudaStream_t st);

// One group-by query of the fused group-by scan (device-resident array).
struct GroupDesc {
  int32_t ngb, nudaf, prog_base;
  const int32_t* code[8];
  int32_t code_child[8];
  int64_t stride[8];
  double* table;
  unsigned long long* counts;
  unsigned char countlike[64];  // UDAF j is a constant c (SUM(c)): derived from the counts
  int32_t nsum;                 // UDAFs that are not countlike
};
cudaError_t launch_groups_fused(const NodeArgs& a, const GroupDesc* descs, int nq, const int32_t* prog_i,
                                const double* prog_d, const int32_t* ioff, const int32_t* doff, cudaStream_t st);
// group-by queries finished at a root child T with a non-unique key (generic.cu k_rev_*)
struct ProgPtrs {
  const int32_t* pi;
  const double* pd;
  const int32_t* io;
  const int32_t* dofs;
  int nout;
};
cudaError_t launch_rev(const NodeArgs& root, const int32_t* fkT, const ProgPtrs& rp, const NodeArgs& t,
                       const int32_t* tkey, const ProgPtrs& tp, const int32_t* pu, double* A, int64_t nkT,
                       const GroupDesc& d, cudaStream_t st);

// Compaction of a dense cell table: present cells (count > 0) in ascending order.
struct DecodeArgs {
  int32_t ngb;
  int64_t cell0;  // the table's first cell (a rank's range of a distributed table)
  const int32_t* dict[8];
  int64_t radix[8];
  int64_t stride[8];
  const double* countcoef;  // per UDAF: c if the UDAF is the constant c (value = c * count), NaN otherwise
};
cudaError_t launch_compact(const double* table, const unsigned long long* counts, int64_t ncells, int nudaf,
                           const DecodeArgs& d, DevBuf& keys, DevBuf& vals, DevBuf& cnts, int64_t& ngroups,
                           cudaStream_t st);

int launches_counter_reset();
void launches_add(int n);

}  // namespace lmfao
