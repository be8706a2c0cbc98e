// prims.cu — device primitives for kernel (a) "sort / remap":
// a stable LSD radix sort of (u32 key, u32 payload) pairs, exclusive scans,
// stream compaction, gathers, and the dense remap of join keys.
//
// P:42 "We sort the relations once"; "We choose the order that is the
// increasing order in the domain sizes of these attributes ... We sort S in this
// order."  These run at load time (lmfao_prepare) and plan time, never in lmfao_run.
#include <mutex>

#include "internal.h"

namespace lmfao {

constexpr int SORT_THREADS = 256;
constexpr int SORT_ITEMS = 8;                       // elements per thread per tile
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 2048
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// ---------------------------------------------------------------- radix sort
// Pass layout: hist[digit * nblocks + block] (digit-major) so one exclusive
// scan over the whole array gives each (digit, block) its output offset and the
// sort is stable across blocks.
__global__ void k_radix_hist(const uint32_t* __restrict__ keys, int64_t n, const unsigned long long* n_dev, int shift,
                             int bits, uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[256];
  if (n_dev) n = min(n, (int64_t)*n_dev);  // device-side size (n = capacity)
  int nd = 1 << bits;
  for (int i = threadIdx.x; i < nd; i += blockDim.x) h[i] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * SORT_TILE;
  for (int i = threadIdx.x; i < SORT_TILE; i += blockDim.x) {
    int64_t idx = base + i;
    if (idx < n) atomicAdd(&h[(keys[idx] >> shift) & (nd - 1)], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < nd; d += blockDim.x) hist[(int64_t)d * nblocks + blockIdx.x] = h[d];
}

// Stable scatter: the tile is consumed in chunks of SORT_THREADS elements (one
// per thread, in order); the rank of an element among equal digits is
// (earlier chunks) + (earlier warps in this chunk) + (earlier lanes in warp).
__global__ void k_radix_scatter(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                uint32_t* __restrict__ okeys, uint32_t* __restrict__ ovals, int64_t n,
                                const unsigned long long* n_dev, int shift, int bits,
                                const uint32_t* __restrict__ offs, int nblocks) {
  if (n_dev) n = min(n, (int64_t)*n_dev);
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[SORT_THREADS / 32][256];
  int nd = 1 << bits;
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < nd; d += blockDim.x) base[d] = offs[(int64_t)d * nblocks + blockIdx.x];
  int64_t tile0 = (int64_t)blockIdx.x * SORT_TILE;
  for (int c = 0; c < SORT_ITEMS; c++) {
    for (int i = threadIdx.x; i < (SORT_THREADS / 32) * nd; i += blockDim.x) (&wcnt[0][0])[(i / nd) * 256 + (i % nd)] = 0;
    __syncthreads();
    int64_t idx = tile0 + (int64_t)c * SORT_THREADS + threadIdx.x;
    bool valid = idx < n;
    uint32_t k = valid ? keys[idx] : 0u;
    uint32_t d = valid ? ((k >> shift) & (nd - 1)) : 0xFFFFFFFFu;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    int rank_in_warp = __popc(peers & ((1u << lane) - 1));
    int leader = __ffs(peers) - 1;
    if (valid && lane == leader) wcnt[warp][d] = __popc(peers);
    __syncthreads();
    uint32_t pos = 0;
    if (valid) {
      uint32_t before = 0;
      for (int w = 0; w < warp; w++) before += wcnt[w][d];
      pos = base[d] + before + rank_in_warp;
      okeys[pos] = k;
      ovals[pos] = vals[idx];
    }
    __syncthreads();
    for (int dd = threadIdx.x; dd < nd; dd += blockDim.x) {
      uint32_t t = 0;
      for (int w = 0; w < SORT_THREADS / 32; w++) t += wcnt[w][dd];
      base[dd] += t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- scans
template <typename T>
__device__ T block_exclusive_scan(T v, T* smem_warp, T& total) {
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : T(0);
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    smem_warp[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  T warp_prefix = warp ? smem_warp[warp - 1] : T(0);
  total = smem_warp[(blockDim.x >> 5) - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

template <typename T>
__global__ void k_scan_tiles(const T* __restrict__ in, T* __restrict__ out, int64_t n, T* __restrict__ tile_sums) {
  __shared__ T sw[32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  T v[SCAN_ITEMS];
  T s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    v[i] = (base + i < n) ? in[base + i] : T(0);
    s += v[i];
  }
  T total;
  T ex = block_exclusive_scan<T>(s, sw, total);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    if (base + i < n) out[base + i] = ex;
    ex += v[i];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ out, int64_t n, const T* __restrict__ tile_offs) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  T add = tile_offs[blockIdx.x];
  for (int i = threadIdx.x; i < SCAN_TILE; i += blockDim.x)
    if (base + i < n) out[base + i] += add;
}

// Load-time scratch (sort / scan temporaries): grow-only per thread and device, reused in
// stream order, so the sort passes need no allocation or synchronisation of their own.
struct Arena {
  int dev = -1;
  DevBuf buf[6];
  void* get(int i, size_t bytes) {
    StreamScope plain(nullptr, false);  // outlives any one context's stream
    int d = 0;
    cudaGetDevice(&d);
    if (d != dev) {
      for (auto& b : buf) b.reset();
      dev = d;
    }
    if (buf[i].bytes < bytes + 256 && buf[i].alloc(bytes + bytes / 4)) return nullptr;
    return buf[i].p;
  }
};
static thread_local Arena g_arena;

template <typename T>
size_t scan_scratch_elems(int64_t n) {  // sums + offs of every recursion level
  size_t tot = 0;
  for (int64_t t = (n + SCAN_TILE - 1) / SCAN_TILE; t > 1; t = (t + SCAN_TILE - 1) / SCAN_TILE) tot += 2 * t;
  return tot;
}

template <typename T>
cudaError_t exclusive_scan_rec(const T* in, T* out, int64_t n, T* scratch, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    k_scan_tiles<T><<<1, SCAN_THREADS, 0, st>>>(in, out, n, nullptr);
    return cudaGetLastError();
  }
  T* sums = scratch;
  T* offs = scratch + tiles;
  k_scan_tiles<T><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, out, n, sums);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(exclusive_scan_rec<T>(sums, offs, tiles, scratch + 2 * tiles, st));
  k_scan_add<T><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(out, n, offs);
  return cudaGetLastError();
}

// stream-ordered: the scratch lives in the arena slot `slot`
template <typename T>
cudaError_t exclusive_scan_t(const T* in, T* out, int64_t n, cudaStream_t st, int slot = 5) {
  T* scratch = (T*)g_arena.get(slot, std::max<size_t>(scan_scratch_elems<T>(n), 1) * sizeof(T));
  if (!scratch) return cudaErrorMemoryAllocation;
  return exclusive_scan_rec<T>(in, out, n, scratch, st);
}

cudaError_t exclusive_scan_u32(const uint32_t* in, uint32_t* out, int64_t n, cudaStream_t st) {
  return exclusive_scan_t<uint32_t>(in, out, n, st);
}
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t* out, int64_t n, cudaStream_t st) {
  return exclusive_scan_t<int64_t>(in, out, n, st);
}

// n_dev (optional): the number of pairs is *n_dev <= n, known on the device only (n is then the
// capacity; launches are sized by it, so the sort needs no host synchronisation)
cudaError_t radix_sort_pairs(uint32_t* keys, uint32_t* vals, int64_t n, int key_bits, cudaStream_t st,
                             const unsigned long long* n_dev) {
  if (n <= 1 || key_bits <= 0) return cudaSuccess;
  int64_t nblocks = (n + SORT_TILE - 1) / SORT_TILE;
  uint32_t* k2 = (uint32_t*)g_arena.get(0, n * 4);
  uint32_t* v2 = (uint32_t*)g_arena.get(1, n * 4);
  uint32_t* hist = (uint32_t*)g_arena.get(2, 256 * nblocks * 4);
  uint32_t* offs = (uint32_t*)g_arena.get(3, 256 * nblocks * 4);
  if (!k2 || !v2 || !hist || !offs) return cudaErrorMemoryAllocation;
  uint32_t *ka = keys, *va = vals, *kb = k2, *vb = v2;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8) {
    int bits = std::min(8, key_bits - shift);
    k_radix_hist<<<(unsigned)nblocks, SORT_THREADS, 0, st>>>(ka, n, n_dev, shift, bits, hist, (int)nblocks);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(exclusive_scan_t<uint32_t>(hist, offs, (int64_t)(1 << bits) * nblocks, st, 4));
    k_radix_scatter<<<(unsigned)nblocks, SORT_THREADS, 0, st>>>(ka, va, kb, vb, n, n_dev, shift, bits, offs,
                                                                 (int)nblocks);
    CUDA_TRY(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
    passes++;
  }
  if (passes & 1) {
    CUDA_TRY(cudaMemcpyAsync(keys, ka, n * 4, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(vals, va, n * 4, cudaMemcpyDeviceToDevice, st));
  }
  return cudaSuccess;  // stream-ordered; callers synchronise before reading results on the host
}

// ---------------------------------------------------------------- small kernels
__global__ void k_iota(uint32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (uint32_t)i;
}

// int32 -> order-preserving u32 (flip the sign bit)
__global__ void k_i32_to_key(const int32_t* __restrict__ in, const uint32_t* __restrict__ perm, uint32_t* out,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = perm ? in[perm[i]] : in[i];
    out[i] = (uint32_t)v ^ 0x80000000u;
  }
}

__global__ void k_gather_u32(const uint32_t* __restrict__ in, const uint32_t* __restrict__ perm, uint32_t* out,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

template <typename T>
__global__ void k_gather(const T* __restrict__ in, const uint32_t* __restrict__ perm, T* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[perm[i]];
}

// flags[i] = 1 if sorted key i starts a new distinct value
__global__ void k_head_flags(const uint32_t* __restrict__ sk, uint32_t* flags, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1u : 0u;
}

// dense id of sorted element i = (#heads up to i) - 1; dict[id] = value at heads
__global__ void k_dense_from_heads(const uint32_t* __restrict__ sk, const uint32_t* __restrict__ flags,
                                   const uint32_t* __restrict__ excl, int32_t* dense_sorted, int32_t* dict,
                                   int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t id = excl[i] + flags[i] - 1;
    if (dense_sorted) dense_sorted[i] = (int32_t)id;
    if (flags[i]) dict[id] = (int32_t)(sk[i] ^ 0x80000000u);
  }
}

// binary search of v in the sorted dictionary: dense id or -1 (dangling)
__global__ void k_lookup(const int32_t* __restrict__ vals, int64_t n, const int32_t* __restrict__ dict, int64_t nd,
                         int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = vals[i];
    int64_t lo = 0, hi = nd;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (dict[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    out[i] = (lo < nd && dict[lo] == v) ? (int32_t)lo : -1;
  }
}

__global__ void k_keep_flags(const int32_t* const* __restrict__ fks, int nfk, uint32_t* flags, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t keep = 1;
    for (int j = 0; j < nfk; j++)
      if (fks[j][i] < 0) keep = 0;
    flags[i] = keep;
  }
}

__global__ void k_compact_index(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ excl,
                                uint32_t* __restrict__ idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) idx[excl[i]] = (uint32_t)i;
}

// segment offsets for a relation sorted by dense key: off[k] = first row with key >= k
__global__ void k_seg_offsets(const int32_t* __restrict__ dkey, int64_t n, int64_t nkeys, int64_t* off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t prev = (i == 0) ? -1 : dkey[i - 1];
    int64_t cur = (i == n) ? nkeys : dkey[i];
    for (int64_t k = prev + 1; k <= cur; k++) off[k] = i;
  }
}

static unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (unsigned)g;
}

cudaError_t iota_u32(uint32_t* a, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_iota<<<grid_for(n), 256, 0, st>>>(a, n);
  return cudaGetLastError();
}

cudaError_t gather_bytes(const void* in, const uint32_t* perm, void* out, int64_t n, int elem_bytes, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (elem_bytes == 4) k_gather<uint32_t><<<grid_for(n), 256, 0, st>>>((const uint32_t*)in, perm, (uint32_t*)out, n);
  else if (elem_bytes == 8) k_gather<uint64_t><<<grid_for(n), 256, 0, st>>>((const uint64_t*)in, perm, (uint64_t*)out, n);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

// Dictionary-encode an int32 column: dict = sorted distinct values, codes[i] = rank.
cudaError_t dict_encode_i32(const int32_t* col, int64_t n, DevBuf& dict, int64_t& ndict, DevBuf* codes,
                            cudaStream_t st) {
  ndict = 0;
  if (n <= 0) {
    CUDA_TRY(dict.alloc(4));
    if (codes) CUDA_TRY(codes->alloc(4));
    return cudaSuccess;
  }
  DevBuf sk, perm, flags, excl, dense_sorted;
  CUDA_TRY(sk.alloc(n * 4));
  CUDA_TRY(perm.alloc(n * 4));
  CUDA_TRY(flags.alloc(n * 4));
  CUDA_TRY(excl.alloc(n * 4));
  k_i32_to_key<<<grid_for(n), 256, 0, st>>>(col, nullptr, sk.as<uint32_t>(), n);
  CUDA_TRY(iota_u32(perm.as<uint32_t>(), n, st));
  CUDA_TRY(radix_sort_pairs(sk.as<uint32_t>(), perm.as<uint32_t>(), n, 32, st));
  k_head_flags<<<grid_for(n), 256, 0, st>>>(sk.as<uint32_t>(), flags.as<uint32_t>(), n);
  CUDA_TRY(exclusive_scan_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), n, st));
  uint32_t last_ex = 0, last_f = 0;
  CUDA_TRY(cudaMemcpyAsync(&last_ex, excl.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&last_f, flags.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  ndict = (int64_t)last_ex + last_f;
  CUDA_TRY(dict.alloc(ndict * 4));
  CUDA_TRY(dense_sorted.alloc(n * 4));
  k_dense_from_heads<<<grid_for(n), 256, 0, st>>>(sk.as<uint32_t>(), flags.as<uint32_t>(), excl.as<uint32_t>(),
                                                  dense_sorted.as<int32_t>(), dict.as<int32_t>(), n);
  CUDA_TRY(cudaGetLastError());
  if (codes) {
    CUDA_TRY(codes->alloc(n * 4));
    k_lookup<<<grid_for(n), 256, 0, st>>>(col, n, dict.as<int32_t>(), ndict, codes->as<int32_t>());
    CUDA_TRY(cudaGetLastError());
  }
  return cudaStreamSynchronize(st);
}

// ---- two-attribute join keys (a, b): order-preserving u64 images, dictionary over the pairs
__global__ void k_pair_key(const int32_t* __restrict__ a, const int32_t* __restrict__ b, uint64_t* __restrict__ out,
                           int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = ((uint64_t)((uint32_t)a[i] ^ 0x80000000u) << 32) | (uint64_t)((uint32_t)b[i] ^ 0x80000000u);
}
__global__ void k_split_u64(const uint64_t* __restrict__ in, const uint32_t* __restrict__ perm, uint32_t* __restrict__ lo,
                            uint32_t* __restrict__ hi, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[perm ? perm[i] : i];
    if (lo) lo[i] = (uint32_t)v;
    if (hi) hi[i] = (uint32_t)(v >> 32);
  }
}
__global__ void k_pair_heads(const uint64_t* __restrict__ in, const uint32_t* __restrict__ perm, uint32_t* flags,
                             int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = (i == 0 || in[perm[i]] != in[perm[i - 1]]) ? 1u : 0u;
}
__global__ void k_pair_dict(const uint64_t* __restrict__ in, const uint32_t* __restrict__ perm,
                            const uint32_t* __restrict__ flags, const uint32_t* __restrict__ excl, uint64_t* dict,
                            int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (flags[i]) dict[excl[i]] = in[perm[i]];
}
__global__ void k_lookup_u64(const uint64_t* __restrict__ vals, int64_t n, const uint64_t* __restrict__ dict, int64_t nd,
                             int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = vals[i];
    int64_t lo = 0, hi = nd;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (dict[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    out[i] = (lo < nd && dict[lo] == v) ? (int32_t)lo : -1;
  }
}

cudaError_t dict_encode_pair(const int32_t* a, const int32_t* b, int64_t n, DevBuf& dict, int64_t& ndict, DevBuf* codes,
                             cudaStream_t st) {
  ndict = 0;
  if (n <= 0) {
    CUDA_TRY(dict.alloc(8));
    if (codes) CUDA_TRY(codes->alloc(4));
    return cudaSuccess;
  }
  DevBuf key, k32, perm, flags, excl;
  CUDA_TRY(key.alloc(n * 8));
  CUDA_TRY(k32.alloc(n * 4));
  CUDA_TRY(perm.alloc(n * 4));
  CUDA_TRY(flags.alloc(n * 4));
  CUDA_TRY(excl.alloc(n * 4));
  k_pair_key<<<grid_for(n), 256, 0, st>>>(a, b, key.as<uint64_t>(), n);
  CUDA_TRY(iota_u32(perm.as<uint32_t>(), n, st));
  // LSD over the two 32-bit halves: low word, then (stably) high word
  k_split_u64<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), nullptr, k32.as<uint32_t>(), nullptr, n);
  CUDA_TRY(radix_sort_pairs(k32.as<uint32_t>(), perm.as<uint32_t>(), n, 32, st));
  k_split_u64<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), perm.as<uint32_t>(), nullptr, k32.as<uint32_t>(), n);
  CUDA_TRY(radix_sort_pairs(k32.as<uint32_t>(), perm.as<uint32_t>(), n, 32, st));
  k_pair_heads<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), perm.as<uint32_t>(), flags.as<uint32_t>(), n);
  CUDA_TRY(exclusive_scan_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), n, st));
  uint32_t last_ex = 0, last_f = 0;
  CUDA_TRY(cudaMemcpyAsync(&last_ex, excl.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&last_f, flags.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  ndict = (int64_t)last_ex + last_f;
  CUDA_TRY(dict.alloc(ndict * 8));
  k_pair_dict<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), perm.as<uint32_t>(), flags.as<uint32_t>(),
                                           excl.as<uint32_t>(), dict.as<uint64_t>(), n);
  CUDA_TRY(cudaGetLastError());
  if (codes) {
    CUDA_TRY(codes->alloc(n * 4));
    k_lookup_u64<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), n, dict.as<uint64_t>(), ndict, codes->as<int32_t>());
    CUDA_TRY(cudaGetLastError());
  }
  return cudaStreamSynchronize(st);
}

cudaError_t lookup_dense_pair(const int32_t* a, const int32_t* b, int64_t n, const uint64_t* dict, int64_t nd,
                              int32_t* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  DevBuf key;
  CUDA_TRY(key.alloc(n * 8));
  k_pair_key<<<grid_for(n), 256, 0, st>>>(a, b, key.as<uint64_t>(), n);
  k_lookup_u64<<<grid_for(n), 256, 0, st>>>(key.as<uint64_t>(), n, dict, nd, out);
  return cudaGetLastError();
}

cudaError_t lookup_dense(const int32_t* vals, int64_t n, const int32_t* dict, int64_t nd, int32_t* out,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_lookup<<<grid_for(n), 256, 0, st>>>(vals, n, dict, nd, out);
  return cudaGetLastError();
}

// Row filter: keep rows whose every fk is >= 0. Returns the kept-row index list.
cudaError_t keep_rows(const std::vector<const int32_t*>& fks, int64_t n, DevBuf& idx, int64_t& nkeep,
                      cudaStream_t st) {
  nkeep = n;
  if (fks.empty() || n <= 0) return cudaSuccess;
  DevBuf dfks, flags, excl;
  CUDA_TRY(dfks.alloc(fks.size() * sizeof(void*)));
  CUDA_TRY(cudaMemcpyAsync(dfks.p, fks.data(), fks.size() * sizeof(void*), cudaMemcpyHostToDevice, st));
  CUDA_TRY(flags.alloc(n * 4));
  CUDA_TRY(excl.alloc(n * 4));
  k_keep_flags<<<grid_for(n), 256, 0, st>>>((const int32_t* const*)dfks.p, (int)fks.size(), flags.as<uint32_t>(), n);
  CUDA_TRY(exclusive_scan_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), n, st));
  uint32_t le = 0, lf = 0;
  CUDA_TRY(cudaMemcpyAsync(&le, excl.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&lf, flags.as<uint32_t>() + n - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  nkeep = (int64_t)le + lf;
  CUDA_TRY(idx.alloc(std::max<int64_t>(nkeep, 1) * 4));
  k_compact_index<<<grid_for(n), 256, 0, st>>>(flags.as<uint32_t>(), excl.as<uint32_t>(), idx.as<uint32_t>(), n);
  CUDA_TRY(cudaGetLastError());
  return cudaStreamSynchronize(st);
}

// Stable sort permutation of n rows by a dense int32 key in [0, nkeys).
cudaError_t sort_perm_by_dense(const int32_t* dense, int64_t n, int64_t nkeys, DevBuf& perm, cudaStream_t st) {
  CUDA_TRY(perm.alloc(std::max<int64_t>(n, 1) * 4));
  if (n <= 0) return cudaSuccess;
  CUDA_TRY(iota_u32(perm.as<uint32_t>(), n, st));
  DevBuf k;
  CUDA_TRY(k.alloc(n * 4));
  CUDA_TRY(cudaMemcpyAsync(k.p, dense, n * 4, cudaMemcpyDeviceToDevice, st));
  int bits = 0;
  while ((int64_t(1) << bits) < nkeys) bits++;
  CUDA_TRY(radix_sort_pairs(k.as<uint32_t>(), perm.as<uint32_t>(), n, bits, st));
  return cudaStreamSynchronize(st);
}

// Composite LSD sort: permutation sorting rows by (keys[0], keys[1], ...) with
// keys[0] most significant; each key is dense in [0, nkeys[j]).
cudaError_t sort_perm_composite(const std::vector<const int32_t*>& keys, const std::vector<int64_t>& nkeys, int64_t n,
                                DevBuf& perm, cudaStream_t st) {
  CUDA_TRY(perm.alloc(std::max<int64_t>(n, 1) * 4));
  if (n <= 0) return cudaSuccess;
  CUDA_TRY(iota_u32(perm.as<uint32_t>(), n, st));
  DevBuf k;
  CUDA_TRY(k.alloc(n * 4));
  for (int j = (int)keys.size() - 1; j >= 0; j--) {
    k_gather_u32<<<grid_for(n), 256, 0, st>>>((const uint32_t*)keys[j], perm.as<uint32_t>(), k.as<uint32_t>(), n);
    CUDA_TRY(cudaGetLastError());
    int bits = 0;
    while ((int64_t(1) << bits) < nkeys[j]) bits++;
    CUDA_TRY(radix_sort_pairs(k.as<uint32_t>(), perm.as<uint32_t>(), n, bits, st));
  }
  return cudaStreamSynchronize(st);
}

cudaError_t segment_offsets(const int32_t* dkey, int64_t n, int64_t nkeys, DevBuf& off, cudaStream_t st) {
  CUDA_TRY(off.alloc((nkeys + 1) * 8));
  if (n == 0) {
    CUDA_TRY(cudaMemsetAsync(off.p, 0, (nkeys + 1) * 8, st));
    return cudaStreamSynchronize(st);
  }
  k_seg_offsets<<<grid_for(n + 1), 256, 0, st>>>(dkey, n, nkeys, off.as<int64_t>());
  CUDA_TRY(cudaGetLastError());
  return cudaStreamSynchronize(st);
}

}  // namespace lmfao

namespace lmfao {
cudaError_t ensure_smem_attr(const void* func, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{dev, func}];
  if (smem > cur) {
    CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cur = smem;
  }
  return cudaSuccess;
}

static int64_t g_launches = 0;
int launches_counter_reset() {
  int r = (int)g_launches;
  g_launches = 0;
  return r;
}
void launches_add(int n) { g_launches += n; }
}  // namespace lmfao
