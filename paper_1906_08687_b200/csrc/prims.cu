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
constexpr int SORT_ITEMS = 16;                      // elements per thread per tile
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 4096
constexpr int SORT_WARP_ITEMS = 32 * SORT_ITEMS;     // a warp's slice of the tile
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// ---------------------------------------------------------------- radix sort
// One pass = histogram per tile, one exclusive scan over hist[digit * ntiles + tile] (digit-
// major, so the scan gives every (digit, tile) its output offset and the sort is stable across
// tiles), then the scatter.  The scatter ranks a tile's elements locally (each warp walks its
// 512-element slice in order, 32 at a time: equal digits by __match_any_sync, running counts
// per warp in shared memory), sorts the tile by digit in shared memory, and writes it out in
// that order, so a digit's elements leave as one contiguous, coalesced run per tile.
#ifndef SORT_HIST_EARLY
#define SORT_HIST_EARLY 1  // 1: k_radix_hist loads a warp's 16 keys per lane before its table updates (C5 run: 9.35 -> 9.18 ms)
#endif
#ifndef SORT_MINB
#define SORT_MINB 4  // resident CTAs per SM the register budget is sized for (C5 run, with the early hist loads: 3 9.18, 4 9.03, 5 9.29, 6 9.44 ms)
#endif
#ifndef SORT_VALS_EARLY
#define SORT_VALS_EARLY 0  // 1: a tile's payloads loaded with its keys (more live registers)
#endif
__global__ void __launch_bounds__(SORT_THREADS) k_radix_hist(const uint32_t* __restrict__ keys, int64_t n,
                                                             const unsigned long long* n_dev, int shift, int bits,
                                                             uint32_t* __restrict__ hist, int nblocks) {
  __shared__ uint32_t h[SORT_THREADS / 32][256];
  if (n_dev) n = min(n, (int64_t)*n_dev);  // device-side size (n = capacity)
  const int nd = 1 << bits, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (SORT_THREADS / 32) * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * SORT_TILE + (int64_t)warp * SORT_WARP_ITEMS;
#if SORT_HIST_EARLY
  uint32_t kk[SORT_ITEMS];  // every key of the warp's slice in flight before the table updates
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    const int64_t idx = base + j * 32 + lane;
    kk[j] = idx < n ? keys[idx] : 0u;
  }
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++)
    if (base + j * 32 + lane < n) atomicAdd(&h[warp][(kk[j] >> shift) & (nd - 1)], 1u);
#else
#pragma unroll 4
  for (int j = 0; j < SORT_ITEMS; j++) {  // per-warp tables (measured: __match_any_sync here is 2x slower)
    const int64_t idx = base + j * 32 + lane;
    if (idx < n) atomicAdd(&h[warp][(keys[idx] >> shift) & (nd - 1)], 1u);
  }
#endif
  __syncthreads();
  for (int d = threadIdx.x; d < nd; d += blockDim.x) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < SORT_THREADS / 32; w++) t += h[w][d];
    hist[(int64_t)d * nblocks + blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(SORT_THREADS, SORT_MINB) k_radix_scatter(const uint32_t* __restrict__ keys,
                                                                const uint32_t* __restrict__ vals,
                                                                uint32_t* __restrict__ okeys, uint32_t* __restrict__ ovals,
                                                                int64_t n, const unsigned long long* n_dev, int shift,
                                                                int bits, const uint32_t* __restrict__ offs, int nblocks) {
  __shared__ uint32_t skey[SORT_TILE];
  __shared__ uint32_t sval[SORT_TILE];
  __shared__ uint32_t wcnt[SORT_THREADS / 32][256];  // per warp: running count, then the warp's offset in the digit
  __shared__ uint32_t dstart[256];                  // the digit's first position in the sorted tile
  __shared__ uint32_t gbase[256];                   // the digit's first output position of this tile
  __shared__ uint32_t wsum[SORT_THREADS / 32];
  if (n_dev) n = min(n, (int64_t)*n_dev);
  const int nd = 1 << bits, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tile0 = (int64_t)blockIdx.x * SORT_TILE;
  if (tile0 >= n) return;
  const int nvalid = (int)min((int64_t)SORT_TILE, n - tile0);
  for (int i = threadIdx.x; i < (SORT_THREADS / 32) * 256; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < nd; d += blockDim.x) gbase[d] = offs[(int64_t)d * nblocks + blockIdx.x];
  __syncthreads();
  uint32_t k[SORT_ITEMS], rk[SORT_ITEMS];
#if SORT_VALS_EARLY
  uint32_t pv[SORT_ITEMS];
#endif
  const int wbase = warp * SORT_WARP_ITEMS;
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    const int e = wbase + j * 32 + lane;
    const bool ok = e < nvalid;
    k[j] = ok ? keys[tile0 + e] : 0u;
#if SORT_VALS_EARLY
    pv[j] = ok ? vals[tile0 + e] : 0u;
#endif
  }
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    const bool ok = wbase + j * 32 + lane < nvalid;
    const uint32_t d = ok ? (k[j] >> shift) & (nd - 1) : 0x100u;  // invalid: a digit of their own
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const uint32_t before = ok ? wcnt[warp][d] : 0u;
    rk[j] = before + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) wcnt[warp][d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: the warps' offsets within the digit, the digit's total; then the digits' starts
  uint32_t tot = 0;
  const int d = threadIdx.x;  // SORT_THREADS == 256 digits at most
  if (d < nd) {
#pragma unroll
    for (int w = 0; w < SORT_THREADS / 32; w++) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = tot;
      tot += c;
    }
  }
  uint32_t x = tot;  // block exclusive scan of the totals over the 256 digits
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; w++) wpre += wsum[w];
  if (d < nd) dstart[d] = wpre + x - tot;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < SORT_ITEMS; j++) {
    if (wbase + j * 32 + lane < nvalid) {
      const uint32_t dd = (k[j] >> shift) & (nd - 1);
      const uint32_t pos = dstart[dd] + wcnt[warp][dd] + rk[j];
      skey[pos] = k[j];
#if SORT_VALS_EARLY
      sval[pos] = pv[j];
#else
      sval[pos] = vals[tile0 + wbase + j * 32 + lane];  // read again (cached): fewer live registers
#endif
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nvalid; i += SORT_THREADS) {
    const uint32_t kk = skey[i];
    const uint32_t dd = (kk >> shift) & (nd - 1);
    const uint32_t o = gbase[dd] + (uint32_t)i - dstart[dd];
    okeys[o] = kk;
    ovals[o] = sval[i];
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
  constexpr int VEC = 16 / sizeof(T);  // 16-byte accesses when the thread's items are whole and aligned
  const bool vec = base + SCAN_ITEMS <= n && ((reinterpret_cast<uintptr_t>(in + base) | reinterpret_cast<uintptr_t>(out + base)) & 15) == 0;
  if (vec) {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i += VEC) *reinterpret_cast<int4*>(&v[i]) = *reinterpret_cast<const int4*>(in + base + i);
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) v[i] = (base + i < n) ? in[base + i] : T(0);
  }
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) s += v[i];
  T total;
  T ex = block_exclusive_scan<T>(s, sw, total);
  if (vec) {
    T o[SCAN_ITEMS];
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      o[i] = ex;
      ex += v[i];
    }
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i += VEC) *reinterpret_cast<int4*>(out + base + i) = *reinterpret_cast<const int4*>(&o[i]);
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) {
      if (base + i < n) out[base + i] = ex;
      ex += v[i];
    }
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ out, int64_t n, const T* __restrict__ tile_offs) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  const T add = tile_offs[blockIdx.x];
  constexpr int VEC = 16 / sizeof(T);
  if (base + SCAN_TILE <= n && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
    for (int i = threadIdx.x * VEC; i < SCAN_TILE; i += blockDim.x * VEC) {
      T w[VEC];
      *reinterpret_cast<int4*>(w) = *reinterpret_cast<const int4*>(out + base + i);
#pragma unroll
      for (int k = 0; k < VEC; k++) w[k] += add;
      *reinterpret_cast<int4*>(out + base + i) = *reinterpret_cast<const int4*>(w);
    }
    return;
  }
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
    k_scan_tiles<T><<<1, SCAN_THREADS, 0, st>>>(in, out, n, nullptr); launches_add(1);
    return cudaGetLastError();
  }
  T* sums = scratch;
  T* offs = scratch + tiles;
  k_scan_tiles<T><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(in, out, n, sums); launches_add(1);
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(exclusive_scan_rec<T>(sums, offs, tiles, scratch + 2 * tiles, st));
  k_scan_add<T><<<(unsigned)tiles, SCAN_THREADS, 0, st>>>(out, n, offs); launches_add(1);
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
    k_radix_hist<<<(unsigned)nblocks, SORT_THREADS, 0, st>>>(ka, n, n_dev, shift, bits, hist, (int)nblocks); launches_add(1);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(exclusive_scan_t<uint32_t>(hist, offs, (int64_t)(1 << bits) * nblocks, st, 4));
    k_radix_scatter<<<(unsigned)nblocks, SORT_THREADS, 0, st>>>(ka, va, kb, vb, n, n_dev, shift, bits, offs,
                                                                 (int)nblocks); launches_add(1);
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
  k_iota<<<grid_for(n), 256, 0, st>>>(a, n); launches_add(1);
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
