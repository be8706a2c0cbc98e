// generic.cu — the general (interpreted) evaluation path for any batch the
// planner accepts: view build (b) per non-root node and the root scan (c) for
// no-group-by and dense group-by queries.  It is the coverage path; the
// specialised kernels (gram.cu, hist.cu) are the performance path for the
// BASELINE.json workloads.
//
// Decomposition (SURVEY §8 notation): for a product p split by the
// planner into the root's own factors p_F and one view slot per child c,
//     Σ_{joined t} p(t) = Σ_{f ∈ root} coef · p_F(f) · Π_c V_c[k_c(f)][slot_c(p)],
//     V_c[k][s] = Σ_{d ∈ c, key(d)=k} p_{c,s}(d) · Π_e V_e[k_e(d)][slot_e(s)]   (Ex. 4.1).
// Slot 0 of every view is the count (empty product), which gives bag semantics.
#include "internal.h"

namespace lmfao {

__device__ __forceinline__ double load_col(const NodeArgs& a, int col, int64_t row) {
  return a.col_is_int[col] ? (double)((const int32_t*)a.cols[col])[row] : ((const double*)a.cols[col])[row];
}

__device__ __forceinline__ double apply_factor(int kind, double x, double t) {
  switch (kind) {
    case LMFAO_F_IDENT: return x;
    case LMFAO_F_LT: return x < t ? 1.0 : 0.0;
    case LMFAO_F_LE: return x <= t ? 1.0 : 0.0;
    case LMFAO_F_GT: return x > t ? 1.0 : 0.0;
    case LMFAO_F_GE: return x >= t ? 1.0 : 0.0;
    case LMFAO_F_EQ: return x == t ? 1.0 : 0.0;
    case LMFAO_F_NE: return x != t ? 1.0 : 0.0;
    case LMFAO_F_IN: return (x >= 0.0 && x <= 52.0 && x == floor(x) && ((unsigned long long)t >> (int)x) & 1ull) ? 1.0 : 0.0;
    default: return t;  // CONST
  }
}

// Evaluates one output (sum of terms) at `row`; kk[c] = dense key of child c.
__device__ double eval_output(const NodeArgs& a, int64_t row, const int32_t* kk, const int32_t* __restrict__ ip,
                              const double* __restrict__ dp) {
  int nt = *ip++;
  double sum = 0.0;
  for (int t = 0; t < nt; t++) {
    int nown = *ip++;
    double v = *dp++;
    for (int f = 0; f < nown; f++) {
      int kind = *ip++;
      int col = *ip++;
      double prm = *dp++;
      double x = kind == LMFAO_F_CONST ? 0.0 : load_col(a, col, row);
      v = v * apply_factor(kind, x, prm);
    }
    for (int c = 0; c < a.nchild; c++) {
      int slot = *ip++;
      if (slot >= 0) v = v * a.V[c][(int64_t)kk[c] * a.W[c] + slot];  // -1: the child is left out
    }
    sum += v;
  }
  return sum;
}

// View build (b): V[k][s] = Σ_{rows d with dense key k} slot_s(d).  The child is sorted by
// its dense key (prepare), so a key's rows are contiguous.  Each warp takes a contiguous range
// of 32-row blocks (lane = row) and sums every slot over the runs of equal keys with a
// segmented warp scan; a run that reaches the end of a block is carried (per slot, in shared
// memory) into the next block, so a Zipf-hot key with thousands of rows costs one update, not
// one per row or per block.  Runs that start and end inside the warp's range are stored
// plainly (no other warp has rows of their key); runs touching the range's edges are added
// atomically.  VAL(row, slot, lane) gives a slot's value for a row (interpreted or linear).
constexpr int VB_WARPS = 8;
constexpr int VB_MAXSLOT = 64;

// lacc (optional, [nslots][32] per warp): lane-private sums of the carried run in blocks where
// no run starts, so a long run costs one add per row and slot, reduced once when it ends.
template <typename Val>
__device__ __forceinline__ void view_seg_warp(int64_t nrows, const int32_t* __restrict__ dense_key, int nslots,
                                              double* __restrict__ V, double* carry, double* lacc, Val&& val) {
  const int lane = threadIdx.x & 31;
  const int64_t nblk = (nrows + 31) / 32;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t b0 = nblk * gw / nw, b1 = nblk * (gw + 1) / nw;
  const int64_t rend = min(nrows, 32 * b1);
  bool cstart = false;  // the carried run (if any) started inside this warp's range
  int last = b0 > 0 ? dense_key[32 * b0 - 1] : -2;  // key of the row before the current block
  for (int s = lane; s < nslots; s += 32) carry[s] = 0.0;  // (a run entering the range starts from 0)
  if (lacc)
    for (int s = 0; s < nslots; s++) lacc[s * 32 + lane] = 0.0;
  bool ldirty = false;  // lacc holds part of the carried run
  __syncwarp();
  auto wsum = [&](double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  for (int64_t b = b0; b < b1; b++) {
    const int64_t row = 32 * b + lane;
    const bool v = row < rend;
    const int key = v ? dense_key[row] : -1;
    int prev = __shfl_up_sync(0xffffffffu, key, 1);
    if (lane == 0) prev = last;
    const int next = __shfl_down_sync(0xffffffffu, key, 1);
    const unsigned heads = __ballot_sync(0xffffffffu, v && key != prev);  // rows that start a run
    const unsigned upto = heads & ((2u << lane) - 1u);
    const int s0 = upto ? 31 - __clz(upto) : 0;
    const int64_t nrem = rend - 32 * b;
    const int nv = nrem < 32 ? (int)nrem : 32;
    const bool lastlane = lane == nv - 1;
    const bool tail = v && (lastlane || next != key);
    // the block's last run goes on past this block (into this range: carry; past it: atomic)
    const bool cont = tail && lastlane && row + 1 < nrows && dense_key[row + 1] == key;
    const bool carry_on = cont && row + 1 < rend;
    const bool first_seg = upto == 0;          // the run carried from the previous block
    const bool started_in = first_seg ? cstart : true;
    if (lacc && heads == 0) {  // the carried run goes on through the block: lane-private sums
      const bool c_on = __any_sync(0xffffffffu, carry_on), c_any = __any_sync(0xffffffffu, cont);
      for (int s = 0; s < nslots; s++) lacc[s * 32 + lane] += v ? val(row, s) : 0.0;
      ldirty = true;
      if (!c_on) {  // the run ends with this block (or leaves the range): emit it
        for (int s = 0; s < nslots; s++) {
          const double t = wsum(lacc[s * 32 + lane]) + carry[s];
          lacc[s * 32 + lane] = 0.0;
          if (lane == nv - 1) {
            double* dst = &V[(int64_t)key * nslots + s];
            if (cstart && !c_any) *dst = t;
            else gred_add(dst, t);
            carry[s] = 0.0;
          }
        }
        ldirty = false;
        cstart = false;
      }
      __syncwarp();
      last = __shfl_sync(0xffffffffu, key, nv - 1);
      continue;
    }
    if (ldirty) {  // a run starts in this block: fold the lane-private sums into the carry
      for (int s = 0; s < nslots; s++) {
        const double t = wsum(lacc[s * 32 + lane]);
        lacc[s * 32 + lane] = 0.0;
        if (lane == 0) carry[s] += t;
      }
      ldirty = false;
      __syncwarp();
    }
    for (int s = 0; s < nslots; s++) {
      double x = v ? val(row, s) : 0.0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, x, d);
        if (lane - d >= s0) x += u;
      }
      if (tail) {
        if (first_seg) x += carry[s];
        if (carry_on) {
          carry[s] = x;
        } else {
          double* dst = &V[(int64_t)key * nslots + s];
          if (started_in && !cont) *dst = x;  // the run lies inside this warp's range
          else gred_add(dst, x);
        }
      }
      __syncwarp();
    }
    // the carried run of the next block: the last run of this one, if it goes on
    const unsigned cm = __ballot_sync(0xffffffffu, carry_on);
    if (cm) {
      const unsigned up_l = __shfl_sync(0xffffffffu, upto, __ffs(cm) - 1);
      cstart = up_l ? true : cstart;
    } else {
      cstart = false;
    }
    last = __shfl_sync(0xffffffffu, key, nv - 1);
  }
}

__global__ void __launch_bounds__(VB_WARPS * 32) k_view_build(NodeArgs a, const int32_t* __restrict__ dense_key,
                                                              const int32_t* __restrict__ prog_i,
                                                              const double* __restrict__ prog_d,
                                                              const int32_t* __restrict__ ioff,
                                                              const int32_t* __restrict__ doff, int nslots,
                                                              double* __restrict__ V, int use_lacc) {
  extern __shared__ double vcarry[];  // [VB_WARPS][nslots] (+ [VB_WARPS][nslots][32] lane sums)
  double* carry = vcarry + (threadIdx.x >> 5) * nslots;
  double* lacc = use_lacc ? vcarry + VB_WARPS * nslots + (threadIdx.x >> 5) * nslots * 32 : nullptr;
  int32_t kk[MAX_CHILD];
  int64_t krow = -1;
  view_seg_warp(a.nrows, dense_key, nslots, V, carry, lacc, [&](int64_t row, int s) {
    if (row != krow) {
      for (int c = 0; c < a.nchild; c++) kk[c] = a.fk[c][row];
      krow = row;
    }
    return eval_output(a, row, kk, prog_i + ioff[s], prog_d + doff[s]);
  });
}

// Linear slots of a leaf child (every slot a product of at most two identity factors on the
// child's own columns): the same segmented pass with the slot values read straight from the
// columns (no interpreter).
__global__ void __launch_bounds__(VB_WARPS * 32) k_view_lin(const __grid_constant__ ViewLinArgs a,
                                                            const int32_t* __restrict__ dense_key,
                                                            double* __restrict__ V) {
  extern __shared__ double lsm[];  // [VB_WARPS][nslots] carries, [VB_WARPS][nslots][32] lane sums
  double* carry = lsm + (threadIdx.x >> 5) * a.nslots;
  double* lacc = lsm + VB_WARPS * a.nslots + (threadIdx.x >> 5) * a.nslots * 32;
  auto col = [&](const void* p, int is_int, int64_t row) -> double {
    if (!p) return 1.0;
    return is_int ? (double)reinterpret_cast<const int32_t*>(p)[row] : reinterpret_cast<const double*>(p)[row];
  };
  view_seg_warp(a.nrows, dense_key, a.nslots, V, carry, lacc, [&](int64_t row, int s) {
    return col(a.ca[s], a.ia[s], row) * col(a.cb[s], a.ib[s], row);
  });
}

// k_view_lin for the common shape — every slot the count or one fp64 column (at most 16
// column slots, at most one count: the (b) view bench; many-to-many children of covariance
// batches): the same segmented pass and the same store/RED rule, in registers, without
// per-slot branches.  Ranges of VLF_CHUNK blocks are dealt round-robin to the warps (Zipf-
// hot keys make some ranges cheap and others expensive: interleaving balances them).  The
// child is sorted by key, so a range whose first and last rows have the same key is one run
// segment: its columns are summed as a stream (16-byte loads, no per-block key logic) — most
// rows of a Zipf-skewed child are in such ranges.  Other ranges go block by block (segmented
// warp sums over the runs of equal keys, lane-private sums while no run starts), the next
// block's key and values loaded before this one is processed.
constexpr int VLF_CHUNK = 16;  // 32-row blocks per range
struct ViewFastArgs {
  int64_t nrows;
  const double* col[16];  // the column slots' columns, in kernel order
  int8_t vslot[17];       // kernel slot s -> V column (the count, if any, is kernel slot NC)
  int nslots;             // V's row width
};
// Sums over the warp of NS <= 16 lane values at once by recursive halving (16 shuffles instead
// of 5 per value): afterwards lanes l and l ^ 1 hold the total of value vl_index(l).
__device__ __forceinline__ int vl_index(int l) { return ((l >> 4) & 1) * 8 + ((l >> 3) & 1) * 4 + ((l >> 2) & 1) * 2 + ((l >> 1) & 1); }
template <int NS>
__device__ __forceinline__ double warp_sums16(const double (&x)[NS], int lane) {
  double v[16];
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = i < NS ? x[i] : 0.0;
#pragma unroll
  for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < h; i++) {
      const double send = up ? v[i] : v[h + i];
      const double keep = up ? v[h + i] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}
template <int NC, bool CNT>
__global__ void __launch_bounds__(256) k_view_lin_fast(const __grid_constant__ ViewFastArgs a,
                                                       const int32_t* __restrict__ dense_key,
                                                       double* __restrict__ V) {
  constexpr int NS = NC + (CNT ? 1 : 0);
  const int lane = threadIdx.x & 31;
  const int64_t nrows = a.nrows, nblk = (nrows + 31) / 32;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nch = (nblk + VLF_CHUNK - 1) / VLF_CHUNK;
  auto wsum = [](double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  auto emit = [&](int key, int s, double t, bool store) {
    double* dst = &V[(int64_t)key * a.nslots + a.vslot[s]];
    if (store) *dst = t;
    else gred_add(dst, t);
  };
  // a range's edge keys (lanes 0-3): the row before it, its first and last rows, the row
  // after it; loaded one range ahead
  auto edge = [&](int64_t ch) -> int {
    if (ch >= nch || lane >= 4) return -4;
    const int64_t e0 = ch * VLF_CHUNK, e1 = min(nblk, e0 + VLF_CHUNK), r0 = 32 * e0, re = min(nrows, 32 * e1);
    if (lane == 0) return r0 > 0 ? dense_key[r0 - 1] : -2;
    if (lane == 1) return dense_key[r0];
    if (lane == 2) return dense_key[re - 1];
    return re < nrows ? dense_key[re] : -3;
  };
  int en = edge(gw);
  for (int64_t ch = gw; ch < nch; ch += nw) {
    const int before = __shfl_sync(0xffffffffu, en, 0), first = __shfl_sync(0xffffffffu, en, 1);
    const int lastk = __shfl_sync(0xffffffffu, en, 2), after = __shfl_sync(0xffffffffu, en, 3);
    en = edge(ch + nw);
    const int64_t b0 = ch * VLF_CHUNK, b1 = min(nblk, b0 + VLF_CHUNK);
    const int64_t r0 = 32 * b0, rend = min(nrows, 32 * b1);
    if (first == lastk) {  // one run segment: stream the columns
      const bool store = before != first && after != first;  // the whole run lies in this range
      const int64_t n = rend - r0;
      double xs[NS];  // lane-private sums of every column over the range, then one warp reduction
#pragma unroll
      for (int s = 0; s < NC; s++) {
        const double* c = a.col[s] + r0;
        double x = 0.0, y = 0.0;
        if (n == 32 * VLF_CHUNK) {
#pragma unroll
          for (int j = 0; j < VLF_CHUNK / 2; j++) {
            const double2 w = reinterpret_cast<const double2*>(c)[lane + 32 * j];
            x += w.x;
            y += w.y;
          }
        } else {
          for (int64_t i = lane; i < n; i += 32) x += c[i];
        }
        xs[s] = x + y;
      }
      if (CNT) xs[NS - 1] = lane == 0 ? (double)n : 0.0;
      const double t = warp_sums16<NS>(xs, lane);
      const int si = vl_index(lane);
      if (!(lane & 1) && si < NS) emit(first, si, t, store);
      continue;
    }
    int last = before;
    double carry[NS], acc[NS];
#pragma unroll
    for (int s = 0; s < NS; s++) carry[s] = acc[s] = 0.0;
    bool cstart = false, ldirty = false;
    auto load = [&](int64_t b, int& k, double (&x)[NS]) {
      const int64_t row = 32 * b + lane;
      const bool v = row < rend;
      k = -1;
      if (v) k = dense_key[row];
#pragma unroll
      for (int s = 0; s < NC; s++) {
        x[s] = 0.0;
        if (v) x[s] = a.col[s][row];
      }
      if (CNT) x[NS - 1] = v ? 1.0 : 0.0;
    };
    int nk;
    double nx[NS];
    load(b0, nk, nx);
    for (int64_t b = b0; b < b1; b++) {
      const int key = nk;
      double x[NS];
#pragma unroll
      for (int s = 0; s < NS; s++) x[s] = nx[s];
      if (b + 1 < b1) load(b + 1, nk, nx);
      const int64_t row = 32 * b + lane;
      const bool v = row < rend;
      const int64_t nrem = rend - 32 * b;
      const int nv = nrem < 32 ? (int)nrem : 32;
      int prev = __shfl_up_sync(0xffffffffu, key, 1);
      if (lane == 0) prev = last;
      int next = __shfl_down_sync(0xffffffffu, key, 1);
      const int k0n = __shfl_sync(0xffffffffu, nk, 0);
      if (lane == 31) next = b + 1 < b1 ? k0n : after;
      const unsigned heads = __ballot_sync(0xffffffffu, v && key != prev);
      const bool lastlane = lane == nv - 1;
      const bool tail = v && (lastlane || next != key);
      const bool cont = tail && lastlane && row + 1 < nrows && next == key;  // the block's last run goes on
      const bool carry_on = cont && row + 1 < rend;                           // ... inside this range
      const bool c_on = __shfl_sync(0xffffffffu, (int)carry_on, nv - 1);
      const bool c_any = __shfl_sync(0xffffffffu, (int)cont, nv - 1);
      if (heads == 0) {  // the carried run goes on through the block: lane-private sums
#pragma unroll
        for (int s = 0; s < NS; s++) acc[s] += x[s];
        ldirty = true;
        if (!c_on) {  // the run ends with this block (or leaves the range): emit it
          const double tt = warp_sums16<NS>(acc, lane);
          const int si = vl_index(lane);
          double cs = 0.0;
#pragma unroll
          for (int s = 0; s < NS; s++) {
            if (s == si) cs = carry[s];
            acc[s] = 0.0;
            carry[s] = 0.0;
          }
          const int k0 = __shfl_sync(0xffffffffu, key, 0);  // the block's key (lanes past the end hold -1)
          if (!(lane & 1) && si < NS) emit(k0, si, tt + cs, cstart && !c_any);
          ldirty = false;
          cstart = false;
        }
        last = __shfl_sync(0xffffffffu, key, nv - 1);
        continue;
      }
      if (ldirty) {  // a run starts in this block: fold the lane-private sums into the carry
        const double tt = warp_sums16<NS>(acc, lane);
#pragma unroll
        for (int s = 0; s < NS; s++) {
          carry[s] += __shfl_sync(0xffffffffu, tt, (s >> 3 & 1) * 16 + (s >> 2 & 1) * 8 + (s >> 1 & 1) * 4 + (s & 1) * 2);
          acc[s] = 0.0;
        }
        ldirty = false;
      }
      const unsigned upto = heads & ((2u << lane) - 1u);
      const int s0 = upto ? 31 - __clz(upto) : 0;
      const bool first_seg = upto == 0;
      const bool started_in = first_seg ? cstart : true;
#pragma unroll
      for (int s = 0; s < NS; s++) {
        double y = x[s];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const double u = __shfl_up_sync(0xffffffffu, y, d);
          if (lane - d >= s0) y += u;
        }
        if (first_seg) y += carry[s];
        if (tail && !carry_on) emit(key, s, y, started_in && !cont);  // store: the run lies inside this range
        carry[s] = c_on ? __shfl_sync(0xffffffffu, y, nv - 1) : 0.0;
      }
      const unsigned up_l = __shfl_sync(0xffffffffu, upto, nv - 1);
      cstart = c_on ? (up_l ? true : cstart) : false;
      last = __shfl_sync(0xffffffffu, key, nv - 1);
    }
  }
}

static unsigned grid_rows(int64_t n, int per_sm = 8) {
  int64_t g = (n + 255) / 256;
  g = std::min<int64_t>(g, 148 * per_sm);
  return (unsigned)std::max<int64_t>(g, 1);
}

cudaError_t launch_view_lin(const ViewLinArgs& a, const int32_t* dense_key, double* V, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  if (a.nslots > VB_MAXSLOT) return cudaErrorInvalidValue;
  bool fast = a.nslots >= 1 && a.nslots <= 16 && !(std::getenv("LMFAO_VIEW_FAST") && std::getenv("LMFAO_VIEW_FAST")[0] == '0');
  int ncnt = 0;
  for (int s = 0; s < a.nslots && fast; s++) {
    fast = !a.cb[s] && (!a.ca[s] || !a.ia[s]) && (reinterpret_cast<uintptr_t>(a.ca[s]) & 15) == 0;  // 16-byte loads
    ncnt += !a.ca[s];
  }
  fast = fast && ncnt <= 1;
  if (fast) {
    ViewFastArgs f{};
    f.nrows = a.nrows;
    f.nslots = a.nslots;
    int nc = 0;
    for (int s = 0; s < a.nslots; s++)
      if (a.ca[s]) {
        f.col[nc] = reinterpret_cast<const double*>(a.ca[s]);
        f.vslot[nc++] = (int8_t)s;
      }
    for (int s = 0; s < a.nslots; s++)
      if (!a.ca[s]) f.vslot[nc] = (int8_t)s;  // the count: kernel slot nc
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    auto grid = [&](const void* fn) {  // one wave of resident CTAs
      int per = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0) || per < 1) per = 1;
      return (unsigned)std::max<int64_t>(1, std::min<int64_t>((a.nrows + 255) / 256, (int64_t)nsm * per));
    };
    switch (nc * 2 + (ncnt ? 1 : 0)) {
#define LMFAO_VLF(n)                                                                                            \
  case 2 * n: k_view_lin_fast<n, false><<<grid((const void*)k_view_lin_fast<n, false>), 256, 0, st>>>(f, dense_key, V); break; \
  case 2 * n + 1: k_view_lin_fast<n, true><<<grid((const void*)k_view_lin_fast<n, true>), 256, 0, st>>>(f, dense_key, V); break;
      LMFAO_VLF(1) LMFAO_VLF(2) LMFAO_VLF(3) LMFAO_VLF(4) LMFAO_VLF(5) LMFAO_VLF(6) LMFAO_VLF(7) LMFAO_VLF(8)
      LMFAO_VLF(9) LMFAO_VLF(10) LMFAO_VLF(11) LMFAO_VLF(12) LMFAO_VLF(13) LMFAO_VLF(14) LMFAO_VLF(15)
#undef LMFAO_VLF
      case 1: k_view_lin_fast<0, true><<<grid((const void*)k_view_lin_fast<0, true>), 256, 0, st>>>(f, dense_key, V); break;
      case 32: k_view_lin_fast<16, false><<<grid((const void*)k_view_lin_fast<16, false>), 256, 0, st>>>(f, dense_key, V); break;
      default: return cudaErrorInvalidValue;
    }
    launches_add(1);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)VB_WARPS * a.nslots * 8 * 33;
  if (smem > 48 * 1024) {
    CUDA_TRY(ensure_smem_attr((const void*)k_view_lin, smem));
  }
  k_view_lin<<<grid_rows(a.nrows), VB_WARPS * 32, smem, st>>>(a, dense_key, V);
  launches_add(1);
  return cudaGetLastError();
}

cudaError_t launch_view_build(const NodeArgs& a, const int32_t* dense_key, const int32_t* prog_i, const double* prog_d,
                              const int32_t* ioff, const int32_t* doff, int nslots, double* V, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  size_t smem = (size_t)VB_WARPS * std::max(nslots, 1) * 8 * 33;  // carries + lane sums
  int use_lacc = 1;
  if (smem > 200 * 1024) {  // many slots: carries only
    use_lacc = 0;
    smem = (size_t)VB_WARPS * std::max(nslots, 1) * 8;
  }
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    CUDA_TRY(ensure_smem_attr((const void*)k_view_build, smem));
  }
  k_view_build<<<grid_rows(a.nrows), VB_WARPS * 32, smem, st>>>(a, dense_key, prog_i, prog_d, ioff, doff, nslots, V,
                                                                use_lacc);
  launches_add(1);
  return cudaGetLastError();
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// No-group-by outputs [o0, o0+nout): each warp reduces every output over its
// rows with shuffles and lane 0 adds into the warp's smem row; the block then
// sums its warps in fixed order.  No atomics, deterministic for a fixed grid.
__global__ void k_root_scalar(NodeArgs a, const int32_t* __restrict__ prog_i, const double* __restrict__ prog_d,
                              const int32_t* __restrict__ ioff, const int32_t* __restrict__ doff, int o0, int nout,
                              int ld, double* __restrict__ partials, unsigned long long* __restrict__ cpart) {
  extern __shared__ double wpart[];  // [nwarps][nout]
  __shared__ unsigned long long wcnt[32];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < nw * nout; i += blockDim.x) wpart[i] = 0.0;
  __syncthreads();
  unsigned long long cnt = 0;
  int32_t kk[MAX_CHILD];
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < a.nrows; base += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = base + threadIdx.x;
    bool valid = row < a.nrows;
    double w = valid ? 1.0 : 0.0;
    for (int c = 0; c < a.nchild; c++) {
      kk[c] = valid ? a.fk[c][row] : 0;
      if (valid) w *= a.V[c][(int64_t)kk[c] * a.W[c]];
    }
    cnt += (unsigned long long)w;
    for (int o = 0; o < nout; o++) {
      double v = valid ? eval_output(a, row, kk, prog_i + ioff[o0 + o], prog_d + doff[o0 + o]) : 0.0;
      v = warp_sum(v);
      if (lane == 0) wpart[warp * nout + o] += v;
    }
  }
  cnt = warp_sum(cnt);
  if (lane == 0) wcnt[warp] = cnt;
  __syncthreads();
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double s = 0.0;
    for (int w2 = 0; w2 < nw; w2++) s += wpart[w2 * nout + o];
    partials[(int64_t)blockIdx.x * ld + o0 + o] = s;
  }
  if (threadIdx.x == 0 && cpart) {
    unsigned long long s = 0;
    for (int w2 = 0; w2 < nw; w2++) s += wcnt[w2];
    cpart[blockIdx.x] = s;
  }
}

cudaError_t launch_root_scalar(const NodeArgs& a, const int32_t* prog_i, const double* prog_d, const int32_t* ioff,
                               const int32_t* doff, int nout, double* partials, unsigned long long* count_partials,
                               int grid, cudaStream_t st) {
  const int threads = 256, chunk = 1024;  // 8 warps x 1024 x 8 B = 64 KB smem per launch
  CUDA_TRY(ensure_smem_attr((const void*)k_root_scalar, 8 * chunk * 8));
  if (nout == 0) {
    k_root_scalar<<<grid, threads, 0, st>>>(a, prog_i, prog_d, ioff, doff, 0, 0, 1, partials, count_partials);
    launches_add(1);
    return cudaGetLastError();
  }
  for (int o0 = 0; o0 < nout; o0 += chunk) {
    int n = std::min(chunk, nout - o0);
    k_root_scalar<<<grid, threads, (size_t)(threads / 32) * n * 8, st>>>(a, prog_i, prog_d, ioff, doff, o0, n, nout,
                                                                         partials, o0 == 0 ? count_partials : nullptr);
    launches_add(1);
    CUDA_TRY(cudaGetLastError());
  }
  return cudaSuccess;
}

__global__ void k_combine(const double* __restrict__ partials, const unsigned long long* __restrict__ cpart, int grid,
                          int nout, double* __restrict__ out, unsigned long long* __restrict__ cout_) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < grid; b++) s += partials[(int64_t)b * nout + o];
    out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && cout_) {
    unsigned long long s = 0;
    for (int b = 0; b < grid; b++) s += cpart[b];
    *cout_ = s;
  }
}

cudaError_t launch_combine_partials(const double* partials, const unsigned long long* cpart, int grid, int nout,
                                    double* out, unsigned long long* count_out, cudaStream_t st) {
  int blocks = std::max(1, std::min(64, (nout + 127) / 128));
  k_combine<<<blocks, 128, 0, st>>>(partials, cpart, grid, nout, out, count_out);
  launches_add(1);
  return cudaGetLastError();
}

__global__ void k_root_group(NodeArgs a, GroupArgs g, const int32_t* __restrict__ prog_i,
                             const double* __restrict__ prog_d, const int32_t* __restrict__ ioff,
                             const int32_t* __restrict__ doff, int nudaf, double* __restrict__ table,
                             unsigned long long* __restrict__ counts) {
  int32_t kk[MAX_CHILD];
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < a.nrows;
       row += (int64_t)gridDim.x * blockDim.x) {
    double w = 1.0;
    for (int c = 0; c < a.nchild; c++) {
      kk[c] = a.fk[c][row];
      w *= a.V[c][(int64_t)kk[c] * a.W[c]];
    }
    if (w == 0.0) continue;
    int64_t cell = 0;
    for (int i = 0; i < g.ngb; i++) {
      int cc = g.code_child[i];
      int32_t code = cc < 0 ? g.code[i][row] : g.code[i][kk[cc]];
      cell += (int64_t)code * g.stride[i];
    }
    gred_add(&counts[cell], (unsigned long long)w);
    for (int j = 0; j < nudaf; j++) {
      double v = eval_output(a, row, kk, prog_i + ioff[j], prog_d + doff[j]);
      if (v != 0.0) gred_add(&table[cell * nudaf + j], v);
    }
  }
}

cudaError_t launch_root_group(const NodeArgs& a, const GroupArgs& g, const int32_t* prog_i, const double* prog_d,
                              const int32_t* ioff, const int32_t* doff, int nudaf, double* table,
                              unsigned long long* counts, cudaStream_t st) {
  if (a.nrows <= 0) return cudaSuccess;
  k_root_group<<<grid_rows(a.nrows, 16), 256, 0, st>>>(a, g, prog_i, prog_d, ioff, doff, nudaf, table, counts);
  launches_add(1);
  return cudaGetLastError();
}

// Fused group-by scan: one pass over the root for every group-by query of the
// batch.  Lanes holding the same (query, cell) are found with __match_any_sync;
// counts are aggregated per warp (popc of the peers when every multiplicity is 1)
// so Zipf-hot cells take one atomic per warp instead of one per row.  UDAFs that
// are constants (SUM(c), e.g. COUNT) are not accumulated at all: the compaction
// derives them from the counts.
__global__ void k_groups_fused(NodeArgs a, const GroupDesc* descs, int nq,
                               const int32_t* __restrict__ prog_i, const double* __restrict__ prog_d,
                               const int32_t* __restrict__ ioff, const int32_t* __restrict__ doff) {
  // the query descriptors live in shared memory (read for every row and query)
  extern __shared__ __align__(16) unsigned char dsm[];
  {
    const int4* src = reinterpret_cast<const int4*>(descs);
    int4* dst = reinterpret_cast<int4*>(dsm);
    const int n16 = (int)((nq * sizeof(GroupDesc) + 15) / 16);
    for (int i = threadIdx.x; i < n16; i += blockDim.x) dst[i] = src[i];
    __syncthreads();
  }
  descs = reinterpret_cast<const GroupDesc*>(dsm);
  int32_t kk[MAX_CHILD];
  const int lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) & ~31ll; base < a.nrows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = base + (threadIdx.x & ~31) + lane;
    const bool valid = row < a.nrows;
    double w = valid ? 1.0 : 0.0;
    for (int c = 0; c < a.nchild; c++) {
      kk[c] = valid ? a.fk[c][row] : 0;
      if (valid) w *= a.V[c][(int64_t)kk[c] * a.W[c]];
    }
    const bool ones = __all_sync(0xffffffffu, !valid || w == 1.0);
    for (int q = 0; q < nq; q++) {
      const GroupDesc& d = descs[q];
      long long cell = -1 - lane;
      if (valid && w != 0.0) {
        cell = 0;
        for (int i = 0; i < d.ngb; i++) {
          const int cc = d.code_child[i];
          const int32_t code = cc < 0 ? d.code[i][row] : d.code[i][kk[cc]];
          cell += (long long)code * d.stride[i];
        }
      }
      if (ones) {
        const unsigned peers = __match_any_sync(0xffffffffu, cell);
        if (cell >= 0 && (__ffs(peers) - 1) == lane) gred_add(&d.counts[cell], (unsigned long long)__popc(peers));
      } else if (cell >= 0) {
        gred_add(&d.counts[cell], (unsigned long long)w);
      }
      // non-constant UDAFs: the root is sorted by its keys, so equal cells mostly sit in
      // runs of adjacent lanes; a segmented warp scan sums each run and its last lane
      // issues one atomic (cells repeated in non-adjacent runs just get several atomics)
      if (d.nsum == 0) continue;
      long long pc = __shfl_up_sync(0xffffffffu, cell, 1);
      const bool head = lane == 0 || pc != cell;
      const unsigned heads = __ballot_sync(0xffffffffu, head);
      const unsigned upto = heads & ((2u << lane) - 1u);
      const int s0 = 31 - __clz(upto);
      long long nc = __shfl_down_sync(0xffffffffu, cell, 1);
      const bool tail = lane == 31 || nc != cell;
      for (int j = 0; j < d.nudaf; j++) {
        if (d.countlike[j]) continue;
        const int o = d.prog_base + j;
        double v = cell >= 0 ? eval_output(a, row, kk, prog_i + ioff[o], prog_d + doff[o]) : 0.0;
#pragma unroll
        for (int dd = 1; dd < 32; dd <<= 1) {
          const double u = __shfl_up_sync(0xffffffffu, v, dd);
          if (lane - dd >= s0) v += u;
        }
        if (tail && cell >= 0 && v != 0.0) gred_add(&d.table[cell * d.nudaf + j], v);
      }
    }
  }
}

cudaError_t launch_groups_fused(const NodeArgs& a, const GroupDesc* descs, int nq, const int32_t* prog_i,
                                const double* prog_d, const int32_t* ioff, const int32_t* doff, cudaStream_t st) {
  if (a.nrows <= 0 || nq == 0) return cudaSuccess;
  const size_t smem = ((size_t)nq * sizeof(GroupDesc) + 15) / 16 * 16;
  if (smem > 48 * 1024) {
    CUDA_TRY(ensure_smem_attr((const void*)k_groups_fused, smem));
  }
  k_groups_fused<<<grid_rows(a.nrows, 16), 256, smem, st>>>(a, descs, nq, prog_i, prog_d, ioff, doff);
  launches_add(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- group-bys at a child
// Group-by attributes of a root child T with a non-unique key (a row of T is not determined
// by a root row): "each aggregate to its own root" — the root side of every
// product is summed per key of T, A[k][p] = Σ_{root rows with T-key k} root_side_p(row)
// (the other children through their views, T left out), and the query is finished at T:
// Σ over T rows t of A[key(t)][p] · T_side_p(t) into the cell of t's group-by codes.
// Output nout-1 of both programs is the count term (multiplicities).
__global__ void k_rev_root(NodeArgs a, const int32_t* __restrict__ fkT, int nout, const int32_t* __restrict__ prog_i,
                           const double* __restrict__ prog_d, const int32_t* __restrict__ ioff,
                           const int32_t* __restrict__ doff, double* __restrict__ A) {
  int32_t kk[MAX_CHILD];
  const int lane = threadIdx.x & 31;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) & ~31ll; base < a.nrows;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = base + (threadIdx.x & ~31) + lane;
    const bool valid = row < a.nrows;
    for (int c = 0; c < a.nchild; c++) kk[c] = valid ? a.fk[c][row] : 0;
    const int key = valid ? fkT[row] : -1 - lane;
    // runs of equal T keys (the root is sorted by its keys): a segmented scan per output,
    // the run's last lane adds it
    const int pk = __shfl_up_sync(0xffffffffu, key, 1);
    const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || pk != key);
    const int s0 = 31 - __clz(heads & ((2u << lane) - 1u));
    const int nk = __shfl_down_sync(0xffffffffu, key, 1);
    const bool tail = lane == 31 || nk != key;
    for (int o = 0; o < nout; o++) {
      double v = valid ? eval_output(a, row, kk, prog_i + ioff[o], prog_d + doff[o]) : 0.0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane - d >= s0) v += u;
      }
      if (tail && valid && v != 0.0) gred_add(&A[(int64_t)key * nout + o], v);
    }
  }
}

__global__ void k_rev_child(NodeArgs t, const int32_t* __restrict__ tkey, int nout, const int32_t* __restrict__ prog_i,
                            const double* __restrict__ prog_d, const int32_t* __restrict__ ioff,
                            const int32_t* __restrict__ doff, const int32_t* __restrict__ pu,
                            const double* __restrict__ A, GroupDesc d) {
  int32_t kk[MAX_CHILD];
  for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < t.nrows;
       row += (int64_t)gridDim.x * blockDim.x) {
    for (int c = 0; c < t.nchild; c++) kk[c] = t.fk[c][row];
    const int64_t k = tkey[row];
    long long cell = 0;
    for (int i = 0; i < d.ngb; i++) cell += (long long)d.code[i][row] * d.stride[i];
    const double* Ak = A + k * nout;
    const double cnt = Ak[nout - 1] * eval_output(t, row, kk, prog_i + ioff[nout - 1], prog_d + doff[nout - 1]);
    if (cnt == 0.0) continue;  // no root row joins this T row (or its subtree is empty)
    gred_add(&d.counts[cell], (unsigned long long)cnt);
    for (int p = 0; p < nout - 1; p++) {
      const int u = pu[p];
      if (d.countlike[u]) continue;
      const double v = Ak[p] * eval_output(t, row, kk, prog_i + ioff[p], prog_d + doff[p]);
      if (v != 0.0) gred_add(&d.table[cell * d.nudaf + u], v);
    }
  }
}

cudaError_t launch_rev(const NodeArgs& root, const int32_t* fkT, const ProgPtrs& rp, const NodeArgs& t,
                       const int32_t* tkey, const ProgPtrs& tp, const int32_t* pu, double* A, int64_t nkT,
                       const GroupDesc& d, cudaStream_t st) {
  const int nout = rp.nout;
  CUDA_TRY(cudaMemsetAsync(A, 0, (size_t)std::max<int64_t>(nkT, 1) * nout * 8, st));
  if (root.nrows > 0) {
    k_rev_root<<<grid_rows(root.nrows, 16), 256, 0, st>>>(root, fkT, nout, rp.pi, rp.pd, rp.io, rp.dofs, A);
    launches_add(1);
  }
  if (t.nrows > 0) {
    k_rev_child<<<grid_rows(t.nrows, 16), 256, 0, st>>>(t, tkey, nout, tp.pi, tp.pd, tp.io, tp.dofs, pu, A, d);
    launches_add(1);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- compaction
__global__ void k_present(const unsigned long long* __restrict__ counts, int64_t n, uint32_t* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flags[i] = counts[i] > 0 ? 1u : 0u;
}

__global__ void k_scatter_groups(const double* __restrict__ table, const unsigned long long* __restrict__ counts,
                                 const uint32_t* __restrict__ flags, const uint32_t* __restrict__ excl, int64_t n,
                                 int nudaf, DecodeArgs d, int32_t* __restrict__ keys, double* __restrict__ vals,
                                 unsigned long long* __restrict__ cnts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!flags[i]) continue;
    int64_t g = excl[i];
    for (int a = 0; a < d.ngb; a++) keys[g * d.ngb + a] = d.dict[a][((i + d.cell0) / d.stride[a]) % d.radix[a]];
    for (int j = 0; j < nudaf; j++)
      vals[g * nudaf + j] = d.countcoef ? (isnan(d.countcoef[j]) ? table[i * nudaf + j] : d.countcoef[j] * (double)counts[i])
                                        : table[i * nudaf + j];
    cnts[g] = counts[i];
  }
}

cudaError_t launch_compact(const double* table, const unsigned long long* counts, int64_t ncells, int nudaf,
                           const DecodeArgs& d, DevBuf& keys, DevBuf& vals, DevBuf& cnts, int64_t& ngroups,
                           cudaStream_t st) {
  ngroups = 0;
  DevBuf flags, excl;
  CUDA_TRY(flags.alloc(ncells * 4));
  CUDA_TRY(excl.alloc(ncells * 4));
  k_present<<<grid_rows(ncells, 16), 256, 0, st>>>(counts, ncells, flags.as<uint32_t>());
  CUDA_TRY(exclusive_scan_u32(flags.as<uint32_t>(), excl.as<uint32_t>(), ncells, st));
  uint32_t le = 0, lf = 0;
  CUDA_TRY(cudaMemcpyAsync(&le, excl.as<uint32_t>() + ncells - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(&lf, flags.as<uint32_t>() + ncells - 1, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  ngroups = (int64_t)le + lf;
  if (keys.bytes < (size_t)std::max<int64_t>(ngroups * d.ngb * 4, 16)) CUDA_TRY(keys.alloc(ngroups * d.ngb * 4));
  if (vals.bytes < (size_t)std::max<int64_t>(ngroups * nudaf * 8, 16)) CUDA_TRY(vals.alloc(ngroups * nudaf * 8));
  if (cnts.bytes < (size_t)std::max<int64_t>(ngroups * 8, 16)) CUDA_TRY(cnts.alloc(ngroups * 8));
  k_scatter_groups<<<grid_rows(ncells, 16), 256, 0, st>>>(table, counts, flags.as<uint32_t>(), excl.as<uint32_t>(),
                                                          ncells, nudaf, d, keys.as<int32_t>(), vals.as<double>(),
                                                          cnts.as<unsigned long long>());
  launches_add(3);
  CUDA_TRY(cudaGetLastError());
  return cudaStreamSynchronize(st);
}

}  // namespace lmfao
