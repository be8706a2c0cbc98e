// rt.cu — the histogram path (§8 row (e)) for regression-tree node batches
// (§3 "Regression trees" P:528-555; BASELINE.json configs[2]):
//   Q_cat(X; Σ w_p)                  one single-attribute group-by per categorical X,
//   Q(Σ w_p · 1[A op t])             a Kronecker-delta predicate per (attribute, threshold),
// with w_p = y^p (p ∈ {0, 1, 2}: SUM(1), SUM(y), SUM(y²)) for one root attribute y.
//
// Every such aggregate is a linear functional of a histogram of w:
//  * a predicate A op t only depends on which "cell" A falls in among the sorted distinct
//    thresholds used with A (cell 2i: t_{i-1} < A < t_i, cell 2i+1: A = t_i), so
//    Σ w_p 1[A op t] = Σ_{cells c ⊨ op t} H_A[c][p] — a prefix/suffix sum of H_A
//    (the paper's 20 buckets; the comparison is exact in IEEE double);
//  * for a root attribute A, H_A is accumulated over the root rows (k_rt_fact);
//  * for an attribute of a primary-key leaf D, Σ over the join = Σ_{k ∈ D} V_D[k] · f(A(k))
//    with the fact→dimension view V_D[k][p] = Σ_{root rows with key k} w_p ("each aggregate
//    to its own root") — V_D by segmented warp scans over the sorted root
//    (k_rt_views), then H_A / group tables at the dimension (k_rt_dims);
//  * group-bys on a root attribute accumulate w per cell (k_rt_fact), on a dimension
//    attribute through V_D (k_rt_dims).
// Assembly (k_rt_assemble) maps histogram cells to the batch's UDAFs with term lists.
#include <cmath>
#include <cstdlib>
#include <map>
#include <set>

#include "ctx.h"

namespace lmfao {
namespace {

constexpr unsigned RFULL = 0xffffffffu;
constexpr int RT_MAX_FACT = 24;   // root attributes with histograms (predicates + small group-bys)
constexpr int RT_MAX_DIM = 64;    // dimension attributes with histograms
constexpr int RT_MAX_LEVELS = 8;  // root children with views
#ifndef RT_HT_BITS  // C3: 2^10 slots 1.233 ms, 2^8 1.211, 2^6 1.50 (too many misses to global REDs)
#define RT_HT_BITS 8
#endif
constexpr int RT_HT = 1 << RT_HT_BITS;  // per-CTA hash slots per view level (Zipf-hot keys)

// A histogram over the root rows: predicate cells of a column, or the codes of a group-by.
struct FactHist {
  const void* col;  // root column (fp64 or int32) for predicates, int32 codes for group-bys
  int is_int;       // predicate column dtype
  int is_code;      // group-by codes (cell = code) instead of threshold cells
  int nthr;         // thresholds (predicates)
  int thr_off;      // into the threshold array
  int ncell;
  int uniform;      // thresholds t_i = t_0 + i h exactly (cell estimate + exact fix-up)
  double t0, inv_h;
  double margin;    // max_i |t_i - (t_0 + i h)| / h + 1e-9: estimates farther than this from an integer are exact
  int64_t goff;     // global offset (doubles) of the [ncell][3] table in the output buffer
};
constexpr int RT_SMALL = 21;  // lane cells of a histogram kept in per-lane private tables
constexpr int RT_FACT_WARPS = 16;
struct RtFactArgs {
  int64_t nrows;
  const double* y;  // null: w = (1, 0, 0)
  const uint8_t* filt;  // path condition per root row (null: every row)
  int nh;           // histograms; CTA (part, h) does histogram h over row part `part`
  int nparts;
  FactHist h[RT_MAX_FACT];
  const double* thr;  // thresholds, all attributes
  double* out;        // global accumulators (TOT at 0)
  int eq_off, tab_off;  // shared memory (doubles): thresholds | equality cells | lane tables
  int wgt[RT_MAX_FACT];   // relative cost per row of each histogram (work split)
  int npieces;            // equal-cost pieces of the (histogram, row) space, taken dynamically
  int* work;              // piece counter (zeroed per pass)
};
#ifndef RT_PIECES_PER_CTA
#define RT_PIECES_PER_CTA 2  // (C3: one static piece per CTA left SM active cycles 32 % apart; 2: 1.053, 4: 1.060, 8: 1.121 ms)
#endif

__device__ __forceinline__ int rt_cell(double x, const double* t, int n) {
  int lo = 0, hi = n;  // lower bound: first t >= x
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (t[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && t[lo] == x) ? 2 * lo + 1 : 2 * lo;
}
// lower bound from an arithmetic-progression estimate, corrected by exact comparisons
__device__ __forceinline__ int rt_cell_uniform(double x, const double* t, int n, double t0, double inv_h) {
  double e = (x - t0) * inv_h + 1.0;
  e = e < 0.0 ? 0.0 : (e > (double)n ? (double)n : e);  // NaN-free inputs
  int lo = (int)e;
  while (lo > 0 && t[lo - 1] >= x) lo--;
  while (lo < n && t[lo] < x) lo++;
  return (lo < n && t[lo] == x) ? 2 * lo + 1 : 2 * lo;
}

// Threshold cell without memory traffic when the estimate is safely between two thresholds:
// with g = (x - t_0) / h and |t_i - (t_0 + i h)| <= μ h, t_i < x iff i < g whenever g is more
// than μ from every integer, so #{t_i < x} = clamp(floor(g + 1), 0, n) and x equals no t_i.
// Rounding of e is ~1e-15 absolute for |e| <= n + 1 (the margin adds 1e-9); the rest take
// the exact fix-up.
__device__ __forceinline__ int rt_cell_fast(double x, const double* t, int n, double t0, double inv_h,
                                            double margin) {
  const double e = (x - t0) * inv_h + 1.0;
  if (fabs(e - rint(e)) > margin && fabs(e) < 1e9) {  // NaN compares false: exact path
    const double f = floor(e);
    const int lo = f < 0.0 ? 0 : (f > (double)n ? n : (int)f);
    return 2 * lo;
  }
  return rt_cell_uniform(x, t, n, t0, inv_h);
}

// k_rt_fact's row loop for one histogram piece.  KIND: 0 fp64 predicate column, 1 group-by
// codes, 2 int32 predicate column; FILT: a path condition filters the rows.
template <int KIND, bool FILT>
__device__ __forceinline__ void rt_fact_rows(const RtFactArgs& a, const FactHist& h, int64_t r0, int64_t r1,
                                             const double* thr, double* eqt, unsigned* tc, double2* ty, int nc,
                                             double& t0, double& t1, double& t2) {
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  constexpr int U = 16;  // rows per lane per step: all loads issued before the table updates
  for (int64_t base = r0 + wib * 32 * U + lane; base < r1; base += (int64_t)nw * 32 * U) {
    double yv[U], xv[U];
    int cv[U];
    bool pv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t row = base + 32 * u;
      const bool v = row < r1;
      const bool pass = v && (!FILT || a.filt[row]);
      yv[u] = 0.0;
      if (pass && a.y) yv[u] = a.y[row];
      pv[u] = pass;
      cv[u] = -1;
      xv[u] = 0.0;
      if (v) {
        if (KIND == 1) cv[u] = reinterpret_cast<const int32_t*>(h.col)[row];
        else if (KIND == 2) xv[u] = (double)reinterpret_cast<const int32_t*>(h.col)[row];
        else xv[u] = reinterpret_cast<const double*>(h.col)[row];
      }
    }
#pragma unroll
    for (int u = 0; u < U; u += 2) {
      int e[2];
      double n[2], yy[2], q[2];
#pragma unroll
      for (int z = 0; z < 2; z++) {
        const bool v = base + 32 * (u + z) < r1;
        int c = cv[u + z];
        bool eq = false;
        if (KIND != 1 && v) {
          c = h.uniform ? rt_cell_fast(xv[u + z], thr, h.nthr, h.t0, h.inv_h, h.margin) : rt_cell(xv[u + z], thr, h.nthr);
          eq = (c & 1) && pv[u + z];
          c >>= 1;
        }
        n[z] = pv[u + z] ? 1.0 : 0.0;  // rows failing the path condition weigh 0
        yy[z] = yv[u + z];
        q[z] = yy[z] * yy[z];
        t0 += n[z];
        t1 += yy[z];
        t2 += q[z];
        if (KIND != 1 && eq) {  // x equals threshold c: rare for continuous data
          double* et = eqt + 3 * c;
          sred_add(et, 1.0);
          sred_add(et + 1, yy[z]);
          sred_add(et + 2, q[z]);
          n[z] = yy[z] = q[z] = 0.0;
        }
        e[z] = (v && !eq ? c : nc) * 32 + lane;
      }
      if (e[0] == e[1]) {  // merge into the first; the second writes its old value back
        n[0] += n[1];
        yy[0] += yy[1];
        q[0] += q[1];
        n[1] = yy[1] = q[1] = 0.0;
      }
      const unsigned c0 = tc[e[0]], c1 = tc[e[1]];
      const double2 w0 = ty[e[0]], w1 = ty[e[1]];
      tc[e[1]] = c1 + (unsigned)n[1];
      ty[e[1]] = make_double2(w1.x + yy[1], w1.y + q[1]);
      tc[e[0]] = c0 + (unsigned)n[0];
      ty[e[0]] = make_double2(w0.x + yy[0], w0.y + q[0]);
    }
  }
}

// Root rows, all histograms: the (histogram, row) space is cut into equal contiguous pieces,
// one per CTA (so every CTA has the same work and at most a few histogram switches, each a
// flush of its tables).  Small histograms (<= RT_SMALL cells) use per-lane private tables in
// shared memory — plain conflict-free read-modify-write, no atomics — with one spare cell for
// rows past the end; rows are taken in pairs whose table updates are issued together (a pair
// in the same cell is merged first), summed over the CTA at each flush.  TOT comes from the
// pieces of histogram 0.
__global__ void __launch_bounds__(RT_FACT_WARPS * 32) k_rt_fact(const __grid_constant__ RtFactArgs a) {
  extern __shared__ double rsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* thr = rsm;
  double* eqt = rsm + a.eq_off;  // [nthr][3] rows equal to a threshold (rare: shared atomics)
  // equal-cost pieces of the (histogram, row) space, histogram h weighing wgt[h], taken
  // dynamically (the weights are estimates)
  const int64_t N = a.nrows;
  int64_t T = 0;
  for (int i = 0; i < a.nh; i++) T += (int64_t)a.wgt[i] * N;
  __shared__ int piece_sh;
  const int64_t P = a.npieces;
  for (;;) {
  if (threadIdx.x == 0) piece_sh = atomicAdd(a.work, 1);
  __syncthreads();
  const int64_t pc = piece_sh;
  __syncthreads();
  if (pc >= P) break;
  const int64_t W0 = T / P * pc + (T % P) * pc / P;
  const int64_t W1 = T / P * (pc + 1) + (T % P) * (pc + 1) / P;
  int64_t hb = 0;  // weighted start of histogram hi
  for (int hi = 0; hi < a.nh; hb += (int64_t)a.wgt[hi] * N, hi++) {
    const int64_t he = hb + (int64_t)a.wgt[hi] * N;
    if (he <= W0 || hb >= W1) continue;
    const int64_t r0 = W0 > hb ? (W0 - hb + a.wgt[hi] - 1) / a.wgt[hi] : 0;
    const int64_t r1 = W1 < he ? (W1 - hb + a.wgt[hi] - 1) / a.wgt[hi] : N;
    if (r0 >= r1) continue;
    const FactHist& h = a.h[hi];
    // lane cells: the group-by codes, or the nthr + 1 intervals between thresholds (cell 2b
    // of the histogram); a row equal to threshold i (cell 2i + 1) goes to eqt
    const int nc = h.is_code ? h.ncell : h.nthr + 1, ncp = nc + 1;  // + the spare cell
    // per warp: [ncp][32] u32 counts, [ncp][32] y, [ncp][32] y^2
    unsigned char* wt = reinterpret_cast<unsigned char*>(rsm + a.tab_off) + (size_t)wib * ncp * 32 * 20;
    unsigned* tc = reinterpret_cast<unsigned*>(wt);
    double2* ty = reinterpret_cast<double2*>(wt + ncp * 32 * 4);  // (Σ y, Σ y²) per (cell, lane)
    __syncthreads();  // the previous piece's flush is done with the tables
    for (int i = threadIdx.x; i < h.nthr; i += blockDim.x) thr[i] = a.thr[h.thr_off + i];
    for (int i = threadIdx.x; i < 3 * h.nthr; i += blockDim.x) eqt[i] = 0.0;
    for (int i = lane; i < ncp * 32; i += 32) {
      tc[i] = 0;
      ty[i] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    double t0 = 0.0, t1 = 0.0, t2 = 0.0;
    // the row loop, specialised by the column kind and the path condition (no per-row checks)
    if (h.is_code) {
      if (a.filt) rt_fact_rows<1, true>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
      else rt_fact_rows<1, false>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
    } else if (h.is_int) {
      if (a.filt) rt_fact_rows<2, true>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
      else rt_fact_rows<2, false>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
    } else {
      if (a.filt) rt_fact_rows<0, true>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
      else rt_fact_rows<0, false>(a, h, r0, r1, thr, eqt, tc, ty, nc, t0, t1, t2);
    }
    if (hi == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        t0 += __shfl_xor_sync(RFULL, t0, o);
        t1 += __shfl_xor_sync(RFULL, t1, o);
        t2 += __shfl_xor_sync(RFULL, t2, o);
      }
      if (lane == 0) {
        gred_add(a.out, t0);
        gred_add(a.out + 1, t1);
        gred_add(a.out + 2, t2);
      }
    }
    __syncthreads();
    // Σ over the CTA's warps and lanes -> global (the spare cell is dropped)
    for (int i = threadIdx.x; i < 3 * h.nthr; i += blockDim.x)
      if (eqt[i] != 0.0) gred_add(a.out + h.goff + 3 * (2 * (i / 3) + 1) + i % 3, eqt[i]);
    const unsigned char* tb = reinterpret_cast<const unsigned char*>(rsm + a.tab_off);
    for (int i = threadIdx.x; i < 3 * nc; i += blockDim.x) {
      const int cell = i / 3, v = i % 3;
      double sum = 0.0;
      for (int w = 0; w < nw; w++) {
        const unsigned char* ww = tb + (size_t)w * ncp * 32 * 20;
        if (v == 0) {
          unsigned long long cs = 0;
          for (int l = 0; l < 32; l++) cs += reinterpret_cast<const unsigned*>(ww)[cell * 32 + l];
          sum += (double)cs;
        } else {
          const double* tv = reinterpret_cast<const double*>(ww + ncp * 32 * 4) + 2 * cell * 32 + (v - 1);
          for (int l = 0; l < 32; l++) sum += tv[2 * l];
        }
      }
      const int oc = h.is_code ? cell : 2 * cell;
      if (sum != 0.0) gred_add(a.out + h.goff + 3 * oc + v, sum);
    }
  }
  }
}

// Root histograms with more than RT_SMALL cells (group-bys on large root domains): one
// table per CTA in shared memory ([ncell] u32 counts, [ncell][2] sums) updated with shared
// atomics when it fits, global atomics otherwise.
struct RtBigArgs {
  int64_t nrows;
  const double* y;
  const uint8_t* filt;
  const int32_t* code;
  int ncell;
  int in_smem;
  double* out;  // [ncell][3] at its goff
};
#ifndef RT_BIG_THREADS
#define RT_BIG_THREADS 512
#endif
#ifndef RT_BIG_U
#define RT_BIG_U 4
#endif
__global__ void __launch_bounds__(RT_BIG_THREADS) k_rt_big(const __grid_constant__ RtBigArgs a) {
  extern __shared__ unsigned char bsm[];
  unsigned* cnt = reinterpret_cast<unsigned*>(bsm);
  double* sums = reinterpret_cast<double*>(bsm + ((a.ncell * 4 + 15) & ~15));
  if (a.in_smem) {
    for (int i = threadIdx.x; i < a.ncell; i += blockDim.x) {
      cnt[i] = 0;
      sums[2 * i] = sums[2 * i + 1] = 0.0;
    }
    __syncthreads();
  }
  // RT_BIG_U rows per thread per step, their loads issued together (one CTA of 16 warps per SM:
  // one row at a time left the warps waiting on their loads, 62 % long-scoreboard stalls)
  constexpr int U = RT_BIG_U;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r0 < a.nrows; r0 += U * stride) {
    double yv[U];
    int cv[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t row = r0 + u * stride;
      ok[u] = row < a.nrows;
      cv[u] = ok[u] ? a.code[row] : 0;
      yv[u] = (ok[u] && a.y) ? a.y[row] : 0.0;
      if (ok[u] && a.filt) ok[u] = a.filt[row] != 0;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
    if (!ok[u]) continue;
    const double y = yv[u];
    const int c = cv[u];
    if (a.in_smem) {
      atomicAdd(&cnt[c], 1u);
      if (a.y) {
        sred_add(&sums[2 * c], y);
        sred_add(&sums[2 * c + 1], y * y);
      }
    } else {
      gred_add(a.out + 3 * (int64_t)c, 1.0);
      if (a.y) {
        gred_add(a.out + 3 * (int64_t)c + 1, y);
        gred_add(a.out + 3 * (int64_t)c + 2, y * y);
      }
    }
    }
  }
  if (!a.in_smem) return;
  __syncthreads();
  for (int i = threadIdx.x; i < a.ncell; i += blockDim.x) {
    if (!cnt[i]) continue;
    gred_add(a.out + 3 * (int64_t)i, (double)cnt[i]);
    gred_add(a.out + 3 * (int64_t)i + 1, sums[2 * i]);
    gred_add(a.out + 3 * (int64_t)i + 2, sums[2 * i + 1]);
  }
}

// Fact -> dimension views V_j[k][p] = Σ_{root rows with key k} w_p, for the root children
// that carry predicate or group-by attributes.  Each warp takes a contiguous row range,
// lane = row; runs of equal keys are summed by a segmented warp scan (the root is sorted
// by its keys, so runs are long at the outer levels) and a run's total is carried across
// blocks until it ends.  Run totals go to a per-CTA open-addressing table in shared
// memory (Zipf-hot keys), to global atomics when a probe misses twice.
constexpr int RT_VCHUNK = 16;  // blocks of 32 rows per dynamically taken chunk (k_rt_views)
struct RtViewArgs {
  int* work;  // chunk counter (zeroed per launch)
  int64_t nrows;
  const double* y;
  const uint8_t* filt;
  int nlev;
  const int32_t* fk[RT_MAX_LEVELS];
  double* V[RT_MAX_LEVELS];  // [nk][3]
};
template <int NLEV>
__global__ void __launch_bounds__(256) k_rt_views(const __grid_constant__ RtViewArgs a) {
  extern __shared__ unsigned char vsm[];
  const int lane = threadIdx.x & 31;
  int* hkey = reinterpret_cast<int*>(vsm);                                     // [nlev][RT_HT]
  double* hval = reinterpret_cast<double*>(vsm + a.nlev * RT_HT * 4 + 16);  // [nlev][RT_HT][3]
  hval = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(hval) + 15) & ~(uintptr_t)15);
  for (int i = threadIdx.x; i < a.nlev * RT_HT; i += blockDim.x) {
    hkey[i] = -1;
    hval[3 * i] = hval[3 * i + 1] = hval[3 * i + 2] = 0.0;
  }
  __syncthreads();
  auto add = [&](int l, int key, double v0, double v1, double v2) {
    unsigned h = ((unsigned)key * 2654435761u) >> (32 - RT_HT_BITS);
#pragma unroll 1
    for (int probe = 0; probe < 2; probe++) {
      int* slot = hkey + l * RT_HT + h;
      int t = *slot;
      if (t == -1) {
        const int old = atomicCAS(slot, -1, key);
        t = old == -1 ? key : old;
      }
      if (t == key) {
        double* e = hval + 3 * (l * RT_HT + h);
        sred_add(e, v0);
        sred_add(e + 1, v1);
        sred_add(e + 2, v2);
        return;
      }
      h = (h + 1) & (RT_HT - 1);
    }
    double* e = a.V[l] + 3 * (int64_t)key;
    gred_add(e, v0);
    gred_add(e + 1, v1);
    gred_add(e + 2, v2);
  };
  // warps take chunks of RT_VCHUNK blocks dynamically (Zipf-hot and -cold regions cost very
  // differently); a run crossing a chunk edge is added in parts (linear)
  const int64_t nblk = (a.nrows + 31) / 32, nchunks = (nblk + RT_VCHUNK - 1) / RT_VCHUNK;
  int64_t b0 = 0, b1 = 0;
  int ckey[NLEV];
  double c0[NLEV], c1[NLEV], c2[NLEV];
  // lane-private sums of the carried run over blocks it goes on through (folded when it ends)
  double p0[NLEV], p1[NLEV], p2[NLEV];
  bool dirty[NLEV];
#pragma unroll
  for (int l = 0; l < NLEV; l++) {
    ckey[l] = -1;
    c0[l] = c1[l] = c2[l] = 0.0;
    p0[l] = p1[l] = p2[l] = 0.0;
    dirty[l] = false;
  }
  // software pipeline: the next block's y and keys are loaded while this block is scanned
  for (;;) {
  {
    int chk = 0;
    if (lane == 0) chk = atomicAdd(a.work, 1);
    chk = __shfl_sync(RFULL, chk, 0);
    if (chk >= nchunks) break;
    b0 = (int64_t)chk * RT_VCHUNK;
    b1 = b0 + RT_VCHUNK < nblk ? b0 + RT_VCHUNK : nblk;
  }
#pragma unroll
  for (int l = 0; l < NLEV; l++) {
    ckey[l] = -1;
    c0[l] = c1[l] = c2[l] = 0.0;
    p0[l] = p1[l] = p2[l] = 0.0;
    dirty[l] = false;
  }
  double ny = 0.0;
  bool npass = false;
  int nkey[NLEV];
  auto load = [&](int64_t b) {
    const int64_t row = 32 * b + lane;
    const bool v = b < b1 && row < a.nrows;
    const bool pass = v && (!a.filt || a.filt[row]);
    ny = pass ? (a.y ? a.y[row] : 0.0) : 0.0;
    npass = pass;
#pragma unroll
    for (int l = 0; l < NLEV; l++) nkey[l] = v ? a.fk[l][row] : -2;
  };
  load(b0);
  for (int64_t b = b0; b < b1; b++) {
    const int64_t row = 32 * b + lane;
    const bool vr = row < a.nrows;
    const int64_t nrem = a.nrows - 32 * b;
    const int nv = nrem < 32 ? (int)nrem : 32;
    const double y = ny;
    const bool rp = npass;
    int keys[NLEV];
#pragma unroll
    for (int l = 0; l < NLEV; l++) keys[l] = nkey[l];
    load(b + 1);
    const double w0 = rp ? 1.0 : 0.0, w1 = y, w2 = y * y;
    const unsigned pm = __ballot_sync(RFULL, rp);  // rows counted (w0 = 1): counts by popc, not scanned
#pragma unroll
    for (int l = 0; l < NLEV; l++) {
      const int key = keys[l];
      int prev = __shfl_up_sync(RFULL, key, 1);
      if (lane == 0) prev = ckey[l];
      const unsigned heads = __ballot_sync(RFULL, vr && key != prev);
      double v0 = w0, v1 = w1, v2 = w2;
      if (heads == 0) {  // the carried run goes on through the block: lane-private sums
        p0[l] += v0;
        p1[l] += v1;
        p2[l] += v2;
        dirty[l] = true;
        continue;
      }
      if (dirty[l]) {  // a run starts here: fold the lane-private sums into the carried run
        double q0 = p0[l], q1 = p1[l], q2 = p2[l];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          q0 += __shfl_xor_sync(RFULL, q0, o);
          q1 += __shfl_xor_sync(RFULL, q1, o);
          q2 += __shfl_xor_sync(RFULL, q2, o);
        }
        c0[l] += q0;
        c1[l] += q1;
        c2[l] += q2;
        p0[l] = p1[l] = p2[l] = 0.0;
        dirty[l] = false;
      }
      // segmented inclusive scan; segment s0 = the run containing the lane
      const unsigned upto = heads & ((2u << lane) - 1u);
      const int s0 = upto ? 31 - __clz(upto) : 0;
      v0 = (double)__popc(pm & ((2u << lane) - 1u) & ~((1u << s0) - 1u));
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double o1 = __shfl_up_sync(RFULL, v1, d), o2 = __shfl_up_sync(RFULL, v2, d);
        if (lane - d >= s0) {
          v1 += o1;
          v2 += o2;
        }
      }
      if (!upto) {  // lanes of the carried run (before the first head)
        v0 += c0[l];
        v1 += c1[l];
        v2 += c2[l];
      }
      // run ends: the lane before a head, and the carried run if the block starts a new one
      const bool ends = vr && lane < 31 && ((heads >> (lane + 1)) & 1u);  // the next row starts a run
      if (ends) add(l, upto ? key : ckey[l], v0, v1, v2);
      if ((heads & 1u) && lane == 0 && ckey[l] >= 0 && (c0[l] != 0.0 || c1[l] != 0.0 || c2[l] != 0.0))
        add(l, ckey[l], c0[l], c1[l], c2[l]);  // the carried run ended with the previous block
      // the last run continues: its total (at lane nv-1) becomes the carry
      c0[l] = __shfl_sync(RFULL, v0, nv - 1);
      c1[l] = __shfl_sync(RFULL, v1, nv - 1);
      c2[l] = __shfl_sync(RFULL, v2, nv - 1);
      ckey[l] = __shfl_sync(RFULL, key, nv - 1);
    }
  }
#pragma unroll
  for (int l = 0; l < NLEV; l++) {
    if (dirty[l]) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        p0[l] += __shfl_xor_sync(RFULL, p0[l], o);
        p1[l] += __shfl_xor_sync(RFULL, p1[l], o);
        p2[l] += __shfl_xor_sync(RFULL, p2[l], o);
      }
      c0[l] += p0[l];
      c1[l] += p1[l];
      c2[l] += p2[l];
    }
    if (lane == 0 && ckey[l] >= 0) add(l, ckey[l], c0[l], c1[l], c2[l]);
  }
  }  // chunks
  __syncthreads();
  for (int i = threadIdx.x; i < a.nlev * RT_HT; i += blockDim.x) {
    const int key = hkey[i];
    if (key < 0) continue;
    const int l = i / RT_HT;
    double* e = a.V[l] + 3 * (int64_t)key;
    gred_add(e, hval[3 * i]);
    gred_add(e + 1, hval[3 * i + 1]);
    gred_add(e + 2, hval[3 * i + 2]);
  }
}

// Dimension side: for every dimension row k of a view level, its V[k] goes to the
// histogram cell of each of its predicate attributes and to the group cell of each of its
// group-by attributes.
struct DimHist {
  int level;
  const void* col;  // dimension column (predicates) or codes per dense key (group-bys)
  int is_int, is_code;
  int nthr, thr_off, ncell;
  int64_t goff;
};
struct RtDimArgs {
  int nh;
  DimHist h[RT_MAX_DIM];
  const double* V[RT_MAX_LEVELS];
  int64_t nk[RT_MAX_LEVELS];
  const double* thr;
  double* out;
};
constexpr int RT_DIM_CELLS = 64;  // histograms up to this many cells: per-warp shared tables
__global__ void __launch_bounds__(256) k_rt_dims(const __grid_constant__ RtDimArgs a) {
  __shared__ double wtab[8][RT_DIM_CELLS * 3];
  const int i = blockIdx.y;
  const DimHist& h = a.h[i];
  const double* V = a.V[h.level];
  const int64_t nk = a.nk[h.level];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const bool small = h.ncell <= RT_DIM_CELLS;  // CTA-uniform
  double* tab = wtab[wib];
  if (small) {
    for (int k = lane; k < h.ncell * 3; k += 32) tab[k] = 0.0;
    __syncwarp();
  }
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < nk; base += stride) {
    const int64_t k = base + lane;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0;
    int c = -1;
    if (k < nk) {
      v0 = V[3 * k];
      if (v0 != 0.0) {
        v1 = V[3 * k + 1];
        v2 = V[3 * k + 2];
        if (h.is_code) {
          c = reinterpret_cast<const int32_t*>(h.col)[k];
        } else {
          const double x = h.is_int ? (double)reinterpret_cast<const int32_t*>(h.col)[k]
                                    : reinterpret_cast<const double*>(h.col)[k];
          c = rt_cell(x, a.thr + h.thr_off, h.nthr);
        }
      }
    }
    if (!small) {  // large domains: few collisions, fire-and-forget global reductions
      if (c >= 0) {
        double* e = a.out + h.goff + 3 * (int64_t)c;
        gred_add(e, v0);
        gred_add(e + 1, v1);
        gred_add(e + 2, v2);
      }
      continue;
    }
    // lanes with the same cell take turns (rank among their peers): plain read-modify-write
    const unsigned peers = __match_any_sync(RFULL, c);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    const int rounds = __reduce_max_sync(RFULL, c >= 0 ? rank + 1 : 0);
    for (int r = 0; r < rounds; r++) {
      if (c >= 0 && rank == r) {
        tab[3 * c] += v0;
        tab[3 * c + 1] += v1;
        tab[3 * c + 2] += v2;
      }
      __syncwarp();
    }
  }
  if (!small) return;
  __syncthreads();
  for (int k = threadIdx.x; k < h.ncell * 3; k += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < 8; w++) s += wtab[w][k];
    if (s != 0.0) gred_add(a.out + h.goff + k, s);
  }
}

// Scalar outputs: out[o] = Σ_t coef_t · acc[idx_t]; group tables: per (query, cell)
// table[cell][j] = Σ_p coef_{j,p} G[cell][p], counts[cell] = G[cell][0].
// Path condition φ = Π_i 1[A_i op_i t_i] shared by every product of the batch (a tree node's
// condition, §3 "Regression trees" P:528-555: α = Π of Kronecker deltas along the
// path): one byte per root row, dimension attributes read through the foreign keys.
constexpr int RT_MAX_PHI = 8;
constexpr int RT_MAX_CLASSES = 16;  // classes of a classification node's group-by attribute
struct RtPhi {
  const void* col;  // root column, or dimension column indexed by dense key
  const int32_t* fk;  // null: root attribute
  int is_int, kind;
  double t;
};
struct RtFilterArgs {
  int64_t nrows;
  int n;
  RtPhi p[RT_MAX_PHI];
  uint8_t* out;
};
__device__ __forceinline__ bool rt_pred(int kind, double x, double t) {
  switch (kind) {
    case LMFAO_F_LT: return x < t;
    case LMFAO_F_LE: return x <= t;
    case LMFAO_F_GT: return x > t;
    case LMFAO_F_GE: return x >= t;
    case LMFAO_F_EQ: return x == t;
    case LMFAO_F_IN: return x >= 0.0 && x <= 52.0 && x == floor(x) && (((unsigned long long)t >> (int)x) & 1ull);
    default: return x != t;
  }
}
__global__ void k_rt_filter(const __grid_constant__ RtFilterArgs a) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < a.nrows; r += (int64_t)gridDim.x * blockDim.x) {
    bool ok = true;
    for (int i = 0; i < a.n; i++) {
      const RtPhi& p = a.p[i];
      const int64_t k = p.fk ? (int64_t)p.fk[r] : r;
      const double x = p.is_int ? (double)reinterpret_cast<const int32_t*>(p.col)[k]
                                : reinterpret_cast<const double*>(p.col)[k];
      ok = ok && rt_pred(p.kind, x, p.t);
    }
    a.out[r] = ok ? 1 : 0;
  }
}

struct RtGroupOut {
  int64_t ncell, goff;
  int nudaf, coff;  // coefficients [nudaf][3] at coef + coff
  double* table;
  unsigned long long* counts;
};
// acc: the sums (under the path condition); cnt: the unconditioned accumulators, whose TOT[0]
// is the join size (the count of the scalar queries)
__global__ void k_rt_scalar(const double* __restrict__ acc, const double* __restrict__ cnt,
                            const int32_t* __restrict__ toff, const int32_t* __restrict__ tidx,
                            const double* __restrict__ tcoef, int nout, double* __restrict__ out,
                            unsigned long long* __restrict__ count) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = toff[o]; t < toff[o + 1]; t++) s += tcoef[t] * acc[tidx[t]];
    out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)cnt[0];
}
// group presence and counts are the join multiplicities (unconditioned, cnt), the UDAF values
// the sums under the path condition (acc)
__global__ void k_rt_groups(const double* __restrict__ acc, const double* __restrict__ cnt,
                            const RtGroupOut* __restrict__ gq, const double* __restrict__ coef) {
  const RtGroupOut g = gq[blockIdx.y];
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < g.ncell; c += (int64_t)gridDim.x * blockDim.x) {
    const double* e = acc + g.goff + 3 * c;
    g.counts[c] = (unsigned long long)cnt[g.goff + 3 * c];
    for (int j = 0; j < g.nudaf; j++) {
      const double* cf = coef + g.coff + 3 * j;
      g.table[c * g.nudaf + j] = cf[0] * e[0] + cf[1] * e[1] + cf[2] * e[2];
    }
  }
}

// Classification node outputs CT(X; α·...): per (query, UDAF) a term list over the
// accumulators of class c's pass (acc + c·nacc); counts from the unconditioned histogram of X.
struct RtCtOut {
  double* table;
  unsigned long long* counts;
  int ncell, nudaf, u;
  int64_t cnt_goff;
};
__global__ void k_rt_ct(const double* __restrict__ acc, int64_t nacc, const double* __restrict__ cnt,
                        const RtCtOut* __restrict__ outs, const int32_t* __restrict__ toff,
                        const int32_t* __restrict__ tidx, const double* __restrict__ tcoef) {
  const RtCtOut o = outs[blockIdx.x];
  for (int c = threadIdx.x; c < o.ncell; c += blockDim.x) {
    double v = 0.0;
    for (int t = toff[blockIdx.x]; t < toff[blockIdx.x + 1]; t++) v += tcoef[t] * acc[c * nacc + tidx[t]];
    o.table[(int64_t)c * o.nudaf + o.u] = v;
    if (o.u == 0) o.counts[c] = (unsigned long long)cnt[o.cnt_goff + 3 * c];
  }
}

// ======================================================================= host
struct FastRT : FastPaths {
  std::vector<int> handled;  // group indices (c->groups) computed here
  std::vector<FactHist> fh;  // small root histograms (k_rt_fact)
  std::vector<FactHist> fbig;  // large root group-bys (k_rt_big)
  int nparts = 1;
  std::vector<DimHist> dh;
  std::vector<double> thr;
  DevBuf dthr, acc, V, toff, tidx, tcoef, gq, gcoef;
  // path condition: the filter, and the unconditioned pass for the join multiplicities
  int nphi = 0;
  RtFilterArgs phi{};
  DevBuf filt, acc_all, V_all, vwork;
  std::vector<FactHist> fh_cnt;  // TOT + root group histograms
  std::vector<DimHist> dh_cnt;   // dimension group histograms
  // classification node: one conditioned pass per class of ct_code
  int ncls = 0, nct = 0;
  RtPhi ct_code{};
  std::vector<FactHist> fh_ct;
  std::vector<DimHist> dh_ct;
  DevBuf acc_cls, ct_outs, ct_toff, ct_tidx, ct_tcoef;
  int64_t nacc = 0;
  int nlev = 0;
  int64_t vnk[RT_MAX_LEVELS];
  int64_t voff[RT_MAX_LEVELS];
  const int32_t* vfk[RT_MAX_LEVELS];
  const double* y = nullptr;
  int nout = 0, ngq = 0;
  size_t fact_smem = 0, view_smem = 0;
  int eq_off = 0, tab_off = 0;
  int64_t vtotal = 0;
  std::string describe() const override {
    char b[200];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"rt\", \"fact_hists\": %zu, \"dim_hists\": %zu, \"views\": %d, \"groups\": %zu, "
                  "\"path_preds\": %d, \"classes\": %d}",
                  fh.size(), dh.size(), nlev, handled.size(), nphi, ncls);
    return b;
  }
  bool handles_group(int g) const override {
    for (int h : handled)
      if (h == g) return true;
    return false;
  }
  bool handles_all_groups() const override { return true; }
  bool skip_generic_views() const override { return true; }
  int run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) override;
  // the row filter takes its predicates from phi at every run: a new path condition needs no
  // re-planning (the unconditioned pass for the join multiplicities is planned with any φ)
  int set_condition(lmfao_ctx* c, int n, const lmfao_factor* f) override {
    if (nphi == 0 || n < 0 || n + (ncls > 0 ? 1 : 0) > RT_MAX_PHI) return -1;
    const Rel& R = c->rels[c->root];
    RtFilterArgs np = phi;
    np.n = n;
    for (int i = 0; i < n; i++) {
      const int a = f[i].attr, kind = f[i].kind;
      if (a < 0 || a >= (int)c->attrs.size() || kind < LMFAO_F_LT || kind > LMFAO_F_IN) return -1;
      const int o = c->owner[a];
      int lv = -1;
      if (o != c->root) {
        for (size_t j = 0; j < R.children.size(); j++)
          if (R.children[j] == o) lv = (int)j;
        if (lv < 0 || !c->rels[o].unique_key) return -1;  // deeper than a root child, or not a primary key
      }
      const Rel& O = lv < 0 ? R : c->rels[o];
      RtPhi& q = np.p[i];
      q.col = O.cols[O.find_attr(a)].buf.p;
      q.fk = lv < 0 ? nullptr : R.fk_dense[lv].as<int32_t>();
      q.is_int = c->attrs[a].dt == LMFAO_INT32;
      q.kind = kind;
      q.t = f[i].param;
    }
    phi = np;
    return 0;
  }
  cudaError_t pass(lmfao_ctx* c, cudaStream_t st, const uint8_t* fp, const double* yp, double* accp, double* Vp,
                   const std::vector<FactHist>& fhl, const std::vector<DimHist>& dhl, bool timed);
};

int FastRT::run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool& scalar_done) {
  const Rel& R = c->rels[c->root];
  const uint8_t* fp = nullptr;
  if (nphi > 0 && R.nrows > 0) {
    RtFilterArgs f = phi;
    f.nrows = R.nrows;
    f.out = filt.as<uint8_t>();
    k_rt_filter<<<148 * 8, 256, 0, st>>>(f);
    launches_add(1);
    fp = filt.as<uint8_t>();
  }
  CUDA_TRY(pass(c, st, fp, y, acc.as<double>(), V.as<double>(), fh, dh, true));
  const double* cnt = acc.as<double>();
  if (nphi > 0) {  // the join multiplicities do not depend on the path condition
    CUDA_TRY(pass(c, st, nullptr, nullptr, acc_all.as<double>(), V_all.as<double>(), fh_cnt, dh_cnt, false));
    cnt = acc_all.as<double>();
  }
  if (ncls > 0 && R.nrows == 0) CUDA_TRY(cudaMemsetAsync(acc_cls.p, 0, (size_t)ncls * nacc * 8, st));
  if (ncls > 0 && R.nrows > 0) {  // classification: the node's condition and X = class, per class
    for (int k = 0; k < ncls; k++) {
      RtFilterArgs f = phi;
      f.n = phi.n + 1;
      f.p[phi.n] = ct_code;
      f.p[phi.n].t = (double)k;
      f.nrows = R.nrows;
      f.out = filt.as<uint8_t>();
      k_rt_filter<<<148 * 8, 256, 0, st>>>(f);
      launches_add(1);
      CUDA_TRY(pass(c, st, filt.as<uint8_t>(), y, acc_cls.as<double>() + k * nacc, V.as<double>(), fh_ct, dh_ct, false));
    }
  }
  if (nct > 0) {
    k_rt_ct<<<nct, 128, 0, st>>>(acc_cls.as<double>(), nacc, cnt, ct_outs.as<RtCtOut>(), ct_toff.as<int32_t>(),
                                 ct_tidx.as<int32_t>(), ct_tcoef.as<double>());
    launches_add(1);
  }
  if (nout > 0) {
    k_rt_scalar<<<(nout + 255) / 256, 256, 0, st>>>(acc.as<double>(), cnt, toff.as<int32_t>(), tidx.as<int32_t>(),
                                                    tcoef.as<double>(), nout, c->scalar_out.as<double>(),
                                                    c->scalar_count.as<unsigned long long>());
    launches_add(1);
    scalar_done = true;
  }
  if (ngq > 0) {
    k_rt_groups<<<dim3(64, (unsigned)ngq), 256, 0, st>>>(acc.as<double>(), cnt, gq.as<RtGroupOut>(),
                                                        gcoef.as<double>());
    launches_add(1);
  }
  return cudaGetLastError();
}

// One pass of the histogram kernels over the root: fp = path-condition filter (null: every
// row), yp = target (null: w = (1, 0, 0)), into the accumulators accp and views Vp.
cudaError_t FastRT::pass(lmfao_ctx* c, cudaStream_t st, const uint8_t* fp, const double* yp, double* accp,
                         double* Vp, const std::vector<FactHist>& fhl, const std::vector<DimHist>& dhl, bool timed) {
  const Rel& R = c->rels[c->root];
  CUDA_TRY(cudaMemsetAsync(accp, 0, nacc * 8, st));
  if (vtotal && !dhl.empty()) CUDA_TRY(cudaMemsetAsync(Vp, 0, vtotal * 24, st));
  RtFactArgs fa{};
  fa.nrows = R.nrows;
  fa.y = yp;
  fa.filt = fp;
  fa.nh = (int)fhl.size();
  fa.nparts = nparts;
  for (size_t i = 0; i < fhl.size(); i++) {
    fa.h[i] = fhl[i];
    fa.wgt[i] = fhl[i].is_code ? 6 : 11;  // measured: a code row costs ~0.55 of a threshold row
  }
  fa.thr = dthr.as<double>();
  fa.eq_off = eq_off;
  fa.tab_off = tab_off;
  fa.out = accp;
  fa.npieces = nparts * RT_PIECES_PER_CTA;
  fa.work = vwork.as<int>() + 1;
  CUDA_TRY(cudaMemsetAsync(vwork.p, 0, 16, st));
  if (timed) scan_timer_begin(c, st);
  if (R.nrows > 0 && fa.nh > 0) {
    k_rt_fact<<<nparts, RT_FACT_WARPS * 32, fact_smem, st>>>(fa);
    launches_add(1);
  }
  if (timed) scan_timer_end(c, st);
  for (auto& h : fbig) {
    if (R.nrows <= 0) break;
    RtBigArgs ba{};
    ba.nrows = R.nrows;
    ba.y = yp;
    ba.filt = fp;
    ba.code = reinterpret_cast<const int32_t*>(h.col);
    ba.ncell = h.ncell;
    const size_t smem = (size_t)((h.ncell * 4 + 15) & ~15) + (size_t)h.ncell * 16;
    ba.in_smem = smem <= 200 * 1024;
    ba.out = accp + h.goff;
    k_rt_big<<<148, RT_BIG_THREADS, ba.in_smem ? smem : 0, st>>>(ba);
    launches_add(1);
  }
  if (nlev > 0 && R.nrows > 0 && !dhl.empty()) {
    RtViewArgs va{};
    CUDA_TRY(cudaMemsetAsync(vwork.p, 0, 16, st));
    va.work = vwork.as<int>();
    va.nrows = R.nrows;
    va.y = yp;
    va.filt = fp;
    va.nlev = nlev;
    for (int l = 0; l < nlev; l++) {
      va.fk[l] = vfk[l];
      va.V[l] = Vp + 3 * voff[l];
    }
    switch (nlev) {
#define VIEWS(n)                                               \
  case n:                                                      \
    k_rt_views<n><<<148 * 2, 256, view_smem, st>>>(va);        \
    break;
      VIEWS(1) VIEWS(2) VIEWS(3) VIEWS(4) VIEWS(5) VIEWS(6) VIEWS(7) VIEWS(8)
#undef VIEWS
    }
    launches_add(1);
  }
  if (!dhl.empty()) {
    RtDimArgs da{};
    da.nh = (int)dhl.size();
    for (size_t i = 0; i < dhl.size(); i++) da.h[i] = dhl[i];
    for (int l = 0; l < nlev; l++) {
      da.V[l] = Vp + 3 * voff[l];
      da.nk[l] = vnk[l];
    }
    da.thr = dthr.as<double>();
    da.out = accp;
    k_rt_dims<<<dim3(16, (unsigned)dhl.size()), 256, 0, st>>>(da);
    launches_add(1);
  }
  return cudaGetLastError();
}

}  // namespace

// Planner hook: every product is coeff · y^p · [at most one predicate on one attribute]
// (p <= 2, y one fp64 root attribute), every group-by query has one group-by attribute
// and predicate-free products; attributes belong to the root or to primary-key leaves
// of the root.  Otherwise nullptr.
// LMFAO_PLAN_DEBUG=1: report where the planner declines a batch
#define RT_DECLINE()                                                                             \
  do {                                                                                           \
    if (const char* e__ = std::getenv("LMFAO_PLAN_DEBUG"))                                       \
      if (e__[0] == '1') std::fprintf(stderr, "[lmfao] plan_rt declines (rt.cu:%d)\n", __LINE__); \
    return nullptr;                                                                              \
  } while (0)
FastPaths* plan_rt(lmfao_ctx* c) {
  const Rel& R = c->rels[c->root];
  for (int ch : R.children)
    if (!c->rels[ch].children.empty() || !c->rels[ch].unique_key) RT_DECLINE();
  auto level_of = [&](int attr) -> int {  // -1 root, j child index, -2 unsupported
    const int o = c->owner[attr];
    if (o == c->root) return -1;
    for (size_t j = 0; j < R.children.size(); j++)
      if (R.children[j] == o) return (int)j;
    return -2;
  };
  struct P {
    double coef;
    int pw;
    int pattr;  // -1: none
    int kind;
    double t;
  };
  int yattr = -1;
  bool any_pred = false;
  auto parse = [&](const QProduct& pr, P& out, bool allow_pred) -> bool {
    out = P{pr.coeff, 0, -1, 0, 0.0};
    for (auto& f : pr.f) {
      if (f.kind == LMFAO_F_CONST) {
        out.coef *= f.param;
      } else if (f.kind == LMFAO_F_IDENT) {
        if (yattr < 0) yattr = f.attr;
        if (f.attr != yattr) return false;
        if (++out.pw > 2) return false;
      } else {
        if (!allow_pred || out.pattr >= 0 || f.kind == LMFAO_F_IN) return false;  // IN: only in a path condition
        out.pattr = f.attr;
        out.kind = f.kind;
        out.t = f.param;
      }
    }
    return true;
  };
  // path condition φ: the predicates that every product of the batch carries (a tree node's
  // condition); each product is φ · (its own part), parsed below without φ
  struct PR {
    int attr, kind;
    double t;
    bool operator<(const PR& o) const {
      return attr != o.attr ? attr < o.attr : (kind != o.kind ? kind < o.kind : t < o.t);
    }
  };
  std::vector<PR> phi;
  {
    bool first = true;
    auto visit = [&](const QProduct& pr) -> bool {
      std::vector<PR> v;
      for (auto& f : pr.f)
        if (f.kind >= LMFAO_F_LT) {
          if (std::isnan(f.param)) return false;
          v.push_back(PR{f.attr, f.kind, f.param});
        }
      std::sort(v.begin(), v.end());
      if (first) {
        phi = v;
        first = false;
      } else {
        std::vector<PR> o;
        std::set_intersection(phi.begin(), phi.end(), v.begin(), v.end(), std::back_inserter(o));
        phi = o;
      }
      return true;
    };
    for (auto& Q : c->queries)
      for (auto& u : Q.udafs)
        for (auto& pr : u)
          if (!visit(pr)) RT_DECLINE();
  }
  if ((int)phi.size() > RT_MAX_PHI) RT_DECLINE();
  auto strip = [&](const QProduct& pr) {  // the product without (one occurrence of each) φ predicate
    QProduct o{pr.coeff, {}};
    std::vector<bool> used(phi.size(), false);
    for (auto& f : pr.f) {
      bool drop = false;
      if (f.kind >= LMFAO_F_LT)
        for (size_t i = 0; i < phi.size() && !drop; i++)
          if (!used[i] && phi[i].attr == f.attr && phi[i].kind == f.kind && phi[i].t == f.param) used[i] = drop = true;
      if (!drop) o.f.push_back(f);
    }
    return o;
  };
  std::vector<std::vector<std::vector<P>>> sq;  // scalar: per query, per udaf, products
  for (int q : c->scalar_queries) {
    std::vector<std::vector<P>> us;
    for (auto& u : c->queries[q].udafs) {
      std::vector<P> ps;
      for (auto& pr0 : u) {
        const QProduct pr = strip(pr0);
        P p;
        if (!parse(pr, p, true)) RT_DECLINE();
        if (p.pattr >= 0) any_pred = true;
        ps.push_back(p);
      }
      us.push_back(ps);
    }
    sq.push_back(us);
  }
  std::vector<std::vector<std::vector<P>>> gqp(c->groups.size());
  std::vector<char> ct(c->groups.size(), 0);  // classification queries: a predicate inside a group-by
  int ct_attr = -1;
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    const Query& Q = c->queries[c->groups[gi].q];
    if (Q.gb.size() != 1) RT_DECLINE();
    if (level_of(Q.gb[0]) == -2) RT_DECLINE();
    for (auto& u : Q.udafs) {
      std::vector<P> ps;
      for (auto& pr0 : u) {
        const QProduct pr = strip(pr0);
        P p;
        if (!parse(pr, p, true)) RT_DECLINE();
        if (p.pattr >= 0) ct[gi] = 1;
        ps.push_back(p);
      }
      gqp[gi].push_back(ps);
    }
    if (ct[gi]) {  // CT(X; α·1[A op t]): one conditioned pass per class of X
      if (ct_attr >= 0 && ct_attr != Q.gb[0]) RT_DECLINE();
      ct_attr = Q.gb[0];
      if (c->groups[gi].ncells > RT_MAX_CLASSES) RT_DECLINE();
    }
  }
  if (!any_pred && c->groups.empty() && phi.empty()) RT_DECLINE();
  for (auto& p : phi)
    if (level_of(p.attr) == -2) RT_DECLINE();
  if (yattr >= 0 && (level_of(yattr) != -1 || c->attrs[yattr].dt != LMFAO_FP64)) RT_DECLINE();
  std::unique_ptr<FastRT> rt(new FastRT());
  if (yattr >= 0) rt->y = (const double*)R.cols[R.find_attr(yattr)].buf.p;
  // predicate attributes and their sorted distinct thresholds
  std::map<int, std::set<double>> thr_of;
  for (auto& us : sq)
    for (auto& ps : us)
      for (auto& p : ps)
        if (p.pattr >= 0) {
          if (level_of(p.pattr) == -2) RT_DECLINE();
          if (std::isnan(p.t)) RT_DECLINE();
          thr_of[p.pattr].insert(p.t);
        }
  for (size_t gi = 0; gi < gqp.size(); gi++)
    if (ct[gi])
      for (auto& ps : gqp[gi])
        for (auto& p : ps)
          if (p.pattr >= 0) {
            if (level_of(p.pattr) == -2 || std::isnan(p.t)) RT_DECLINE();
            thr_of[p.pattr].insert(p.t);
        }
  // accumulator layout: [TOT 3] [fact / dim histograms] [group tables]
  int64_t nacc = 3;
  std::map<int, int64_t> hoff;  // predicate attr -> offset of its [ncell][3]
  std::map<int, int> hthr;      // attr -> thr offset
  std::vector<int> levels_used(R.children.size(), 0);
  for (auto& kv : thr_of) {
    const int a = kv.first, lv = level_of(a);
    const int thr_off = (int)rt->thr.size();
    for (double t : kv.second) rt->thr.push_back(t);
    const int nthr = (int)kv.second.size(), ncell = 2 * nthr + 1;
    hoff[a] = nacc;
    hthr[a] = thr_off;
    if (lv == -1) {
      FactHist h{};
      h.col = R.cols[R.find_attr(a)].buf.p;
      h.is_int = c->attrs[a].dt == LMFAO_INT32;
      h.is_code = 0;
      h.nthr = nthr;
      h.thr_off = thr_off;
      h.ncell = ncell;
      h.goff = nacc;
      if (nthr >= 2) {  // near-arithmetic thresholds: O(1) cell estimate (exact fix-up either way)
        const double t0 = *kv.second.begin(), tl = *kv.second.rbegin();
        const double step = (tl - t0) / (nthr - 1);
        bool ok = step > 0.0 && std::isfinite(step);
        int i = 0;
        double mu = 0.0;
        for (double t : kv.second) mu = std::max(mu, std::fabs(t - (t0 + i++ * step)) / step);
        ok = ok && mu <= 0.25;
        if (ok) {
          h.uniform = 1;
          h.t0 = t0;
          h.inv_h = 1.0 / step;
          h.margin = mu + 1e-9;
        }
      }
      if (nthr + 1 <= RT_SMALL) rt->fh.push_back(h);
      else rt->fbig.push_back(h);  // (predicate with > 20 thresholds: not expected; handled below)
    } else {
      const Rel& D = c->rels[R.children[lv]];
      DimHist h{};
      h.level = lv;
      h.col = D.cols[D.find_attr(a)].buf.p;
      h.is_int = c->attrs[a].dt == LMFAO_INT32;
      h.is_code = 0;
      h.nthr = nthr;
      h.thr_off = thr_off;
      h.ncell = ncell;
      h.goff = nacc;
      rt->dh.push_back(h);
      levels_used[lv] = 1;
    }
    nacc += 3 * (int64_t)ncell;
  }
  // group-by queries
  std::vector<RtGroupOut> gouts;
  std::vector<std::pair<int, int64_t>> ct_goff;  // classification queries: (group, offset of its count histogram)
  std::map<int, int64_t> code_goff;  // group-by attribute -> offset of its histogram
  std::vector<double> gcoef;
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    GroupPlan& gp = c->groups[gi];
    const Query& Q = c->queries[gp.q];
    const int a = Q.gb[0], lv = level_of(a);
    const int64_t ncell = gp.ncells;
    // one histogram of w per group-by attribute, shared by the queries grouping by it
    auto seen = code_goff.find(a);
    const bool fresh = seen == code_goff.end();
    const int64_t goff = fresh ? nacc : seen->second;
    if (!fresh) {
    } else if (lv == -1) {
      FactHist h{};
      h.col = gp.g.code[0];
      h.is_code = 1;
      h.ncell = (int)std::min<int64_t>(ncell, INT32_MAX);
      h.goff = nacc;
      if (ncell <= RT_SMALL) rt->fh.push_back(h);
      else rt->fbig.push_back(h);
    } else {
      DimHist h{};
      h.level = lv;
      h.col = gp.g.code[0];  // codes indexed by the child's dense key
      h.is_code = 1;
      h.ncell = (int)std::min<int64_t>(ncell, INT32_MAX);
      h.goff = nacc;
      rt->dh.push_back(h);
      levels_used[lv] = 1;
    }
    if (fresh) {
      code_goff[a] = nacc;
      nacc += 3 * ncell;
    }
    if (ct[gi]) {  // classification query: values from the per-class passes, counts from here
      rt->handled.push_back((int)gi);
      ct_goff.push_back({(int)gi, goff});
      continue;
    }
    RtGroupOut go{};
    go.ncell = ncell;
    go.goff = goff;
    go.nudaf = gp.nudaf;
    go.coff = (int)gcoef.size();
    go.table = gp.table.as<double>();
    go.counts = gp.counts.as<unsigned long long>();
    for (auto& ps : gqp[gi]) {
      double cf[3] = {0, 0, 0};
      for (auto& p : ps) cf[p.pw] += p.coef;
      gcoef.insert(gcoef.end(), cf, cf + 3);
    }
    gouts.push_back(go);
    rt->handled.push_back((int)gi);
  }
  if ((int)rt->fh.size() > RT_MAX_FACT || (int)rt->dh.size() > RT_MAX_DIM) RT_DECLINE();
  for (auto& h : rt->fbig)
    if (!h.is_code) RT_DECLINE();  // predicates with more than 20 distinct thresholds: generic path
  if (rt->fh.empty()) {  // TOT still comes from k_rt_fact: a one-cell histogram of the first root column
    FactHist h{};
    h.col = R.cols.empty() ? nullptr : R.cols[0].buf.p;
    if (!h.col) RT_DECLINE();
    h.is_int = R.cols[0].dt == LMFAO_INT32;
    h.ncell = 1;
    h.goff = nacc;
    nacc += 3;
    rt->fh.push_back(h);
  }
  // path condition: the filter's predicates, and the unconditioned pass (TOT + group histograms)
  rt->nphi = (int)phi.size();
  rt->phi.n = rt->nphi;
  for (int i = 0; i < rt->nphi; i++) {
    RtPhi& q = rt->phi.p[i];
    const int lv = level_of(phi[i].attr);
    const Rel& O = lv < 0 ? R : c->rels[R.children[lv]];
    q.col = O.cols[O.find_attr(phi[i].attr)].buf.p;
    q.fk = lv < 0 ? nullptr : R.fk_dense[lv].as<int32_t>();
    q.is_int = c->attrs[phi[i].attr].dt == LMFAO_INT32;
    q.kind = phi[i].kind;
    q.t = phi[i].t;
  }
  if (rt->nphi > 0) {
    for (auto& h : rt->fh)
      if (h.is_code) rt->fh_cnt.push_back(h);
    if (rt->fh_cnt.empty() || rt->fh_cnt[0].is_code) {  // TOT from a one-cell histogram in front
      FactHist h{};
      h.col = R.cols[0].buf.p;
      h.is_int = R.cols[0].dt == LMFAO_INT32;
      h.ncell = 1;
      h.goff = nacc;
      nacc += 3;
      rt->fh_cnt.insert(rt->fh_cnt.begin(), h);
    }
    for (auto& h : rt->dh)
      if (h.is_code) rt->dh_cnt.push_back(h);
  }
  if (!ct_goff.empty()) {  // classification: the class code per row, and the predicate histograms
    if (rt->nphi + 1 > RT_MAX_PHI) RT_DECLINE();
    const GroupPlan& gp = c->groups[ct_goff[0].first];
    const int lv = level_of(ct_attr);
    rt->ct_code.col = gp.g.code[0];  // codes: per root row, or per dense key of the child
    rt->ct_code.fk = lv < 0 ? nullptr : R.fk_dense[lv].as<int32_t>();
    rt->ct_code.is_int = 1;
    rt->ct_code.kind = LMFAO_F_EQ;
    rt->ncls = (int)gp.ncells;
    {
      FactHist h{};  // TOT of the class pass, in front
      h.col = R.cols[0].buf.p;
      h.is_int = R.cols[0].dt == LMFAO_INT32;
      h.ncell = 1;
      h.goff = nacc;
      nacc += 3;
      rt->fh_ct.push_back(h);
    }
    for (auto& h : rt->fh)
      if (!h.is_code && h.ncell > 1) rt->fh_ct.push_back(h);
    for (auto& h : rt->dh)
      if (!h.is_code) rt->dh_ct.push_back(h);
    if ((int)rt->fh_ct.size() > RT_MAX_FACT) RT_DECLINE();
  }
  rt->nacc = nacc;
  {  // one CTA per SM over equal pieces of the (histogram, row) space (the tables fill shared memory)
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    rt->nparts = nsm;
  }
  {
    int maxthr = 0;
    for (auto& h : rt->fh) maxthr = std::max(maxthr, h.nthr);
    rt->eq_off = (maxthr + 1) & ~1;
    rt->tab_off = rt->eq_off + ((3 * maxthr + 1) & ~1);
    rt->fact_smem = (size_t)rt->tab_off * 8 + (size_t)RT_FACT_WARPS * (RT_SMALL + 1) * 32 * 20;
  }
  // views
  int64_t vt = 0;
  for (size_t j = 0; j < R.children.size(); j++) {
    if (!levels_used[j]) continue;
    if (rt->nlev == RT_MAX_LEVELS) RT_DECLINE();
    const int l = rt->nlev++;
    rt->vfk[l] = R.fk_dense[j].as<int32_t>();
    rt->vnk[l] = c->rels[R.children[j]].nkeys;
    rt->voff[l] = vt;
    vt += rt->vnk[l];
    for (auto& h : rt->dh)
      if (h.level == (int)j) h.level = l;
    for (auto& h : rt->dh_cnt)
      if (h.level == (int)j) h.level = l;
    for (auto& h : rt->dh_ct)
      if (h.level == (int)j) h.level = l;
  }
  rt->vtotal = vt;
  rt->view_smem = (size_t)rt->nlev * RT_HT * 4 + 32 + (size_t)rt->nlev * RT_HT * 24;
  if (rt->view_smem > 200 * 1024) RT_DECLINE();
  // scalar outputs: term lists over the accumulators
  std::vector<int32_t> toff{0}, tidx;
  std::vector<double> tcoef;
  auto truth = [](int kind, int q, int cell) -> bool {  // predicate `op t_q` on cell
    switch (kind) {
      case LMFAO_F_LT: return cell <= 2 * q;
      case LMFAO_F_LE: return cell <= 2 * q + 1;
      case LMFAO_F_GT: return cell >= 2 * q + 2;
      case LMFAO_F_GE: return cell >= 2 * q + 1;
      case LMFAO_F_EQ: return cell == 2 * q + 1;
      default: return cell != 2 * q + 1;  // NE
    }
  };
  for (auto& us : sq)
    for (auto& ps : us) {
      for (auto& p : ps) {
        if (p.pattr < 0) {
          tidx.push_back(p.pw);
          tcoef.push_back(p.coef);
          continue;
        }
        const std::set<double>& ts = thr_of[p.pattr];
        const int q = (int)std::distance(ts.begin(), ts.find(p.t));
        const int ncell = 2 * (int)ts.size() + 1;
        for (int cell = 0; cell < ncell; cell++)
          if (truth(p.kind, q, cell)) {
            tidx.push_back((int32_t)(hoff[p.pattr] + 3 * cell + p.pw));
            tcoef.push_back(p.coef);
          }
      }
      toff.push_back((int32_t)tidx.size());
    }
  rt->nout = (int)toff.size() - 1;
  rt->ngq = (int)gouts.size();
  // classification outputs: per (query, UDAF) term lists over a class pass's accumulators
  std::vector<RtCtOut> couts;
  std::vector<int32_t> ctoff{0}, ctidx;
  std::vector<double> ctcoef;
  for (auto& cg : ct_goff) {
    GroupPlan& gp = c->groups[cg.first];
    for (int u = 0; u < gp.nudaf; u++) {
      for (auto& p : gqp[cg.first][u]) {
        if (p.pattr < 0) {
          ctidx.push_back(p.pw);
          ctcoef.push_back(p.coef);
          continue;
        }
        const std::set<double>& ts = thr_of[p.pattr];
        const int q = (int)std::distance(ts.begin(), ts.find(p.t));
        for (int cell = 0; cell < 2 * (int)ts.size() + 1; cell++)
          if (truth(p.kind, q, cell)) {
            ctidx.push_back((int32_t)(hoff[p.pattr] + 3 * cell + p.pw));
            ctcoef.push_back(p.coef);
          }
      }
      ctoff.push_back((int32_t)ctidx.size());
      couts.push_back(RtCtOut{gp.table.as<double>(), gp.counts.as<unsigned long long>(), (int)gp.ncells, gp.nudaf, u,
                              cg.second});
    }
  }
  rt->nct = (int)couts.size();
  cudaStream_t st = c->stream;
  auto up = [&](DevBuf& b, const void* src, size_t bytes) -> bool {
    if (b.alloc(std::max<size_t>(bytes, 16))) return false;
    if (bytes && cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, st)) return false;
    return true;
  };
  if (!up(rt->dthr, rt->thr.data(), rt->thr.size() * 8) || !up(rt->toff, toff.data(), toff.size() * 4) ||
      !up(rt->tidx, tidx.data(), tidx.size() * 4) || !up(rt->tcoef, tcoef.data(), tcoef.size() * 8) ||
      !up(rt->gq, gouts.data(), gouts.size() * sizeof(RtGroupOut)) ||
      !up(rt->gcoef, gcoef.data(), gcoef.size() * 8) ||
      !up(rt->ct_outs, couts.data(), couts.size() * sizeof(RtCtOut)) || !up(rt->ct_toff, ctoff.data(), ctoff.size() * 4) ||
      !up(rt->ct_tidx, ctidx.data(), ctidx.size() * 4) || !up(rt->ct_tcoef, ctcoef.data(), ctcoef.size() * 8))
    RT_DECLINE();
  if (rt->ncls > 0 && rt->acc_cls.alloc((size_t)rt->ncls * nacc * 8)) RT_DECLINE();
  if (rt->acc.alloc(nacc * 8) || rt->vwork.alloc(16)) RT_DECLINE();
  if (rt->V.alloc(std::max<int64_t>(vt, 1) * 24)) RT_DECLINE();
  if (rt->nphi > 0 && (rt->acc_all.alloc(nacc * 8) || rt->V_all.alloc(std::max<int64_t>(vt, 1) * 24))) RT_DECLINE();
  if ((rt->nphi > 0 || rt->ncls > 0) && rt->filt.alloc(std::max<int64_t>(R.nrows, 1))) RT_DECLINE();
  if (cudaStreamSynchronize(st)) RT_DECLINE();
  if (cudaFuncSetAttribute(k_rt_fact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rt->fact_smem) ||
      cudaFuncSetAttribute(k_rt_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024))
    RT_DECLINE();
  {
    cudaError_t e = cudaSuccess;
#define VATTR(n) \
  if (!e) e = cudaFuncSetAttribute(k_rt_views<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rt->view_smem);
    VATTR(1) VATTR(2) VATTR(3) VATTR(4) VATTR(5) VATTR(6) VATTR(7) VATTR(8)
#undef VATTR
    if (e) RT_DECLINE();
  }
  return rt.release();
}

}  // namespace lmfao
