// cube.cu — the histogram path (§8 row (e)(iii)) for group-by batches whose aggregates are
// linear in root measures: SUM(c_0 + Σ_j c_j · m_j) GROUP BY attributes of the root and of
// its primary-key children (§3 "Data cubes": one query per subset of
// the cube dimensions, each with SUM(m) for every measure; BASELINE.json configs[4]).
//
// The root is sorted by its children's dense keys in increasing domain order (levels
// 0..R-1), so for a cuboid whose deepest group-by attribute lives at level d, every
// maximal run of rows with equal keys at levels 0..d ("level-d run") falls into one cell.
// Per 32-row block a warp takes segmented sums of (1, m_1..m_M) over the level-d runs of
// every level d some cuboid needs, carries a run that continues into the next block, and at
// each run end adds the run's totals once to each of the level's cuboids (one atomic per
// UDAF and one for the count) — "cuboid cells updated once per run at the level of their
// deepest group-by attribute", instead of once per row.  Cuboids
// with root attributes use level R: runs of equal keys and equal root group-by codes.
// With primary-key leaves and no dangling rows (dropped at prepare) every root row joins
// exactly one row per child, so the join multiplicity of a row is 1.
#include <cstdlib>
#include <map>
#include <set>

#include "comm.h"
#include "ctx.h"

namespace lmfao {
namespace {

constexpr int CB_LEV = 8;     // root children
constexpr int CB_MEAS = 8;    // measure attributes per scan (more: one scan per group of 8)
constexpr int CB_MAXM = 64;   // distinct measure attributes of a batch
constexpr int CB_GB = 8;      // group-by attributes per cuboid
constexpr int CB_ATTR = 8;    // distinct group-by attributes of the batch
constexpr int CB_TERMS = 512; // UDAF terms of the batch (shared memory)
constexpr int CB_QD = 16;     // cuboids per level
constexpr int CB_ITEMS = 1024;  // (cuboid, non-constant UDAF) pairs of the batch
constexpr int CB_WARPS = 8;
constexpr unsigned BFULL = 0xffffffffu;

struct Cuboid {
  long long stride[CB_GB];
  int8_t aslot[CB_GB];          // group-by attribute i -> batch attribute slot
  int ngb, nudaf;
  int sparse, derived;          // derived: rolled up from a sparse cuboid's groups (finish_sparse), not flushed
  double* table;                // [cells][nudaf]; constant UDAFs are left to the compaction (countcoef)
  unsigned long long* counts;
  // sparse cuboid (too many cells for a dense table): one record per run end, sorted and
  // reduced after the scan: rkey[slot] = cell, rval[slot * (M + 1) + j] = S_j (a record's sums
  // contiguous); a work chunk's records start at rbase[chunk] (counted at plan time: the run
  // ends depend on the sorted keys only), so slots need no atomics and their order is fixed
  unsigned* rkey;
  double* rval;
  const long long* rbase;
  long long rcap;
  int smoff;                    // >= 0: a small table kept per CTA in shared memory at smoff (doubles):
  int sncell;                   //   [sncell][nudaf] doubles, then the counts [sncell] (u64)
};
static_assert(sizeof(Cuboid) % 16 == 0, "cuboids are copied to shared memory in 16-byte units");
// (cuboid, UDAF) pair of a level: value = Σ_{t in [t0, t1)} tc[t] · S_{tj[t]}
struct CubeItem {
  int16_t qk;  // cuboid within its level
  int16_t u;
  int16_t t0, t1;
  int32_t j1;  // single-term UDAF (t1 == t0 + 1): S index and coefficient, no term loop
  int32_t pad_;
  double c1;
};
struct CubeArgs {
  int64_t nrows;
  int R, M, nattr, nq, nterm, nitem;
  unsigned dmask;               // levels (0..R) with cuboids
  int nkey;                     // dense keys read per row (levels 0..nkey-1)
  int64_t chunk;                // rows per work unit (multiple of 32), taken dynamically
  int* work;                    // chunk counter (zeroed per run)
  const int32_t* key[CB_LEV];   // dense keys, level order
  const void* meas[CB_MEAS];
  int meas_i32[CB_MEAS];
  const int32_t* midx[CB_MEAS];  // dimension measure: its row per root row (the dense foreign key); null: root
  const int32_t* acode[CB_ATTR];  // codes per child dense key (level < R) or per root row (level R)
  int alvl[CB_ATTR];
  int qbeg[CB_LEV + 2];         // cuboids sorted by depth: depth d = [qbeg[d], qbeg[d + 1])
  int ibeg[CB_LEV + 2];         // items sorted by depth
  const Cuboid* q;
  const CubeItem* items;
  const int8_t* tj;             // [nterm] S index (0 = count, 1 + measure)
  const double* tc;             // [nterm] coefficient
  int ablate;                   // LMFAO_CUBE_ABLATE (profiling): 1 no flush, 2 counts only
  int nocount;                  // a later measure group's scan: the counts come from the first
  int nsmall;                   // doubles of the per-CTA small tables (shared memory)
  int slevel;                   // the sparse cuboids' level (-1: none)
  int count_only;               // plan time: count each chunk's run ends at slevel into tails[chunk]
  long long* tails;
  // k_cube_rec (the scan keeps only the sparse cuboids' level: C5's {A,B,C}, every other cuboid
  // rolled up from it): the records' cuboids
  int nrec;
  const long long* rbase;
  struct RecOut {
    unsigned* rkey;
    double* rval;
    const unsigned* part[CB_LEV];  // per level: the cell's part from that level's key (null: none)
    int ngb;                       // root group-by attributes (level R): slot, stride
    int8_t aslot[CB_GB];
    long long stride[CB_GB];
  } rec[4];
  int meas_plain;               // every measure an fp64 root column, no root group-by attribute
};

unsigned cgrid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

__device__ __forceinline__ double seg_scan(double v, int lane, int s0) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double u = __shfl_up_sync(BFULL, v, d);
    if (lane - d >= s0) v += u;
  }
  return v;
}

// shared memory: [cuboids | items | tj | tc | per warp: S[32][CB_MEAS+1], carry[CB_LEV+1][CB_MEAS+1],
// cells[32][CB_QD], codes[32][CB_ATTR]]
struct CubeSmem {
  size_t q, items, tj, tc, warps, per_warp, small;
  __host__ __device__ CubeSmem(int nq, int nitem, int nterm, int nsmall = 0) {
    q = 0;
    items = (nq * sizeof(Cuboid) + 15) / 16 * 16;
    tj = items + (nitem * sizeof(CubeItem) + 15) / 16 * 16;
    tc = tj + (nterm + 15) / 16 * 16;
    warps = tc + (size_t)nterm * 8;
    per_warp = (32 * (CB_MEAS + 1) + (CB_LEV + 1) * (CB_MEAS + 1) + 32 * CB_QD) * 8 + 32 * CB_ATTR * 4;
    small = warps + CB_WARPS * per_warp;
    nsm = nsmall;
  }
  int nsm;
  size_t total() const { return small + (size_t)nsm * 8; }
};

__global__ void __launch_bounds__(CB_WARPS * 32) k_cube(const __grid_constant__ CubeArgs a) {
  extern __shared__ __align__(16) unsigned char csm[];
  const CubeSmem L(a.nq, a.nitem, a.nterm, a.nsmall);
  double* stab = reinterpret_cast<double*>(csm + L.small);  // the small tables of this CTA
  for (int i = threadIdx.x; i < a.nsmall; i += blockDim.x) stab[i] = 0.0;
  const Cuboid* sq = reinterpret_cast<const Cuboid*>(csm + L.q);
  const CubeItem* items = reinterpret_cast<const CubeItem*>(csm + L.items);
  const int8_t* tj = reinterpret_cast<const int8_t*>(csm + L.tj);
  const double* tc = reinterpret_cast<const double*>(csm + L.tc);
  {
    const int4* src = reinterpret_cast<const int4*>(a.q);
    int4* dst = reinterpret_cast<int4*>(csm + L.q);
    for (int i = threadIdx.x; i < (int)(a.nq * sizeof(Cuboid) / 16); i += blockDim.x) dst[i] = src[i];
    for (int i = threadIdx.x; i < a.nitem; i += blockDim.x) reinterpret_cast<CubeItem*>(csm + L.items)[i] = a.items[i];
    for (int i = threadIdx.x; i < a.nterm; i += blockDim.x) {
      reinterpret_cast<int8_t*>(csm + L.tj)[i] = a.tj[i];
      reinterpret_cast<double*>(csm + L.tc)[i] = a.tc[i];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int M1 = a.M + 1;
  unsigned char* wsm = csm + L.warps + (size_t)wib * L.per_warp;
  double* S = reinterpret_cast<double*>(wsm);               // run totals of the level's run ends [tail][j]
  double* carry = S + 32 * (CB_MEAS + 1);                   // the run open at the previous block's end [d][j]
  long long* cells = reinterpret_cast<long long*>(carry + (CB_LEV + 1) * (CB_MEAS + 1));  // [tail][cuboid]
  int* codes = reinterpret_cast<int*>(cells + 32 * CB_QD);  // [tail][attr]
  const int64_t nchunks = (a.nrows + a.chunk - 1) / a.chunk;
  for (;;) {
    int ch = 0;
    if (lane == 0) ch = atomicAdd(a.work, 1);
    ch = __shfl_sync(BFULL, ch, 0);
    if (ch >= nchunks) break;
    const int64_t r0 = (int64_t)ch * a.chunk;
    const int64_t r1 = r0 + a.chunk < a.nrows ? r0 + a.chunk : a.nrows;
    for (int i = lane; i < (CB_LEV + 1) * (CB_MEAS + 1); i += 32) carry[i] = 0.0;
    __syncwarp();
    long long rdone = 0;  // this chunk's records so far (run ends at slevel)
    long long rb = 0;
    if (a.slevel >= 0 && !a.count_only) rb = sq[a.qbeg[a.slevel]].rbase[ch];
    for (int64_t base = r0; base < r1; base += 32) {
      const int64_t row = base + lane;
      const bool v = row < r1;
      const bool vn = row + 1 < r1;  // the next row exists in this chunk
      // level-d run starts of this row (st) and of the next row (stn); a row beyond the
      // chunk starts runs everywhere
      unsigned st = 0, stn = 0;  // bit d
      int key[CB_LEV];
      {
        bool chg = false, chgn = false;
#pragma unroll
        for (int l = 0; l < CB_LEV; l++) {
          if (l >= a.nkey) break;
          const int k = v ? a.key[l][row] : -1;
          key[l] = k;
          int kp = __shfl_up_sync(BFULL, k, 1);
          if (lane == 0) kp = base > r0 ? a.key[l][base - 1] : -2;
          int kn = __shfl_down_sync(BFULL, k, 1);
          if (lane == 31) kn = vn ? a.key[l][row + 1] : -3;
          chg |= kp != k;
          chgn |= !vn || kn != k;
          if (chg) st |= 1u << l;
          if (chgn) stn |= 1u << l;
        }
        if (a.dmask >> a.R & 1u) {  // level R: equal keys and equal root group-by codes
#pragma unroll
          for (int i = 0; i < CB_ATTR; i++) {
            if (i >= a.nattr) break;
            if (a.alvl[i] != a.R) continue;
            const int c = v ? a.acode[i][row] : -1;
            int cp = __shfl_up_sync(BFULL, c, 1);
            if (lane == 0) cp = base > r0 ? a.acode[i][base - 1] : -2;
            int cn = __shfl_down_sync(BFULL, c, 1);
            if (lane == 31) cn = vn ? a.acode[i][row + 1] : -3;
            chg |= cp != c;
            chgn |= !vn || cn != c;
          }
          if (chg) st |= 1u << a.R;
          if (chgn) stn |= 1u << a.R;
        }
        if (!v) st = stn = ~0u;
      }
      // the row's values: S_0 = 1 (count), S_j = m_j
      double xm[CB_MEAS + 1];
      xm[0] = v ? 1.0 : 0.0;
#pragma unroll
      for (int j = 0; j < CB_MEAS; j++) {
        xm[j + 1] = 0.0;
        if (j < a.M && v && !a.count_only) {
          const int64_t mr = a.midx[j] ? (int64_t)a.midx[j][row] : row;
          xm[j + 1] = a.meas_i32[j] ? (double)reinterpret_cast<const int32_t*>(a.meas[j])[mr]
                                    : reinterpret_cast<const double*>(a.meas[j])[mr];
        }
      }
      for (int d = a.R; d >= 0; d--) {
        if (!(a.dmask >> d & 1u)) continue;
        const bool s = st >> d & 1u, tail = v && (stn >> d & 1u);
        const unsigned starts = __ballot_sync(BFULL, s) | 1u;
        const int s0 = 31 - __clz(starts & ((2u << lane) - 1u));
        const bool cont0 = !__shfl_sync(BFULL, (int)s, 0);  // lane 0 continues the carried run
        const bool carry_out = !__shfl_sync(BFULL, (int)(stn >> d & 1u), 31);
        const unsigned T = __ballot_sync(BFULL, tail);  // run ends, compacted by rank
        const int nt = __popc(T), rank = __popc(T & ((1u << lane) - 1u));
        if (a.count_only) {
          if (d == a.slevel) rdone += nt;
          continue;
        }
        double* cd = carry + d * (CB_MEAS + 1);
#pragma unroll
        for (int j = 0; j <= CB_MEAS; j++) {
          if (j >= M1) break;
          double x = xm[j];
          if (lane == 0 && cont0) x += cd[j];
          x = seg_scan(x, lane, s0);
          if (tail) S[rank * (CB_MEAS + 1) + j] = x;
          __syncwarp();
          if (lane == 31) cd[j] = carry_out ? x : 0.0;
        }
        __syncwarp();
        if (nt && !(a.ablate & 1)) {
          // (0) each run end's group-by codes (attributes at levels <= d), loaded once
          if (tail) {
            int* cl = codes + rank * CB_ATTR;
#pragma unroll
            for (int i = 0; i < CB_ATTR; i++) {
              if (i >= a.nattr) break;
              const int l = a.alvl[i];
              if (l > d) continue;
              int idx = 0;
#pragma unroll
              for (int t = 0; t < CB_LEV; t++)
                if (t == l) idx = key[t];
              cl[i] = l >= a.R ? a.acode[i][row] : a.acode[i][idx];
            }
          }
          __syncwarp();
          // (1) per (run end, cuboid): the cell, the count, or a record of a sparse cuboid;
          // lanes split as tp run ends x nqd cuboids
          const int q0 = a.qbeg[d], nqd = a.qbeg[d + 1] - q0;
          {
            const int tp = 32 / nqd, sub = lane / nqd, qk = lane - sub * nqd;
            for (int tb = 0; tb < nt; tb += tp) {
              const int t = tb + sub;
              const bool act = sub < tp && t < nt;
              const Cuboid& q = sq[q0 + (act ? qk : 0)];
              long long cell = 0;
              if (act && !q.derived) {
                for (int i = 0; i < q.ngb; i++) cell += (long long)codes[t * CB_ATTR + q.aslot[i]] * q.stride[i];
                cells[t * CB_QD + qk] = cell;
                if (!q.sparse && !a.nocount) {
                  const unsigned long long n = (unsigned long long)S[t * (CB_MEAS + 1)];
                  if (q.smoff >= 0)
                    atomicAdd(reinterpret_cast<unsigned long long*>(stab + q.smoff + q.sncell * q.nudaf) + cell, n);
                  else gred_add(&q.counts[cell], n);
                }
              }
              if (act && q.sparse) {  // the t-th run end of this block: slot fixed at plan time
                const long long slot = rb + rdone + t;
                if (slot < q.rcap) {
                  q.rkey[slot] = (unsigned)cell;
                  for (int j = 0; j < M1; j++) q.rval[slot * M1 + j] = S[t * (CB_MEAS + 1) + j];
                }
              }
            }
          }
          __syncwarp();
          // (2) per (run end, non-constant UDAF of a dense cuboid): one reduction each
          if (!(a.ablate & 2)) {
            const int i0 = a.ibeg[d], nid = a.ibeg[d + 1] - i0;
            if (nid > 0 && nid <= 32) {
              const int tp = 32 / nid, sub = lane / nid, it = lane - sub * nid;
              const CubeItem e = items[i0 + it];
              const Cuboid& q = sq[q0 + e.qk];
              for (int tb = 0; tb < nt; tb += tp) {
                const int t = tb + sub;
                if (sub < tp && t < nt) {
                  double val = 0.0;
                  if (e.t1 == e.t0 + 1) val = e.c1 * S[t * (CB_MEAS + 1) + e.j1];
                  else
                    for (int k = e.t0; k < e.t1; k++) val = fma(tc[k], S[t * (CB_MEAS + 1) + tj[k]], val);
                  if (val != 0.0) {
                    const long long at = cells[t * CB_QD + e.qk] * q.nudaf + e.u;
                    if (q.smoff >= 0) sred_add(stab + q.smoff + at, val);
                    else gred_add(q.table + at, val);
                  }
                }
              }
            } else if (nid > 32) {
              for (int t = 0; t < nt; t++)
                for (int it = lane; it < nid; it += 32) {
                  const CubeItem e = items[i0 + it];
                  const Cuboid& q = sq[q0 + e.qk];
                  double val = 0.0;
                  if (e.t1 == e.t0 + 1) val = e.c1 * S[t * (CB_MEAS + 1) + e.j1];
                  else
                    for (int k = e.t0; k < e.t1; k++) val = fma(tc[k], S[t * (CB_MEAS + 1) + tj[k]], val);
                  if (val != 0.0) {
                    const long long at = cells[t * CB_QD + e.qk] * q.nudaf + e.u;
                    if (q.smoff >= 0) sred_add(stab + q.smoff + at, val);
                    else gred_add(q.table + at, val);
                  }
                }
            }
          }
        }
        if (d == a.slevel) rdone += nt;
        __syncwarp();
      }
    }
    if (a.count_only && lane == 0) a.tails[ch] = rdone;
  }
  if (a.nsmall == 0) return;
  __syncthreads();  // the CTA's small tables -> the global ones, nonzero entries only
  for (int k = 0; k < a.nq; k++) {
    const Cuboid& q = sq[k];
    if (q.smoff < 0) continue;
    const int nd = q.sncell * q.nudaf;  // [cells][nudaf] doubles, then the counts
    for (int i = threadIdx.x; i < nd; i += blockDim.x)
      if (stab[q.smoff + i] != 0.0) gred_add(q.table + i, stab[q.smoff + i]);
    const unsigned long long* sc = reinterpret_cast<const unsigned long long*>(stab + q.smoff + nd);
    for (int i = threadIdx.x; i < q.sncell; i += blockDim.x)
      if (sc[i]) gred_add(&q.counts[i], sc[i]);
  }
}

// The scan when only the sparse cuboids' level is left (every dense cuboid rolled up from a
// sparse one's groups; C5): per 32-row block, the run starts at that level from the keys
// (the previous row's keys carried in registers), segmented sums of the M1 values, and at each
// run end one record per sparse cuboid — its cell from the run's group-by codes and its sums —
// in the slot fixed at plan time.  Same chunks and run ends as k_cube's count mode.  The next
// block's keys, codes and measures are loaded before this block is processed (its row 0's
// keys are also this block's row 31's successors).
constexpr int REC_LEV = 4;   // k_cube_rec: key levels read
constexpr int REC_ATTR = 4;  // ... and root group-by attributes (level R)
// a record's cell = Σ_l part_l[key_l] (+ the root group-by codes × strides at level R), the
// per-level parts tabulated at plan time (k_cell_part): no per-attribute code lookups per row
// PLAIN: every measure an fp64 root column and no root group-by attribute
template <int M1, bool PLAIN>
struct RecRow {
  int k[REC_LEV], c[REC_ATTR];  // dense keys; root group-by codes
  unsigned cell;                // rec[0]'s cell (the parts from the keys)
  double x[M1];
  __device__ __forceinline__ void load(const CubeArgs& a, int64_t row, bool v) {
#pragma unroll
    for (int l = 0; l < REC_LEV; l++) k[l] = (l < a.nkey && v) ? a.key[l][row] : -1;
#pragma unroll
    for (int i = 0; i < REC_ATTR; i++) c[i] = (!PLAIN && a.slevel == a.R && i < a.nattr && a.alvl[i] == a.R && v) ? a.acode[i][row] : -1;
    cell = 0;
#pragma unroll
    for (int l = 0; l < REC_LEV; l++)
      if (l < a.nkey && a.rec[0].part[l] && v) cell += a.rec[0].part[l][k[l]];
    x[0] = v ? 1.0 : 0.0;
#pragma unroll
    for (int j = 1; j < M1; j++) {
      x[j] = 0.0;
      if (PLAIN) {
        if (v) x[j] = reinterpret_cast<const double*>(a.meas[j - 1])[row];
      } else if (v) {
        const int64_t mr = a.midx[j - 1] ? (int64_t)a.midx[j - 1][row] : row;
        x[j] = a.meas_i32[j - 1] ? (double)reinterpret_cast<const int32_t*>(a.meas[j - 1])[mr]
                                 : reinterpret_cast<const double*>(a.meas[j - 1])[mr];
      }
    }
  }
};
#ifndef REC_MINB
#define REC_MINB 3
#endif
template <int M1, bool PLAIN>
__global__ void __launch_bounds__(256, REC_MINB) k_cube_rec(const __grid_constant__ CubeArgs a) {
  const int lane = threadIdx.x & 31;
  const int d = a.slevel;
  const int64_t nchunks = (a.nrows + a.chunk - 1) / a.chunk;
  for (;;) {
    int ch = 0;
    if (lane == 0) ch = atomicAdd(a.work, 1);
    ch = __shfl_sync(BFULL, ch, 0);
    if (ch >= nchunks) break;
    const int64_t r0 = (int64_t)ch * a.chunk;
    const int64_t r1 = r0 + a.chunk < a.nrows ? r0 + a.chunk : a.nrows;
    long long slot0 = a.rbase[ch];
    double carry[M1];
#pragma unroll
    for (int j = 0; j < M1; j++) carry[j] = 0.0;
    int pk[REC_LEV], pc[REC_ATTR];  // the previous block's last row: keys, root group-by codes
#pragma unroll
    for (int l = 0; l < REC_LEV; l++) pk[l] = -2;
#pragma unroll
    for (int i = 0; i < REC_ATTR; i++) pc[i] = -2;
    RecRow<M1, PLAIN> cur, nxt;
    cur.load(a, r0 + lane, r0 + lane < r1);
    for (int64_t base = r0; base < r1; base += 32) {
      const int64_t row = base + lane;
      const bool v = row < r1;
      const bool vn = row + 1 < r1;
      if (base + 32 < r1) nxt.load(a, row + 32, row + 32 < r1);
      bool chg = false, chgn = false;
#pragma unroll
      for (int l = 0; l < REC_LEV; l++) {
        if (l >= a.nkey) continue;
        const int k = cur.k[l];
        int kp = __shfl_up_sync(BFULL, k, 1);
        if (lane == 0) kp = pk[l];
        int kn = __shfl_down_sync(BFULL, k, 1);
        const int k0n = __shfl_sync(BFULL, nxt.k[l], 0);
        if (lane == 31) kn = vn ? k0n : -3;
        pk[l] = __shfl_sync(BFULL, k, 31);
        chg |= kp != k;
        chgn |= !vn || kn != k;
      }
      if (!PLAIN && d == a.R) {  // level R: equal keys and equal root group-by codes
#pragma unroll
        for (int i = 0; i < REC_ATTR; i++) {
          if (i >= a.nattr || a.alvl[i] != a.R) continue;
          const int c = cur.c[i];
          int cp = __shfl_up_sync(BFULL, c, 1);
          if (lane == 0) cp = pc[i];
          int cn = __shfl_down_sync(BFULL, c, 1);
          const int c0n = __shfl_sync(BFULL, nxt.c[i], 0);
          if (lane == 31) cn = vn ? c0n : -3;
          pc[i] = __shfl_sync(BFULL, c, 31);
          chg |= cp != c;
          chgn |= !vn || cn != c;
        }
      }
      if (!v) chg = chgn = true;
      const bool tail = v && chgn;
      const unsigned starts = __ballot_sync(BFULL, chg) | 1u;
      const int s0 = 31 - __clz(starts & ((2u << lane) - 1u));
      const bool end31 = __shfl_sync(BFULL, (int)chgn, 31);  // lane 31 closes its run: no carry
      double x[M1];
#pragma unroll
      for (int j = 0; j < M1; j++) {
        x[j] = cur.x[j];
        if (lane == 0 && !chg) x[j] += carry[j];
        x[j] = seg_scan(x[j], lane, s0);
        const double c31 = __shfl_sync(BFULL, x[j], 31);
        carry[j] = end31 ? 0.0 : c31;
      }
      const unsigned T = __ballot_sync(BFULL, tail);
      if (tail) {
        const long long slot = slot0 + __popc(T & ((1u << lane) - 1u));
        for (int r = 0; r < a.nrec; r++) {
          const CubeArgs::RecOut& o = a.rec[r];
          unsigned cell = cur.cell;
          if (r > 0) {
            cell = 0;
#pragma unroll
            for (int l = 0; l < REC_LEV; l++)
              if (l < a.nkey && o.part[l]) cell += o.part[l][cur.k[l]];
          }
          for (int i = 0; i < (PLAIN ? 0 : o.ngb); i++) {  // root group-by attributes (level R)
            int code = 0;
#pragma unroll
            for (int t = 0; t < REC_ATTR; t++)
              if (t == o.aslot[i]) code = cur.c[t];
            cell += (unsigned)((long long)code * o.stride[i]);
          }
          o.rkey[slot] = cell;
          double* rv = o.rval + slot * M1;
#pragma unroll
          for (int j = 0; j < M1; j++) rv[j] = x[j];
        }
      }
      slot0 += __popc(T);
      cur = nxt;
    }
  }
}
// part[k] += code_i[k] * stride_i over a level's group-by attributes (plan time)
__global__ void k_cell_part(unsigned* part, const int32_t* code, long long stride, int64_t nkeys) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nkeys; k += (int64_t)gridDim.x * blockDim.x)
    part[k] += (unsigned)((long long)code[k] * stride);
}

// ---- sparse cuboids: run records -> sorted -> reduced groups, sizes on the device only
//
// World > 1: the cells are owned by the ranks in contiguous ranges
// (owner_range); each rank reduces its own records, and the reduce kernel writes every local
// group straight into its owner's receive buffer in peer memory (NVLink P2P stores, slot by a
// remote atomic on the owner's counter) — compute and exchange fused, no host round trip — then
// the owner sorts and reduces what it received: its range of the output, in canonical order.
// Two receive buffers (by run parity) and epoch flags order successive runs: a sender waits
// until the owner released the buffer of its parity, the owner until every sender signalled.
struct XHdr {                  // a rank's exchange header (mapped by every rank)
  unsigned long long cnt[2];   // records received, per run parity
  unsigned long long done[2];  // senders finished (cumulative over the runs of that parity)
  long long freed[2];          // the parity's buffer may be written by runs >= freed[b]
  long long epoch;             // runs started (identical on every rank: runs are collective)
  int err;                     // a wait timed out / a buffer overflowed
  int pad_;
};
static_assert(sizeof(XHdr) == 64, "exchange header layout");
struct XArgs {
  XHdr* const* hdr;            // [world] every rank's header
  unsigned* const* keys;       // [world] every rank's keys [2][capr]
  double* const* vals;         // [world] every rank's vals [2][capr][M1]
  long long capr;
  long long chunk;             // owner of a cell: cell / chunk
  int rank, world;
};
__device__ __forceinline__ long long x_epoch(const XHdr* h) { return *(volatile const long long*)&h->epoch - 1; }
__device__ bool x_spin(const volatile long long* p, long long target, XHdr* own) {  // *p >= target, 60 s at most
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*p < target) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) {
      atomicExch(&own->err, 1);
      return false;
    }
    __nanosleep(200);
  }
  return true;
}
__global__ void k_x_begin(XArgs x) {  // a new run; wait until every owner released this parity
  XHdr* own = x.hdr[x.rank];
  own->epoch += 1;
  __threadfence_system();
  const long long e = own->epoch - 1;
  for (int p = 0; p < x.world; p++) x_spin(&x.hdr[p]->freed[e & 1], e, own);
  __threadfence_system();
}
__global__ void k_x_signal(XArgs x) {  // this rank's groups are all in their owners' buffers
  const long long e = x_epoch(x.hdr[x.rank]);
  __threadfence_system();
  for (int p = 0; p < x.world; p++) atomicAdd(&x.hdr[p]->done[e & 1], 1ull);
}
__global__ void k_x_wait(XArgs x, unsigned long long* nrecv) {  // every sender of this run has signalled
  XHdr* own = x.hdr[x.rank];
  const long long e = x_epoch(own);
  const int b = (int)(e & 1);
  x_spin((const volatile long long*)&own->done[b], (long long)x.world * ((e >> 1) + 1), own);
  __threadfence_system();
  *nrecv = min(*(volatile unsigned long long*)&own->cnt[b], (unsigned long long)x.capr);
}
__global__ void k_x_take(XArgs x, const unsigned long long* nrecv, unsigned* __restrict__ rkey,
                         uint32_t* __restrict__ perm) {
  const long long n = (long long)*nrecv;
  const unsigned* src = x.keys[x.rank] + (size_t)(x_epoch(x.hdr[x.rank]) & 1) * x.capr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    rkey[i] = src[i];
    perm[i] = (uint32_t)i;
  }
}
__global__ void k_x_release(XArgs x) {  // the received records are consumed: free the parity
  XHdr* own = x.hdr[x.rank];
  const long long e = x_epoch(own);
  own->cnt[e & 1] = 0;
  __threadfence_system();
  *(volatile long long*)&own->freed[e & 1] = e + 2;
}

__global__ void k_rec_heads(const unsigned* __restrict__ key, int64_t cap, const unsigned long long* n_dev,
                            uint32_t* __restrict__ head) {
  const int64_t n = min(cap, (int64_t)*n_dev);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cap; i += (int64_t)gridDim.x * blockDim.x)
    head[i] = (i < n && (i == 0 || key[i] != key[i - 1])) ? 1u : 0u;
}
// group g's records are [gstart[g], gstart[g + 1]); *ng = the number of groups
__global__ void k_rec_starts(const uint32_t* __restrict__ head, const uint32_t* __restrict__ excl,
                             const unsigned long long* n_dev, int64_t cap, uint32_t* __restrict__ gstart,
                             unsigned long long* __restrict__ ng) {
  const int64_t n = min(cap, (int64_t)*n_dev);
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    gstart[0] = 0;
    *ng = 0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (head[i]) gstart[excl[i]] = (uint32_t)i;
    if (i == n - 1) {
      const uint32_t tot = excl[i] + head[i];
      gstart[tot] = (uint32_t)n;
      *ng = tot;
    }
  }
}
struct RecReduce {
  const unsigned* key;
  const uint32_t* perm;
  const uint32_t* gstart;  // [groups + 1] first record of each group (k_rec_starts)
  const unsigned long long* ng;  // groups (device)
  const double* rval;  // records' sums [.][M1] (merge: the own receive buffer, both parities)
  long long rcap;
  int64_t cap;
  const unsigned long long* n_dev;
  int M1, nudaf;
  const double* coef;  // [nudaf][M1]
  DecodeArgs d;
  int32_t* okeys;
  double* ovals;
  unsigned long long* ocnts;
  int nder;
  const struct Rollup* der;
  int send;            // world > 1, local groups: to their owners (x), not decoded
  int merge;           // world > 1, received groups: rval = own vals, parity from the epoch
  int sorted;          // rval is already in sorted order (k_rec_gather): perm not used
  unsigned* gcell;     // (merge rollups) the groups' cells
  double rinv[CB_GB];  // 1 / radix of Y's attributes (decode by reciprocal, corrected)
  size_t smem;         // dynamic shared memory: the coefficients and the rollups (0: read from global)
  XArgs x;
  int ablate;          // diagnostics only (LMFAO_CUBE_ABLATE=1, results invalid): no non-prefix rollup REDs
};
// A dense cuboid X at the sparse cuboid Y's level whose attributes are a subset of Y's: its
// cells are sums of Y's groups (X = Σ over Y's other attributes), added per reduced group of Y
// instead of per run end.
struct Rollup {
  double* table;
  unsigned long long* counts;
  const double* coef;  // [nudaf][M1]
  int nudaf, ngb;
  int pos[CB_GB];      // X's attribute i is Y's attribute pos[i]
  long long stride[CB_GB];
  unsigned long long cmask;
  int prefix;          // X's attributes are the first ngb of Y's: X's cells are runs of consecutive groups
  int same;            // X's UDAFs are Y's (same coefficient rows): X's values are the group's
  long long xstr_y[CB_GB];  // X's stride of Y's attribute t (0: X drops it)
};
// The records' sums in sorted order: sval[i][j] = rval[perm[i]][j], one thread per (i, j), so the
// M1 threads of a record read its M1 doubles together (a record per two 32-byte sectors instead
// of a sector per double when each group's thread followed perm itself) and the reduce below
// reads consecutive records.
__global__ void k_rec_gather(const __grid_constant__ RecReduce r, double* __restrict__ sval) {
  const int64_t n = min(r.cap, (int64_t)*r.n_dev);
  const double* rval = r.rval;
  if (r.merge) rval += (size_t)(x_epoch(r.x.hdr[r.x.rank]) & 1) * r.x.capr * r.M1;
  const int64_t tot = n * r.M1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / r.M1;
    const int j = (int)(t - i * r.M1);
    sval[t] = rval[(int64_t)r.perm[i] * r.M1 + j];
  }
}
// X = Σ of a dense cuboid Y over Y's attributes X lacks (X's attributes a subset of Y's, both
// rolled up from the same sparse cuboid): one thread per (X cell, column, slice of the dropped
// index space), plain loads of Y, one RED per thread (no per-group atomics for X).
struct DenseRollup {
  const double* ytab;
  const unsigned long long* ycnt;
  double* xtab;
  unsigned long long* xcnt;
  int nudaf, xngb, nd;           // X's UDAF columns (= Y's), X's attributes, dropped attributes
  long long xcells, dcells;      // X cells, dropped index space
  long long xstride[CB_GB];      // X's attribute i: stride in X
  long long xradix[CB_GB];
  long long ystride_x[CB_GB];    // ... and in Y
  long long dradix[CB_GB];       // dropped attribute j: radix, stride in Y
  long long dstride[CB_GB];
  int split;
};
__global__ void k_dense_rollup(const __grid_constant__ DenseRollup d) {
  const int ncol = d.nudaf + 1;  // + the count
  const long long tot = d.xcells * ncol * d.split;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const long long xc = t % d.xcells;
    const int col = (int)((t / d.xcells) % ncol);
    const int sl = (int)(t / (d.xcells * ncol));
    long long ybase = 0;
    for (int i = 0; i < d.xngb; i++) ybase += ((xc / d.xstride[i]) % d.xradix[i]) * d.ystride_x[i];
    const long long d0 = d.dcells * sl / d.split, d1 = d.dcells * (sl + 1) / d.split;
    double sv = 0.0;
    unsigned long long sc = 0;
    for (long long di = d0; di < d1; di++) {
      long long yc = ybase, rem = di;
      for (int j = d.nd - 1; j >= 0; j--) {
        yc += (rem % d.dradix[j]) * d.dstride[j];
        rem /= d.dradix[j];
      }
      if (col < d.nudaf) sv += d.ytab[yc * d.nudaf + col];
      else sc += d.ycnt[yc];
    }
    if (col < d.nudaf) {
      if (sv != 0.0) gred_add(&d.xtab[xc * d.nudaf + col], sv);
    } else if (sc) {
      gred_add(&d.xcnt[xc], sc);
    }
  }
}
// One lane per group (consecutive lanes: consecutive groups, in canonical order): the group's
// sums over its records, its output row (or, world > 1, its owner's buffer), and its share of
// the cuboids rolled up from it.  A rolled-up cuboid X whose attributes are the first of Y's
// (C5: {A,B} of {A,B,C}) has its cells on runs of consecutive groups: summed over the run by
// a segmented warp scan, one RED per run and warp instead of one per group.
// X = Σ of the sparse cuboid Y's groups over the attributes X drops, without atomics to global
// memory (world 1; X's UDAFs = Y's).  Y's groups are sorted by Y's cell; let p be the position
// of the last attribute X drops.  Groups with equal Y-attributes 0..p form a segment, sorted
// within by the suffix (Y's attributes after p, all kept by X); X's other attributes (kept,
// before p) are constant in a segment.  A tile = one value P of those kept prefix attributes and
// a range [lo, hi) of the suffix: its groups are, in every segment consistent with P (one per
// combination of the dropped attributes), the contiguous run with suffix in [lo, hi) — found by
// binary search — summed into a shared-memory table of the tile's cells and written once.
// C5: {B,C} (drop A: 50 segments per tile) and {A,C} (drop B: 1000) from {A,B,C}.
constexpr int MR_W = 1024;     // suffix cells per tile
constexpr int MR_SEG = 1024;   // segments per tile (more: per-group REDs instead)
struct MergeRollup {
  const unsigned* gcell;       // Y's groups' cells, ascending
  const unsigned long long* ng;
  const double* yvals;         // [g][nudaf]
  const unsigned long long* ycnt;
  double* xtab;
  unsigned long long* xcnt;
  int nudaf;
  int nseg;                    // combinations of the dropped attributes
  long long npre;              // values P of the kept prefix attributes
  long long suffix;            // suffix cells (Y's stride of attribute p)
  long long ntile_s;           // tiles per P
  // Y's attributes 0..p: radix, Y stride, role (0 dropped, 1 kept prefix), X stride (kept)
  int np;
  int role[CB_GB];
  long long radix[CB_GB], ystr[CB_GB], xstr[CB_GB];
  // suffix attributes (Y's after p): radix, Y stride, X stride
  int ns;
  long long sradix[CB_GB], systr[CB_GB], sxstr[CB_GB];
};
__device__ __forceinline__ int64_t lower_bound_u32(const unsigned* a, int64_t n, unsigned long long v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((unsigned long long)a[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__global__ void __launch_bounds__(256) k_merge_rollup(const __grid_constant__ MergeRollup m) {
  extern __shared__ __align__(16) unsigned char msm[];
  double* tv = reinterpret_cast<double*>(msm);                                        // [MR_W][nudaf]
  unsigned long long* tc = reinterpret_cast<unsigned long long*>(tv + (size_t)MR_W * m.nudaf);  // [MR_W]
  uint32_t* sbeg = reinterpret_cast<uint32_t*>(tc + MR_W);                            // [MR_SEG]
  uint32_t* soff = sbeg + MR_SEG;                                                     // [MR_SEG + 1]
  unsigned long long* sbase = reinterpret_cast<unsigned long long*>(soff + MR_SEG + 2);  // [MR_SEG]
  __shared__ uint32_t wsum[8];
  const int64_t ng = (int64_t)*m.ng;
  const int64_t ntiles = m.npre * m.ntile_s;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long P = tile / m.ntile_s;
    const long long lo = (tile - P * m.ntile_s) * MR_W;
    const long long hi = min(lo + MR_W, m.suffix);
    for (int i = threadIdx.x; i < MR_W * m.nudaf; i += blockDim.x) tv[i] = 0.0;
    for (int i = threadIdx.x; i < MR_W; i += blockDim.x) tc[i] = 0ull;
    // segment s: Y's prefix cell from P (kept attributes) and s (dropped ones)
    for (int sg = threadIdx.x; sg < m.nseg; sg += blockDim.x) {
      unsigned long long base = 0;
      long long rp = P, rs = sg;
      for (int i = m.np - 1; i >= 0; i--) {
        long long code;
        if (m.role[i]) {
          code = rp % m.radix[i];
          rp /= m.radix[i];
        } else {
          code = rs % m.radix[i];
          rs /= m.radix[i];
        }
        base += (unsigned long long)code * m.ystr[i];
      }
      const int64_t b = lower_bound_u32(m.gcell, ng, base + lo);
      const int64_t e = lower_bound_u32(m.gcell + b, ng - b, base + hi) + b;
      sbeg[sg] = (uint32_t)b;
      soff[sg] = (uint32_t)(e - b);
      sbase[sg] = base + lo;
    }
    __syncthreads();
    // exclusive scan of the slice lengths (one thread per segment chunk)
    {
      const int per = (m.nseg + blockDim.x - 1) / blockDim.x;
      const int s0 = threadIdx.x * per, s1 = min(m.nseg, s0 + per);
      uint32_t loc = 0;
      for (int sg = s0; sg < s1; sg++) loc += soff[sg];
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      uint32_t x = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(BFULL, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[warp] = x;
      __syncthreads();
      uint32_t pre = x - loc;
      for (int w = 0; w < warp; w++) pre += wsum[w];
      __syncthreads();
      for (int sg = s0; sg < s1; sg++) {
        const uint32_t l = soff[sg];
        soff[sg] = pre;
        pre += l;
      }
      if (threadIdx.x == blockDim.x - 1) soff[m.nseg] = pre;
    }
    __syncthreads();
    const uint32_t total = soff[m.nseg];
    for (uint32_t it = threadIdx.x; it < total; it += blockDim.x) {
      int a = 0, b = m.nseg;  // the segment: last s with soff[s] <= it
      while (b - a > 1) {
        const int mid = (a + b) >> 1;
        if (soff[mid] <= it) a = mid;
        else b = mid;
      }
      const int64_t g = (int64_t)sbeg[a] + (it - soff[a]);
      const int r = (int)(m.gcell[g] - sbase[a]);
      const double* yv = m.yvals + g * m.nudaf;
      for (int u = 0; u < m.nudaf; u++) sred_add(&tv[r * m.nudaf + u], yv[u]);
      atomicAdd(&tc[r], m.ycnt[g]);
    }
    __syncthreads();
    // write the tile's cells (each X cell belongs to one tile: plain stores)
    for (int r = threadIdx.x; r < hi - lo; r += blockDim.x) {
      const unsigned long long cnt = tc[r];
      if (!cnt) continue;
      long long xc = 0, rp = P, rr = lo + r;
      for (int i = m.np - 1; i >= 0; i--)
        if (m.role[i]) {
          xc += (rp % m.radix[i]) * m.xstr[i];
          rp /= m.radix[i];
        }
      for (int i = 0; i < m.ns; i++) xc += (rr / m.systr[i] % m.sradix[i]) * m.sxstr[i];
      m.xcnt[xc] = cnt;
      for (int u = 0; u < m.nudaf; u++) m.xtab[xc * m.nudaf + u] = tv[r * m.nudaf + u];
    }
    __syncthreads();
  }
}
inline size_t merge_smem(int nudaf) { return (size_t)MR_W * nudaf * 8 + MR_W * 8 + MR_SEG * 4 + (MR_SEG + 2) * 4 + MR_SEG * 8; }

__device__ __forceinline__ unsigned div_rinv(unsigned n, unsigned d, double rinv, unsigned& rem) {
  unsigned q = (unsigned)((double)n * rinv);  // within one of the quotient
  long long r = (long long)n - (long long)q * d;
  if (r < 0) {
    q--;
    r += d;
  } else if (r >= (long long)d) {
    q++;
    r -= d;
  }
  rem = (unsigned)r;
  return q;
}
#ifndef REC_RED_MINB
#define REC_RED_MINB 5  // resident CTAs per SM the register budget is sized for (C5 run, same box: 1 9.59, 5 9.21, 6 9.37 ms)
#endif
__global__ void __launch_bounds__(256, REC_RED_MINB) k_rec_reduce(const __grid_constant__ RecReduce r) {
  // the UDAF coefficients and the rollups in shared memory (read by every group)
  extern __shared__ __align__(16) unsigned char rsm[];
  const Rollup* der = r.der;
  const double* ycoef = r.coef;
  if (r.smem) {
    Rollup* sd = reinterpret_cast<Rollup*>(rsm);
    double* sc = reinterpret_cast<double*>(rsm + r.nder * sizeof(Rollup));
    for (int i = threadIdx.x; i < r.nudaf * r.M1; i += blockDim.x) sc[i] = r.coef[i];
    double* xc0 = sc + r.nudaf * r.M1;
    for (int x = 0; x < r.nder; x++) {
      if (threadIdx.x == 0) sd[x] = r.der[x];
      for (int i = threadIdx.x; i < r.der[x].nudaf * r.M1; i += blockDim.x) xc0[i] = r.der[x].coef[i];
      __syncthreads();
      if (threadIdx.x == 0) sd[x].coef = xc0;
      xc0 += r.der[x].nudaf * r.M1;
    }
    __syncthreads();
    der = sd;
    ycoef = sc;
  }
  const int64_t ng = (int64_t)*r.ng;
  const double* rval = r.rval;
  int b = 0;
  if (r.send || r.merge) b = (int)(x_epoch(r.x.hdr[r.x.rank]) & 1);
  if (r.merge && !r.sorted) rval += (size_t)b * r.x.capr * r.M1;
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g0 = wid * 32; g0 < ng; g0 += nw * 32) {
    const int64_t g = g0 + lane;
    const bool act = g < ng;
    double S[CB_MEAS + 1];
#pragma unroll
    for (int j = 0; j <= CB_MEAS; j++) S[j] = 0.0;
    unsigned cell = 0;
    unsigned code[CB_GB];
#pragma unroll
    for (int a = 0; a < CB_GB; a++) code[a] = 0;
    if (act) {
      const int64_t t0 = r.gstart[g], t1 = r.gstart[g + 1];
      for (int64_t t = t0; t < t1; t++) {
        const int64_t p = r.sorted ? t : (int64_t)r.perm[t];
        const double* rv = rval + p * r.M1;
        if (!(r.M1 & 1)) {  // 16-byte aligned record: pairs
#pragma unroll
          for (int j = 0; j < CB_MEAS; j += 2)
            if (j < r.M1) {
              const double2 w = *reinterpret_cast<const double2*>(rv + j);
              S[j] += w.x;
              S[j + 1] += w.y;
            }
        } else {
#pragma unroll
          for (int j = 0; j <= CB_MEAS; j++)
            if (j < r.M1) S[j] += rv[j];
        }
      }
      cell = r.key[t0];  // sparse cuboids have < 2^32 cells: 32-bit decode
      unsigned rest = cell;  // row-major: the last attribute varies fastest
#pragma unroll
      for (int a = CB_GB - 1; a >= 0; a--)
        if (a < r.d.ngb) rest = div_rinv(rest, (unsigned)r.d.radix[a], r.rinv[a], code[a]);
      if (r.send) {  // fused exchange: the group goes straight to its owner's buffer (peer memory)
        const int o = (int)(cell / (unsigned long long)r.x.chunk);
        const unsigned long long slot = atomicAdd(&r.x.hdr[o]->cnt[b], 1ull);
        if (slot < (unsigned long long)r.x.capr) {
          const size_t at = (size_t)b * r.x.capr + slot;
          r.x.keys[o][at] = cell;
#pragma unroll
          for (int j = 0; j <= CB_MEAS; j++)
            if (j < r.M1) r.x.vals[o][at * r.M1 + j] = S[j];
        } else {
          atomicExch(&r.x.hdr[r.x.rank]->err, 2);
        }
      } else {
#pragma unroll
        for (int a = 0; a < CB_GB; a++)
          if (a < r.d.ngb) r.okeys[g * r.d.ngb + a] = r.d.dict[a][code[a]];
        for (int u = 0; u < r.nudaf; u++) {
          double v = 0.0;
#pragma unroll
          for (int j = 0; j <= CB_MEAS; j++)
            if (j < r.M1) v = fma(ycoef[u * r.M1 + j], S[j], v);
          r.ovals[g * r.nudaf + u] = v;
        }
        r.ocnts[g] = (unsigned long long)S[0];
        if (r.gcell) r.gcell[g] = cell;
      }
    }
    for (int x = 0; x < r.nder; x++) {
      const Rollup& X = der[x];
      long long xc = -1 - lane;  // idle lanes: cells of their own
      if (act) {
        xc = 0;
#pragma unroll
        for (int t = 0; t < CB_GB; t++)
          if (t < r.d.ngb) xc += (long long)code[t] * X.xstr_y[t];
      }
      const double* xcoef = X.same ? ycoef : X.coef;
      if (X.prefix) {
        const long long xp = __shfl_up_sync(BFULL, xc, 1), xn = __shfl_down_sync(BFULL, xc, 1);
        const unsigned starts = __ballot_sync(BFULL, lane == 0 || xp != xc) | 1u;
        const int s0 = 31 - __clz(starts & ((2u << lane) - 1u));
        const bool tail = act && (lane == 31 || xn != xc);
        const double cnt = seg_scan(S[0], lane, s0);
        if (tail) gred_add(&X.counts[xc], (unsigned long long)cnt);
        for (int u = 0; u < X.nudaf; u++) {
          if (X.cmask >> u & 1ull) continue;
          double v = 0.0;
#pragma unroll
          for (int j = 0; j <= CB_MEAS; j++)
            if (j < r.M1) v = fma(xcoef[u * r.M1 + j], S[j], v);
          v = seg_scan(v, lane, s0);
          if (tail && v != 0.0) gred_add(&X.table[xc * X.nudaf + u], v);
        }
      } else if (act && !r.ablate) {
        gred_add(&X.counts[xc], (unsigned long long)S[0]);
        for (int u = 0; u < X.nudaf; u++) {
          if (X.cmask >> u & 1ull) continue;
          double v = 0.0;
#pragma unroll
          for (int j = 0; j <= CB_MEAS; j++)
            if (j < r.M1) v = fma(xcoef[u * r.M1 + j], S[j], v);
          if (v != 0.0) gred_add(&X.table[xc * X.nudaf + u], v);
        }
      }
    }
  }
}

// exchange buffer layout: [XHdr | keys [2][capr] (u32) | vals [2][capr][M1] (f64)]
inline size_t xoff_keys() { return 256; }
inline size_t xoff_vals(long long capr) { return (256 + (size_t)2 * capr * 4 + 255) / 256 * 256; }
inline size_t xbytes(long long capr, int M1) { return xoff_vals(capr) + (size_t)2 * capr * M1 * 8; }

struct SparseOut {  // per sparse cuboid: record buffers and sort temporaries
  int gi = -1, coff = 0, bits = 1;
  long long cap = 0;
  DevBuf key, val, n, perm, head, excl, gstart, ngl;
  std::vector<Rollup> der;  // dense cuboids rolled up from this one's groups
  DevBuf dder;
  // world > 1: the exchange
  long long capr = 0;
  DevBuf xbuf;                 // [XHdr | keys [2][capr] | vals [2][capr][M1]], mapped by every rank
  std::vector<void*> peers;    // every rank's xbuf
  DevBuf xptrs;                // [3][world] device pointers: headers, keys, vals
  DevBuf rkey, rperm, rhead, rexcl, rgstart, nrecv;
  DevBuf sval;                 // records' sums in sorted order (k_rec_gather), local then received
  std::vector<DenseRollup> dense_rollups;  // derived cuboids summed from a larger derived one, after the reduce
  std::vector<MergeRollup> merges;        // derived cuboids merged from the sorted groups (world 1), after the reduce
  size_t reduce_smem = 0;                 // k_rec_reduce's shared memory (coefficients and rollups)
  XArgs x{};
  Comm* comm = nullptr;
  SparseOut() = default;
  SparseOut(SparseOut&&) = default;
  ~SparseOut() {
    if (comm && !peers.empty()) comm->unmap_peers(peers);
  }
};

struct FastCube : FastPaths {
  CubeArgs ca{};
  std::vector<CubeArgs> parts;  // one scan per group of up to CB_MEAS measures
  std::vector<DevBuf> pbuf;     // per part: items, tj, tc
  DevBuf dq, dcoef, ditems, dtj, dtc, dwork, rbase;
  std::vector<SparseOut> sparse;
  int nq = 0, grid = 148, rec_grid = 148;
  DevBuf parts_tab[4 * CB_LEV];  // k_cube_rec: per record cuboid and level, the cell parts
  bool rec_only = false;  // k_cube_rec
  bool gather_first = false;
  size_t smem = 0;
  bool graph_ok() const override { return true; }  // device-side sizes: no host synchronisation
  std::string describe() const override {
    char b[160];
    int m = 0;
    for (auto& p : parts) m += p.M;
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"cube\", \"cuboids\": %d, \"sparse\": %d, \"measures\": %d, \"scans\": %d, \"levels\": %d, "
                  "\"scan\": \"%s\"}",
                  nq, (int)sparse.size(), m, (int)parts.size(), ca.R, rec_only ? "records" : "levels");
    return b;
  }
  bool handles_group(int) const override { return true; }
  bool handles_all_groups() const override { return true; }
  bool skip_generic_views() const override { return true; }
  int run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool&) override {
    for (auto& gp : c->groups) {
      if (gp.direct) continue;
      CUDA_TRY(cudaMemsetAsync(gp.counts.p, 0, gp.ncells * 8, st));
      CUDA_TRY(cudaMemsetAsync(gp.table.p, 0, gp.table.bytes, st));
    }
    for (size_t pi = 0; pi < parts.size(); pi++) {
      CUDA_TRY(cudaMemsetAsync(dwork.as<int>() + pi, 0, 4, st));
      CubeArgs a = parts[pi];
      a.nrows = c->rels[c->root].nrows;
      a.work = dwork.as<int>() + pi;
      if (a.nrows > 0) {
        const int64_t nch = (a.nrows + a.chunk - 1) / a.chunk;
        if (rec_only) {
          const int64_t g = std::min<int64_t>((nch + 7) / 8, rec_grid);
          CUDA_TRY(launch_rec(a, (unsigned)g, st));
        } else {
          const int64_t g = std::min<int64_t>((nch + CB_WARPS - 1) / CB_WARPS, grid);
          k_cube<<<(unsigned)g, CB_WARPS * 32, smem, st>>>(a);
        }
        launches_add(1);
      }
    }
    CUDA_TRY(cudaGetLastError());
    for (auto& sp : sparse) CUDA_TRY(finish_sparse(c, sp, st));
    return cudaSuccess;
  }
  static cudaError_t launch_rec(const CubeArgs& a, unsigned g, cudaStream_t st) {
    switch (a.M + 1) {
#define LMFAO_REC(m)                                       \
  case m:                                                  \
    if (a.meas_plain) k_cube_rec<m, true><<<g, 256, 0, st>>>(a); \
    else k_cube_rec<m, false><<<g, 256, 0, st>>>(a);       \
    break;
      LMFAO_REC(1) LMFAO_REC(2) LMFAO_REC(3) LMFAO_REC(4) LMFAO_REC(5) LMFAO_REC(6) LMFAO_REC(7) LMFAO_REC(8) LMFAO_REC(9)
#undef LMFAO_REC
      default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
  // sort the records by cell, reduce equal cells: the groups in canonical order (world 1), or,
  // world > 1, every local group to its owner (peer memory) and the owner's merge of what it
  // received.  Sizes stay on the device (record count, groups): no host synchronisation.
  cudaError_t finish_sparse(lmfao_ctx* c, SparseOut& sp, cudaStream_t st) {
    GroupPlan& gp = c->groups[sp.gi];
    const bool dist = c->world > 1;
    if (dist) {
      k_x_begin<<<1, 1, 0, st>>>(sp.x);
      launches_add(1);
    }
    const int64_t cap = sp.cap;
    CUDA_TRY(iota_u32(sp.perm.as<uint32_t>(), cap, st));
    CUDA_TRY(radix_sort_pairs(sp.key.as<uint32_t>(), sp.perm.as<uint32_t>(), cap, sp.bits, st,
                              sp.n.as<unsigned long long>()));
    k_rec_heads<<<cgrid(cap), 256, 0, st>>>(sp.key.as<unsigned>(), cap, sp.n.as<unsigned long long>(),
                                            sp.head.as<uint32_t>());
    CUDA_TRY(exclusive_scan_u32(sp.head.as<uint32_t>(), sp.excl.as<uint32_t>(), cap, st));
    RecReduce r{};
    r.key = sp.key.as<unsigned>();
    r.perm = sp.perm.as<uint32_t>();
    k_rec_starts<<<cgrid(cap), 256, 0, st>>>(sp.head.as<uint32_t>(), sp.excl.as<uint32_t>(), sp.n.as<unsigned long long>(),
                                             cap, sp.gstart.as<uint32_t>(),
                                             dist ? sp.ngl.as<unsigned long long>() : gp.ngroups_dev.as<unsigned long long>());
    r.gstart = sp.gstart.as<uint32_t>();
    r.ng = dist ? sp.ngl.as<unsigned long long>() : gp.ngroups_dev.as<unsigned long long>();
    r.rval = sp.val.as<double>();
    r.rcap = sp.cap;
    r.cap = cap;
    r.n_dev = sp.n.as<unsigned long long>();
    r.M1 = ca.M + 1;
    r.nudaf = gp.nudaf;
    r.coef = dcoef.as<double>() + sp.coff;
    for (int a = 0; a < gp.d.ngb; a++) r.rinv[a] = 1.0 / (double)gp.d.radix[a];
    r.smem = sp.reduce_smem;
    r.d = gp.d;
    r.okeys = gp.rkeys.as<int32_t>();
    r.ovals = gp.rvals.as<double>();
    r.ocnts = gp.rcnts.as<unsigned long long>();
    r.nder = (int)sp.der.size();
    r.der = sp.dder.as<Rollup>();
    r.send = dist;
    r.x = sp.x;
    r.ablate = [] {
      const char* e = std::getenv("LMFAO_CUBE_ABLATE");
      return e && e[0] == '1' ? 1 : 0;
    }();
    if (gather_first) {  // LMFAO_CUBE_GATHER=1: the records' sums permuted first (round-2 A/B)
      k_rec_gather<<<cgrid(cap * r.M1), 256, 0, st>>>(r, sp.sval.as<double>());
      r.rval = sp.sval.as<double>();
      r.sorted = 1;
    }
    r.gcell = sp.merges.empty() || dist ? nullptr : sp.excl.as<unsigned>();  // excl is free after k_rec_starts
    k_rec_reduce<<<cgrid(cap), 256, r.smem, st>>>(r);
    for (auto& mr : sp.merges) {
      MergeRollup m = mr;
      m.gcell = sp.excl.as<unsigned>();
      m.ng = gp.ngroups_dev.as<unsigned long long>();
      const long long nt = m.npre * m.ntile_s;
      k_merge_rollup<<<(unsigned)std::max<long long>(1, std::min<long long>(nt, 148 * 4)), 256, merge_smem(m.nudaf), st>>>(m);
    }
    launches_add((int)sp.merges.size());
    for (auto& dr : sp.dense_rollups) {
      const long long tot = dr.xcells * (dr.nudaf + 1) * dr.split;
      k_dense_rollup<<<(unsigned)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 148 * 16)), 256, 0, st>>>(dr);
    }
    launches_add(3 + (gather_first ? 1 : 0) + (int)sp.dense_rollups.size());  // heads, starts, (gather), reduce, rollups
    CUDA_TRY(cudaGetLastError());
    if (!dist) return cudaSuccess;
    // world > 1: signal the owners, then merge what this rank received
    k_x_signal<<<1, 1, 0, st>>>(sp.x);
    if (c->comm->phase(st)) return cudaErrorUnknown;  // loopback: every rank has sent
    const int64_t capr = sp.capr;
    unsigned long long* nrecv = sp.nrecv.as<unsigned long long>();
    k_x_wait<<<1, 1, 0, st>>>(sp.x, nrecv);
    k_x_take<<<cgrid(capr), 256, 0, st>>>(sp.x, nrecv, sp.rkey.as<unsigned>(), sp.rperm.as<uint32_t>());
    CUDA_TRY(radix_sort_pairs(sp.rkey.as<uint32_t>(), sp.rperm.as<uint32_t>(), capr, sp.bits, st, nrecv));
    k_rec_heads<<<cgrid(capr), 256, 0, st>>>(sp.rkey.as<unsigned>(), capr, nrecv, sp.rhead.as<uint32_t>());
    CUDA_TRY(exclusive_scan_u32(sp.rhead.as<uint32_t>(), sp.rexcl.as<uint32_t>(), capr, st));
    RecReduce m = r;
    m.key = sp.rkey.as<unsigned>();
    m.perm = sp.rperm.as<uint32_t>();
    k_rec_starts<<<cgrid(capr), 256, 0, st>>>(sp.rhead.as<uint32_t>(), sp.rexcl.as<uint32_t>(), nrecv, capr,
                                              sp.rgstart.as<uint32_t>(), gp.ngroups_dev.as<unsigned long long>());
    m.gstart = sp.rgstart.as<uint32_t>();
    m.ng = gp.ngroups_dev.as<unsigned long long>();
    m.rval = reinterpret_cast<const double*>(sp.xbuf.as<char>() + xoff_vals(sp.capr));
    m.rcap = capr;
    m.cap = capr;
    m.n_dev = nrecv;
    m.nder = 0;  // the rollups were added from the local groups
    m.send = 0;
    m.merge = 1;
    m.sorted = 0;
    k_rec_gather<<<cgrid(capr * m.M1), 256, 0, st>>>(m, sp.sval.as<double>());
    m.rval = sp.sval.as<double>();
    m.sorted = 1;
    m.smem = 0;
    k_rec_reduce<<<cgrid(capr), 256, 0, st>>>(m);
    k_x_release<<<1, 1, 0, st>>>(sp.x);
    launches_add(8);
    return cudaGetLastError();
  }
};

}  // namespace

// Planner hook: every group-by query's UDAFs are sums of products of constants and at most
// one identity factor on a root attribute, the root's children are primary-key leaves, and
// the batch's measures, levels and attributes fit the kernel's limits.  Otherwise nullptr.
FastPaths* plan_cube(lmfao_ctx* c) {
  if (c->groups.empty()) return nullptr;
  const Rel& R = c->rels[c->root];
  const int nlev = (int)R.children.size();
  if (nlev > CB_LEV) return nullptr;
  for (int ch : R.children)
    if (!c->rels[ch].children.empty() || !c->rels[ch].unique_key) return nullptr;
  std::vector<int> lvl_of_child(nlev, -1);
  for (size_t p = 0; p < c->levels.size(); p++) lvl_of_child[c->levels[p]] = (int)p;
  std::unique_ptr<FastCube> fc(new FastCube());
  CubeArgs& a = fc->ca;
  a.R = nlev;
  for (int l = 0; l < nlev; l++) a.key[l] = R.fk_dense[c->levels[l]].as<int32_t>();
  std::vector<int> meas;  // attr ids
  auto meas_slot = [&](int attr) -> int {
    for (size_t i = 0; i < meas.size(); i++)
      if (meas[i] == attr) return (int)i;
    if (meas.size() == (size_t)CB_MAXM) return -1;
    meas.push_back(attr);
    return (int)meas.size() - 1;
  };
  for (auto& gp : c->groups)
    for (auto& u : c->queries[gp.q].udafs)
      for (auto& p : u) {
        int nid = 0;
        for (auto& f : p.f) {
          if (f.kind == LMFAO_F_CONST) continue;
          if (f.kind != LMFAO_F_IDENT || ++nid > 1) return nullptr;
          const int o = c->owner[f.attr];
          if (o != c->root && c->rels[o].parent != c->root) return nullptr;  // root or a (primary-key leaf) child
          if (meas_slot(f.attr) < 0) return nullptr;
        }
      }
  const int M = (int)meas.size(), M1 = M + 1;
  std::map<int, int> aslot;  // group-by attribute -> slot
  struct QInfo {
    Cuboid q;
    int gi, depth;
    std::vector<std::vector<std::pair<int, double>>> terms;  // per UDAF (j, coef), empty: constant
    std::vector<double> dense;                               // [nudaf][M1] (sparse reduce)
  };
  std::vector<QInfo> qs;
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    GroupPlan& gp = c->groups[gi];
    const Query& Q = c->queries[gp.q];
    if (Q.gb.size() > (size_t)CB_GB || gp.nudaf > 64) return nullptr;
    QInfo qi{};
    qi.gi = (int)gi;
    Cuboid& q = qi.q;
    q.ngb = (int)Q.gb.size();
    for (int i = 0; i < q.ngb; i++) {
      const int cc = gp.g.code_child[i];
      const int l = cc < 0 ? nlev : lvl_of_child[cc];
      auto it = aslot.find(Q.gb[i]);
      if (it == aslot.end()) {
        if ((int)aslot.size() == CB_ATTR) return nullptr;
        const int sl = (int)aslot.size();
        aslot[Q.gb[i]] = sl;
        a.acode[sl] = gp.g.code[i];
        a.alvl[sl] = l;
        it = aslot.find(Q.gb[i]);
      }
      q.aslot[i] = (int8_t)it->second;
      q.stride[i] = gp.g.stride[i];
      qi.depth = std::max(qi.depth, l);
    }
    q.nudaf = gp.nudaf;
    q.table = gp.table.as<double>();
    q.counts = gp.counts.as<unsigned long long>();
    for (int u = 0; u < gp.nudaf; u++) {
      std::vector<double> row(M1, 0.0);
      bool constant = true;
      for (auto& p : Q.udafs[u]) {
        double v = p.coeff;
        int j = 0;
        for (auto& f : p.f) {
          if (f.kind == LMFAO_F_CONST) v *= f.param;
          else j = 1 + meas_slot(f.attr), constant = false;
        }
        row[j] += v;
      }
      std::vector<std::pair<int, double>> t;
      if (!constant)
        for (int j = 0; j < M1; j++)
          if (row[j] != 0.0) t.push_back({j, row[j]});
      qi.terms.push_back(t);
      qi.dense.insert(qi.dense.end(), row.begin(), row.end());
    }
    a.dmask |= 1u << qi.depth;
    qs.push_back(std::move(qi));
  }
  std::stable_sort(qs.begin(), qs.end(), [](const QInfo& x, const QInfo& y) { return x.depth < y.depth; });
  for (int d = 0, k = 0; d <= CB_LEV + 1; d++) {
    while (k < (int)qs.size() && qs[k].depth < d) k++;
    a.qbeg[d] = k;
  }
  a.M = std::min(M, CB_MEAS);
  std::vector<const void*> mptr(M);
  std::vector<int> mi32(M);
  std::vector<const int32_t*> midx(M);
  for (int j = 0; j < M; j++) {
    const int o = c->owner[meas[j]];
    const Rel& O = c->rels[o];
    const Column& col = O.cols[O.find_attr(meas[j])];
    mptr[j] = col.buf.p;
    mi32[j] = col.dt == LMFAO_INT32;
    midx[j] = nullptr;
    if (o != c->root)  // a dimension measure: read through the dense foreign key
      for (size_t ch = 0; ch < R.children.size(); ch++)
        if (R.children[ch] == o) midx[j] = R.fk_dense[ch].as<int32_t>();
  }
  const int nparts = std::max(1, (M + CB_MEAS - 1) / CB_MEAS);
  a.nattr = (int)aslot.size();
  a.nq = (int)qs.size();
  a.chunk = 32 * 32;
  if (const char* ab = std::getenv("LMFAO_CUBE_ABLATE")) a.ablate = std::atoi(ab);
  for (int d = 0; d <= CB_LEV; d++)
    if (a.qbeg[d + 1] - a.qbeg[d] > CB_QD) return nullptr;
  // cuboids with more cells than 2^25 (C5's {A,B,C}: 5·10^8) keep no dense table: their
  // run records are sorted and reduced after the scan (single GPU; LMFAO_CUBE_DENSE=1: off)
  const char* dn = std::getenv("LMFAO_CUBE_DENSE");
  const bool allow_sparse = nparts == 1 && !(dn && dn[0] == '1') && (c->world == 1 || c->comm);
  const int64_t nrows = R.nrows, nchunks = (nrows + a.chunk - 1) / a.chunk;
  const char* smin = std::getenv("LMFAO_CUBE_SPARSE_CELLS");  // tests: lower the threshold
  const int64_t sparse_min = smin ? std::atoll(smin) : ((int64_t)1 << 25);
  std::vector<Cuboid> hq;
  std::vector<double> dense;
  a.slevel = -1;
  if (const char* gf = std::getenv("LMFAO_CUBE_GATHER")) fc->gather_first = gf[0] == '1';
  std::vector<int> coffs, sparse_of(qs.size(), -1);
  for (size_t k = 0; k < qs.size(); k++) {
    hq.push_back(qs[k].q);
    const int coff = (int)dense.size();
    coffs.push_back(coff);
    dense.insert(dense.end(), qs[k].dense.begin(), qs[k].dense.end());
    GroupPlan& gp = c->groups[qs[k].gi];
    if (!allow_sparse || gp.ncells <= sparse_min || gp.ncells > ((int64_t)1 << 32)) continue;
    if (a.slevel >= 0 && qs[k].depth != a.slevel) continue;  // one level's run ends give the slots
    a.slevel = qs[k].depth;
    SparseOut sp;
    sp.gi = qs[k].gi;
    sp.coff = coff;
    sp.cap = nrows + nchunks + 64;
    while (sp.bits < 32 && ((int64_t)1 << sp.bits) < gp.ncells) sp.bits++;
    if (sp.key.alloc(sp.cap * 4) || sp.val.alloc((size_t)sp.cap * M1 * 8) || sp.n.alloc(8) || sp.perm.alloc(sp.cap * 4) ||
        sp.head.alloc(sp.cap * 4) || sp.excl.alloc(sp.cap * 4) || sp.gstart.alloc((sp.cap + 1) * 4) || sp.ngl.alloc(8) ||
        gp.ngroups_dev.alloc(8))
      return nullptr;
    int64_t ocap = std::min<int64_t>(sp.cap, gp.ncells);  // groups this rank outputs
    if (c->world > 1) {
      // receive capacity: every rank's groups are distinct cells, so at most world x (own
      // cells), and at most the records of the whole root
      const int64_t G = c->world, chunk = (gp.ncells + G - 1) / G;
      const int64_t nch_all = (c->root_rows_global + a.chunk - 1) / a.chunk;
      sp.capr = std::min<int64_t>(c->root_rows_global + G * (nch_all + 64), G * chunk);
      ocap = std::min<int64_t>(sp.capr, chunk);
      {
        StreamScope plain(nullptr, false);  // CUDA IPC needs cudaMalloc memory (not the stream-ordered pool)
        if (sp.xbuf.alloc(xbytes(sp.capr, M1))) return nullptr;
      }
      XHdr h{};
      h.freed[0] = 0;
      h.freed[1] = 1;
      if (cudaMemsetAsync(sp.xbuf.p, 0, 256, c->stream) ||
          cudaMemcpyAsync(sp.xbuf.p, &h, sizeof h, cudaMemcpyHostToDevice, c->stream) ||
          cudaStreamSynchronize(c->stream))
        return nullptr;
      if (c->comm->map_peers(sp.xbuf.p, sp.peers, c->stream)) return nullptr;  // collective
      std::vector<void*> ptr(3 * G);
      for (int r = 0; r < G; r++) {
        ptr[r] = sp.peers[r];
        ptr[G + r] = (char*)sp.peers[r] + xoff_keys();
        ptr[2 * G + r] = (char*)sp.peers[r] + xoff_vals(sp.capr);
      }
      if (sp.xptrs.alloc(ptr.size() * sizeof(void*)) ||
          cudaMemcpyAsync(sp.xptrs.p, ptr.data(), ptr.size() * sizeof(void*), cudaMemcpyHostToDevice, c->stream))
        return nullptr;
      sp.x.hdr = (XHdr* const*)sp.xptrs.p;
      sp.x.keys = (unsigned* const*)(sp.xptrs.as<void*>() + G);
      sp.x.vals = (double* const*)(sp.xptrs.as<void*>() + 2 * G);
      sp.x.capr = sp.capr;
      sp.x.chunk = chunk;
      sp.x.rank = c->rank;
      sp.x.world = (int)G;
      sp.comm = c->comm.get();
      if (sp.rkey.alloc(sp.capr * 4) || sp.rperm.alloc(sp.capr * 4) || sp.rhead.alloc(sp.capr * 4) ||
          sp.rexcl.alloc(sp.capr * 4) || sp.rgstart.alloc((sp.capr + 1) * 4) || sp.nrecv.alloc(8))
        return nullptr;
    }
    if (gp.rkeys.alloc(std::max<int64_t>(ocap, 1) * gp.d.ngb * 4) || gp.rvals.alloc(std::max<int64_t>(ocap, 1) * gp.nudaf * 8) ||
        gp.rcnts.alloc(std::max<int64_t>(ocap, 1) * 8) ||
        ((c->world > 1 || fc->gather_first) && sp.sval.alloc((size_t)std::max<int64_t>(sp.cap, sp.capr) * M1 * 8)))
      return nullptr;
    gp.ngroups_on_device = true;
    Cuboid& q = hq[k];
    q.sparse = 1;
    q.rkey = sp.key.as<unsigned>();
    q.rval = sp.val.as<double>();
    q.rcap = sp.cap;
    sparse_of[k] = (int)fc->sparse.size();
    fc->sparse.push_back(std::move(sp));
  }
  // dense cuboids over a subset of a sparse cuboid's attributes: rolled up from its reduced
  // groups (one update per group, not per run end), at any level — every join row falls in
  // exactly one of Y's groups, so X's cells are sums of Y's.  C5: all seven cuboids from
  // {A,B,C}, so the scan keeps only {A,B,C}'s level.  LMFAO_CUBE_ROLLUP=0: off.
  std::vector<std::vector<int>> der_coff(fc->sparse.size()), der_k(fc->sparse.size());
  const char* ru = std::getenv("LMFAO_CUBE_ROLLUP");
  const char* rmin = std::getenv("LMFAO_CUBE_ROLLUP_MIN");  // cuboids with fewer cells stay on the scan
  const int64_t rollup_min = rmin ? std::atoll(rmin) : 0;
  if (!(ru && ru[0] == '0'))
    for (size_t k = 0; k < qs.size(); k++) {
      if (hq[k].sparse || c->groups[qs[k].gi].ncells < rollup_min) continue;
      for (size_t y = 0; y < qs.size(); y++) {
        if (sparse_of[y] < 0) continue;
        Rollup ro{};
        bool sub = true;
        for (int i = 0; i < hq[k].ngb && sub; i++) {
          int p = -1;
          for (int t = 0; t < hq[y].ngb; t++)
            if (hq[y].aslot[t] == hq[k].aslot[i]) p = t;
          sub = p >= 0;
          ro.pos[i] = p;
          ro.stride[i] = hq[k].stride[i];
        }
        if (!sub) continue;
        ro.prefix = 1;  // X's attributes = Y's first ngb (as a set)
        for (int i = 0; i < hq[k].ngb; i++) ro.prefix &= ro.pos[i] < hq[k].ngb;
        ro.table = hq[k].table;
        ro.counts = hq[k].counts;
        ro.nudaf = hq[k].nudaf;
        ro.ngb = hq[k].ngb;
        for (int u = 0; u < hq[k].nudaf; u++)
          if (qs[k].terms[u].empty()) ro.cmask |= 1ull << u;
        hq[k].derived = 1;
        fc->sparse[sparse_of[y]].der.push_back(ro);
        der_coff[sparse_of[y]].push_back(coffs[k]);
        der_k[sparse_of[y]].push_back((int)k);
        break;
      }
    }
  // a derived cuboid X whose attributes are a proper subset of another derived cuboid Y's (same
  // sparse source, same UDAFs) is summed from Y's dense table after the reduce instead of from
  // every group (C5: {C} from {A,C}: 50 loads per cell instead of 6 REDs per {A,B,C} group)
  for (size_t y = 0; y < fc->sparse.size(); y++) {
    SparseOut& sp = fc->sparse[y];
    std::vector<Rollup> keep;
    std::vector<int> keep_coff, keep_k;
    auto contains = [&](int ky, int kx) {  // attrs(X) ⊊ attrs(Y), same UDAFs
      if (hq[ky].ngb <= hq[kx].ngb || qs[ky].dense != qs[kx].dense) return false;
      for (int i = 0; i < hq[kx].ngb; i++) {
        bool f = false;
        for (int t = 0; t < hq[ky].ngb; t++) f |= hq[ky].aslot[t] == hq[kx].aslot[i];
        if (!f) return false;
      }
      return true;
    };
    std::vector<char> maximal(sp.der.size(), 1);  // rolled up from the groups in any case
    for (size_t xi = 0; xi < sp.der.size(); xi++)
      for (size_t yi = 0; yi < sp.der.size(); yi++)
        if (yi != xi && contains(der_k[y][yi], der_k[y][xi])) maximal[xi] = 0;
    for (size_t xi = 0; xi < sp.der.size(); xi++) {
      const int kx = der_k[y][xi];
      const GroupPlan& gx = c->groups[qs[kx].gi];
      int best = -1;
      for (size_t yi = 0; yi < sp.der.size(); yi++) {
        const int ky = der_k[y][yi];
        if (yi == xi || !maximal[yi] || !contains(ky, kx)) continue;
        if (best < 0 || c->groups[qs[ky].gi].ncells < c->groups[qs[der_k[y][best]].gi].ncells) best = (int)yi;
      }
      if (best < 0) {
        keep.push_back(sp.der[xi]);
        keep_coff.push_back(der_coff[y][xi]);
        keep_k.push_back(kx);
        continue;
      }
      const int ky = der_k[y][best];
      const GroupPlan& gy = c->groups[qs[ky].gi];
      DenseRollup d{};
      d.ytab = gy.table.as<double>();
      d.ycnt = gy.counts.as<unsigned long long>();
      d.xtab = const_cast<GroupPlan&>(gx).table.as<double>();
      d.xcnt = const_cast<GroupPlan&>(gx).counts.as<unsigned long long>();
      d.nudaf = gx.nudaf;
      d.xngb = hq[kx].ngb;
      d.xcells = gx.ncells;
      for (int i = 0; i < hq[kx].ngb; i++) {
        d.xstride[i] = hq[kx].stride[i];
        d.xradix[i] = gx.d.radix[i];
        for (int t = 0; t < hq[ky].ngb; t++)
          if (hq[ky].aslot[t] == hq[kx].aslot[i]) d.ystride_x[i] = hq[ky].stride[t];
      }
      d.dcells = 1;
      for (int t = 0; t < hq[ky].ngb; t++) {
        bool in_x = false;
        for (int i = 0; i < hq[kx].ngb; i++) in_x |= hq[ky].aslot[t] == hq[kx].aslot[i];
        if (in_x) continue;
        d.dradix[d.nd] = gy.d.radix[t];
        d.dstride[d.nd] = hq[ky].stride[t];
        d.dcells *= gy.d.radix[t];
        d.nd++;
      }
      d.split = (int)std::max<long long>(1, std::min<long long>(d.dcells, (d.dcells + 63) / 64));
      sp.dense_rollups.push_back(d);
    }
    if (keep.size() != sp.der.size() && !sp.dense_rollups.empty()) {
      // every Y must be rolled up from the groups: a Y that became dense-rolled keeps its entry
      sp.der = keep;
      der_coff[y] = keep_coff;
      der_k[y] = keep_k;
    }
    // world 1: a non-prefix rollup with Y's UDAFs and few segments per tile can be merged from
    // the sorted groups (k_merge_rollup) instead of per-group REDs.  Opt-in (LMFAO_CUBE_MERGE=1):
    // on C5 it measured 4.1 ms for {A,C} + {B,C} against ~1.1 ms of REDs (the per-tile binary
    // searches and the latency-bound slice walks dominate).
    const char* mg = std::getenv("LMFAO_CUBE_MERGE");
    int ky = -1;
    for (size_t k = 0; k < qs.size(); k++)
      if (sparse_of[k] == (int)y) ky = (int)k;
    if (c->world == 1 && ky >= 0 && mg && mg[0] == '1') {
      const GroupPlan& gy = c->groups[qs[ky].gi];
      std::vector<Rollup> left;
      std::vector<int> left_coff, left_k;
      for (size_t xi = 0; xi < sp.der.size(); xi++) {
        const Rollup& ro = sp.der[xi];
        const int kx = der_k[y][xi];
        const int ngy = hq[ky].ngb;
        std::vector<int> xpos_of(ngy, -1);  // Y position -> X attribute index
        for (int i = 0; i < ro.ngb; i++) xpos_of[ro.pos[i]] = i;
        int p = -1;
        for (int t = 0; t < ngy; t++)
          if (xpos_of[t] < 0) p = t;
        MergeRollup m{};
        m.nudaf = ro.nudaf;
        m.nseg = 1;
        m.npre = 1;
        bool ok = !ro.prefix && p >= 0 && qs[kx].dense == qs[ky].dense && ro.nudaf == gy.nudaf;
        if (ok) {
          m.suffix = hq[ky].stride[p];
          m.np = p + 1;
          for (int t = 0; t <= p; t++) {
            m.role[t] = xpos_of[t] >= 0;
            m.radix[t] = gy.d.radix[t];
            m.ystr[t] = hq[ky].stride[t];
            m.xstr[t] = m.role[t] ? hq[kx].stride[xpos_of[t]] : 0;
            if (m.role[t]) m.npre *= gy.d.radix[t];
            else m.nseg = (int)std::min<long long>((long long)m.nseg * gy.d.radix[t], 1 << 30);
          }
          for (int t = p + 1; t < ngy; t++) {
            m.sradix[m.ns] = gy.d.radix[t];
            m.systr[m.ns] = hq[ky].stride[t];
            m.sxstr[m.ns] = hq[kx].stride[xpos_of[t]];
            m.ns++;
          }
          m.ntile_s = (m.suffix + MR_W - 1) / MR_W;
          const char* mm = std::getenv("LMFAO_CUBE_MERGE_MIN");  // tests: small suffix spaces too
          ok = m.nseg <= MR_SEG && m.suffix >= (mm ? std::atoll(mm) : 256) && merge_smem(m.nudaf) <= 160 * 1024;
        }
        if (!ok) {
          left.push_back(ro);
          left_coff.push_back(der_coff[y][xi]);
          left_k.push_back(kx);
          continue;
        }
        m.yvals = gy.rvals.as<double>();
        m.ycnt = gy.rcnts.as<unsigned long long>();
        m.xtab = ro.table;
        m.xcnt = ro.counts;
        sp.merges.push_back(m);
      }
      sp.der = left;
      der_coff[y] = left_coff;
      der_k[y] = left_k;
    }
  }
  // small dense tables (C5-like cubes over tiny domains; a root categorical's group-bys, whose
  // runs end at nearly every row): one copy per CTA in shared memory, flushed once at the end —
  // REDs from every SM on a handful of global addresses serialise in L2.  LMFAO_CUBE_SMALL=0: off.
  {
    const char* sm = std::getenv("LMFAO_CUBE_SMALL");
    const bool on = !(sm && sm[0] == '0');
    int used = 0;
    for (size_t k = 0; k < hq.size(); k++) {
      hq[k].smoff = -1;
      hq[k].sncell = 0;
      const GroupPlan& g = c->groups[qs[k].gi];
      const int64_t need = g.ncells * (hq[k].nudaf + 1);
      if (!on || hq[k].sparse || hq[k].derived || need > 1024 || used + need > 4096) continue;
      hq[k].smoff = used;
      hq[k].sncell = (int)g.ncells;
      used += (int)need;
    }
    a.nsmall = used;
  }
  // the scan's levels: those of the cuboids it still updates (derived ones are not), and the
  // dense keys it needs to find their runs
  a.dmask = 0;
  for (size_t k = 0; k < qs.size(); k++)
    if (!hq[k].derived) a.dmask |= 1u << qs[k].depth;
  a.nkey = (a.dmask >> a.R & 1u) ? a.R : std::min(a.R, 32 - __builtin_clz(a.dmask | 1u));
  // items: (cuboid, non-constant UDAF) pairs of the dense cuboids, by level, with their terms;
  // with more than CB_MEAS measures one scan per group of CB_MEAS, each with the terms of its
  // measures (the count term and the counts with the first)
  std::vector<std::vector<CubeItem>> pitems(nparts);
  std::vector<std::vector<int8_t>> ptj(nparts);
  std::vector<std::vector<double>> ptc(nparts);
  for (int pt = 0; pt < nparts; pt++) {
    CubeArgs ap = a;
    const int m0 = pt * CB_MEAS, m1 = std::min(M, m0 + CB_MEAS);
    ap.M = m1 - m0;
    for (int j = m0; j < m1; j++) {
      ap.meas[j - m0] = mptr[j];
      ap.meas_i32[j - m0] = mi32[j];
      ap.midx[j - m0] = midx[j];
    }
    ap.nocount = pt > 0;
    auto& items = pitems[pt];
    auto& tj = ptj[pt];
    auto& tc = ptc[pt];
    for (int d = 0; d <= CB_LEV; d++) {
      ap.ibeg[d] = (int)items.size();
      for (int k = a.qbeg[d]; k < a.qbeg[d + 1]; k++) {
        if (hq[k].sparse || hq[k].derived) continue;
        for (size_t u = 0; u < qs[k].terms.size(); u++) {
          const auto& t = qs[k].terms[u];
          if (t.empty()) continue;  // constant UDAF: from the count at compaction
          std::vector<std::pair<int, double>> lt;  // this part's terms, local S indices
          for (auto& jt : t) {
            if (jt.first == 0 && pt == 0) lt.push_back(jt);
            else if (jt.first >= 1 + m0 && jt.first < 1 + m1) lt.push_back({jt.first - m0, jt.second});
          }
          if (lt.empty()) continue;
          CubeItem e{(int16_t)(k - a.qbeg[d]), (int16_t)u, (int16_t)tj.size(), 0, lt[0].first, 0, lt[0].second};
          for (auto& jt : lt) {
            tj.push_back((int8_t)jt.first);
            tc.push_back(jt.second);
          }
          e.t1 = (int16_t)tj.size();
          items.push_back(e);
        }
      }
    }
    ap.ibeg[CB_LEV + 1] = (int)items.size();
    if ((int)tj.size() > CB_TERMS || (int)items.size() > CB_ITEMS) return nullptr;
    ap.nterm = (int)tj.size();
    ap.nitem = (int)items.size();
    fc->parts.push_back(ap);
  }
  a = fc->parts[0];
  fc->nq = a.nq;
  cudaStream_t st = c->stream;
  if (fc->dq.alloc(hq.size() * sizeof(Cuboid)) || fc->dcoef.alloc(std::max<size_t>(dense.size(), 1) * 8) ||
      fc->dwork.alloc(16 * 4))
    return nullptr;
  if (nparts > 16) return nullptr;
  if (cudaMemcpyAsync(fc->dq.p, hq.data(), hq.size() * sizeof(Cuboid), cudaMemcpyHostToDevice, st)) return nullptr;
  if (!dense.empty() && cudaMemcpyAsync(fc->dcoef.p, dense.data(), dense.size() * 8, cudaMemcpyHostToDevice, st))
    return nullptr;
  fc->pbuf.resize(3 * nparts);
  int max_item = 0, max_term = 0;
  for (int pt = 0; pt < nparts; pt++) {
    DevBuf& bi = fc->pbuf[3 * pt];
    DevBuf& bj = fc->pbuf[3 * pt + 1];
    DevBuf& bc = fc->pbuf[3 * pt + 2];
    const auto& items = pitems[pt];
    const auto& tj = ptj[pt];
    const auto& tc = ptc[pt];
    if (bi.alloc(std::max<size_t>(items.size(), 1) * sizeof(CubeItem)) || bj.alloc(std::max<size_t>(tj.size(), 1)) ||
        bc.alloc(std::max<size_t>(tc.size(), 1) * 8))
      return nullptr;
    if (!items.empty() && cudaMemcpyAsync(bi.p, items.data(), items.size() * sizeof(CubeItem), cudaMemcpyHostToDevice, st))
      return nullptr;
    if (!tj.empty() && (cudaMemcpyAsync(bj.p, tj.data(), tj.size(), cudaMemcpyHostToDevice, st) ||
                        cudaMemcpyAsync(bc.p, tc.data(), tc.size() * 8, cudaMemcpyHostToDevice, st)))
      return nullptr;
    CubeArgs& ap = fc->parts[pt];
    ap.q = fc->dq.as<Cuboid>();
    ap.items = bi.as<CubeItem>();
    ap.tj = bj.as<int8_t>();
    ap.tc = bc.as<double>();
    max_item = std::max(max_item, ap.nitem);
    max_term = std::max(max_term, ap.nterm);
  }
  for (size_t y = 0; y < fc->sparse.size(); y++) {
    SparseOut& sp = fc->sparse[y];
    for (size_t x = 0; x < sp.der.size(); x++) sp.der[x].coef = fc->dcoef.as<double>() + der_coff[y][x];
    {  // rollup cells from Y's codes; X's UDAFs identical to Y's; the reduce's shared memory
      int ky = -1;
      for (size_t k = 0; k < qs.size(); k++)
        if (sparse_of[k] == (int)y) ky = (int)k;
      const GroupPlan& gy = c->groups[qs[ky].gi];
      size_t sm = (size_t)gy.nudaf * M1 * 8;
      for (size_t x = 0; x < sp.der.size(); x++) {
        Rollup& ro = sp.der[x];
        const int kx = der_k[y][x];
        for (int t = 0; t < CB_GB; t++) ro.xstr_y[t] = 0;
        for (int i = 0; i < ro.ngb; i++) ro.xstr_y[ro.pos[i]] = ro.stride[i];
        ro.same = qs[kx].dense == qs[ky].dense;
        sm += sizeof(Rollup) + (size_t)ro.nudaf * M1 * 8;
      }
      sp.reduce_smem = sm <= 96 * 1024 ? sm : 0;
      if (sp.reduce_smem > 48 * 1024 && ensure_smem_attr((const void*)k_rec_reduce, sp.reduce_smem)) return nullptr;
    }
    if (sp.dder.alloc(std::max<size_t>(sp.der.size(), 1) * sizeof(Rollup))) return nullptr;
    if (!sp.der.empty() &&
        cudaMemcpyAsync(sp.dder.p, sp.der.data(), sp.der.size() * sizeof(Rollup), cudaMemcpyHostToDevice, st))
      return nullptr;
  }
  fc->ca = fc->parts[0];
  fc->smem = CubeSmem(a.nq, max_item, max_term, a.nsmall).total();
  if (fc->smem > 227 * 1024) return nullptr;
  if (fc->smem > 48 * 1024 &&
      cudaFuncSetAttribute(k_cube, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fc->smem))
    return nullptr;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cube, CB_WARPS * 32, fc->smem) || per_sm < 1) per_sm = 1;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
  fc->grid = nsm * per_sm;
  for (auto& sp : fc->sparse)
    for (auto& m : sp.merges)
      if (ensure_smem_attr((const void*)k_merge_rollup, merge_smem(m.nudaf)))
        return nullptr;
  if (!fc->sparse.empty()) {
    // the sparse cuboids' record slots: each work chunk's run ends at slevel, counted by the
    // scan itself in count mode (keys only), then an exclusive scan gives the chunks' bases
    // and the total the sort and reduce read
    if (fc->rbase.alloc((nchunks + 1) * 8) || fc->dwork.alloc(16 * 4)) return nullptr;
    CubeArgs ca = fc->parts[0];
    ca.count_only = 1;
    ca.tails = fc->rbase.as<long long>();
    ca.nrows = nrows;
    ca.work = fc->dwork.as<int>();
    if (cudaMemsetAsync(fc->dwork.p, 0, 4, st) || cudaMemsetAsync(fc->rbase.p, 0, (nchunks + 1) * 8, st)) return nullptr;
    if (nrows > 0) {
      const int64_t g = std::min<int64_t>((nchunks + CB_WARPS - 1) / CB_WARPS, fc->grid);
      k_cube<<<(unsigned)g, CB_WARPS * 32, fc->smem, st>>>(ca);
    }
    if (exclusive_scan_i64(fc->rbase.as<int64_t>(), fc->rbase.as<int64_t>(), nchunks + 1, st)) return nullptr;
    for (auto& sp : fc->sparse)
      if (cudaMemcpyAsync(sp.n.p, fc->rbase.as<long long>() + nchunks, 8, cudaMemcpyDeviceToDevice, st)) return nullptr;
    for (int k = a.qbeg[a.slevel]; k < a.qbeg[a.slevel + 1]; k++) hq[k].rbase = fc->rbase.as<long long>();
    if (cudaMemcpyAsync(fc->dq.p, hq.data(), hq.size() * sizeof(Cuboid), cudaMemcpyHostToDevice, st)) return nullptr;
    // only the sparse level left to scan, no dense cuboid updated by the scan: k_cube_rec
    CubeArgs& p0 = fc->parts[0];
    bool rec = fc->parts.size() == 1 && p0.dmask == (1u << p0.slevel) && p0.nitem == 0 && p0.nkey <= REC_LEV &&
               p0.nattr <= REC_ATTR &&
               !(std::getenv("LMFAO_CUBE_REC") && std::getenv("LMFAO_CUBE_REC")[0] == '0');
    for (int k = a.qbeg[a.slevel]; k < a.qbeg[a.slevel + 1] && rec; k++) rec = hq[k].sparse || hq[k].derived;
    int nr = 0;
    for (int k = a.qbeg[a.slevel]; k < a.qbeg[a.slevel + 1] && rec; k++) {
      if (!hq[k].sparse) continue;
      if (nr == 4) {
        rec = false;
        break;
      }
      CubeArgs::RecOut& o = p0.rec[nr++];
      o.rkey = hq[k].rkey;
      o.rval = hq[k].rval;
      // per level: the part of the cell its key determines (the codes of the level's
      // attributes × strides), tabulated over the level's dense keys
      for (int i = 0; i < hq[k].ngb && rec; i++) {
        const int sl = hq[k].aslot[i], l = p0.alvl[sl];
        if (l >= p0.R) {
          o.aslot[o.ngb] = (int8_t)sl;
          o.stride[o.ngb++] = hq[k].stride[i];
          continue;
        }
        const int64_t nk = c->rels[R.children[c->levels[l]]].nrows;
        DevBuf& pb = fc->parts_tab[(nr - 1) * CB_LEV + l];
        if (!pb.p) {
          if (pb.alloc(std::max<int64_t>(nk, 1) * 4) || cudaMemsetAsync(pb.p, 0, std::max<int64_t>(nk, 1) * 4, st)) return nullptr;
        }
        if (nk > 0)
          k_cell_part<<<cgrid(nk), 256, 0, st>>>(pb.as<unsigned>(), p0.acode[sl], hq[k].stride[i], nk);
        o.part[l] = pb.as<unsigned>();
      }
    }
    if (rec) {
      p0.nrec = nr;
      p0.meas_plain = 1;
      for (int j = 0; j < p0.M; j++) p0.meas_plain &= !p0.midx[j] && !p0.meas_i32[j];
      if (p0.slevel == p0.R) p0.meas_plain = 0;
      p0.rbase = fc->rbase.as<long long>();
      fc->rec_only = true;
      int per = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cube_rec<CB_MEAS + 1, false>, 256, 0) || per < 1) per = 1;
      fc->rec_grid = nsm * per;
    }
  }
  if (cudaStreamSynchronize(st)) return nullptr;
  for (auto& sp : fc->sparse) {  // no dense table for these
    GroupPlan& gp = c->groups[sp.gi];
    gp.direct = true;
    gp.table.reset();
    gp.counts.reset();
  }
  return fc.release();
}

}  // namespace lmfao
