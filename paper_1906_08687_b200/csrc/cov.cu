// cov.cu — the covariance batch's fused root scan, B200 version 3 (k_cov).
//
// Same mathematics as gram.cu (§3 "covariance matrix" P:397-402: every
// aggregate is an entry of G = Σ_f u(f) u(f)^T with u = [1, x, s_L, s_A, s_B]),
// evaluated over the root sorted by its foreign keys in increasing domain size
// with the multi-output trie registration of P:1020-1214:
//   per row          x⊗x, x⊗s_L                 (DMMA m8n8k4; x⊗s_L8/9 by DFMA in cold blocks)
//   per level-A run  R_A⊗s_A, R_A = Σ_run [x, s_L, 1]   ("intermediate aggregates": run sums
//                    carried per lane, one DMMA per tile per run) — or, in blocks where many
//                    short runs end (the Zipf tail), the same sum row by row (linearity)
//   per level-B run  R_B⊗s_B, R_B = Σ_{A-runs} [R_A, n·s_A]  (record list, finished off-scan)
//   dimension side   Σ_k H_r[k] s_r(k) s_r(k)^T  ("each aggregate to its own root")
// Design on B200 (measurements in DESIGN.md §2):
//  * the FP64 pipe (DMMA and DFMA share it: 18.5 T FMA/s) is the scarce unit next to issue:
//    x⊗x and x⊗s_L0..7 are one DMMA m8n8k4 each per 4 rows (the k = 4 sums the rows), the
//    thin x⊗[s_L8, s_L9] a third DMMA in fast blocks and two DFMA per lane and group in cold
//    blocks, where s_L8/9 are loaded anyway (COV_XT_DFMA); x⊗x as DFMA (lane (m, k) forming
//    x_m·x_{m+d}, COV_XX_DMMA=0) saves FP64 pipe cycles but measured slower (issue);
//  * run boundaries are structural (like the trie): the scan layout built at plan
//    time carries a run-start flag in bit 31 of every dense key, so a block's boundary masks
//    are one ballot per level;
//  * work is static: each warp scans a contiguous chunk of 32-row blocks, chunks of equal
//    estimated cost (plan time, from the flags), and writes its partial sums and its level-B
//    records to fixed slots — the result is bit-identical from run to run;
//  * each warp streams its chunk with `cp.async.bulk` (one 2432-byte block per copy into a
//    3-deep shared ring) and gathers the view rows s_L[k_L] (96-byte rows, L2-resident) one
//    block ahead with 16-byte `cp.async` (a TMA `tile::gather4` measured 0.60 vs 0.367 ms);
//  * H_L (root rows per L key, for s_L⊗s_L) is counted in a per-CTA open-addressing table in
//    shared memory (Zipf-hot keys would serialise global atomics), spilling to global REDs.
// Runs split at block / chunk boundaries are exact (every update is linear in the run sums).
#include <cuda.h>

#include <cstdlib>
#include <set>

#include <functional>
#include <type_traits>

#include "ctx.h"

namespace lmfao {
namespace {

constexpr int GP = 12;       // doubles per view row (cols >= n are 0; col 10 = 1.0)
#ifndef COV_HT_BITS  // per-CTA H_L slots: only the Zipf-hottest keys need them, the rest go to global
#define COV_HT_BITS 6   // REDs over many addresses (C2 scan: 2^12 0.355, 2^10 0.346, 2^8 0.343, 2^6 0.342,
#endif                  // 2^5 0.345 ms, round 1)
constexpr int HT = 1 << COV_HT_BITS;
constexpr int SBLK = 256 * 8 + 3 * 32 * 4;     // scan-layout bytes per 32-row block: x in DMMA order + 3 key rows
constexpr int STG_G = 32 * GP * 8;             // 3072 B of gathered view rows per block (2 slots)
constexpr int NPART = 384;   // per-warp partial: XX[8][8] | XL[8][10] | RA[24][10]
constexpr int BRW = 36;      // doubles per B record
constexpr int NFIN = 640 + 3 * 256;  // RBM[40][16] | ML[16][16] | MA[16][16] | MB[16][16]
#ifndef COV_FIN_BLOCKS
#define COV_FIN_BLOCKS 296
#endif
#ifndef COV_FIN_U
#define COV_FIN_U 4  // k_cov_fin: key groups (4 keys each) whose loads are in flight together per warp
#endif
#ifndef COV_SUM_SP  // k_cov_sum: the scan's per-item partial rows in SUM_SP chunks, the fin partials in
#define COV_SUM_SP 16  // SUM_SF chunks (one CTA per chunk and 32 elements; 12 x 16 + 44 x 2 = 280 CTAs, one
#endif                 // wave), the chunk sums added again by k_cov_assemble (was 8 and 8: 57 x 8 CTAs)
#ifndef COV_SUM_SF
#define COV_SUM_SF 2
#endif
constexpr int FIN_BLOCKS = COV_FIN_BLOCKS;
constexpr int SUM_SP = COV_SUM_SP, SUM_SF = COV_SUM_SF;
constexpr int SUM_CTAS = (NPART / 32) * SUM_SP + (NFIN / 32) * SUM_SF;
constexpr int SRC_N = SUM_SP * NPART + SUM_SF * NFIN;  // src: [SUM_SP][NPART] | [SUM_SF][NFIN]
static_assert(NPART % 32 == 0 && NFIN % 32 == 0, "k_cov_sum: whole 32-element columns");
constexpr unsigned FULL = 0xffffffffu;
constexpr int KEYMASK = 0x3fffffff;  // dense key; bit 31 = a run starts at this row (at this level),
constexpr int RUN_END = 0x40000000;  // bit 30 = the run (at this level) ends after this row
#ifndef COV_W
#define COV_W 12  // warps per CTA of the scan (one CTA per SM)
#endif
#ifndef COV_XT_DFMA  // x⊗[s_L8, s_L9] (with COV_XX_DMMA): 0 a third DMMA per group (B = [s_L8, s_L9, 1, 0..]),
#define COV_XT_DFMA 2   // 1 two DFMA per lane and group, 2 DFMA in cold blocks (which load s_L8/9 anyway) and
#endif                  // the DMMA elsewhere (C2 scan: 0 0.3072, 1 0.3044, 2 0.3032 ms)
#ifndef COV_XX_DMMA  // 1: x⊗x and x⊗[s_L8, s_L9, 1] as two more DMMA per 4-row group; 0: 7 DFMA (x_m·x_{m+d})
#define COV_XX_DMMA 1   // (C2 scan: DFMA 0.334, DMMA 0.296 ms with the same static split: issue-bound)
#endif
// Work split (plan time): one static chunk per warp over the first (100 - COV_TAIL) % of the
// estimated cost, chunks of equal cost (a block with level-A run starts inside costs COV_COST_COLD,
// others COST_FAST), then COV_TB-block items grabbed dynamically — the dynamic tail absorbs what
// the cost model gets wrong, per-item partials keep the sums in a fixed order.
constexpr int COST_FAST = 3;
#ifndef COV_COST_COLD
#define COV_COST_COLD 6  // (C2, static chunks only: 3 0.395, 4 0.358, 5 0.334, 6 0.296, 7 0.391 ms)
#endif
#ifndef COV_TB
#define COV_TB 8
#endif
#ifndef COV_TAIL
#define COV_TAIL 10
#endif

static_assert(SBLK % 128 == 0 && STG_G % 128 == 0, "TMA / cp.async alignment");

struct CovArgs {
  int64_t nblk;
  const unsigned char* scan;  // [nblk][SBLK] scan layout of the root
  const double* VL;           // [nkL + 1 x GP]
  const double* VA;           // [nkA + 1 x GP] (a zero row if absent)
  unsigned* HL;
  unsigned* HA;
  double* brec;               // level-B records, [rec_base[NW]][BRW]
  const int* item;            // [nitems + 1] first block of each work item (plan time)
  int nitems;
  int nstatic;                // items [0, nstatic): warp gw's first item is item gw (cost-balanced
                              // static chunks); the rest are grabbed dynamically
  int* work;                  // item counter (dynamic schedule), cleared every run
  const int* rec_base;        // [nitems + 1] first level-B record slot of each item
  double* partials;           // [nitems][NPART] per-item partials (summed in item order: deterministic)
  int ablate;  // diagnostics only (LMFAO_COV_ABLATE, results invalid): 1 no gathers, 8 no H_L,
               // 16 no compute at all (pipeline only), 32 every block on the fast path
  int cold_all;  // LMFAO_COV_COLD_ALL=1 (tests): every block on the per-row level-A path (exact)
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n W_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W_%=;\n}" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b))
               : "memory");
}
__device__ __forceinline__ void cp16full(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double red4(double v) {
  v += __shfl_xor_sync(FULL, v, 1);
  v += __shfl_xor_sync(FULL, v, 2);
  return v;
}
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
// Programmatic dependent launch (the run's kernel chain dims -> scan -> fin -> sum -> assemble):
// a kernel launched with the PDL attribute may start while its predecessor drains; it runs only
// work on plan-time data before pdl_wait(), which returns once the predecessor grid has completed
// and its writes are visible.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Scan layout of the root (built once at plan time, like the sort at prepare): per
// 32-row block b, x in the DMMA lane order [group j][lane 4m+k] = x_m[32b+4j+k] (0 for
// m >= nx or rows >= N), then the dense keys [level][32] of L, A, B.  Bit 31 of a key is
// the run-start flag of its level in the sorted root: a B run starts where the B key
// changes, an A run where the A or B key changes, an L run where any of them changes
// (so A runs nest in B runs and L runs in A runs), and every level starts at row 0 and at
// row N (the padding rows past N carry the key of a zero row appended to each view).  One
// contiguous bulk copy per block; conflict-free shared reads.
struct LayoutArgs {
  const double* x[8];
  const int32_t* key[3];
  int pad[3];  // key of rows >= N per level: the zero row appended to the level's view (0: no level)
  int nx, nlev;
  int64_t N, nblk;
  unsigned char* out;
};
__global__ void k_cov_layout(LayoutArgs a) {
  const int64_t tot = a.nblk * (SBLK / 8);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / (SBLK / 8);
    const int o = (int)(i % (SBLK / 8));
    if (o < 256) {
      const int j = o >> 5, l = o & 31, m = l >> 2, kk = l & 3;
      const int64_t row = 32 * b + 4 * j + kk;
      reinterpret_cast<double*>(a.out)[i] = (m < a.nx && row < a.N) ? a.x[m][row] : 0.0;
    } else {
      const int e = 2 * (o - 256), lv = e >> 5, r = e & 31;
      int v[2] = {0, 0};
      if (lv < a.nlev) {
        auto starts = [&](int64_t row) {  // a run starts at `row` at level lv
          if (row == 0 || row >= a.N) return true;
          for (int l = lv; l < a.nlev; l++)
            if (a.key[l][row] != a.key[l][row - 1]) return true;
          return false;
        };
#pragma unroll
        for (int h = 0; h < 2; h++) {
          const int64_t row = 32 * b + r + h;
          if (row < a.N) {
            v[h] = a.key[lv][row] | (starts(row) ? (int)0x80000000u : 0) | (starts(row + 1) ? RUN_END : 0);
          } else {
            v[h] = a.pad[lv] | (row == a.N ? (int)0x80000000u : 0) | (row == 32 * a.nblk - 1 ? RUN_END : 0);
          }
        }
      }
      reinterpret_cast<int2*>(a.out)[i] = make_int2(v[0], v[1]);
    }
  }
}

// Plan time, per block (one warp per block): bits 0..5 the number of level-B run starts in it, bit
// 6 its row 0 starts a B run, bit 7 level-A runs start inside it (the per-row path).
__global__ void k_cov_bstats(const unsigned char* __restrict__ scan, int64_t nblk, int NS, uint32_t* __restrict__ st) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w0; b < nblk; b += nw) {
    const int* ks = reinterpret_cast<const int*>(scan + b * SBLK + 2048);
    const unsigned mA = NS >= 1 ? __ballot_sync(FULL, ks[32 + lane] < 0) : 0u;
    const unsigned mB = NS == 2 ? __ballot_sync(FULL, ks[64 + lane] < 0) : 0u;
    if (lane == 0) st[b] = (uint32_t)__popc(mB) | ((mB & 1u) << 6) | ((mA & ~1u) ? 128u : 0u);
  }
}

// Plan time, the work split on the device (no per-block data to the host): a block's cost
// (COST_FAST, or `cold` when level-A runs start inside it); the static chunk boundaries, chunk w
// ending at the first block whose cost prefix reaches stat·w/NW; the level-B records of each work
// item (its blocks' B run starts, plus one if its row 0 does not start a B run).
__global__ void k_cov_cost(const uint32_t* __restrict__ st, int64_t n, uint32_t cold, uint32_t* __restrict__ cost) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= n; b += (int64_t)gridDim.x * blockDim.x)
    cost[b] = b < n ? ((st[b] & 128u) ? cold : (uint32_t)COST_FAST) : 0u;
}
__global__ void k_cov_static(const uint32_t* __restrict__ cc, int64_t n, int NW, int tail, int32_t* __restrict__ it) {
  const uint64_t stat = (uint64_t)cc[n] * (uint64_t)(100 - tail) / 100;  // cost of the static part
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= NW; w += gridDim.x * blockDim.x) {
    const uint64_t target = stat * (uint64_t)w / (uint64_t)NW;
    int64_t lo = 0, hi = n + 1;  // first b with cc[b] >= target
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((uint64_t)cc[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    it[w] = w == 0 ? 0 : (int32_t)lo;
  }
}
__global__ void k_cov_recs(const uint32_t* __restrict__ st, const int32_t* __restrict__ it, int nitems,
                           uint32_t* __restrict__ rc) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nitems; i += gridDim.x * blockDim.x) {
    uint32_t r = 0;
    if (i < nitems) {
      for (int64_t b = it[i]; b < it[i + 1]; b++) r += st[b] & 63u;
      if (it[i + 1] > it[i] && !(st[it[i]] & 64u)) r += 1;
    }
    rc[i] = r;
  }
}

template <int W>
struct CovCfg {
  static constexpr int CF = 3;                           // fact-block ring slots per warp
  static constexpr int WB = CF * SBLK + 2 * STG_G + 128;  // + barriers
  static constexpr int SMEM = 128 + HT * 8 + W * WB;      // [CTA counters | H_L table | warps]
  static_assert(SMEM <= 232448, "shared memory budget");
};

// NS = number of featured levels above L (0: L only, 1: A and L, 2: B, A and L); W warps per CTA.
// The per-warp state and per-block work of the scan: lane (m, k)
// = (lane / 4, lane % 4) holds, for DMMA group j (rows 4j..4j+3), feature m of row 4j + k.
// Paths by the block's level-A / level-B run starts (flags of the scan layout):
//  * fast (no A run starts inside): per-row products; v = [x, s_L0..7, (s_L8, s_L9, 1)] is
//    summed per lane into the open A run's carry C; when the run ends (at a block end) the
//    carry times the run's s_A row is one DMMA per tile (the DMMA's k = 4 sums the lanes'
//    rows) plus DFMA for s_A8/9;
//  * cold (A run starts inside, no B start): every row's v times its own s_A row (the same
//    sum by linearity: Σ_run (Σ_rows v) ⊗ s_A = Σ_rows v ⊗ s_A(row)), no segments;
//  * slow (B run starts inside; rare): the cold product once per B segment, masked to its rows.
template <int NS>
struct CovWarp {
  const CovArgs& g;
  const int lane, k, m, tcol;
  int* hkey;
  unsigned* hcnt;
  int rec = 0;           // the current item's next level-B record slot
  bool carried = false;  // C holds rows of the open level-A run
  // accumulators
  double aXL[2] = {0, 0};                              // x ⊗ s_L0..7 (DMMA)
  double aXX[2] = {0, 0}, aXT[2] = {0, 0};             // COV_XX_DMMA: x ⊗ x, x ⊗ [s_L8, s_L9, 1] (DMMA)
  double xx0 = 0, xx1 = 0, xx2 = 0, xx3 = 0, xx4 = 0;  // x_m · x_{(m+d)%8}, d = 0..4 (COV_XX_DMMA=0)
  double x8 = 0, x9 = 0;                               // x_m · s_L8, x_m · s_L9 (COV_XX_DMMA=0)
  double C0 = 0, C1 = 0, C2 = 0;                       // open A run: Σ x_m, Σ s_L_m, Σ t_m (this lane's rows)
  double aRA0[2] = {0, 0}, aRA1[2] = {0, 0}, aRA2[2] = {0, 0};  // [x | s_L0..7 | t] ⊗ s_A0..7 (DMMA)
  double r8x = 0, r9x = 0, r8l = 0, r9l = 0, r8t = 0, r9t = 0;   // ... ⊗ s_A8, s_A9
  double tA8 = 0, tA9 = 0;                                       // s_L8 · s_A_m, s_L9 · s_A_m (per row)
  double SB0 = 0, SB1 = 0, SB2 = 0, SBn = 0, SBn8 = 0, SBn9 = 0;  // open B run: Σ v, Σ s_A

  __device__ __forceinline__ CovWarp(const CovArgs& g_, int lane_, int* hk, unsigned* hc)
      : g(g_), lane(lane_), k(lane_ & 3), m(lane_ >> 2), tcol((lane_ >> 2) < 3 ? 8 + (lane_ >> 2) : 11), hkey(hk),
        hcnt(hc) {}

  __device__ __forceinline__ void hl_add(int key, unsigned len) {  // two probes, straight-line; full: global RED
    unsigned h = ((unsigned)key * 2654435761u) >> (32 - COV_HT_BITS);
    int t = hkey[h];
    if (t == -1) {
      const int old = atomicCAS(&hkey[h], -1, key);
      t = old == -1 ? key : old;
    }
    if (t != key) {
      h = (h + 1) & (HT - 1);
      t = hkey[h];
      if (t == -1) {
        const int old = atomicCAS(&hkey[h], -1, key);
        t = old == -1 ? key : old;
      }
    }
    if (t == key) atomicAdd(&hcnt[h], len);
    else gred_add(&g.HL[key], len);
  }
  __device__ __forceinline__ void push_B(int keyB) {  // the open B run's record -> the item's next slot
    const double v0 = red4(SB0), v1 = red4(SB1), v2 = red4(SB2), v3 = red4(SBn), v4 = red4(SBn8), v5 = red4(SBn9);
    double* r = g.brec + (size_t)rec * BRW;
    if (k == 0) {
      r[m] = v0;
      r[8 + m] = v1;
      r[16 + m] = v2;
      r[24 + m] = v3;
    }
    if (lane == 0) {
      r[32] = v4;
      r[33] = v5;
      r[34] = (double)keyB;
      r[35] = 0.0;
    }
    rec++;
    SB0 = SB1 = SB2 = SBn = SBn8 = SBn9 = 0.0;
  }
  // the carried rows of the A run with key keyA: C ⊗ s_A(keyA), into the B sums, H_A
  __device__ __forceinline__ void flush_carry(int keyA) {
    const double* ar = g.VA + (size_t)(unsigned)keyA * GP;
    const double b0v = ar[m];
    const double2 b89 = ld2(ar + 8);
    dmma(aRA0, C0, b0v);
    dmma(aRA1, C1, b0v);
    dmma(aRA2, C2, b0v);
    r8x = fma(C0, b89.x, r8x);
    r9x = fma(C0, b89.y, r9x);
    r8l = fma(C1, b89.x, r8l);
    r9l = fma(C1, b89.y, r9l);
    r8t = fma(C2, b89.x, r8t);
    r9t = fma(C2, b89.y, r9t);
    SB0 += C0;
    SB1 += C1;
    SB2 += C2;
    const double n = __shfl_sync(FULL, red4(C2), 8);  // the carried rows: the "1" row (m == 2) of t
    const double nq = k == 0 ? n : 0.0;               // once per quad (SBn* are summed over k at push_B)
    SBn = fma(nq, b0v, SBn);
    SBn8 = fma(nq, b89.x, SBn8);
    SBn9 = fma(nq, b89.y, SBn9);
    if (NS >= 1 && lane == 0 && n > 0.0) gred_add(&g.HA[keyA], (unsigned)n);
    C0 = C1 = C2 = 0.0;
  }
  // the item's partial (every entry written; both triangles of XX); then the accumulators restart
  __device__ __forceinline__ void store_partial(int item) {
    const double q0 = red4(xx0), q1 = red4(xx1), q2 = red4(xx2), q3 = red4(xx3), q4 = red4(xx4);
    const double q8 = red4(x8), q9 = red4(x9);
    const double s8x = red4(r8x), s9x = red4(r9x), s8l = red4(r8l), s9l = red4(r9l), s8t = red4(r8t), s9t = red4(r9t);
    const double a8 = red4(tA8), a9 = red4(tA9);
    double* out = g.partials + (size_t)item * NPART;
    if (k == 0) {
      const double qd[5] = {q0, q1, q2, q3, q4};
#pragma unroll
      for (int d = 0; d < 5; d++) {
        const int n = (m + d) & 7;
        if (d < 4 || m < 4) {
          out[m * 8 + n] = qd[d];
          out[n * 8 + m] = qd[d];
        }
      }
      out[64 + m * 10 + 8] = q8;
      out[64 + m * 10 + 9] = q9;
      out[144 + m * 10 + 8] = s8x;
      out[144 + m * 10 + 9] = s9x;
      out[144 + (8 + m) * 10 + 8] = s8l;
      out[144 + (8 + m) * 10 + 9] = s9l;
      out[144 + (16 + m) * 10 + 8] = s8t;
      out[144 + (16 + m) * 10 + 9] = s9t;
    }
    out[64 + m * 10 + 2 * k] = aXL[0];
    out[64 + m * 10 + 2 * k + 1] = aXL[1];
    if (COV_XX_DMMA) {
      __syncwarp();
      out[m * 8 + 2 * k] = aXX[0];
      out[m * 8 + 2 * k + 1] = aXX[1];
      if (k == 0 && COV_XT_DFMA == 0) {
        out[64 + m * 10 + 8] = aXT[0];
        out[64 + m * 10 + 9] = aXT[1];
      }
      if (k == 0 && COV_XT_DFMA == 2) {  // the DMMA part (fast and slow blocks) + the DFMA part (cold)
        out[64 + m * 10 + 8] = aXT[0] + q8;
        out[64 + m * 10 + 9] = aXT[1] + q9;
      }
    }
    // t rows 0, 1 (s_L8, s_L9) of RA: the carried DMMA part plus the per-row DFMA part (on lane m
    // for column m: moved to the fragment's owner, lane (row, column / 2))
    const double a8c0 = __shfl_sync(FULL, a8, 8 * k), a8c1 = __shfl_sync(FULL, a8, 8 * k + 4);
    const double a9c0 = __shfl_sync(FULL, a9, 8 * k), a9c1 = __shfl_sync(FULL, a9, 8 * k + 4);
    const double e0 = m == 0 ? a8c0 : (m == 1 ? a9c0 : 0.0), e1 = m == 0 ? a8c1 : (m == 1 ? a9c1 : 0.0);
    out[144 + m * 10 + 2 * k] = aRA0[0];
    out[144 + m * 10 + 2 * k + 1] = aRA0[1];
    out[144 + (8 + m) * 10 + 2 * k] = aRA1[0];
    out[144 + (8 + m) * 10 + 2 * k + 1] = aRA1[1];
    out[144 + (16 + m) * 10 + 2 * k] = aRA2[0] + e0;
    out[144 + (16 + m) * 10 + 2 * k + 1] = aRA2[1] + e1;
    aXL[0] = aXL[1] = aXX[0] = aXX[1] = aXT[0] = aXT[1] = 0.0;
    xx0 = xx1 = xx2 = xx3 = xx4 = x8 = x9 = 0.0;
    aRA0[0] = aRA0[1] = aRA1[0] = aRA1[1] = aRA2[0] = aRA2[1] = 0.0;
    r8x = r9x = r8l = r9l = r8t = r9t = tA8 = tA9 = 0.0;
    __syncwarp();
  }

  // One 32-row block: st = its scan-layout block, gs = its gathered view rows [32][GP].  An item's
  // first row starts runs at every level, its last row ends them.
  __device__ __forceinline__ void block(const unsigned char* st, const double* gs, bool first_of_item,
                                        bool last_of_item) {
    const double* xs = reinterpret_cast<const double*>(st);
    const int* ks = reinterpret_cast<const int*>(st + 2048);
    const int klr = ks[lane];
    const int kar = NS >= 1 ? ks[32 + lane] : 0;
    const int kbr = NS == 2 ? ks[64 + lane] : 0;
    const int kl = klr & KEYMASK, ka = kar & KEYMASK, kb = kbr & KEYMASK;
    const unsigned first = first_of_item ? 1u : 0u;
    const unsigned mL = __ballot_sync(FULL, klr < 0) | first;
    const unsigned mA = (NS >= 1 ? __ballot_sync(FULL, kar < 0) : 0u) | first;
    const unsigned mB = (NS == 2 ? __ballot_sync(FULL, kbr < 0) : 0u) | first;
    // does the run open at this block's end end here? (the row-31 end flags, or the item's end)
    const int ends = __shfl_sync(FULL, (kar & RUN_END ? 1 : 0) | (kbr & RUN_END ? 2 : 0), 31);
    const bool endA = last_of_item || (NS >= 1 && (ends & 1));
    const bool endB = last_of_item || (NS == 2 && (ends & 2));
    if (!(g.ablate & 8) && (((mL >> lane) & 1u) || lane == 0)) {  // H_L: each L run's rows in the block
      const unsigned above = mL & ~((2u << lane) - 1u);
      hl_add(kl, (unsigned)((above ? __ffs(above) - 1 : 32) - lane));
    }
    const double* gl = gs + k * GP;
    // per-row products of group j; returns the lane's operands for the run-level work
    auto rowpart = [&](int j, double& xa, double& sv, double2& s89, double& tv, bool cold) {
      xa = xs[32 * j + lane];
      const double* gr = gl + j * 4 * GP;
      sv = gr[m];
      tv = gr[tcol];
      if (COV_XX_DMMA) {
        dmma(aXX, xa, xa);
        dmma(aXL, xa, sv);
        if (COV_XT_DFMA == 1 || (COV_XT_DFMA == 2 && cold)) {  // (2: DFMA where the cold path loads s89 anyway)
          s89 = ld2(gr + 8);
          x8 = fma(xa, s89.x, x8);
          x9 = fma(xa, s89.y, x9);
        } else {
          dmma(aXT, xa, tv);
          s89 = make_double2(0.0, 0.0);
        }
        return;
      }
      s89 = ld2(gr + 8);
      const double xd1 = xs[32 * j + ((lane + 4) & 31)];
      const double xd2 = xs[32 * j + ((lane + 8) & 31)];
      const double xd3 = xs[32 * j + ((lane + 12) & 31)];
      const double xd4 = xs[32 * j + ((lane + 16) & 31)];
      dmma(aXL, xa, sv);
      xx0 = fma(xa, xa, xx0);
      xx1 = fma(xa, xd1, xx1);
      xx2 = fma(xa, xd2, xx2);
      xx3 = fma(xa, xd3, xx3);
      xx4 = fma(xa, xd4, xx4);
      x8 = fma(xa, s89.x, x8);
      x9 = fma(xa, s89.y, x9);
    };
    // row-level A products of group j (rows masked to [lo, hi) when MASK)
    auto cold_group = [&](auto mask_tag, int j, double xa, double sv, double2 s89, double tv, double sam,
                          double2 sa89, int lo, int hi) {
      constexpr bool MASK = decltype(mask_tag)::value;
      if (MASK) {
        const int r = 4 * j + k;
        const double mk = (r >= lo && r < hi) ? 1.0 : 0.0;
        xa *= mk;
        sv *= mk;
        tv *= mk;
        s89.x *= mk;
        s89.y *= mk;
        sa89.x *= mk;
        sa89.y *= mk;
        sam *= mk;
      }
      if (COV_XX_DMMA && COV_XT_DFMA == 0 && !MASK) s89 = ld2(gl + j * 4 * GP + 8);
      dmma(aRA0, xa, sam);
      dmma(aRA1, sv, sam);
      tA8 = fma(s89.x, sam, tA8);
      tA9 = fma(s89.y, sam, tA9);
      r8x = fma(xa, sa89.x, r8x);
      r9x = fma(xa, sa89.y, r9x);
      r8l = fma(sv, sa89.x, r8l);
      r9l = fma(sv, sa89.y, r9l);
      r8t = fma(tv, sa89.x, r8t);
      r9t = fma(tv, sa89.y, r9t);
      SB0 += xa;
      SB1 += sv;
      SB2 += tv;
      SBn += sam;
      SBn8 += sa89.x;
      SBn9 += sa89.y;
    };
    // s_A rows of this lane's rows in groups 4h .. 4h+3 (loads in flight together)
    auto load_sa = [&](int h, double (&sam)[4], double2 (&sa89)[4]) {
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const unsigned key = (unsigned)__shfl_sync(FULL, ka, 4 * (4 * h + jj) + k);
        const double* ar = g.VA + (size_t)key * GP;
        sam[jj] = ar[m];
        sa89[jj] = ld2(ar + 8);
      }
    };
    // H_A: each A run's rows in this block (the carried rows were added by flush_carry)
    auto ha_runs = [&]() {
      if (((mA >> lane) & 1u) || lane == 0) {
        const unsigned above = mA & ~((2u << lane) - 1u);
        gred_add(&g.HA[ka], (unsigned)((above ? __ffs(above) - 1 : 32) - lane));
      }
    };
    const unsigned mBi = NS == 2 ? (mB & ~1u) : 0u;
    if (NS >= 1 && mBi) {
      // slow: level-B runs start inside the block
      if (carried) flush_carry(__shfl_sync(FULL, ka, 0));
      carried = false;
      ha_runs();
#pragma unroll
      for (int j = 0; j < 8; j++) {
        double xa, sv, tv;
        double2 s89;
        rowpart(j, xa, sv, s89, tv, false);
      }
      unsigned bits = mBi;
      int lo = 0;
      while (true) {
        const int hi = bits ? __ffs(bits) - 1 : 32;
#pragma unroll 1
        for (int h = 0; h < 2; h++) {
          double sam[4];
          double2 sa89[4];
          load_sa(h, sam, sa89);
#pragma unroll
          for (int jj = 0; jj < 4; jj++) {
            const int j = 4 * h + jj;
            const double* gr = gl + j * 4 * GP;
            cold_group(std::true_type{}, j, xs[32 * j + lane], gr[m], ld2(gr + 8), gr[tcol], sam[jj], sa89[jj], lo, hi);
          }
        }
        if (hi == 32) break;
        push_B(__shfl_sync(FULL, kb, hi - 1));
        lo = hi;
        bits &= bits - 1;
      }
    } else if (NS >= 1 && ((mA & ~1u) || g.cold_all) && !(g.ablate & 32)) {
      // cold: level-A runs start inside the block; every row times its own s_A row
      if (carried) flush_carry(__shfl_sync(FULL, ka, 0));
      carried = false;
      ha_runs();
#pragma unroll
      for (int h = 0; h < 2; h++) {
        double sam[4];
        double2 sa89[4];
        load_sa(h, sam, sa89);
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          double xa, sv, tv;
          double2 s89;
          rowpart(4 * h + jj, xa, sv, s89, tv, true);
          cold_group(std::false_type{}, 4 * h + jj, xa, sv, s89, tv, sam[jj], sa89[jj], 0, 32);
        }
      }
    } else {
      // fast: the open A run goes on through the block
#pragma unroll
      for (int j = 0; j < 8; j++) {
        double xa, sv, tv;
        double2 s89;
        rowpart(j, xa, sv, s89, tv, false);
        C0 += xa;
        C1 += sv;
        C2 += tv;
      }
      carried = !endA;
      if (endA) flush_carry(__shfl_sync(FULL, ka, 31));
    }
    if (endB) push_B(__shfl_sync(FULL, kb, 31));
  }
};

// view rows s_L[k_L(row)] of a landed fact block -> a gather slot [32 rows x 96 B]; 16-byte chunk
// c = 32 i + lane (row c / 6), so each instruction covers ~5 whole rows (coalesced)
__device__ __forceinline__ void gather_rows(const CovArgs& g, const unsigned char* fact, uint32_t dst_slot, int lane) {
  const int kl = reinterpret_cast<const int*>(fact + 2048)[lane] & KEYMASK;
  const char* vl = reinterpret_cast<const char*>(g.VL);
  const uint32_t dst = dst_slot + 16 * lane;
#pragma unroll
  for (int i = 0; i < 6; i++) {
    const int c = 32 * i + lane;
    const unsigned key = (unsigned)__shfl_sync(FULL, kl, c / 6);
    cp16full(dst + 512 * i, vl + key * (unsigned)(GP * 8) + (unsigned)((c % 6) * 16));
  }
}

// The scan, every warp its own pipeline: the CF-deep fact ring (bulk copies), the view-row
// gathers one block ahead (cp.async), and the work schedule — item gw (a static chunk), then
// items grabbed dynamically — all in the computing warp.
template <int NS, int W>
__global__ void __launch_bounds__(W * 32, 1) k_cov(const __grid_constant__ CovArgs g) {
  using Cfg = CovCfg<W>;
  constexpr int CF = Cfg::CF;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int gw = blockIdx.x * W + wib;
  extern __shared__ __align__(1024) unsigned char sm[];
  int* cta_done = reinterpret_cast<int*>(sm);
  int* hkey = reinterpret_cast<int*>(sm + 128);
  unsigned* hcnt = reinterpret_cast<unsigned*>(sm + 128 + HT * 4);
  unsigned char* wbase = sm + 128 + HT * 8 + wib * Cfg::WB;
  unsigned char* gbase = wbase + CF * SBLK;  // 2 gather slots
  uint64_t* bar_f = reinterpret_cast<uint64_t*>(gbase + 2 * STG_G);
  int* ring = reinterpret_cast<int*>(bar_f + 4);  // [8] item ids grabbed by this warp, in order

  for (int i = threadIdx.x; i < HT; i += blockDim.x) {
    hkey[i] = -1;
    hcnt[i] = 0;
  }
  if (threadIdx.x == 0) *cta_done = 0;
  if (lane == 0) {
    for (int s = 0; s < CF; s++) mbar_init(&bar_f[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  CovWarp<NS> w(g, lane, hkey, hcnt);

  // ---- schedule: item gw (a static chunk), then items grabbed dynamically; this warp's items in
  // grab order in a ring.  Every item has at least CF blocks (plan), so the fact look-ahead (CF
  // blocks) is never more than one item ahead of the block being processed.
  const int nitems = g.nitems;
  int nring = 0;
  auto grab = [&]() {  // the static chunk first; dynamic items when needed (no grab ahead: a
                       // prefetched tail item would wait behind the warp's current one)
    int it = 0;
    if (lane == 0) it = nring == 0 && gw < g.nstatic ? gw : g.nstatic + atomicAdd(g.work, 1);
    it = __shfl_sync(FULL, it, 0);
    if (lane == 0) ring[nring & 7] = it;
    nring++;
    __syncwarp();
  };
  auto issue_fact = [&](int64_t b, int stage) {
    if (lane == 0) {  // the slot was only read (generic proxy) since its last fill: no proxy fence needed
      mbar_expect(&bar_f[stage], SBLK);
      bulk_load(wbase + stage * SBLK, g.scan + b * SBLK, SBLK, &bar_f[stage]);
    }
  };
  auto issue_gather = [&](int stage, int gslot) {
    if (!(g.ablate & 1)) gather_rows(g, wbase + stage * SBLK, sa(gbase + gslot * STG_G), lane);
  };

  // ---- pipeline prologue: the first CF blocks of the sequence in flight, gathers of block 0.
  // A warp without a static chunk takes its first item from the work counter, which k_cov_dims
  // clears: it waits for that grid first; the others issue their first fact loads before.
  const bool dyn_first = gw >= g.nstatic;
  if (dyn_first) pdl_wait();
  grab();
  int pslot = 0, pitem = ring[0];  // the block being processed: pb of item pitem = [pbeg, pend)
  int pb = 0, pbeg = 0, pend = 0;
  if (pitem < nitems) {
    pb = pbeg = g.item[pitem];
    pend = g.item[pitem + 1];
    w.rec = g.rec_base[pitem];
  }
  int fslot = 0, fitem = pitem, fb = pb, fend = pend;  // the next block to load (look-ahead)
  auto f_advance = [&]() {
    if (fitem >= nitems) return;
    if (++fb < fend) return;
    if (++fslot >= nring) grab();
    fitem = ring[fslot & 7];
    if (fitem < nitems) {
      fb = g.item[fitem];
      fend = g.item[fitem + 1];
    }
  };
  for (int s = 0; s < CF; s++) {
    if (fitem < nitems) issue_fact(fb, s);
    f_advance();
  }
  if (!dyn_first) pdl_wait();  // the view rows (k_cov_dims) and the cleared H / work buffers
  if (pitem < nitems) {
    mbar_wait(&bar_f[0], 0);
    issue_gather(0, 0);
  }
  cp_commit();
  int fs = 0;  // position in the sequence % CF
  uint32_t fph = 0;
  for (int i = 0; pitem < nitems; i++) {
    const bool next_in_item = pb + 1 < pend;
    const int nitem = next_in_item ? pitem : ring[(pslot + 1) & 7];  // (grabbed by the look-ahead)
    const bool has_next = nitem < nitems;
    const int fs1 = fs + 1 == CF ? 0 : fs + 1;
    const uint32_t fph1 = fs + 1 == CF ? fph ^ 1u : fph;
    if (has_next) {  // gathers of the next block (its keys land first)
      mbar_wait(&bar_f[fs1], fph1);
      issue_gather(fs1, (i + 1) & 1);
    }
    cp_commit();
    cp_wait1();  // this block's gathers have landed
    __syncwarp();
    if (!(g.ablate & 16))
      w.block(wbase + fs * SBLK, reinterpret_cast<const double*>(gbase + (i & 1) * STG_G), pb == pbeg, !next_in_item);
    __syncwarp();
    if (fitem < nitems) issue_fact(fb, fs);  // the slot just consumed takes the block CF ahead
    f_advance();
    if (next_in_item) {
      pb++;
    } else {  // the item is done: its partial -> partials[item], accumulators cleared
      w.store_partial(pitem);
      pslot++;
      pitem = nitem;
      if (has_next) {
        pb = pbeg = g.item[pitem];
        pend = g.item[pitem + 1];
        w.rec = g.rec_base[pitem];
      }
    }
    fs = fs1;
    fph = fph1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  pdl_trigger();

  // ---- the CTA's last warp to finish moves the H_L table to global
  __threadfence_block();
  int ticket = 0;
  if (lane == 0) ticket = atomicAdd(cta_done, 1);
  ticket = __shfl_sync(FULL, ticket, 0);
  if (ticket == W - 1) {
    __threadfence_block();
    for (int i = lane; i < HT; i += 32) {
      const int key = hkey[i];
      if (key != -1 && hcnt[i]) gred_add(&g.HL[key], hcnt[i]);
    }
  }
}



// V[k][f] = col_f[k] for f < n, 0 for n <= f < GP, except V[k][10] = 1 (the constant of the
// scan's t tile; primary-key leaf: row k has dense key k).
struct DimTables {
  const double* cols[3][GP];   // by value in the parameter space: no dependent pointer loads
  const int32_t* idx[3][GP];   // per feature: row of its relation per dimension key (null: the key's own row)
  int n[3];
  int64_t nk[3];
  double* V[3];
  unsigned* z;  // the run's cleared words (work counter, H_A, H_L): zeroed here instead of a memset node
  int64_t nz;
};
__global__ void k_cov_dims(const __grid_constant__ DimTables d) {
  pdl_trigger();  // k_cov's prologue (fact loads) may start on SMs this grid frees
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.nz; i += (int64_t)gridDim.x * blockDim.x)
    d.z[i] = 0u;
  const int64_t n0 = d.nk[0], n1 = d.nk[1], n2 = d.nk[2];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n0 + n1 + n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int l = i < n0 ? 0 : (i < n0 + n1 ? 1 : 2);
    const int64_t kk = i - (l == 0 ? 0 : (l == 1 ? n0 : n0 + n1));
    const int n = d.n[l];
    double v[GP];
#pragma unroll
    for (int f = 0; f < GP; f++) {
      if (f < n) {
        const int32_t* ix = d.idx[l][f];
        v[f] = d.cols[l][f][ix ? (int64_t)ix[kk] : kk];
      } else {
        v[f] = f == 10 ? 1.0 : 0.0;
      }
    }
    double2* out = reinterpret_cast<double2*>(d.V[l] + kk * GP);
#pragma unroll
    for (int f = 0; f < GP / 2; f++) out[f] = make_double2(v[2 * f], v[2 * f + 1]);
  }
}

// Off-scan finishing with DMMA tiles (4 keys / records per m8n8k4), per warp over
// contiguous ranges of: the L keys (weights H_L), the A keys (H_A), the B records
// (R_B ⊗ [s_B, 1] and the B moments weighted by the record counts).  With
// s' = [s_0..s_9, 1] (index 10 = the constant), a level's moments are the 16x16
// matrix Σ_k w_k s'(k) s'(k)^T; the records give RBM[40][16] = Σ_rec rec ⊗ s'_B.
struct FinArgs {
  const double* brec;
  const int* bcount;
  int bcap;
  const double* VB;
  const unsigned* HL;
  const double* VL;
  int64_t nkL;
  const unsigned* HA;
  const double* VA;
  int64_t nkA;
  double* partials;  // [grid][NFIN]
};
__global__ void __launch_bounds__(256) k_cov_fin(FinArgs a) {
  const int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2, w = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 8 + w, GW = (int64_t)gridDim.x * 8;
  pdl_wait();
  pdl_trigger();
  double mL[4][2] = {}, mA[4][2] = {}, mB[4][2] = {}, rb[5][2][2] = {};
  auto srow = [&](const double* V, int64_t kk, bool v, double& s0, double& s1) {
    const double* row = V + (size_t)kk * GP;
    s0 = v ? row[m] : 0.0;
    s1 = v ? (m < 2 ? row[8 + m] : (m == 2 ? 1.0 : 0.0)) : 0.0;
  };
  auto moments = [&](const unsigned* H, const double* V, int64_t nk, double (&acc)[4][2]) {
    const int64_t ng = (nk + 3) / 4, g0 = gw * ng / GW, g1 = (gw + 1) * ng / GW;
    constexpr int U = COV_FIN_U;  // groups whose loads are in flight together
    for (int64_t gb = g0; gb < g1; gb += U) {
      double h[U], s0[U], s1[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t kk = (gb + u) * 4 + k;
        const bool v = gb + u < g1 && kk < nk;
        h[u] = v ? (double)H[kk] : 0.0;
        srow(V, v ? kk : 0, v, s0[u], s1[u]);
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        dmma(acc[0], h[u] * s0[u], s0[u]);
        dmma(acc[1], h[u] * s0[u], s1[u]);
        dmma(acc[2], h[u] * s1[u], s0[u]);
        dmma(acc[3], h[u] * s1[u], s1[u]);
      }
    }
  };
  moments(a.HL, a.VL, a.nkL, mL);
  moments(a.HA, a.VA, a.nkA, mA);
  {
    const int64_t nrec = min(*a.bcount, a.bcap);
    const int64_t ng = (nrec + 3) / 4, g0 = gw * ng / GW, g1 = (gw + 1) * ng / GW;
    for (int64_t gi = g0; gi < g1; gi++) {
      const int64_t r = gi * 4 + k;
      const bool v = r < nrec;
      const double* rec = a.brec + (size_t)(v ? r : 0) * BRW;
      const double n = v ? rec[18] : 0.0;
      double s0, s1;
      srow(a.VB, v ? (int64_t)(int)rec[34] : 0, v, s0, s1);
#pragma unroll
      for (int t = 0; t < 5; t++) {
        const double av = (v && 8 * t + m < 34) ? rec[8 * t + m] : 0.0;
        dmma(rb[t][0], av, s0);
        dmma(rb[t][1], av, s1);
      }
      dmma(mB[0], n * s0, s0);
      dmma(mB[1], n * s0, s1);
      dmma(mB[2], n * s1, s0);
      dmma(mB[3], n * s1, s1);
    }
  }
  // each warp stores its fragments into its own slice (every element exactly once), then one
  // barrier and a fixed-order sum over the 8 slices
  extern __shared__ __align__(16) double fred[];  // [8][NFIN]
  double* red = fred + (size_t)w * NFIN;
  auto put = [&](int base, int t1, int t2, const double (&c)[2]) {
    const int i = base + (8 * t1 + m) * 16 + 8 * t2 + 2 * k;
    *reinterpret_cast<double2*>(red + i) = make_double2(c[0], c[1]);
  };
#pragma unroll
  for (int t = 0; t < 5; t++) {
    put(0, t, 0, rb[t][0]);
    put(0, t, 1, rb[t][1]);
  }
#pragma unroll
  for (int q = 0; q < 4; q++) {
    put(640, q >> 1, q & 1, mL[q]);
    put(896, q >> 1, q & 1, mA[q]);
    put(1152, q >> 1, q & 1, mB[q]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NFIN; i += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ww++) t += fred[(size_t)ww * NFIN + i];
    a.partials[(size_t)blockIdx.x * NFIN + i] = t;
  }
}

// src[0:NPART] = Σ_warp scan partials; src[NPART:NPART+NFIN] = Σ_b fin partials.  A CTA per 32
// consecutive outputs: lane = output (coalesced rows), warp r of 32 sums rows r, r + 32, ...;
// then a fixed-order sum over the warps (deterministic).
// src = chunk sums of the partial rows, per element e: the scan's (e < NPART) in SUM_SP chunks,
// the fin's in SUM_SF chunks.  A CTA per (chunk, 32 consecutive elements): lane = element
// (coalesced rows), warp r of 32 sums rows r, r + 32, ... of the chunk, then a fixed-order sum
// over the warps (deterministic).
__global__ void __launch_bounds__(1024) k_cov_sum(const double* __restrict__ p1, int n1, const double* __restrict__ p2,
                                                  int n2, double* __restrict__ src) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
  int b = blockIdx.x;
  const double* p;
  int n, w, split, g, e;
  double* dst;
  if (b < (NPART / 32) * SUM_SP) {  // the heavy part first (scheduled first)
    g = b / (NPART / 32);
    e = (b % (NPART / 32)) * 32 + lane;
    p = p1, n = n1, w = NPART, split = SUM_SP;
    dst = src + (size_t)g * NPART + e;
  } else {
    b -= (NPART / 32) * SUM_SP;
    g = b / (NFIN / 32);
    e = (b % (NFIN / 32)) * 32 + lane;
    p = p2, n = n2, w = NFIN, split = SUM_SF;
    dst = src + (size_t)SUM_SP * NPART + (size_t)g * NFIN + e;
  }
  const int b0 = (int)((int64_t)n * g / split), b1 = (int)((int64_t)n * (g + 1) / split);
  double s = 0.0;
#pragma unroll 4
  for (int i = b0 + r; i < b1; i += 32) s += p[(size_t)i * w + e];
  __shared__ double red[32][33];
  red[r][lane] = s;
  __syncthreads();
  if (r == 0) {
    double t = 0.0;
    for (int i = 0; i < 32; i++) t += red[i][lane];
    *dst = t;
  }
}
__device__ __forceinline__ double cov_src(const double* __restrict__ src, int e) {
  double t = 0.0;
  if (e < NPART) {
#pragma unroll
    for (int g = 0; g < SUM_SP; g++) t += src[(size_t)g * NPART + e];
  } else {
#pragma unroll
    for (int g = 0; g < SUM_SF; g++) t += src[(size_t)SUM_SP * NPART + (size_t)g * NFIN + e - NPART];
  }
  return t;
}

__global__ void k_cov_assemble(const double* __restrict__ src, const int32_t* __restrict__ toff,
                               const int32_t* __restrict__ tidx, const double* __restrict__ tcoef, int nout,
                               double* __restrict__ out, int count_idx, unsigned long long* __restrict__ count) {
  pdl_wait();
  // a warp per output: lane (half, g) takes chunk g of every other term, then a fixed-order
  // butterfly sum over the lanes (all loads of an output in flight together; deterministic)
  static_assert(SUM_SP <= 16 && SUM_SF <= 16, "k_cov_assemble: one lane per chunk");
  const int lane = threadIdx.x & 31, g = lane & 15, half = lane >> 4;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < nout; o += nw) {
    double s = 0.0;
    const int t1 = toff[o + 1];
    for (int t = toff[o] + half; t < t1; t += 2) {
      const int e = tidx[t];
      double v = 0.0;
      if (e < NPART) {
        if (g < SUM_SP) v = src[(size_t)g * NPART + e];
      } else if (g < SUM_SF) {
        v = src[(size_t)SUM_SP * NPART + (size_t)g * NFIN + e - NPART];
      }
      s = fma(tcoef[t], v, s);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(FULL, s, d);
    if (lane == 0) out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)cov_src(src, count_idx);
}

// ======================================================================= host
struct CovLevel {
  int child = -1, rel = -1;
  std::vector<int> attrs;
  int64_t nk = 0;
  DevBuf V;
  std::vector<const double*> hcols;  // the features' columns (k_cov_dims parameters)
  std::vector<const int32_t*> hidx;
  std::vector<DevBuf> idx;  // composed foreign-key chains to the features of deeper relations
};

struct FastCov : FastPaths {
  int NS = 0, nF = 0;
  std::vector<int> fattrs;
  CovLevel L, A, B;
  DevBuf zeros;  // one zero view row (absent levels)
  DevBuf zbuf;   // [pad] [HA] [HL], cleared every run
  size_t off_HA = 0, off_HL = 0, zbytes = 0;
  DevBuf brec, partials, finp, src, toff, tidx, tcoef;
  DevBuf scan;   // scan layout of the root (k_cov_layout), built at plan time
  DevBuf items;  // [nitems + 1] first block of each work item (plan time)
  DevBuf rbase;  // [nitems + 1] first level-B record slot of each item; rbase[nitems] = records
  int64_t nblk = 0, nrec = 0;
  int nitems = 0, nstatic = 0;
  int grid = 148, nout = 0;
  bool only_scalar = true;

  std::string describe() const override {
    char b[320];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"cov\", \"NS\": %d, \"nF\": %d, \"nL\": %zu, \"nA\": %zu, \"nB\": %zu, \"grid\": %d, "
                  "\"threads\": %d, \"stages\": %d, \"static_chunks\": %d, \"items\": %d, \"b_records\": %lld}",
                  NS, nF, L.attrs.size(), A.attrs.size(), B.attrs.size(), grid, COV_W * 32, CovCfg<COV_W>::CF,
                  nstatic, nitems, (long long)nrec);
    return b;
  }
  bool skip_generic_views() const override { return only_scalar; }
  int run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) override;
};



template <int W>
cudaError_t cov_kernel_attr(int NS) {  // per device: called at plan time on the ctx's device
  constexpr int smem = CovCfg<W>::SMEM;
  if (NS == 0) return cudaFuncSetAttribute(k_cov<0, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (NS == 1) return cudaFuncSetAttribute(k_cov<1, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return cudaFuncSetAttribute(k_cov<2, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}
// launch with the programmatic-stream-serialization attribute (LMFAO_PDL=0: plain launches)
bool pdl_on() {
  static const int on = [] {
    const char* e = std::getenv("LMFAO_PDL");
    return e && e[0] == '0' ? 0 : 1;
  }();
  return on;
}
template <typename... KA, typename... A>
cudaError_t launch_pdl(void (*kern)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}
template <int W>
cudaError_t launch_cov_w(int NS, const CovArgs& g, int grid, cudaStream_t st) {
  constexpr int smem = CovCfg<W>::SMEM;
  if (NS == 0) return launch_pdl(k_cov<0, W>, grid, W * 32, smem, st, g);
  if (NS == 1) return launch_pdl(k_cov<1, W>, grid, W * 32, smem, st, g);
  return launch_pdl(k_cov<2, W>, grid, W * 32, smem, st, g);
}
cudaError_t launch_cov(int NS, const CovArgs& g, int grid, cudaStream_t st) { return launch_cov_w<COV_W>(NS, g, grid, st); }

}  // namespace

int FastCov::run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool& scalar_done) {
  const Rel& R = c->rels[c->root];
  {  // (b) dimension views of the featured PK leaves
    DimTables d{};
    d.z = zbuf.as<unsigned>();
    d.nz = (int64_t)(zbytes / 4);
    CovLevel* lv[3] = {&L, &A, &B};
    int64_t tot = 0;
    for (int i = 0; i < 3; i++) {
      for (size_t f = 0; f < lv[i]->hcols.size(); f++) {
        d.cols[i][f] = lv[i]->hcols[f];
        d.idx[i][f] = lv[i]->hidx[f];
      }
      d.n[i] = (int)lv[i]->attrs.size();
      d.nk[i] = lv[i]->rel >= 0 ? lv[i]->nk : 0;
      d.V[i] = lv[i]->V.as<double>();
      tot += d.nk[i] * GP;
    }
    const int64_t nth = std::max<int64_t>(tot / GP, d.nz);
    k_cov_dims<<<(unsigned)std::min<int64_t>((nth + 255) / 256, 148 * 16), 256, 0, st>>>(d);
    launches_add(1);
  }
  CovArgs g{};
  g.nblk = nblk;
  g.scan = scan.as<unsigned char>();
  g.VL = L.V.as<double>();
  g.VA = NS >= 1 ? A.V.as<double>() : zeros.as<double>();
  char* z = zbuf.as<char>();
  g.HA = reinterpret_cast<unsigned*>(z + off_HA);
  g.HL = reinterpret_cast<unsigned*>(z + off_HL);
  {
    const char* ab = std::getenv("LMFAO_COV_ABLATE");
    g.ablate = ab ? std::atoi(ab) : 0;
    const char* cd = std::getenv("LMFAO_COV_COLD_ALL");
    g.cold_all = cd && cd[0] == '1';
  }
  g.brec = brec.as<double>();
  g.item = items.as<int>();
  g.nitems = nitems;
  g.nstatic = nstatic;
  g.work = reinterpret_cast<int*>(z);
  g.rec_base = rbase.as<int>();
  g.partials = partials.as<double>();
  scan_timer_begin(c, st);
  cudaError_t e = launch_cov(NS, g, grid, st);
  scan_timer_end(c, st);
  if (e) return e;
  launches_add(1);
  FinArgs f{};
  f.brec = brec.as<double>();
  f.bcount = g.rec_base + nitems;
  f.bcap = (int)nrec;
  f.VB = NS == 2 ? B.V.as<double>() : zeros.as<double>();
  f.HL = g.HL;
  f.VL = L.V.as<double>();
  f.nkL = L.nk;
  f.HA = g.HA;
  f.VA = g.VA;
  f.nkA = NS >= 1 ? A.nk : 0;
  f.partials = finp.as<double>();
  CUDA_TRY(launch_pdl(k_cov_fin, FIN_BLOCKS, 256, 8 * NFIN * 8, st, f));
  CUDA_TRY(launch_pdl(k_cov_sum, SUM_CTAS, 1024, 0, st,
                      (const double*)partials.as<double>(), (int)nitems, (const double*)finp.as<double>(),
                      (int)FIN_BLOCKS, src.as<double>()));
  CUDA_TRY(launch_pdl(k_cov_assemble, (nout + 7) / 8 + 1, 256, 0, st, (const double*)src.as<double>(),
                      (const int32_t*)toff.as<int32_t>(), (const int32_t*)tidx.as<int32_t>(),
                      (const double*)tcoef.as<double>(), (int)nout, c->scalar_out.as<double>(),
                      (int)(NPART + 18 * 16 + 10), c->scalar_count.as<unsigned long long>()));
  launches_add(3);
  scalar_done = true;
  return cudaGetLastError();
}

// Planner hook: the batch is a covariance-shaped scalar batch (products of at most
// two identity factors) over fp64 features of the root (<= 8) and of at most three
// primary-key leaf dimensions (<= 10 each).  Otherwise nullptr (gram.cu / generic).
FastPaths* plan_cov(lmfao_ctx* c) {
  if (c->scalar_queries.empty()) return nullptr;
  const Rel& R = c->rels[c->root];
  if (R.children.empty()) return nullptr;
  // every non-root relation unique-keyed: a root row joins one row of each (snowflake PK chains,
  // dangling rows dropped at prepare), so a dimension key determines its subtree's features
  for (size_t u = 0; u < c->rels.size(); u++)
    if ((int)u != c->root && !c->rels[u].unique_key) return nullptr;
  auto root_child_of = [&](int rel) {  // the root child whose subtree holds rel
    while (c->rels[rel].parent != c->root) rel = c->rels[rel].parent;
    return rel;
  };
  struct Term {
    double coef;
    int a, b;
  };
  std::vector<std::vector<Term>> outs;
  std::set<int> feats;
  for (int q : c->scalar_queries) {
    for (auto& u : c->queries[q].udafs) {
      std::vector<Term> ts;
      for (auto& p : u) {
        double coef = p.coeff;
        std::vector<int> fa;
        for (auto& f : p.f) {
          if (f.kind == LMFAO_F_CONST) coef *= f.param;
          else if (f.kind == LMFAO_F_IDENT) fa.push_back(f.attr);
          else return nullptr;
        }
        if (fa.size() > 2) return nullptr;
        for (int a : fa) feats.insert(a);
        while (fa.size() < 2) fa.insert(fa.begin(), -1);
        ts.push_back(Term{coef, fa[0], fa[1]});
      }
      outs.push_back(ts);
    }
  }
  PhaseTrace tr("plan_cov");
  std::unique_ptr<FastCov> fc(new FastCov());
  fc->only_scalar = c->groups.empty();
  std::vector<std::vector<int>> lf(R.children.size());
  for (int a : feats) {
    if (c->attrs[a].dt != LMFAO_FP64) return nullptr;
    int o = c->owner[a];
    if (o == c->root) {
      fc->fattrs.push_back(a);
      continue;
    }
    bool found = false;
    for (size_t j = 0; j < R.children.size(); j++)
      if (R.children[j] == root_child_of(o)) {
        lf[j].push_back(a);
        found = true;
      }
    if (!found) return nullptr;
  }
  fc->nF = (int)fc->fattrs.size();
  if (fc->nF > 8) return nullptr;
  std::vector<int> featured;  // root children in sort order that carry features
  for (int j : c->levels)
    if (!lf[j].empty()) featured.push_back(j);
  if (featured.empty() || featured.size() > 3) return nullptr;
  for (int j : featured)
    if (lf[j].size() > 10) return nullptr;
  auto setup = [&](CovLevel& l, int j) {
    l.child = j;
    l.rel = R.children[j];
    l.attrs = lf[j];
    l.nk = c->rels[l.rel].nkeys;
  };
  setup(fc->L, featured.back());
  fc->NS = (int)featured.size() - 1;
  if (fc->L.nk * GP * 8 >= ((int64_t)1 << 32)) return nullptr;  // 32-bit view-row offsets in the scan
  if (fc->NS >= 1) setup(fc->A, featured[featured.size() - 2]);
  if (fc->NS == 2) setup(fc->B, featured[0]);
  // buffers
  if (fc->zeros.alloc(GP * 8)) return nullptr;
  if (cudaMemsetAsync(fc->zeros.p, 0, fc->zeros.bytes, c->stream)) return nullptr;
  CovLevel* lv[3] = {&fc->L, &fc->A, &fc->B};
  for (int i = 0; i < 3; i++) {
    CovLevel& l = *lv[i];
    if (l.rel < 0) continue;
    // + one zero row (index nk): the key of the scan layout's padding rows
    if (l.V.alloc((size_t)(l.nk + 1) * GP * 8)) return nullptr;
    if (cudaMemsetAsync(l.V.p, 0, l.V.bytes, c->stream)) return nullptr;
    std::vector<const double*> cp;
    std::vector<const int32_t*> ip;
    std::map<int, const int32_t*> chain;  // relation -> row per dimension key (composed foreign keys)
    std::function<const int32_t*(int)> row_of = [&](int rel) -> const int32_t* {
      if (rel == l.rel) return nullptr;
      auto it = chain.find(rel);
      if (it != chain.end()) return it->second;
      const int par = c->rels[rel].parent;
      const Rel& P = c->rels[par];
      int j = 0;
      while (P.children[j] != rel) j++;
      const int32_t* fk = P.fk_dense[j].as<int32_t>();  // the parent's rows -> this relation's rows
      const int32_t* up = row_of(par);
      const int32_t* out = fk;
      if (up) {  // compose: key -> parent row -> this relation's row
        l.idx.emplace_back();
        DevBuf& b = l.idx.back();
        if (b.alloc((size_t)std::max<int64_t>(l.nk, 1) * 4)) return nullptr;
        if (l.nk > 0 && gather_bytes(fk, reinterpret_cast<const uint32_t*>(up), b.p, l.nk, 4, c->stream)) return nullptr;
        out = b.as<int32_t>();
      }
      chain[rel] = out;
      return out;
    };
    for (int a : l.attrs) {
      const int o = c->owner[a];
      const Rel& O = c->rels[o];
      cp.push_back((const double*)O.cols[O.find_attr(a)].buf.p);
      const int32_t* ix = row_of(o);
      if (o != l.rel && !ix) return nullptr;
      ip.push_back(ix);
    }
    if (cp.size() > (size_t)GP) return nullptr;
    l.hcols = cp;
    l.hidx = ip;
  }
  const int64_t nkA = fc->NS >= 1 ? fc->A.nk : 0;
  fc->off_HA = 16;
  fc->off_HL = (fc->off_HA + (size_t)(nkA + 1) * 4 + 15) / 16 * 16;  // + the padding rows' key
  fc->zbytes = fc->off_HL + (size_t)(fc->L.nk + 1) * 4;
  if (fc->zbuf.alloc(fc->zbytes)) return nullptr;
  tr.mark("terms + buffers", c->stream);
  {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) == cudaSuccess && sms > 0) fc->grid = sms;
  }
  const int NW = fc->grid * COV_W;
  fc->nblk = (R.nrows + 31) / 32;
  if (fc->finp.alloc((size_t)FIN_BLOCKS * NFIN * 8)) return nullptr;
  if (fc->src.alloc((size_t)SRC_N * 8)) return nullptr;
  {  // scan layout of the root: x in DMMA lane order + dense keys with run-start flags, one
     // 2432-byte block per 32 rows
    if (fc->scan.alloc((size_t)std::max<int64_t>(fc->nblk, 1) * SBLK)) return nullptr;
    LayoutArgs la{};
    for (int i = 0; i < 8; i++) la.x[i] = i < fc->nF ? (const double*)R.cols[R.find_attr(fc->fattrs[i])].buf.p : nullptr;
    la.key[0] = R.fk_dense[fc->L.child].as<int32_t>();
    la.key[1] = fc->NS >= 1 ? R.fk_dense[fc->A.child].as<int32_t>() : nullptr;
    la.key[2] = fc->NS == 2 ? R.fk_dense[fc->B.child].as<int32_t>() : nullptr;
    la.nx = fc->nF;
    la.nlev = 1 + fc->NS;
    la.N = R.nrows;
    la.nblk = fc->nblk;
    la.pad[0] = (int)fc->L.nk;
    la.pad[1] = fc->NS >= 1 ? (int)fc->A.nk : 0;
    la.pad[2] = fc->NS == 2 ? (int)fc->B.nk : 0;
    la.out = fc->scan.as<unsigned char>();
    if (fc->nblk > 0) {
      k_cov_layout<<<148 * 8, 256, 0, c->stream>>>(la);
      if (cudaGetLastError() != cudaSuccess) return nullptr;
    }
  }
  tr.mark("scan layout", c->stream);
  {  // work items and their level-B record slots (see COV_TAIL)
    const int64_t n = fc->nblk;
    DevBuf bst;
    if (bst.alloc((size_t)std::max<int64_t>(n, 1) * 4)) return nullptr;
    if (n > 0)
      k_cov_bstats<<<(unsigned)std::min<int64_t>((n + 7) / 8, 148 * 16), 256, 0, c->stream>>>(
          fc->scan.as<unsigned char>(), n, fc->NS, bst.as<uint32_t>());
    int cold = COV_COST_COLD, tb = COV_TB, tail = COV_TAIL;
    if (const char* e = std::getenv("LMFAO_COV_COST_COLD")) cold = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LMFAO_COV_TB")) tb = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("LMFAO_COV_TAIL")) tail = std::min(100, std::max(0, std::atoi(e)));
    cudaStream_t st = c->stream;
    const bool stat_chunks = n >= 8 * (int64_t)NW;  // every static chunk non-empty (>= 3 blocks)
    if (!stat_chunks) tb = (int)std::min<int64_t>(tb, n / (2 * (int64_t)NW));  // dynamic items only, ~two per warp
    constexpr int CFb = CovCfg<COV_W>::CF;  // k_cov needs items of at least CF blocks
    tb = std::max(tb, CFb);
    // the static chunks' boundaries on the device; the host reads back where they end
    int32_t static_end = 0;
    DevBuf cost, cc;
    if (stat_chunks) {
      if (cost.alloc((size_t)(n + 1) * 4) || cc.alloc((size_t)(n + 1) * 4) || fc->items.alloc((size_t)(NW + 1) * 4 + 4))
        return nullptr;
      k_cov_cost<<<(unsigned)std::min<int64_t>((n + 256) / 256, 148 * 8), 256, 0, st>>>(bst.as<uint32_t>(), n,
                                                                                       (uint32_t)cold, cost.as<uint32_t>());
      if (exclusive_scan_u32(cost.as<uint32_t>(), cc.as<uint32_t>(), n + 1, st)) return nullptr;
      k_cov_static<<<(NW + 256) / 256, 256, 0, st>>>(cc.as<uint32_t>(), n, NW, tail, fc->items.as<int32_t>());
      if (cudaMemcpyAsync(&static_end, fc->items.as<int32_t>() + NW, 4, cudaMemcpyDeviceToHost, st) ||
          cudaStreamSynchronize(st) || cudaGetLastError())
        return nullptr;
      fc->nstatic = NW;
    } else {
      fc->nstatic = 0;
    }
    std::vector<int32_t> tl{static_end};  // the dynamic items after the static part
    while (tl.back() < n) {
      const int64_t e = std::min<int64_t>(tl.back() + tb, n);
      if (n - e < CFb) {  // the remainder is too short for an item of its own
        tl.push_back((int32_t)n);
        break;
      }
      tl.push_back((int32_t)e);
    }
    const int nst = fc->nstatic;
    fc->nitems = nst + (int)tl.size() - 1;
    DevBuf items_all, rc;
    if (items_all.alloc((size_t)(fc->nitems + 1) * 4) || rc.alloc((size_t)(fc->nitems + 1) * 4) ||
        fc->rbase.alloc((size_t)(fc->nitems + 1) * 4))
      return nullptr;
    if ((nst && cudaMemcpyAsync(items_all.p, fc->items.p, (size_t)nst * 4, cudaMemcpyDeviceToDevice, st)) ||
        cudaMemcpyAsync(items_all.as<int32_t>() + nst, tl.data(), tl.size() * 4, cudaMemcpyHostToDevice, st))
      return nullptr;
    fc->items = std::move(items_all);
    k_cov_recs<<<(fc->nitems + 256) / 256, 256, 0, st>>>(bst.as<uint32_t>(), fc->items.as<int32_t>(), fc->nitems,
                                                         rc.as<uint32_t>());
    if (exclusive_scan_u32(rc.as<uint32_t>(), fc->rbase.as<uint32_t>(), fc->nitems + 1, st)) return nullptr;
    uint32_t tot = 0;
    if (cudaMemcpyAsync(&tot, fc->rbase.as<uint32_t>() + fc->nitems, 4, cudaMemcpyDeviceToHost, st) ||
        cudaStreamSynchronize(st) || cudaGetLastError())
      return nullptr;

    fc->nrec = tot;
    if (fc->partials.alloc((size_t)std::max(fc->nitems, 1) * NPART * 8)) return nullptr;  // one partial per item
    if (fc->brec.alloc((size_t)std::max<uint32_t>(tot, 1) * BRW * 8)) return nullptr;
  }
  tr.mark("scan layout", c->stream);
  // source index of G[a][b] (a, b: attr id or -1 = "1"); see the layout above k_cov_sum
  auto fidx = [](const std::vector<int>& v, int a) {
    for (size_t i = 0; i < v.size(); i++)
      if (v[i] == a) return (int)i;
    return -1;
  };
  // fin layout (k_cov_fin): RBM[40][16] (rec row r x [s_B(0..9), 1 at col 10]), then 16x16 moment
  // matrices of L, A, B over s' = [s_0..s_9, 1]
  const int F0 = NPART, RBM = F0, MLM = F0 + 640, MAM = F0 + 896, MBM = F0 + 1152;
  auto TOT = [&](int r) { return RBM + r * 16 + 10; };
  auto lvl = [&](int x) -> int {  // 0 = "1", 1 = fact, 2 = L, 3 = A, 4 = B
    if (x < 0) return 0;
    if (fidx(fc->fattrs, x) >= 0) return 1;
    if (fidx(fc->L.attrs, x) >= 0) return 2;
    if (fc->NS >= 1 && fidx(fc->A.attrs, x) >= 0) return 3;
    return 4;
  };
  auto pos = [&](int x, int l) -> int {
    switch (l) {
      case 1: return fidx(fc->fattrs, x);
      case 2: return fidx(fc->L.attrs, x);
      case 3: return fidx(fc->A.attrs, x);
      case 4: return fidx(fc->B.attrs, x);
    }
    return 0;
  };
  auto src_of = [&](int a, int b) -> int {
    int la = lvl(a), lb = lvl(b);
    if (la > lb) {
      std::swap(a, b);
      std::swap(la, lb);
    }
    const int i = pos(a, la), j = pos(b, lb);
    switch (la * 5 + lb) {
      case 0: return TOT(18);                  // 1·1 = count
      case 1: return TOT(j);                   // 1·x
      case 2: return TOT(8 + j);               // 1·s_L
      case 3: return TOT(24 + j);              // 1·s_A
      case 4: return MBM + j * 16 + 10;        // 1·s_B
      case 6: return i * 8 + j;                // x·x
      case 7: return 64 + i * 10 + j;          // x·s_L
      case 8: return 144 + i * 10 + j;         // x·s_A
      case 9: return RBM + i * 16 + j;         // x·s_B
      case 12: return MLM + i * 16 + j;        // s_L·s_L
      case 13: return 144 + (8 + i) * 10 + j;  // s_L·s_A
      case 14: return RBM + (8 + i) * 16 + j;  // s_L·s_B
      case 18: return MAM + i * 16 + j;        // s_A·s_A
      case 19: return RBM + (24 + i) * 16 + j; // s_A·s_B
      case 24: return MBM + i * 16 + j;        // s_B·s_B
    }
    return -1;
  };
  std::vector<int32_t> toff{0}, tidx;
  std::vector<double> tcoef;
  for (auto& ts : outs) {
    for (auto& t : ts) {
      int s = src_of(t.a, t.b);
      if (s < 0) return nullptr;
      tidx.push_back(s);
      tcoef.push_back(t.coef);
    }
    toff.push_back((int32_t)tidx.size());
  }
  fc->nout = (int)outs.size();
  if (fc->toff.alloc(toff.size() * 4) || fc->tidx.alloc(std::max<size_t>(tidx.size(), 1) * 4) ||
      fc->tcoef.alloc(std::max<size_t>(tcoef.size(), 1) * 8))
    return nullptr;
  cudaStream_t st = c->stream;
  cudaMemcpyAsync(fc->toff.p, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice, st);
  if (!tidx.empty()) {
    cudaMemcpyAsync(fc->tidx.p, tidx.data(), tidx.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(fc->tcoef.p, tcoef.data(), tcoef.size() * 8, cudaMemcpyHostToDevice, st);
  }
  if (cudaStreamSynchronize(st)) return nullptr;
  if (cudaFuncSetAttribute(k_cov_fin, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * NFIN * 8)) return nullptr;
  if (cov_kernel_attr<COV_W>(fc->NS)) return nullptr;
  return fc.release();
}

}  // namespace lmfao
