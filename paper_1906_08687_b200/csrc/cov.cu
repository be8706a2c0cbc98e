// cov.cu — the covariance batch's fused root scan, B200 version 2 (k_cov).
//
// Same mathematics as gram.cu (§3 "covariance matrix" P:397-402: every
// aggregate is an entry of G = Σ_f u(f) u(f)^T with u = [1, x, s_L, s_A, s_B]),
// evaluated over the root sorted by its foreign keys in increasing domain size
// with the multi-output trie registration of P:1020-1214:
//   per row          x⊗x, x⊗s_L                (FP64 DMMA m8n8k4 on 4-row groups)
//   per level-A run  R_A⊗s_A, R_A = Σ_run [x, s_L, 1]  (4 runs per DMMA, "intermediate aggregates")
//   per level-B run  R_B⊗s_B, R_B = Σ_{A-runs} [R_A, n·s_A]  (record list, finished off-scan)
//   dimension side   Σ_k H_r[k] s_r(k) s_r(k)^T  ("each aggregate to its own root")
// What changed against gram.cu, and why (all measured on B200):
//  * the kernel is specialised at compile time for ≤ 8 fact features and ≤ 10
//    features per dimension level (C1, C2, C5's covariance), so the hot loop has
//    no runtime shape logic (the v12 kernel spent 45 warp-instructions per row);
//  * every warp runs its own TMA pipeline: `cp.async.bulk` of the fact columns and
//    keys of a 32-row block into a CF-deep shared-memory ring, and 16-byte
//    `cp.async` gathers of the view rows s_L[k_L] (96-byte rows, L2-resident),
//    issued one block ahead — no operand prefetch lives in registers (a TMA
//    `tile::gather4` per 4 rows instead was measured at 0.60 vs 0.367 ms per scan);
//  * level-A run records are stored unreduced (per lane) in shared memory and
//    reduced four at a time straight into the DMMA A-operand layout;
//  * level-B records go to a device list and are finished by a small kernel;
//  * H_L (root rows per L key, for s_L⊗s_L) is counted in a per-CTA open-
//    addressing table in shared memory (Zipf-hot keys would serialise global
//    atomics), spilling to global atomics when a probe misses twice.
// Runs split at block / item boundaries are exact (every update is linear in the
// run sums), so any row order is correct; the sort only makes runs long.
#include <cuda.h>

#include <cstdlib>
#include <set>

#include <functional>

#include "ctx.h"

namespace lmfao {
namespace {

#ifndef COV_IB  // C2 scan by item size: 8 0.359, 16 0.342, 24 0.335, 32 0.335, 40 0.342, 48 0.358, 64 0.373 ms
#define COV_IB 24
#endif
constexpr int IB = COV_IB;   // 32-row blocks per dynamically scheduled item (at most; fewer for small roots)
#ifndef COV_TAIL_PCT  // the last COV_TAIL_PCT % of the blocks go in 2-block items (C2: 4 % 0.348, 10 % 0.335, 20 % 0.348 ms)
#define COV_TAIL_PCT 10
#endif
constexpr int GP = 12;       // doubles per view row (cols >= n are 0)
#ifndef COV_HT_BITS  // per-CTA H_L slots: only the Zipf-hottest keys need them, the rest go to global
#define COV_HT_BITS 6   // REDs over many addresses (C2 scan: 2^12 0.355, 2^10 0.346, 2^8 0.343, 2^6 0.342,
#endif                  // 2^5 0.345 ms)
constexpr int HT = 1 << COV_HT_BITS;
constexpr int SBLK = 256 * 8 + 3 * 32 * 4;     // scan-layout bytes per 32-row block: x in DMMA order + 3 key rows
constexpr int STG_G = 32 * GP * 8;             // 3072 B of gathered view rows per block (2 slots)
constexpr int NPART = 384;   // per-CTA partial: XX[8][8] | XL[8][10] | RA[24][10]
constexpr int BRW = 36;      // doubles per B record
constexpr int NFIN = 640 + 3 * 256;  // RBM[40][16] | ML[16][16] | MA[16][16] | MB[16][16]
constexpr int FIN_BLOCKS = 296;
constexpr int SUM_SPLIT = 8;  // k_cov_sum: partial rows in SUM_SPLIT chunks (grid y), summed again by k_cov_assemble
constexpr unsigned FULL = 0xffffffffu;

static_assert(SBLK % 128 == 0 && STG_G % 128 == 0, "TMA / cp.async alignment");

struct CovArgs {
  int64_t nrows, nblk;
  const unsigned char* scan;  // [nblk][SBLK] scan layout of the root
  const double* VL;           // [nkL x GP]
  const double* VA;           // [nkA x GP] (a zero row if absent)
  unsigned* HL;
  unsigned* HA;
  double* brec;
  int* bcount;
  int bcap;
  double* partials;  // [grid * W][NPART] per-warp partials
  int* work;
  int ablate;  // diagnostics only (LMFAO_COV_ABLATE, results invalid): 1 no gathers, 2 no record DMMA, 8 no H_L,
               // 16 no compute at all (pipeline only), 32 every block on the fast path, 64 no wait for gathers
  int cold;    // blocks with at least this many level-A run starts (and no level-B start inside) take
               // the per-row level-A path; 0: never (LMFAO_COV_COLD)
  int ib;      // blocks per work item before the 2-block tail: IB, or 2 for small roots (template IBK)
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
// 16-byte L1-allocating async copy; src_bytes = 0 writes zeros (ragged tail rows)
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
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

// Scan layout of the root (built once at plan time, like the sort at prepare):
// per 32-row block b, x in the DMMA lane order [group j][lane 4m+k] = x_m[32b+4j+k]
// (0 for m >= nx or rows >= N), then the dense keys [level][32] of L, A, B.  One
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
      int2 v = make_int2(0, 0);
      const int64_t row = 32 * b + r;
      if (lv < a.nlev) {
        v.x = row < a.N ? a.key[lv][row] : a.pad[lv];
        v.y = row + 1 < a.N ? a.key[lv][row + 1] : a.pad[lv];
      }
      reinterpret_cast<int2*>(a.out)[i] = v;
    }
  }
}

constexpr int COV_W = 12;     // warps per CTA of the scan (one CTA per SM; 168 registers with the per-row path)
constexpr int COV_COLD = 1;  // level-A run starts from which a block takes the per-row path (C2 scan: 1 0.333, 2 0.335, 3 0.338, 4 0.339, never 0.383 ms)

template <int W>
#ifndef COV_CF12  // 3: a smaller carve-out leaves 60 KB of L1 for the view-row gathers (0.359 -> 0.357 ms vs 4)
#define COV_CF12 3
#endif
struct CovCfg {
  static constexpr int CF = W >= 16 ? 3 : (W >= 12 ? COV_CF12 : 7);  // fact-block ring slots per warp
  static constexpr int WB = CF * SBLK + 2 * STG_G + 512;       // + barriers, item ring, segment table
  static constexpr int SMEM = 128 + HT * 8 + W * WB;  // [CTA counters | H_L table | warps]
  static_assert(SMEM <= 232448, "shared memory budget");
};

// NS = number of featured levels above L (0: L only, 1: A and L, 2: B, A and L); W warps per CTA.
//
// Per 32-row block (lane = row for keys; DMMA layout lane = 4m + k for values):
//  * x⊗x, x⊗s_L0..7 and x⊗[s_L8, s_L9, 1] (B = the t tile) as three DMMA m8n8k4 per 4-row group;
//  * the open level-A run's sums of v = [x, s_L0..7, (s_L8, s_L9, 1)] are carried per lane (C,
//    DADD) across blocks in which no run ends (62% of C2's blocks: Zipf-hot keys make long runs);
//  * in a block where runs end, the run ("segment") sums come from DMMA against a 0/1
//    segment-indicator operand, D_t[f][s] += Σ_k v_t[f](row k) [seg(row k) = s], in windows of 8
//    segments; each window's records (partial runs are exact by linearity) are two DMMA passes
//    against the s_A rows (lane (m,k) holds segments 2k and 2k+1), DFMA for s_A8/9 and n·s_A,
//    and H_A;
//  * level-B records (run totals and Σ n·s_A) go to the device record list at B-run ends.
template <int NS, int W, int IBK>
__global__ void __launch_bounds__(W * 32, 1) k_cov(const __grid_constant__ CovArgs g) {
  using Cfg = CovCfg<W>;
  constexpr int CF = Cfg::CF;
  const int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2, wib = threadIdx.x >> 5;
  extern __shared__ __align__(1024) unsigned char sm[];
  int* cta_done = reinterpret_cast<int*>(sm);
  int* hkey = reinterpret_cast<int*>(sm + 128);
  unsigned* hcnt = reinterpret_cast<unsigned*>(sm + 128 + HT * 4);
  unsigned char* wbase = sm + 128 + HT * 8 + wib * Cfg::WB;
  unsigned char* gbase = wbase + CF * SBLK;  // 2 gather slots
  uint64_t* bar_f = reinterpret_cast<uint64_t*>(gbase + 2 * STG_G);
  int* ring = reinterpret_cast<int*>(bar_f + 8);  // 8 grabbed item ids
  int* segst = ring + 8;                          // [34] segment start rows of the current block
  int* segkey = segst + 40;                       // [33] their A keys

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

  // work items: blocks [0, NB) in items of IB blocks, the last ~10% in items of 2 blocks (a
  // short tail for the dynamic schedule)
  const int64_t N = g.nrows, NB = g.nblk;
  constexpr int ib = IBK;
  const int nbig = (int)(NB * (100 - COV_TAIL_PCT) / 100 / ib);
  const int nitems = nbig + (int)((NB - (int64_t)nbig * ib + 1) / 2);
  auto item_first = [&](int it) { return it < nbig ? (int64_t)it * ib : (int64_t)nbig * ib + 2 * (int64_t)(it - nbig); };
  auto item_blocks = [&](int it) {
    const int64_t f = item_first(it), r = NB - f;
    const int64_t cap = it < nbig ? ib : 2;
    return (int)(r < cap ? r : cap);
  };

  // cursors over this warp's block sequence (items grabbed dynamically, in order)
  int nring = 0;
  int next_item = lane == 0 ? atomicAdd(g.work, 1) : 0;  // one grab in flight ahead of use
  auto grab = [&]() {
    const int it = __shfl_sync(FULL, next_item, 0);
    if (lane == 0) {
      ring[nring & 7] = it;
      next_item = atomicAdd(g.work, 1);
    }
    nring++;
    __syncwarp();
  };
  struct Cur {
    int slot, b, item, nb;  // nb: blocks of the item
    int64_t gb0;            // its first block
    int rows;               // rows of the item
  };
  auto set_item = [&](Cur& c) {
    c.item = ring[c.slot & 7];
    if (c.item < nitems) {
      c.gb0 = item_first(c.item);
      c.nb = item_blocks(c.item);
      const int64_t r = N - c.gb0 * 32;
      c.rows = (int)(r < 32 * c.nb ? r : 32 * c.nb);
    }
  };
  auto advance = [&](Cur& c, bool may_grab) {
    if (c.item >= nitems) return;
    if (++c.b < c.nb) return;
    c.b = 0;
    c.slot++;
    if (may_grab && c.slot >= nring) grab();
    set_item(c);
  };
  auto gblock = [&](const Cur& c) { return c.gb0 + c.b; };
  auto issue_fact = [&](const Cur& c, int stage) {
    __syncwarp();
    if (c.item >= nitems) return;
    if (lane == 0) {  // the slot was only read (generic proxy) since its last fill: no proxy fence needed
      mbar_expect(&bar_f[stage], SBLK);
      bulk_load(wbase + stage * SBLK, g.scan + gblock(c) * SBLK, SBLK, &bar_f[stage]);
    }
  };
  // view rows s_L[k_L(row)] of a landed fact block -> gather slot [32 rows x 96 B]; 16-byte
  // chunk c = 32 i + lane (row c / 6), so each instruction covers ~5 whole rows (coalesced)
  int ch_row[6], ch_off[6];
#pragma unroll
  for (int i = 0; i < 6; i++) {
    const int c = 32 * i + lane;
    ch_row[i] = c / 6;
    ch_off[i] = (c % 6) * 16;
  }
  auto issue_gather = [&](const Cur& c, int fslot, int gslot) {
    if (c.item < nitems && !(g.ablate & 1)) {
      // every block is full: rows past N carry the zero row's key (no per-chunk bounds)
      const int* kls = reinterpret_cast<const int*>(wbase + fslot * SBLK + 2048);
      const char* vl = reinterpret_cast<const char*>(g.VL);
      const uint32_t dst = sa(gbase + gslot * STG_G) + 16 * lane;
#pragma unroll
      for (int i = 0; i < 6; i++) {
        const unsigned off = (unsigned)kls[ch_row[i]] * (unsigned)(GP * 8) + (unsigned)ch_off[i];
        cp16full(dst + 512 * i, vl + off);
      }
    }
    cp_commit();
  };

  // ---- accumulators
  double aXX[2] = {0, 0}, aXL[2] = {0, 0}, aXT[2] = {0, 0};
  double aRA[3][2] = {{0, 0}, {0, 0}, {0, 0}}, r8[3] = {0, 0, 0}, r9[3] = {0, 0, 0};
  double SB0 = 0, SB1 = 0, SB2 = 0, SBn = 0, SBn8 = 0, SBn9 = 0;
  double C0 = 0, C1 = 0, C2 = 0;  // this lane's rows of the open level-A run (since its last fold)
  bool openB = false;
  int curB = 0;
  int prevL = -1, prevA = -1, prevB = -1;
  const int tcol = m < 3 ? 8 + m : 11;  // t tile: s_L8, s_L9, 1 (view column 10 holds 1.0), 0

  auto hl_add = [&](int key, unsigned len) {  // two probes, straight-line; full: global RED
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
  };
  auto push_B = [&](int keyB) {
    const double v0 = red4(SB0), v1 = red4(SB1), v2 = red4(SB2), v3 = red4(SBn), v4 = red4(SBn8), v5 = red4(SBn9);
    int slot = 0;
    if (lane == 0) slot = atomicAdd(g.bcount, 1);
    slot = __shfl_sync(FULL, slot, 0);
    if (slot < g.bcap) {
      double* rec = g.brec + (size_t)slot * BRW;
      if (k == 0) {
        rec[m] = v0;
        rec[8 + m] = v1;
        rec[16 + m] = v2;
        rec[24 + m] = v3;
      }
      if (lane == 0) {
        rec[32] = v4;
        rec[33] = v5;
        rec[34] = (double)keyB;
        rec[35] = 0.0;
      }
    }
    SB0 = SB1 = SB2 = SBn = SBn8 = SBn9 = 0.0;
  };

  // ---- pipeline prologue: fact blocks 0..CF-1 in flight, gathers of block 0
  grab();
  Cur cc{0, 0, 0, 0, 0, 0};
  set_item(cc);
  Cur cf = cc;
  for (int s = 0; s < CF; s++) {
    issue_fact(cf, s);
    advance(cf, true);
  }
  if (cc.item < nitems) mbar_wait(&bar_f[0], 0);
  issue_gather(cc, 0, 0);
  int blk = 0, fs = 0, fph = 0;  // fs = blk % CF, fph = (blk / CF) & 1
  while (cc.item < nitems) {
    Cur cn = cc;
    advance(cn, false);
    const bool has_next = cn.item < nitems;
    const int fs1 = fs + 1 == CF ? 0 : fs + 1;
    {  // gathers of the next block (its keys have landed)
      const int fph1 = fs + 1 == CF ? fph ^ 1 : fph;
      if (has_next) mbar_wait(&bar_f[fs1], (uint32_t)fph1);
      issue_gather(cn, fs1, (blk + 1) & 1);
    }
    if (cc.b == 0) prevL = prevA = prevB = -1;  // a new item: row 0 starts runs at every level
    if (!(g.ablate & 64)) cp_wait1();
    __syncwarp();
    if (g.ablate & 16) {
      issue_fact(cf, fs);
      advance(cf, true);
      cc = cn;
      blk++;
      fs = fs1;
      if (fs == 0) fph ^= 1;
      continue;
    }
    const unsigned char* st = wbase + fs * SBLK;
    const double* xs = reinterpret_cast<const double*>(st);
    const int* ks = reinterpret_cast<const int*>(st + 2048);
    const double* gs = reinterpret_cast<const double*>(gbase + (blk & 1) * STG_G);
    // rows past N (the last block's tail) are padding in the scan layout: x = 0 and the keys of
    // the zero rows appended to the views, in runs of their own — they add exact zeros
    constexpr int nv = 32;
    constexpr bool vr = true;
    const int kl = vr ? ks[lane] : -1;
    const int ka = vr ? (NS >= 1 ? ks[32 + lane] : 0) : -1;
    const int kb = vr ? (NS == 2 ? ks[64 + lane] : 0) : -1;
    int pl = __shfl_up_sync(FULL, kl, 1), pa = __shfl_up_sync(FULL, ka, 1), pb = __shfl_up_sync(FULL, kb, 1);
    if (lane == 0) {
      pl = prevL;
      pa = prevA;
      pb = prevB;
    }
    const bool dB = vr && kb != pb;
    const bool dA = vr && (dB || ka != pa);
    const bool lead = vr && (dA || kl != pl || lane == 0);
    const unsigned mB = __ballot_sync(FULL, dB), mA = __ballot_sync(FULL, dA), mLd = __ballot_sync(FULL, lead);
    prevL = __shfl_sync(FULL, kl, nv - 1);
    prevA = __shfl_sync(FULL, ka, nv - 1);
    prevB = __shfl_sync(FULL, kb, nv - 1);
    // does the run open at this block's end end here? (the next block is another item, or
    // its row 0 has other A / B keys)
    bool endA = true, endB = true;
    if (has_next && cn.b != 0) {
      const int* kn = reinterpret_cast<const int*>(wbase + fs1 * SBLK + 2048);
      const int na = NS >= 1 ? kn[32] : 0, nb2 = NS == 2 ? kn[64] : 0;
      endB = nb2 != prevB;
      endA = endB || na != prevA;
    }
    if (lead && !(g.ablate & 8)) {
      const unsigned above = mLd & ~((2u << lane) - 1u);
      const int end = above ? __ffs(above) - 1 : nv;
      hl_add(kl, (unsigned)(end - lane));
    }
    if (mB & 1u) {  // a level-B run starts at row 0
      openB = true;
      curB = __shfl_sync(FULL, kb, 0);
    }
    const unsigned mAx = mA & ~1u;  // run starts inside the block (row 0 always opens segment 0)
    const double* gl = gs + k * GP;
    if ((mAx == 0 && !endA) || (g.ablate & 32)) {
      // fast path: the open run continues through the block
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const double xa = xs[32 * j + lane];
        const double* gr = gl + j * 4 * GP;
        const double sv = gr[m];
        const double tv = gr[tcol];
        dmma(aXX, xa, xa);
        dmma(aXL, xa, sv);
        dmma(aXT, xa, tv);  // x ⊗ [s_L8, s_L9, 1]: B[k][n] = t_n(row k) from lane 4n + k
        C0 += xa;
        C1 += sv;
        C2 += tv;
      }
    } else if (NS >= 1 && g.cold > 0 && __popc(mAx) >= g.cold && !(mB & ~1u)) {
      // cold block (many short level-A runs, no level-B run starting inside): instead of run
      // ("segment") sums times the run's s_A row, every row's v = [x, s_L, (s_L8, s_L9, 1)]
      // times its own s_A row — the same sum by linearity, Σ_run (Σ_rows v) ⊗ s_A =
      // Σ_rows v ⊗ s_A(row) — without segment windows, records or their s_A loads.
      const int* kas = ks + 32;
      double nc = 0.0;
      if (!(mA & 1u)) {  // row 0 continues the run open at the previous block's end: its rows from
                         // earlier blocks (carried in C) with the run's s_A row (row 0's key)
        const int key0 = __shfl_sync(FULL, ka, 0);
        const double* ar = g.VA + (size_t)(unsigned)key0 * GP;
        const double b0 = ar[m];
        const double2 b89 = *reinterpret_cast<const double2*>(ar + 8);
        dmma(aRA[0], C0, b0);
        dmma(aRA[1], C1, b0);
        dmma(aRA[2], C2, b0);
        r8[0] = fma(C0, b89.x, r8[0]);
        r9[0] = fma(C0, b89.y, r9[0]);
        r8[1] = fma(C1, b89.x, r8[1]);
        r9[1] = fma(C1, b89.y, r9[1]);
        r8[2] = fma(C2, b89.x, r8[2]);
        r9[2] = fma(C2, b89.y, r9[2]);
        SB0 += C0;
        SB1 += C1;
        SB2 += C2;
        // carried rows: their count is the constant row (m == 2) of the t tile
        nc = __shfl_sync(FULL, red4(C2), 8);
        const double nq = k == 0 ? nc : 0.0;  // once per quad (SBn* are summed over k at push_B)
        SBn = fma(nq, b0, SBn);
        SBn8 = fma(nq, b89.x, SBn8);
        SBn9 = fma(nq, b89.y, SBn9);
        C0 = C1 = C2 = 0.0;
      }
      // H_A: each run's rows in this block (and the carried rows for row 0's run)
      if (vr && (dA || lane == 0) && !(g.ablate & 2)) {
        const unsigned above = mA & ~((2u << lane) - 1u);
        const int end = above ? __ffs(above) - 1 : nv;
        gred_add(&g.HA[ka], (unsigned)(end - lane) + (lane == 0 ? (unsigned)nc : 0u));
      }
#pragma unroll
      for (int h = 0; h < 2; h++) {
        double sam[4], s8[4], s9[4];  // the s_A rows of this lane's next 4 rows, loads in flight together
#pragma unroll
        for (int jj = 0; jj < 4; jj++) {
          const int r = 4 * (4 * h + jj) + k;
          const double* ar = g.VA + (size_t)(unsigned)(r < nv ? kas[r] : 0) * GP;
          const double2 a89 = *reinterpret_cast<const double2*>(ar + 8);
          sam[jj] = r < nv ? ar[m] : 0.0;
          s8[jj] = r < nv ? a89.x : 0.0;
          s9[jj] = r < nv ? a89.y : 0.0;
        }
#pragma unroll
      for (int jj = 0; jj < 4; jj++) {
        const int j = 4 * h + jj;
        const double xa = xs[32 * j + lane];
        const double* gr = gl + j * 4 * GP;
        const double sv = gr[m];
        const double tv = gr[tcol];
        dmma(aXX, xa, xa);
        dmma(aXL, xa, sv);
        dmma(aXT, xa, tv);  // x ⊗ [s_L8, s_L9, 1]: B[k][n] = t_n(row k) from lane 4n + k
        dmma(aRA[0], xa, sam[jj]);
        dmma(aRA[1], sv, sam[jj]);
        dmma(aRA[2], tv, sam[jj]);
        r8[0] = fma(xa, s8[jj], r8[0]);
        r9[0] = fma(xa, s9[jj], r9[0]);
        r8[1] = fma(sv, s8[jj], r8[1]);
        r9[1] = fma(sv, s9[jj], r9[1]);
        r8[2] = fma(tv, s8[jj], r8[2]);
        r9[2] = fma(tv, s9[jj], r9[2]);
        SB0 += xa;
        SB1 += sv;
        SB2 += tv;
        SBn += sam[jj];
        SBn8 += s8[jj];
        SBn9 += s9[jj];
      }
      }
    } else {
      // segments of the block: segment 0 starts at row 0, segment s >= 1 at the s-th run start
      const int R = __popc(mAx);
      {
        const int sr = __popc(mAx & ((2u << lane) - 1u));
        if (lane == 0 || ((mAx >> lane) & 1u)) {
          segst[sr] = lane;
          segkey[sr] = ka;
        }
        if (lane == 0) segst[R + 1] = nv;
        __syncwarp();
      }
      int sb = 0;  // first segment of the current window of 8
      double D[3][2] = {{0, 0}, {0, 0}, {0, 0}};
      // this lane's record slots: segments s0 = sb + 2k (pass 0) and s0 + 1 (pass 1)
      int key0 = 0, key1 = 0;
      double b0 = 0, b1 = 0;
      double2 b089 = make_double2(0, 0), b189 = make_double2(0, 0);
      auto load_window = [&]() {  // keys and s_A rows of the window's segments
        const int s0 = sb + 2 * k, s1 = s0 + 1;
        const bool v0 = s0 <= R, v1 = s1 <= R;
        key0 = v0 ? segkey[s0] : 0;
        key1 = v1 ? segkey[s1] : 0;
        const double* row0 = g.VA + (size_t)(unsigned)key0 * GP;
        const double* row1 = g.VA + (size_t)(unsigned)key1 * GP;
        b0 = v0 ? row0[m] : 0.0;
        b1 = v1 ? row1[m] : 0.0;
        b089 = v0 ? *reinterpret_cast<const double2*>(row0 + 8) : make_double2(0, 0);
        b189 = v1 ? *reinterpret_cast<const double2*>(row1 + 8) : make_double2(0, 0);
      };
      // the window's (partial) level-A records ⊗ s_A, and level B; segments before s_end are
      // complete here (s_end itself may continue into the next window)
      auto flush_window = [&](int s_end) {
        const int s0 = sb + 2 * k, s1 = s0 + 1;
        // row counts of the slots (incl. rows carried from earlier blocks) = the t tile's "1" row
        const double n0 = __shfl_sync(FULL, D[2][0], 8 + k), n1 = __shfl_sync(FULL, D[2][1], 8 + k);
        if (!(g.ablate & 2)) {
#pragma unroll
          for (int t = 0; t < 3; t++) {
            dmma(aRA[t], D[t][0], b0);
            dmma(aRA[t], D[t][1], b1);
            r8[t] = fma(D[t][0], b089.x, fma(D[t][1], b189.x, r8[t]));
            r9[t] = fma(D[t][0], b089.y, fma(D[t][1], b189.y, r9[t]));
          }
          if (NS >= 1 && m == 0) {
            if (n0 > 0.0) gred_add(&g.HA[key0], (unsigned)n0);
            if (n1 > 0.0) gred_add(&g.HA[key1], (unsigned)n1);
          }
        }
        auto add_segs = [&](int lo, int hi) {  // segments [lo, hi) of the window -> the open B run
          const bool u0 = s0 >= lo && s0 < hi, u1 = s1 >= lo && s1 < hi;
          const double d0 = u0 ? 1.0 : 0.0, d1 = u1 ? 1.0 : 0.0;
          SB0 = fma(d0, D[0][0], fma(d1, D[0][1], SB0));
          SB1 = fma(d0, D[1][0], fma(d1, D[1][1], SB1));
          SB2 = fma(d0, D[2][0], fma(d1, D[2][1], SB2));
          const double w0 = u0 ? n0 : 0.0, w1 = u1 ? n1 : 0.0;
          SBn = fma(w0, b0, fma(w1, b1, SBn));
          SBn8 = fma(w0, b089.x, fma(w1, b189.x, SBn8));
          SBn9 = fma(w0, b089.y, fma(w1, b189.y, SBn9));
        };
        int lo = sb;
        unsigned bb = mB & ~1u;
        while (bb) {  // level-B run starts inside the block (rare)
          const int p = __ffs(bb) - 1;
          bb &= bb - 1;
          const int sp = __popc(mAx & ((2u << p) - 1u));
          if (sp <= sb || sp > s_end) continue;  // handled by the window that completes segment sp - 1
          add_segs(lo, sp);
          push_B(curB);
          curB = __shfl_sync(FULL, kb, p);
          lo = sp;
        }
        add_segs(lo, sb + 8);
#pragma unroll
        for (int t = 0; t < 3; t++) D[t][0] = D[t][1] = 0.0;
      };
      load_window();
      {  // the carried part of segment 0 (rows of earlier blocks) -> slot 0
        const double f0 = red4(C0), f1 = red4(C1), f2 = red4(C2);
        if (k == 0) {
          D[0][0] = f0;
          D[1][0] = f1;
          D[2][0] = f2;
        }
        C0 = C1 = C2 = 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const double xa = xs[32 * j + lane];
        const double* gr = gl + j * 4 * GP;
        const double sv = gr[m];
        const double tv = gr[tcol];
        dmma(aXX, xa, xa);
        dmma(aXL, xa, sv);
        dmma(aXT, xa, tv);  // x ⊗ [s_L8, s_L9, 1]: B[k][n] = t_n(row k) from lane 4n + k
        const int slast = __popc(mAx & ((2u << (4 * j + 3)) - 1u));
        if (slast - sb >= 8) {  // the group reaches past the window: flush it, restart at the group's first segment
          const int s4j = __popc(mAx & ((2u << (4 * j)) - 1u));
          flush_window(s4j);
          sb = s4j;
          load_window();
        }
        const int sr = __popc(mAx & ((2u << (4 * j + k)) - 1u));
        const double ind = (sr - sb == m) ? 1.0 : 0.0;
        dmma(D[0], xa, ind);
        dmma(D[1], sv, ind);
        dmma(D[2], tv, ind);
      }
      if (endA) {
        flush_window(64);
      } else {  // the last segment continues into the next block: keep it open (carried in C)
        const int sl = R - sb;  // its slot
        {
          // take it out of D before the flush: its value moves to lane (m, 0) of C
          double e0 = 0, e1 = 0, e2 = 0;
          if (k == (sl >> 1)) {
            e0 = (sl & 1) ? D[0][1] : D[0][0];
            e1 = (sl & 1) ? D[1][1] : D[1][0];
            e2 = (sl & 1) ? D[2][1] : D[2][0];
            if (sl & 1) D[0][1] = D[1][1] = D[2][1] = 0.0;
            else D[0][0] = D[1][0] = D[2][0] = 0.0;
          }
          C0 = __shfl_sync(FULL, e0, 4 * m + (sl >> 1));
          C1 = __shfl_sync(FULL, e1, 4 * m + (sl >> 1));
          C2 = __shfl_sync(FULL, e2, 4 * m + (sl >> 1));
          if (k != 0) C0 = C1 = C2 = 0.0;
        }
        flush_window(64);
      }
    }
    if (endB && openB) {  // the level-B run ends with this block
      push_B(curB);
      openB = false;
    }
    issue_fact(cf, fs);  // the slot just consumed takes the block CF ahead
    advance(cf, true);
    cc = cn;
    blk++;
    fs = fs1;
    if (fs == 0) fph ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");

  // ---- this warp's partial -> partials[CTA * W + warp] (no CTA barrier: warps finish unevenly)
#pragma unroll
  for (int t = 0; t < 3; t++) {
    r8[t] = red4(r8[t]);
    r9[t] = red4(r9[t]);
  }
  double* out = g.partials + ((size_t)blockIdx.x * W + wib) * NPART;
  out[m * 8 + 2 * k] = aXX[0];
  out[m * 8 + 2 * k + 1] = aXX[1];
  out[64 + m * 10 + 2 * k] = aXL[0];
  out[64 + m * 10 + 2 * k + 1] = aXL[1];
  if (k == 0) {
    out[64 + m * 10 + 8] = aXT[0];
    out[64 + m * 10 + 9] = aXT[1];
  }
#pragma unroll
  for (int t = 0; t < 3; t++) {
    out[144 + (8 * t + m) * 10 + 2 * k] = aRA[t][0];
    out[144 + (8 * t + m) * 10 + 2 * k + 1] = aRA[t][1];
    if (k == 0) {
      out[144 + (8 * t + m) * 10 + 8] = r8[t];
      out[144 + (8 * t + m) * 10 + 9] = r9[t];
    }
  }
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
  const double* const* cols[3];
  const int32_t* const* idx[3];  // per feature: row of its relation per dimension key (null: the key's own row)
  int n[3];
  int64_t nk[3];
  double* V[3];
};
__global__ void k_cov_dims(DimTables d) {
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
  double mL[4][2] = {}, mA[4][2] = {}, mB[4][2] = {}, rb[5][2][2] = {};
  auto srow = [&](const double* V, int64_t kk, bool v, double& s0, double& s1) {
    const double* row = V + (size_t)kk * GP;
    s0 = v ? row[m] : 0.0;
    s1 = v ? (m < 2 ? row[8 + m] : (m == 2 ? 1.0 : 0.0)) : 0.0;
  };
  auto moments = [&](const unsigned* H, const double* V, int64_t nk, double (&acc)[4][2]) {
    const int64_t ng = (nk + 3) / 4, g0 = gw * ng / GW, g1 = (gw + 1) * ng / GW;
    constexpr int U = 4;  // groups whose loads are in flight together
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
// src[g][e] = Σ of chunk g (of SUM_SPLIT) of the partial rows of element e, fixed order
__global__ void __launch_bounds__(1024) k_cov_sum(const double* __restrict__ p1, int n1, const double* __restrict__ p2,
                                                  int n2, double* __restrict__ src) {
  const int e = blockIdx.x * 32 + (threadIdx.x & 31), r = threadIdx.x >> 5, g = blockIdx.y;
  double s = 0.0;
  if (e < NPART) {
    const int b0 = n1 * g / SUM_SPLIT, b1 = n1 * (g + 1) / SUM_SPLIT;
#pragma unroll 4
    for (int b = b0 + r; b < b1; b += 32) s += p1[(size_t)b * NPART + e];
  } else if (e < NPART + NFIN) {
    const int b0 = n2 * g / SUM_SPLIT, b1 = n2 * (g + 1) / SUM_SPLIT;
#pragma unroll 4
    for (int b = b0 + r; b < b1; b += 32) s += p2[(size_t)b * NFIN + e - NPART];
  }
  __shared__ double red[32][33];
  red[r][threadIdx.x & 31] = s;
  __syncthreads();
  if (r == 0 && e < NPART + NFIN) {
    double t = 0.0;
    for (int i = 0; i < 32; i++) t += red[i][threadIdx.x];
    src[(size_t)g * (NPART + NFIN) + e] = t;
  }
}
__device__ __forceinline__ double cov_src(const double* __restrict__ src, int e) {
  double t = 0.0;
#pragma unroll
  for (int g = 0; g < SUM_SPLIT; g++) t += src[(size_t)g * (NPART + NFIN) + e];
  return t;
}

__global__ void k_cov_assemble(const double* __restrict__ src, const int32_t* __restrict__ toff,
                               const int32_t* __restrict__ tidx, const double* __restrict__ tcoef, int nout,
                               double* __restrict__ out, int count_idx, unsigned long long* __restrict__ count) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = toff[o]; t < toff[o + 1]; t++) s += tcoef[t] * cov_src(src, tidx[t]);
    out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)cov_src(src, count_idx);
}

// ======================================================================= host
struct CovLevel {
  int child = -1, rel = -1;
  std::vector<int> attrs;
  int64_t nk = 0;
  DevBuf V, colptrs, idxptrs;
  std::vector<DevBuf> idx;  // composed foreign-key chains to the features of deeper relations
};

struct FastCov : FastPaths {
  int NS = 0, nF = 0;
  std::vector<int> fattrs;
  CovLevel L, A, B;
  DevBuf zeros;  // one zero view row (absent levels)
  DevBuf zbuf;   // [work | bcount | pad] [HA] [HL], cleared every run
  size_t off_HA = 0, off_HL = 0, zbytes = 0;
  DevBuf brec, partials, finp, src, toff, tidx, tcoef;
  DevBuf scan;  // scan layout of the root (k_cov_layout), built at plan time
  int64_t nblk = 0;
  int bcap = 0, grid = 148, nout = 0, ib = IB;
  bool only_scalar = true;

  std::string describe() const override {
    char b[256];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"cov\", \"NS\": %d, \"nF\": %d, \"nL\": %zu, \"nA\": %zu, \"nB\": %zu, \"grid\": %d, "
                  "\"threads\": %d, \"stages\": %d, \"item\": %d}",
                  NS, nF, L.attrs.size(), A.attrs.size(), B.attrs.size(), grid, COV_W * 32, CovCfg<COV_W>::CF, 32 * ib);
    return b;
  }
  bool skip_generic_views() const override { return only_scalar; }
  int run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) override;
};

int cov_warps() { return COV_W; }  // (16 warps per CTA spilled at 128 registers; measured slower)

template <int W, int IBK>
cudaError_t launch_cov_w(int NS, const CovArgs& g, int grid, cudaStream_t st) {
  static bool attr[3] = {false, false, false};
  auto go = [&](auto kern) -> cudaError_t {
    constexpr int smem = CovCfg<W>::SMEM;
    if (!attr[NS]) {
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      attr[NS] = true;
    }
    kern<<<grid, W * 32, smem, st>>>(g);
    return cudaGetLastError();
  };
  if (NS == 0) return go(k_cov<0, W, IBK>);
  if (NS == 1) return go(k_cov<1, W, IBK>);
  return go(k_cov<2, W, IBK>);
}
cudaError_t launch_cov(int NS, const CovArgs& g, int grid, cudaStream_t st) {
  return g.ib == IB ? launch_cov_w<COV_W, IB>(NS, g, grid, st) : launch_cov_w<COV_W, 2>(NS, g, grid, st);
}

}  // namespace

int FastCov::run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool& scalar_done) {
  const Rel& R = c->rels[c->root];
  CUDA_TRY(cudaMemsetAsync(zbuf.p, 0, zbytes, st));
  {  // (b) dimension views of the featured PK leaves
    DimTables d{};
    CovLevel* lv[3] = {&L, &A, &B};
    int64_t tot = 0;
    for (int i = 0; i < 3; i++) {
      d.cols[i] = (const double* const*)lv[i]->colptrs.p;
      d.idx[i] = (const int32_t* const*)lv[i]->idxptrs.p;
      d.n[i] = (int)lv[i]->attrs.size();
      d.nk[i] = lv[i]->rel >= 0 ? lv[i]->nk : 0;
      d.V[i] = lv[i]->V.as<double>();
      tot += d.nk[i] * GP;
    }
    if (tot > 0) {
      k_cov_dims<<<(unsigned)std::min<int64_t>((tot / GP + 255) / 256, 148 * 16), 256, 0, st>>>(d);
      launches_add(1);
    }
  }
  CovArgs g{};
  g.nrows = R.nrows;
  g.nblk = nblk;
  g.scan = scan.as<unsigned char>();
  g.VL = L.V.as<double>();
  g.VA = NS >= 1 ? A.V.as<double>() : zeros.as<double>();
  char* z = zbuf.as<char>();
  g.work = reinterpret_cast<int*>(z);
  g.bcount = reinterpret_cast<int*>(z + 4);
  g.HA = reinterpret_cast<unsigned*>(z + off_HA);
  g.HL = reinterpret_cast<unsigned*>(z + off_HL);
  {
    const char* ab = std::getenv("LMFAO_COV_ABLATE");
    g.ablate = ab ? std::atoi(ab) : 0;
    const char* cd = std::getenv("LMFAO_COV_COLD");
    g.cold = cd ? std::atoi(cd) : COV_COLD;
  }
  g.brec = brec.as<double>();
  g.bcap = bcap;
  g.ib = ib;
  g.partials = partials.as<double>();
  scan_timer_begin(c, st);
  cudaError_t e = launch_cov(NS, g, grid, st);
  scan_timer_end(c, st);
  if (e) return e;
  launches_add(1);
  FinArgs f{};
  f.brec = brec.as<double>();
  f.bcount = g.bcount;
  f.bcap = bcap;
  f.VB = NS == 2 ? B.V.as<double>() : zeros.as<double>();
  f.HL = g.HL;
  f.VL = L.V.as<double>();
  f.nkL = L.nk;
  f.HA = g.HA;
  f.VA = g.VA;
  f.nkA = NS >= 1 ? A.nk : 0;
  f.partials = finp.as<double>();
  k_cov_fin<<<FIN_BLOCKS, 256, 8 * NFIN * 8, st>>>(f);
  k_cov_sum<<<dim3((NPART + NFIN + 31) / 32, SUM_SPLIT), 1024, 0, st>>>(partials.as<double>(), grid * cov_warps(), finp.as<double>(),
                                                      FIN_BLOCKS, src.as<double>());
  k_cov_assemble<<<(nout + 127) / 128 + 1, 128, 0, st>>>(src.as<double>(), toff.as<int32_t>(), tidx.as<int32_t>(),
                                                         tcoef.as<double>(), nout, c->scalar_out.as<double>(),
                                                         NPART + 18 * 16 + 10, c->scalar_count.as<unsigned long long>());
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
    if (l.colptrs.alloc(std::max<size_t>(cp.size(), 1) * sizeof(void*)) ||
        l.idxptrs.alloc(std::max<size_t>(ip.size(), 1) * sizeof(void*)))
      return nullptr;
    if (!cp.empty() &&
        (cudaMemcpyAsync(l.colptrs.p, cp.data(), cp.size() * sizeof(void*), cudaMemcpyHostToDevice, c->stream) ||
         cudaMemcpyAsync(l.idxptrs.p, ip.data(), ip.size() * sizeof(void*), cudaMemcpyHostToDevice, c->stream)))
      return nullptr;
  }
  const int64_t nkA = fc->NS >= 1 ? fc->A.nk : 0;
  fc->off_HA = 16;
  fc->off_HL = (fc->off_HA + (size_t)(nkA + 1) * 4 + 15) / 16 * 16;  // + the padding rows' key
  fc->zbytes = fc->off_HL + (size_t)(fc->L.nk + 1) * 4;
  if (fc->zbuf.alloc(fc->zbytes)) return nullptr;
  tr.mark("terms + buffers", c->stream);
  fc->nblk = (R.nrows + 31) / 32;
  // work items as k_cov defines them: ib-block items, then 2-block items for the last ~10 %;
  // ib = IB unless the root has fewer than 2 such items per warp; then 2 (C1, 625 blocks:
  // 0.057 ms in 24-block items, 0.045 in 16, 0.030 in 2)
  fc->ib = fc->nblk >= (int64_t)fc->grid * COV_W * 2 * IB ? IB : 2;
  const int64_t nbig = fc->nblk * (100 - COV_TAIL_PCT) / 100 / fc->ib;
  const int64_t nitems = nbig + (fc->nblk - nbig * fc->ib + 1) / 2;
  // level-B records: one per (B run, item) pair <= B runs + items
  fc->bcap = (int)std::min<int64_t>((fc->NS == 2 ? fc->B.nk : 0) + nitems + 64, INT32_MAX / BRW);
  if (fc->brec.alloc((size_t)fc->bcap * BRW * 8)) return nullptr;
  if (fc->partials.alloc((size_t)fc->grid * 16 * NPART * 8)) return nullptr;  // one partial per warp
  if (fc->finp.alloc((size_t)FIN_BLOCKS * NFIN * 8)) return nullptr;
  if (fc->src.alloc((size_t)SUM_SPLIT * (NPART + NFIN) * 8)) return nullptr;
  {  // scan layout of the root: x in DMMA lane order + dense keys, one 2432-byte block per 32 rows
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
      if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess) return nullptr;
    }
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
  return fc.release();
}

}  // namespace lmfao
