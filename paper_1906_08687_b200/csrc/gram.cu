// gram.cu — the covariance-batch path: fused root scan (c) with FP64 DMMA Gram
// tiles (d) and run-level factorisation (the MOO intermediate aggregates /
// running sums of P:1186-1214), plus the dimension-side finishing of the
// "each aggregate to its own root" blocks.
//
// Applies when every no-group-by product has at most two identity factors
// (after folding constants), over the root's features and the features of
// primary-key dimensions that are leaves of the root.  With u = [1, x, s_1..s_R]
// (x: root features; s_r: features of dimension r looked up by the root's
// foreign key) every aggregate is an entry of G = Σ_f u(f) u(f)^T.
//
// The root is sorted by its foreign keys in increasing domain size:
// levels B (shallowest featured), A, L (deepest featured).  Blocks of G:
//   x⊗x, x⊗s_L, x⊗1          per row: 4-row DMMA m8n8k4 groups, A = x, B = [x, s_L, 1]
//   [x, s_L, 1]⊗s_A          per level-A run: run sums ("records") ⊗ s_A, DMMA over 4 records
//   s_B⊗s_A                  per level-A run: n·s_B ⊗ s_A
//   [x, s_L, 1]⊗s_B          per level-B run (sum of its level-A records) ⊗ s_B
//   1⊗s_r, s_r⊗s_r, count    dimension side: Σ_k H_r[k] s_r(k), Σ_k H_r[k] s_r(k) s_r(k)^T
// where H_r[k] counts root rows with key k (run lengths).  Runs split at warp
// boundaries are exact (every update is linear in the run sums).
//
// DMMA fragment layout (PTX mma.m8n8k4 .f64): lane = 4*m + k; A[m][k] = a0,
// B[k][n=m] = b0, C[m][2k+i] = c_i.  Here k indexes the 4 rows (or 4 records)
// of a group and m the feature: lane (m, k) holds feature m of row k.
#include <set>

#include "ctx.h"

namespace lmfao {

struct GramArgs {
  int64_t nrows;
  int nF, nL, nA, nB;
  const double* x[8];
  const int32_t* kL;
  const double* VL;
  int WL;
  const int32_t* kA;
  const double* VA;
  int WA;
  const int32_t* kB;
  const double* VB;
  int WB;
  unsigned* HL;
  unsigned* HA;
  unsigned* HB;
  double* partials;
  int WG;             // gathered row stride in smem (doubles, even): [s_L | pad | 1 | 0]
  int cn;             // B / record column holding the constant 1 (the count)
  int* work;          // dynamic work-item counter (zeroed before each launch)
  int smem_per_warp;  // bytes
};

constexpr int CH = 32;   // rows per warp chunk (one 32-row block)
constexpr int GRAM_THREADS = 384;  // 12 warps per CTA, one CTA per SM
constexpr int ITEM = 512; // rows per dynamically scheduled work item (multiple of CH)
constexpr int HCACHE_BITS = 6, HCACHE = 1 << HCACHE_BITS;
constexpr int XST = 36;  // smem column stride (doubles): 16-B aligned, conflict-free DMMA-layout reads

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr unsigned FULL = 0xffffffffu;

template <int NB, int NS, int NTS>
struct GramTiles {
  static constexpr int TA = NS >= 1 ? NB * NTS : 0;
  static constexpr int T12 = NS == 2 ? NTS * NTS : 0;
  static constexpr int TB = NS == 2 ? NB * NTS : 0;
  static constexpr int TOT = NB + TA + T12 + TB;
};

template <int NB, int NS, int NTS>
__global__ void __launch_bounds__(GRAM_THREADS, 1) k_gram(GramArgs g) {
  using T = GramTiles<NB, NS, NTS>;
  constexpr int TOT = T::TOT;
  const int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2;
  const int wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int cn = g.cn;
  const int tn = cn >> 3, mn = cn & 7;
  const int WG = g.WG;
  const int64_t N = g.nrows;
  const int nitems = (int)((N + ITEM - 1) / ITEM);

  double acc[TOT][2];
#pragma unroll
  for (int t = 0; t < TOT; t++) acc[t][0] = acc[t][1] = 0.0;
  // per-lane (row phase k) prefix sums of the B columns over the current item, and the
  // prefix at the start of the open level-A run: a run's record = P(end) - P(start)
  double P[NB], Ps[NB], sumB[NB];
#pragma unroll
  for (int t = 0; t < NB; t++) P[t] = Ps[t] = sumB[t] = 0.0;
  double preA[NTS], preAB[NTS], preB[NTS];
#pragma unroll
  for (int t = 0; t < NTS; t++) preA[t] = preAB[t] = preB[t] = 0.0;
  int npA = 0, npB = 0;
  bool runA_ne = false, runB_ne = false;
  int curA = -1, curB = -1;
  int prevL = -1, prevA = -1, prevB = -1;
  int runL_start = 0;  // row index within the item

  // ---- per-warp shared memory
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* wp = smem_raw + (size_t)wib * g.smem_per_warp;
  double* xs = reinterpret_cast<double*>(wp);  // [3][8][XST]
  wp += 3 * 8 * XST * 8;
  double* gsb = reinterpret_cast<double*>(wp);  // [2][CH][WG]
  wp += 2 * CH * WG * 8;
  double* recA = reinterpret_cast<double*>(wp);  // [4][NB][32]
  wp += 4 * NB * 32 * 8;
  double* recB = reinterpret_cast<double*>(wp);  // [4][NB][32]
  wp += 4 * NB * 32 * 8;
  unsigned long long* hcache = reinterpret_cast<unsigned long long*>(wp);
  wp += HCACHE * 8;
  uint64_t* bars = reinterpret_cast<uint64_t*>(wp);
  wp += 4 * 8;
  int32_t* rkey = reinterpret_cast<int32_t*>(wp);  // [0..3] A keys, [8..11] B keys
  wp += 16 * 4;
  int32_t* ks = reinterpret_cast<int32_t*>(wp);  // [3][3][CH]
  wp += 3 * 3 * CH * 4;
  double* cst = reinterpret_cast<double*>(wp);  // 0.0, 1.0
  for (int i = lane; i < HCACHE; i += 32) hcache[i] = 0xFFFFFFFF00000000ull;
  if (lane == 0) {
    cst[0] = 0.0;
    cst[1] = 1.0;
  }
  const int gch = (g.nL + 1) / 2;
  for (int i = lane; i < 2 * CH; i += 32)
    for (int c2 = 2 * gch; c2 < WG; c2++) gsb[(size_t)i * WG + c2] = (c2 == cn - g.nF) ? 1.0 : 0.0;
  const uint32_t cst0 = smem_u32(cst);
  const int nkeycols = 1 + (NS >= 1) + (NS == 2);
  if (lane == 0) {
    for (int s = 0; s < 3; s++) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // per-lane operand addressing (relative to a stage): A = x column m (or 0); B col 8t+m
  const bool isx0 = m < g.nF;
  uint32_t boff[NB], bstep[NB];  // byte offset within the gathered buffer or -1 markers
  int bkind[NB];
#pragma unroll
  for (int t = 0; t < NB; t++) {
    const int col = 8 * t + m;
    const int gc = col - g.nF;
    bkind[t] = col < g.nF ? 0 : (gc < WG ? 1 : 2);
    boff[t] = bkind[t] == 1 ? (uint32_t)((k * WG + gc) * 8) : 0u;
    bstep[t] = bkind[t] == 0 ? 32u : (bkind[t] == 1 ? (uint32_t)(4 * WG * 8) : 0u);
  }

  // ---------------------------------------------------------------- H_L
  auto hl_flush_lanes = [&](bool fl, int key, unsigned len) {
    if (!__any_sync(FULL, fl)) return;
    const unsigned peers = __match_any_sync(FULL, fl ? key : -1 - lane);
    unsigned sum = len;
    if (fl && __popc(peers) > 1) {
      unsigned s2 = 0, pm = peers;
      while (pm) {
        const int src = __ffs(pm) - 1;
        pm &= pm - 1;
        s2 += __shfl_sync(peers, len, src);
      }
      sum = s2;
    }
    const bool leader = fl && (__ffs(peers) - 1) == lane;
    const unsigned slot = leader ? (((unsigned)key * 2654435761u) >> (32 - HCACHE_BITS)) : 0xFFFFFFFFu - lane;
    const unsigned spe = __match_any_sync(FULL, slot);
    if (leader) {
      if (__popc(spe) == 1) {
        const unsigned long long e = hcache[slot];
        if ((int)(e >> 32) == key) {
          hcache[slot] = e + sum;
        } else {
          if ((unsigned)(e >> 32) != 0xFFFFFFFFu) atomicAdd(&g.HL[(unsigned)(e >> 32)], (unsigned)e);
          hcache[slot] = ((unsigned long long)(unsigned)key << 32) | sum;
        }
      } else {
        atomicAdd(&g.HL[key], sum);
      }
    }
    __syncwarp();
  };

  // ---------------------------------------------------------------- records
  auto process_A = [&]() {
    __syncwarp();
    const bool rv = k < npA;
    double a[NB];
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const double* r = recA + ((size_t)k * NB + t) * 32 + 4 * m;
      a[t] = rv ? (r[0] + r[1]) + (r[2] + r[3]) : 0.0;
    }
    double nk_own = 0.0;
#pragma unroll
    for (int t = 0; t < NB; t++)
      if (t == tn) nk_own = a[t];
    const double nk = __shfl_sync(FULL, nk_own, mn * 4 + k);
#pragma unroll
    for (int t = 0; t < NB; t++)
#pragma unroll
      for (int t2 = 0; t2 < NTS; t2++) dmma(acc[NB + t * NTS + t2], a[t], preA[t2]);
    if constexpr (NS == 2) {
#pragma unroll
      for (int t1 = 0; t1 < NTS; t1++)
#pragma unroll
        for (int t2 = 0; t2 < NTS; t2++) dmma(acc[NB + T::TA + t1 * NTS + t2], nk * preAB[t1], preA[t2]);
    }
    if (rv && m == mn) atomicAdd(&g.HA[rkey[k]], (unsigned)nk);
#pragma unroll
    for (int t = 0; t < NTS; t++) preA[t] = preAB[t] = 0.0;
    npA = 0;
    __syncwarp();
  };
  auto process_B = [&]() {
    __syncwarp();
    const bool rv = k < npB;
    double a[NB];
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const double* r = recB + ((size_t)k * NB + t) * 32 + 4 * m;
      a[t] = rv ? (r[0] + r[1]) + (r[2] + r[3]) : 0.0;
    }
    double nk_own = 0.0;
#pragma unroll
    for (int t = 0; t < NB; t++)
      if (t == tn) nk_own = a[t];
#pragma unroll
    for (int t = 0; t < NB; t++)
#pragma unroll
      for (int t1 = 0; t1 < NTS; t1++) dmma(acc[NB + T::TA + T::T12 + t * NTS + t1], a[t], preB[t1]);
    if (rv && m == mn) atomicAdd(&g.HB[rkey[8 + k]], (unsigned)nk_own);
#pragma unroll
    for (int t = 0; t < NTS; t++) preB[t] = 0.0;
    npB = 0;
    __syncwarp();
  };
  auto push_B = [&](int keyB) {  // record = sumB (per lane, unreduced)
#pragma unroll
    for (int t = 0; t < NB; t++) recB[((size_t)npB * NB + t) * 32 + lane] = sumB[t];
    if (lane == 0) rkey[8 + npB] = keyB;
    if (k == npB) {
      const double* row = g.VB + (unsigned)keyB * (unsigned)g.WB;
      preB[0] = m < g.nB ? row[m] : 0.0;
      if constexpr (NTS == 2) preB[1] = 8 + m < g.nB ? row[8 + m] : 0.0;
    }
    if (++npB == 4) process_B();
  };
  auto push_A = [&](const double* rec, int keyA, int keyB) {
#pragma unroll
    for (int t = 0; t < NB; t++) recA[((size_t)npA * NB + t) * 32 + lane] = rec[t];
    if (lane == 0) rkey[npA] = keyA;
    if (k == npA) {
      const double* row = g.VA + (unsigned)keyA * (unsigned)g.WA;
      preA[0] = m < g.nA ? row[m] : 0.0;
      if constexpr (NTS == 2) preA[1] = 8 + m < g.nA ? row[8 + m] : 0.0;
      if constexpr (NS == 2) {
        const double* rowb = g.VB + (unsigned)keyB * (unsigned)g.WB;
        preAB[0] = m < g.nB ? rowb[m] : 0.0;
        if constexpr (NTS == 2) preAB[1] = 8 + m < g.nB ? rowb[8 + m] : 0.0;
      }
    }
    if constexpr (NS == 2) {
#pragma unroll
      for (int t = 0; t < NB; t++) sumB[t] += rec[t];
      runB_ne = true;
    }
    if (++npA == 4) process_A();
  };
  // close the open runs of an item ending at row-within-item `end`
  auto flush_item = [&](int end) {
    if constexpr (NS >= 1) {
      if (runA_ne) {
        double rec[NB];
#pragma unroll
        for (int t = 0; t < NB; t++) rec[t] = P[t] - Ps[t];
        push_A(rec, curA, curB);
      }
      if constexpr (NS == 2) {
        if (runB_ne) push_B(curB);
      }
    }
    hl_flush_lanes(lane == 0 && end > runL_start && prevL >= 0, prevL, (unsigned)(end - runL_start));
#pragma unroll
    for (int t = 0; t < NB; t++) P[t] = Ps[t] = sumB[t] = 0.0;
    runA_ne = runB_ne = false;
    prevL = prevA = prevB = -1;
  };

  // ---------------------------------------------------------------- work items, staging
  int ring[4] = {0, 0, 0, 0};
  int nring = 0;
  auto grab = [&]() {
    int it = 0;
    if (lane == 0) it = atomicAdd(g.work, 1);
    it = __shfl_sync(FULL, it, 0);
#pragma unroll
    for (int i = 0; i < 4; i++)
      if ((nring & 3) == i) ring[i] = it;
    nring++;
  };
  auto ring_at = [&](int slot) {
    int it = ring[0];
#pragma unroll
    for (int i = 1; i < 4; i++)
      if ((slot & 3) == i) it = ring[i];
    return it;
  };
  // cursor over (item, chunk) with a chunk sequence number for stage selection
  int tm_slot = 0, tm_c = 0, tm_seq = 0, tm_item;   // TMA cursor (2 ahead)
  int ga_slot = 0, ga_c = 0, ga_seq = 0, ga_item;   // gather cursor (1 ahead)
  int ct_c = 0, ct_seq = 0, ct_slot = 0, ct_item;   // compute cursor
  auto item_rows = [&](int it) {
    const int64_t r = (int64_t)it * ITEM;
    return (int)(N - r < ITEM ? N - r : ITEM);
  };
  auto adv = [&](int& slot, int& c, int& seq, int& item, bool may_grab) {
    seq++;
    if ((c + 1) * CH < item_rows(item)) {
      c++;
    } else {
      c = 0;
      slot++;
      if (may_grab && slot >= nring) grab();
      item = ring_at(slot);
    }
  };
  const double* xcol = g.x[0];
#pragma unroll
  for (int i = 1; i < 8; i++)
    if (lane == i) xcol = g.x[i];
  const int32_t* kcl = lane == 8 ? g.kL : (lane == 9 ? g.kA : g.kB);
  auto issue_tma = [&](int item, int c, int seq) {
    const int s = seq % 3;
    const int64_t r = (int64_t)item * ITEM + c * CH;
    const int n = min(CH, item_rows(item) - c * CH);
    const uint32_t bx = (uint32_t)((n * 8 + 15) & ~15), bk = (uint32_t)((n * 4 + 15) & ~15);
    if (lane == 0) {
      fence_proxy_async();
      mbar_expect_tx(&bars[s], bx * g.nF + bk * nkeycols);
    }
    __syncwarp();
    if (lane < g.nF) tma_load_1d(xs + ((size_t)s * 8 + lane) * XST, xcol + r, bx, &bars[s]);
    else if (lane >= 8 && lane < 8 + nkeycols) tma_load_1d(ks + ((size_t)s * 3 + (lane - 8)) * CH, kcl + r, bk, &bars[s]);
  };
  auto wait_tma = [&](int seq) { mbar_wait(&bars[seq % 3], (uint32_t)((seq / 3) & 1)); };
  const int q32 = gch ? 32 / gch : 0, r32 = gch ? 32 % gch : 0;
  const int rr0 = gch ? lane / gch : 0, pc0 = gch ? lane % gch : 0;
  const unsigned WL = (unsigned)g.WL;
  auto issue_gather = [&](int item, int c, int seq) {
    const int s = seq % 3;
    const int n = min(CH, item_rows(item) - c * CH);
    double* dst = gsb + (size_t)(seq & 1) * CH * WG;
    const int32_t* kk = ks + (size_t)s * 3 * CH;
    int rr = rr0, pc = pc0;
    while (rr < n) {
      cp_async16(dst + rr * WG + 2 * pc, g.VL + ((unsigned)kk[rr] * WL + 2 * pc));
      rr += q32;
      pc += r32;
      if (pc >= gch) {
        pc -= gch;
        rr++;
      }
    }
    cp_async_commit();
  };

  grab();
  tm_item = ga_item = ct_item = ring_at(0);
  if (ct_item < nitems) {
    issue_tma(tm_item, tm_c, tm_seq);
    adv(tm_slot, tm_c, tm_seq, tm_item, true);
    if (tm_item < nitems) {
      issue_tma(tm_item, tm_c, tm_seq);
      adv(tm_slot, tm_c, tm_seq, tm_item, true);
    }
    wait_tma(ga_seq);
    if (gch) issue_gather(ga_item, ga_c, ga_seq);
    adv(ga_slot, ga_c, ga_seq, ga_item, false);
  }
  int prev_item_rows = -1;
  while (ct_item < nitems) {
    const bool more = ga_item < nitems;
    if (more) {
      wait_tma(ga_seq);
      if (gch) issue_gather(ga_item, ga_c, ga_seq);
    }
    if (tm_item < nitems) issue_tma(tm_item, tm_c, tm_seq);
    if (more) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncwarp();
    const int irows = item_rows(ct_item);
    if (ct_c == 0) {
      if (prev_item_rows >= 0) flush_item(prev_item_rows);
      runL_start = 0;
      prev_item_rows = irows;
    }
    const int ro = ct_c * CH;  // row offset within the item
    const int nval = min(CH, irows - ro);
    const int s = ct_seq % 3;
    const double* xsc = xs + (size_t)s * 8 * XST;
    const int32_t* ksc = ks + (size_t)s * 3 * CH;
    double* gsc = gsb + (size_t)(ct_seq & 1) * CH * WG;
    // -- row lanes: keys and boundary masks of the 32-row chunk
    const bool vr = lane < nval;
    const int kl = vr ? ksc[lane] : -1;
    const int ka = (NS >= 1 && vr) ? ksc[CH + lane] : -1;
    const int kb = (NS == 2 && vr) ? ksc[2 * CH + lane] : -1;
    int pl = __shfl_up_sync(FULL, kl, 1), pa = __shfl_up_sync(FULL, ka, 1), pb = __shfl_up_sync(FULL, kb, 1);
    if (lane == 0) {
      pl = prevL;
      pa = prevA;
      pb = prevB;
    }
    const bool dB = NS == 2 && vr && kb != pb;
    const bool dA = NS >= 1 && vr && (dB || ka != pa);
    const bool dL = vr && (dA || kl != pl);
    const unsigned mB = __ballot_sync(FULL, dB);
    const unsigned mA = __ballot_sync(FULL, dA);
    const unsigned mL = __ballot_sync(FULL, dL);
    prevL = __shfl_sync(FULL, kl, nval - 1);
    prevA = __shfl_sync(FULL, ka, nval - 1);
    prevB = __shfl_sync(FULL, kb, nval - 1);
    {  // H_L: lane i with a boundary flushes the run ending at row i-1 (key pl)
      const unsigned before = mL & ((1u << lane) - 1u);
      const int st = before ? ro + (31 - __clz(before)) : runL_start;
      const int len = ro + lane - st;
      hl_flush_lanes(dL && len > 0 && pl >= 0, pl, (unsigned)len);
      if (mL) runL_start = ro + (31 - __clz(mL));
    }
    if (nval < CH) {  // the table's final partial chunk: zero its invalid rows in smem
      if (lane >= nval) {
        for (int f = 0; f < g.nF; f++) const_cast<double*>(xsc)[f * XST + lane] = 0.0;
        for (int c2 = 0; c2 < WG; c2++) gsc[lane * WG + c2] = 0.0;
      }
      __syncwarp();
    }
    uint32_t xaddr = isx0 ? smem_u32(xsc + m * XST + k) : cst0;
    const uint32_t xstep = isx0 ? 32u : 0u;
    const uint32_t gbase = smem_u32(gsc);
    uint32_t baddr[NB];
#pragma unroll
    for (int t = 0; t < NB; t++) baddr[t] = bkind[t] == 0 ? xaddr : (bkind[t] == 1 ? gbase + boff[t] : cst0);
    const int ngr = (nval + 3) >> 2;
#pragma unroll 1
    for (int j = 0; j < ngr; j++) {
      const double xa = lds64(xaddr);
      xaddr += xstep;
      double b[NB];
#pragma unroll
      for (int t = 0; t < NB; t++) {
        b[t] = lds64(baddr[t]);
        baddr[t] += bstep[t];
      }
#pragma unroll
      for (int t = 0; t < NB; t++) dmma(acc[t], xa, b[t]);
      if constexpr (NS >= 1) {
        const unsigned nib = (mA >> (4 * j)) & 0xFu;
        if (nib) {
          unsigned bits = nib;
          while (bits) {
            const int p = __ffs(bits) - 1;
            bits &= bits - 1;
            double rec[NB];
#pragma unroll
            for (int t = 0; t < NB; t++) {
              const double pb2 = P[t] + (k < p ? b[t] : 0.0);  // prefix just before row p
              rec[t] = pb2 - Ps[t];
              Ps[t] = pb2;
            }
            if (runA_ne) push_A(rec, curA, curB);
            runA_ne = true;
            if constexpr (NS == 2) {
              if ((mB >> (4 * j + p)) & 1u) {
                if (runB_ne) push_B(curB);
#pragma unroll
                for (int t = 0; t < NB; t++) sumB[t] = 0.0;
                runB_ne = false;
              }
            }
            curA = __shfl_sync(FULL, ka, 4 * j + p);
            curB = __shfl_sync(FULL, kb, 4 * j + p);
          }
        }
#pragma unroll
        for (int t = 0; t < NB; t++) P[t] += b[t];
      }
    }
    if (nval < CH) {  // restore the gathered count column of the zero-filled rows
      if (lane >= nval)
        for (int c2 = 2 * gch; c2 < WG; c2++) gsc[lane * WG + c2] = (c2 == cn - g.nF) ? 1.0 : 0.0;
    }
    __syncwarp();
    adv(ct_slot, ct_c, ct_seq, ct_item, false);
    if (more) adv(ga_slot, ga_c, ga_seq, ga_item, false);
    if (tm_item < nitems) adv(tm_slot, tm_c, tm_seq, tm_item, true);
  }
  if (prev_item_rows >= 0) flush_item(prev_item_rows);
  if constexpr (NS == 2) {
    if (npB > 0) process_B();
  }
  if constexpr (NS >= 1) {
    if (npA > 0) process_A();
  }
  __syncwarp();
  for (int i = lane; i < HCACHE; i += 32) {
    const unsigned long long e = hcache[i];
    if ((unsigned)(e >> 32) != 0xFFFFFFFFu) atomicAdd(&g.HL[(unsigned)(e >> 32)], (unsigned)e);
  }

  // deterministic CTA reduction (warps in order), then one partial per CTA
  __shared__ double red[TOT * 64];
  for (int i = threadIdx.x; i < TOT * 64; i += blockDim.x) red[i] = 0.0;
  __syncthreads();
  for (int w = 0; w < nwb; w++) {
    if (wib == w) {
#pragma unroll
      for (int t = 0; t < TOT; t++) {
        red[t * 64 + m * 8 + 2 * k] += acc[t][0];
        red[t * 64 + m * 8 + 2 * k + 1] += acc[t][1];
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < TOT * 64; i += blockDim.x) g.partials[(int64_t)blockIdx.x * TOT * 64 + i] = red[i];
}


__global__ void k_sum_partials(const double* __restrict__ partials, int nparts, int n, double* __restrict__ out) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; b++) s += partials[(int64_t)b * n + e];
    out[e] = s;
  }
}

// Dimension-side moments: out = [Σ H, Σ H s_f (n), Σ H s_f s_g (n*n)] per block.
__global__ void k_moments(const unsigned* __restrict__ H, const double* __restrict__ V, int64_t nk, int W, int n,
                          double* __restrict__ partials) {
  const int nout = 1 + n + n * n;
  const int64_t per = (nk + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = blockIdx.x * per, k1 = min(nk, k0 + per);
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    int f = -1, g2 = -1;
    if (o >= 1 && o <= n) f = o - 1;
    if (o > n) {
      f = (o - 1 - n) / n;
      g2 = (o - 1 - n) % n;
    }
    double s = 0.0;
    for (int64_t kk = k0; kk < k1; kk++) {
      double h = (double)H[kk];
      if (h == 0.0) continue;
      double v = h;
      if (f >= 0) v *= V[kk * W + f];
      if (g2 >= 0) v *= V[kk * W + g2];
      s += v;
    }
    partials[(int64_t)blockIdx.x * nout + o] = s;
  }
}

// Dimension feature table V[k][f] = col_f[k] (primary-key leaf: row k has dense key k).
__global__ void k_dim_table(const double* const* __restrict__ cols, int n, int64_t nk, int W, double* __restrict__ V) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk * W; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t kk = i / W;
    int f = (int)(i % W);
    V[i] = f < n ? cols[f][kk] : 0.0;
  }
}

// out[o] = Σ_terms coef * src[idx]; count = (u64) src[count_idx]
__global__ void k_assemble(const double* __restrict__ src, const int32_t* __restrict__ toff,
                           const int32_t* __restrict__ tidx, const double* __restrict__ tcoef, int nout,
                           double* __restrict__ out, int count_idx, unsigned long long* __restrict__ count) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = toff[o]; t < toff[o + 1]; t++) s += tcoef[t] * src[tidx[t]];
    out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)src[count_idx];
}

// ======================================================================= host
namespace {

struct Level {
  int child = -1;        // index into root's children
  int rel = -1;
  std::vector<int> attrs;  // featured attributes (ids), in feature order
  int64_t nk = 0;
  int W = 0;
  DevBuf V, H, colptrs;
  int moff = -1;  // offset of its moments in src
  int nmom = 0;
  DevBuf mom_partials;
};

struct FastGram : FastPaths {
  int NB = 1, NS = 0, NTS = 1, TOT = 0;
  int nF = 0;
  std::vector<int> fattrs;  // fact feature attr ids
  Level L, A, B;
  int grid = 148, threads = 256;
  int smem_per_warp = 0;
  int cn = 0, WG = 2;
  DevBuf partials, src, toff, tidx, tcoef, work;
  int nsrc = 0, count_idx = 0, nout = 0;
  int mom_blocks = 148 * 2;

  std::string describe() const override {
    char b[256];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"gram\", \"NB\": %d, \"NS\": %d, \"NTS\": %d, \"tiles\": %d, \"nF\": %d, \"nL\": %zu, "
                  "\"nA\": %zu, \"nB\": %zu, \"grid\": %d, \"threads\": %d}",
                  NB, NS, NTS, TOT, nF, L.attrs.size(), A.attrs.size(), B.attrs.size(), grid, threads);
    return b;
  }
  bool only_scalar = true;  // no group-by queries in the batch: generic views are not needed
  bool skip_generic_views() const override { return only_scalar; }
  int run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) override;
};

int tiles_for(int nb, int ns, int nts) {
  int ta = ns >= 1 ? nb * nts : 0, t12 = ns == 2 ? nts * nts : 0, tb = ns == 2 ? nb * nts : 0;
  return nb + ta + t12 + tb;
}

template <int NB, int NS, int NTS>
cudaError_t launch_gram_t(const GramArgs& g, int grid, int threads, cudaStream_t st) {
  size_t smem = (size_t)g.smem_per_warp * (threads / 32);
  static size_t set = 0;
  if (smem > set) {
    CUDA_TRY(cudaFuncSetAttribute(k_gram<NB, NS, NTS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set = smem;
  }
  k_gram<NB, NS, NTS><<<grid, threads, smem, st>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_gram(int NB, int NS, int NTS, const GramArgs& g, int grid, int threads, cudaStream_t st) {
#define GRAM_CASE(nb, ns, nts) \
  if (NB == nb && NS == ns && NTS == nts) return launch_gram_t<nb, ns, nts>(g, grid, threads, st);
  GRAM_CASE(1, 0, 1) GRAM_CASE(2, 0, 1) GRAM_CASE(3, 0, 1)
  GRAM_CASE(1, 1, 1) GRAM_CASE(2, 1, 1) GRAM_CASE(3, 1, 1)
  GRAM_CASE(1, 1, 2) GRAM_CASE(2, 1, 2) GRAM_CASE(3, 1, 2)
  GRAM_CASE(1, 2, 1) GRAM_CASE(2, 2, 1) GRAM_CASE(3, 2, 1)
  GRAM_CASE(1, 2, 2) GRAM_CASE(2, 2, 2) GRAM_CASE(3, 2, 2)
#undef GRAM_CASE
  return cudaErrorInvalidValue;
}

}  // namespace

int FastGram::run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) {
  const Rel& R = c->rels[c->root];
  // (b) dimension feature tables (PK leaves: a copy into row-major [nk x W])
  Level* lv[3] = {&L, &A, &B};
  int nlev = 1 + (NS >= 1) + (NS == 2);
  for (int i = 0; i < nlev; i++) {
    Level& l = *lv[i];
    if (l.nk > 0) {
      k_dim_table<<<(unsigned)std::min<int64_t>((l.nk * l.W + 255) / 256, 148 * 8), 256, 0, st>>>(
          (const double* const*)l.colptrs.p, (int)l.attrs.size(), l.nk, l.W, l.V.as<double>());
      launches_add(1);
    }
    cudaError_t e = cudaMemsetAsync(l.H.p, 0, l.H.bytes, st);
    if (e) return e;
  }
  GramArgs g{};
  g.nrows = R.nrows;
  g.nF = nF;
  for (int i = 0; i < nF; i++) g.x[i] = (const double*)R.cols[R.find_attr(fattrs[i])].buf.p;
  for (int i = nF; i < 8; i++) g.x[i] = g.x[0];
  g.nL = (int)L.attrs.size();
  g.kL = R.fk_dense[L.child].as<int32_t>();
  g.VL = L.V.as<double>();
  g.WL = L.W;
  g.HL = L.H.as<unsigned>();
  if (NS >= 1) {
    g.nA = (int)A.attrs.size();
    g.kA = R.fk_dense[A.child].as<int32_t>();
    g.VA = A.V.as<double>();
    g.WA = A.W;
    g.HA = A.H.as<unsigned>();
  }
  if (NS == 2) {
    g.nB = (int)B.attrs.size();
    g.kB = R.fk_dense[B.child].as<int32_t>();
    g.VB = B.V.as<double>();
    g.WB = B.W;
    g.HB = B.H.as<unsigned>();
  }
  g.partials = partials.as<double>();
  g.WG = WG;
  g.cn = cn;
  g.smem_per_warp = smem_per_warp;
  g.work = work.as<int>();
  {
    cudaError_t e0 = cudaMemsetAsync(work.p, 0, 4, st);
    if (e0) return e0;
  }
  scan_timer_begin(c, st);
  cudaError_t e = launch_gram(NB, NS, NTS, g, grid, threads, st);
  scan_timer_end(c, st);
  if (e) return e;
  launches_add(1);
  // tile sums -> src[0 : TOT*64]
  k_sum_partials<<<(TOT * 64 + 127) / 128, 128, 0, st>>>(partials.as<double>(), grid, TOT * 64, src.as<double>());
  launches_add(1);
  for (int i = 0; i < nlev; i++) {
    Level& l = *lv[i];
    int n = (int)l.attrs.size();
    k_moments<<<mom_blocks, 128, 0, st>>>(l.H.as<unsigned>(), l.V.as<double>(), l.nk, l.W, n,
                                          l.mom_partials.as<double>());
    k_sum_partials<<<(l.nmom + 127) / 128, 128, 0, st>>>(l.mom_partials.as<double>(), mom_blocks, l.nmom,
                                                         src.as<double>() + l.moff);
    launches_add(2);
  }
  k_assemble<<<(nout + 127) / 128 + 1, 128, 0, st>>>(src.as<double>(), toff.as<int32_t>(), tidx.as<int32_t>(),
                                                      tcoef.as<double>(), nout, c->scalar_out.as<double>(), count_idx,
                                                      c->scalar_count.as<unsigned long long>());
  launches_add(1);
  scalar_done = true;
  return cudaGetLastError();
}

// Planner hook: recognise the Gram shape, else nullptr (generic path).
FastPaths* plan_gram(lmfao_ctx* c) {
  if (c->scalar_queries.empty()) return nullptr;
  const Rel& R = c->rels[c->root];
  if (R.children.empty()) return nullptr;
  for (int ch : R.children) {
    const Rel& D = c->rels[ch];
    if (!D.children.empty() || !D.unique_key) return nullptr;
  }
  // collect products: (coef, feature a, feature b); feature = attr id or -1 for "1"
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
        for (int a : fa) {
          feats.insert(a);
        }
        while (fa.size() < 2) fa.insert(fa.begin(), -1);
        ts.push_back(Term{coef, fa[0], fa[1]});
      }
      outs.push_back(ts);
    }
  }
  auto* fg = new FastGram();
  fg->only_scalar = c->groups.empty();
  std::unique_ptr<FastGram> hold(fg);
  // features per level (root children in sort order)
  std::vector<std::vector<int>> lf(R.children.size());
  for (int a : feats) {
    int o = c->owner[a];
    if (o == c->root) {
      fg->fattrs.push_back(a);
    } else {
      bool found = false;
      for (size_t j = 0; j < R.children.size(); j++)
        if (R.children[j] == o) {
          lf[j].push_back(a);
          found = true;
        }
      if (!found) return nullptr;
      if (c->attrs[a].dt != LMFAO_FP64) return nullptr;  // v1: dim features are fp64 columns
    }
  }
  for (int a : fg->fattrs)
    if (c->attrs[a].dt != LMFAO_FP64) return nullptr;
  fg->nF = (int)fg->fattrs.size();
  if (fg->nF > 8) return nullptr;
  std::vector<int> featured;  // children indices in sort order with features
  for (int j : c->levels)
    if (!lf[j].empty()) featured.push_back(j);
  if (featured.empty() || featured.size() > 3) return nullptr;
  auto setup_level = [&](Level& l, int j) {
    l.child = j;
    l.rel = R.children[j];
    l.attrs = lf[j];
    l.nk = c->rels[l.rel].nkeys;
    l.W = ((int)l.attrs.size() + 3) / 4 * 4;
  };
  setup_level(fg->L, featured.back());
  fg->NS = (int)featured.size() - 1;
  if (fg->NS >= 1) setup_level(fg->A, featured[featured.size() - 2]);
  if (fg->NS == 2) setup_level(fg->B, featured[0]);
  int nL = (int)fg->L.attrs.size();
  const int nLe = (nL + 1) / 2 * 2;  // s_L columns rounded to whole 16-byte pieces
  const int cn = fg->nF + nLe;       // the count column "1" of B / records
  fg->cn = cn;
  fg->WG = nLe + 2;
  fg->NB = (cn + 1 + 7) / 8;
  if (fg->NB > 3) return nullptr;
  int maxs = std::max(fg->NS >= 1 ? (int)fg->A.attrs.size() : 0, fg->NS == 2 ? (int)fg->B.attrs.size() : 0);
  fg->NTS = maxs <= 8 ? 1 : 2;
  if (maxs > 16) return nullptr;
  fg->TOT = tiles_for(fg->NB, fg->NS, fg->NTS);
  {
    fg->smem_per_warp = 3 * 8 * XST * 8 + 2 * CH * fg->WG * 8 + 2 * 4 * fg->NB * 32 * 8 + HCACHE * 8 + 4 * 8 + 16 * 4 +
                        3 * 3 * CH * 4 + 16;
    fg->smem_per_warp = (fg->smem_per_warp + 127) / 128 * 128;
    int warps = GRAM_THREADS / 32;
    while (warps > 1 && warps * fg->smem_per_warp > 212 * 1024) warps--;
    fg->threads = warps * 32;
  }
  cudaStream_t st = c->stream;
  // buffers
  Level* lv[3] = {&fg->L, &fg->A, &fg->B};
  int nlev = 1 + (fg->NS >= 1) + (fg->NS == 2);
  int off = fg->TOT * 64;
  for (int i = 0; i < nlev; i++) {
    Level& l = *lv[i];
    int n = (int)l.attrs.size();
    if (l.V.alloc(std::max<int64_t>(l.nk, 1) * l.W * 8 + 256)) return nullptr;
    if (l.H.alloc(std::max<int64_t>(l.nk, 1) * 4)) return nullptr;
    std::vector<const double*> cp;
    const Rel& D = c->rels[l.rel];
    for (int a : l.attrs) cp.push_back((const double*)D.cols[D.find_attr(a)].buf.p);
    if (l.colptrs.alloc(std::max<size_t>(cp.size(), 1) * sizeof(void*))) return nullptr;
    if (!cp.empty() && cudaMemcpy(l.colptrs.p, cp.data(), cp.size() * sizeof(void*), cudaMemcpyHostToDevice))
      return nullptr;
    l.nmom = 1 + n + n * n;
    l.moff = off;
    off += l.nmom;
    if (l.mom_partials.alloc((size_t)fg->mom_blocks * l.nmom * 8)) return nullptr;
  }
  fg->nsrc = off;
  fg->count_idx = fg->L.moff;
  if (fg->partials.alloc((size_t)fg->grid * fg->TOT * 64 * 8)) return nullptr;
  if (fg->work.alloc(16)) return nullptr;
  if (fg->src.alloc((size_t)fg->nsrc * 8)) return nullptr;
  // source index of G[a][b] (a, b: attr id or -1 = "1")
  auto fidx = [](const std::vector<int>& v, int a) {
    for (size_t i = 0; i < v.size(); i++)
      if (v[i] == a) return (int)i;
    return -1;
  };
  // record/B-operand column of a feature in [x | s_L | 1]
  auto colx = [&](int a) -> int {
    if (a < 0) return cn;
    int i = fidx(fg->fattrs, a);
    if (i >= 0) return i;
    i = fidx(fg->L.attrs, a);
    if (i >= 0) return fg->nF + i;
    return -1;
  };
  const int NB = fg->NB, NTS = fg->NTS, TA = fg->NS >= 1 ? NB * NTS : 0, T12 = fg->NS == 2 ? NTS * NTS : 0;
  auto tile_el = [](int tile, int mrow, int ncol) { return tile * 64 + mrow * 8 + ncol; };
  auto src_of = [&](int a, int b) -> int {
    if (a == b && a < 0) return fg->L.moff;  // count
    // order so that a is "more fact-like"
    auto lvl = [&](int x) -> int {  // 0 = 1, 1 = fact, 2 = L, 3 = A, 4 = B
      if (x < 0) return 0;
      if (fidx(fg->fattrs, x) >= 0) return 1;
      if (fidx(fg->L.attrs, x) >= 0) return 2;
      if (fg->NS >= 1 && fidx(fg->A.attrs, x) >= 0) return 3;
      return 4;
    };
    int la = lvl(a), lb = lvl(b);
    if (la > lb) {
      std::swap(a, b);
      std::swap(la, lb);
    }
    if (lb <= 2) {
      // per-row tiles: A operand = x (x⊗x, x⊗s_L); x⊗1 is the count column of B
      if (la == 0 && lb == 1) return tile_el(cn / 8, fidx(fg->fattrs, b), cn % 8);
      if (la == 1) {
        int i = fidx(fg->fattrs, a), col = colx(b);
        return tile_el(col / 8, i, col % 8);
      }
      // 1⊗s_L or s_L⊗s_L -> moments of L
      if (la == 0) return fg->L.moff + 1 + fidx(fg->L.attrs, b);
      int n = (int)fg->L.attrs.size();
      return fg->L.moff + 1 + n + fidx(fg->L.attrs, a) * n + fidx(fg->L.attrs, b);
    }
    if (lb == 3) {
      int g2 = fidx(fg->A.attrs, b);
      int n = (int)fg->A.attrs.size();
      if (la == 3) return fg->A.moff + 1 + n + fidx(fg->A.attrs, a) * n + g2;
      int col = colx(a);  // 1, x or s_L
      return tile_el(NB + (col / 8) * NTS + g2 / 8, col % 8, g2 % 8);
    }
    // lb == 4 (level B)
    int g1 = fidx(fg->B.attrs, b);
    int n = (int)fg->B.attrs.size();
    if (la == 4) return fg->B.moff + 1 + n + fidx(fg->B.attrs, a) * n + g1;
    if (la == 3) {  // s_A ⊗ s_B: acc12[t1 = B feature][t2 = A feature]
      int g2 = fidx(fg->A.attrs, a);
      return tile_el(NB + TA + (g1 / 8) * NTS + g2 / 8, g1 % 8, g2 % 8);
    }
    int col = colx(a);
    return tile_el(NB + TA + T12 + (col / 8) * NTS + g1 / 8, col % 8, g1 % 8);
  };
  std::vector<int32_t> toff{0}, tidx;
  std::vector<double> tcoef;
  for (auto& ts : outs) {
    for (auto& t : ts) {
      tidx.push_back(src_of(t.a, t.b));
      tcoef.push_back(t.coef);
    }
    toff.push_back((int32_t)tidx.size());
  }
  fg->nout = (int)outs.size();
  if (fg->toff.alloc(toff.size() * 4) || fg->tidx.alloc(std::max<size_t>(tidx.size(), 1) * 4) ||
      fg->tcoef.alloc(std::max<size_t>(tcoef.size(), 1) * 8))
    return nullptr;
  cudaMemcpyAsync(fg->toff.p, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice, st);
  if (!tidx.empty()) {
    cudaMemcpyAsync(fg->tidx.p, tidx.data(), tidx.size() * 4, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(fg->tcoef.p, tcoef.data(), tcoef.size() * 8, cudaMemcpyHostToDevice, st);
  }
  if (cudaStreamSynchronize(st)) return nullptr;
  return hold.release();
}

}  // namespace lmfao
