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
#include <cuda.h>

#include <set>

#include "ctx.h"

namespace lmfao {

struct GramArgs {
  CUtensorMap tmL;  // gather4 tensor map over the deepest view V_L [nk x WL] (must stay first: 64-B aligned)
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
  int nLe;            // s_L columns staged per gathered row (nL rounded to 16 bytes)
  int gslot;          // doubles per gather4 destination slot (4 rows, 128-B multiple)
  int cn;             // B / record column holding the constant 1 (the count)
  int* work;          // dynamic work-item counter (zeroed before each launch)
  int smem_per_warp;  // bytes
};

constexpr int GW = 8;       // warps per CTA (one CTA per SM; 8 or 12 divide the 4 sub-partitions evenly)
constexpr int ITEM = 512;   // rows per dynamically scheduled work item (per warp)
constexpr int NSX = 3;      // stages of TMA-staged fact columns + keys (one 32-row block each)
constexpr int NSG = 2;      // stages of gather4-staged s_L rows
constexpr int XS = 36;      // smem column stride of a staged block (doubles): 16-B aligned, conflict-free
constexpr int RCAP = 4;     // pending A records per DMMA batch
constexpr int HCACHE_BITS = 6, HCACHE = 1 << HCACHE_BITS;


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

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, int col, int r0, int r1, int r2, int r3,
                                            uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(b))
      : "memory");
}

template <int NB, int NS, int NTS>
struct GramTiles {
  static constexpr int TA = NS >= 1 ? NB * NTS : 0;
  static constexpr int T12 = NS == 2 ? NTS * NTS : 0;
  static constexpr int TB = NS == 2 ? NB * NTS : 0;
  static constexpr int TOT = NB + TA + T12 + TB;
};

// Per warp: contiguous work items of ITEM rows (dynamic), processed in 32-row
// blocks.  While a block is processed, every lane prefetches the NEXT block's
// operands into registers directly in the DMMA lane layout -- x_m of row k, the
// view values s_L[key(row k)][col] (L2-resident) -- and the keys two blocks
// ahead; at the start of the block it parks them in its slots of a per-warp
// shared buffer [group][tile][lane].  The group loop is deliberately not unrolled
// and reads its operands from those slots, which keeps the kernel small for the
// instruction cache (the hot loop, boundary and record code exist once).
template <int NB, int NS, int NTS>
__global__ void __launch_bounds__(GW * 32, 1) k_gram(const __grid_constant__ GramArgs g) {
  using T = GramTiles<NB, NS, NTS>;
  constexpr int TREG = NB + T::TA + T::T12;
  constexpr int TOT = T::TOT;
  const int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2;
  const int wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cn = g.cn;
  const int64_t N = g.nrows;
  const int nitems = (int)((N + ITEM - 1) / ITEM);
  const int nB = g.nB;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  double* bacc = reinterpret_cast<double*>(smem_raw) + (size_t)wib * 24 * 16;  // [nw][24][16]
  unsigned char* wp = smem_raw + (size_t)nw * 24 * 16 * 8 + (size_t)wib * g.smem_per_warp;
  double* ob = reinterpret_cast<double*>(wp);  // operand slots [8 groups][NB][32 lanes]
  wp += 8 * NB * 32 * 8;
  double* recA = reinterpret_cast<double*>(wp);  // [RCAP][24]
  wp += RCAP * 24 * 8;
  double* recB = reinterpret_cast<double*>(wp);  // [24]
  wp += 24 * 8;
  unsigned long long* hcache = reinterpret_cast<unsigned long long*>(wp);
  wp += HCACHE * 8;
  int32_t* rkey = reinterpret_cast<int32_t*>(wp);  // A keys of pending records
  for (int i = lane; i < 24 * 16; i += 32) bacc[i] = 0.0;
  for (int i = lane; i < HCACHE; i += 32) hcache[i] = 0xFFFFFFFF00000000ull;
  __syncwarp();

  // B operand column 8t+m: x (t = 0, m < nF) | staged s_L column | constant (1 for the count column)
  const bool isx0 = m < g.nF;
  bool isg[NB];
  int gcol[NB];
  double onev[NB];
#pragma unroll
  for (int t = 0; t < NB; t++) {
    const int col = 8 * t + m;
    const int gc = col - g.nF;
    isg[t] = col >= g.nF && gc < g.nL;
    gcol[t] = isg[t] ? gc : 0;
    onev[t] = col == cn ? 1.0 : 0.0;
  }
  const double* xcolm = g.x[0];
#pragma unroll
  for (int i = 1; i < 8; i++)
    if (m == i) xcolm = g.x[i];
  const unsigned WL = (unsigned)g.WL;

  double acc[TREG][2];
#pragma unroll
  for (int t = 0; t < TREG; t++) acc[t][0] = acc[t][1] = 0.0;
  double P[NB], Ps[NB], sumB[NB];
#pragma unroll
  for (int t = 0; t < NB; t++) P[t] = Ps[t] = sumB[t] = 0.0;
  double preA[NTS], preAB[NTS];
#pragma unroll
  for (int t = 0; t < NTS; t++) preA[t] = preAB[t] = 0.0;
  int npA = 0;
  bool runA_ne = false, runB_ne = false;
  int curA = -1, curB = -1;
  int prevL = -1, prevA = -1, prevB = -1;
  int runL_start = 0;

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
  auto reduce4 = [&](double v) {
    v += __shfl_xor_sync(FULL, v, 1);
    v += __shfl_xor_sync(FULL, v, 2);
    return v;
  };
  auto process_A = [&]() {
    __syncwarp();
    const bool rv = k < npA;
    double a[NB];
#pragma unroll
    for (int t = 0; t < NB; t++) a[t] = rv ? recA[k * 24 + 8 * t + m] : 0.0;
    const double nk = rv ? recA[k * 24 + cn] : 0.0;
#pragma unroll
    for (int t = 0; t < NB; t++)
#pragma unroll
      for (int t2 = 0; t2 < NTS; t2++) dmma(acc[NB + t * NTS + t2], a[t], rv ? preA[t2] : 0.0);
    if constexpr (NS == 2) {
#pragma unroll
      for (int t1 = 0; t1 < NTS; t1++)
#pragma unroll
        for (int t2 = 0; t2 < NTS; t2++)
          dmma(acc[NB + T::TA + t1 * NTS + t2], rv ? nk * preAB[t1] : 0.0, rv ? preA[t2] : 0.0);
    }
    if (rv && m == 0) atomicAdd(&g.HA[rkey[k]], (unsigned)nk);
#pragma unroll
    for (int t = 0; t < NTS; t++) preA[t] = preAB[t] = 0.0;
    npA = 0;
    __syncwarp();
  };
  // level-B record (rare): reduced sums (x) s_B into this warp's shared block
  auto push_B = [&](int keyB) {
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const double v = reduce4(sumB[t]);
      if (k == 0) recB[8 * t + m] = v;
    }
    __syncwarp();
    const double* row = g.VB + (unsigned)keyB * (unsigned)g.WB;
    for (int e = lane; e < 24 * nB; e += 32) {
      const int c = e / nB, f = e % nB;
      bacc[c * 16 + f] += recB[c] * row[f];
    }
    if (lane == 0) atomicAdd(&g.HB[keyB], (unsigned)recB[cn]);
    __syncwarp();
  };
  auto push_A = [&](const double* rec, int keyA, int keyB) {
#pragma unroll
    for (int t = 0; t < NB; t++) {
      const double v = reduce4(rec[t]);
      if (k == 0) recA[npA * 24 + 8 * t + m] = v;
    }
    if (lane == 0) rkey[npA] = keyA;
    if (k == npA) {
      const double* row = g.VA + (unsigned)keyA * (unsigned)g.WA;
      preA[0] = m < g.nA ? row[m] : 0.0;
      if constexpr (NTS == 2) preA[1] = 8 + m < g.nA ? row[8 + m] : 0.0;
      if constexpr (NS == 2) {
        const double* rowb = g.VB + (unsigned)keyB * (unsigned)g.WB;
        preAB[0] = m < nB ? rowb[m] : 0.0;
        if constexpr (NTS == 2) preAB[1] = 8 + m < nB ? rowb[8 + m] : 0.0;
      }
    }
    if constexpr (NS == 2) {
#pragma unroll
      for (int t = 0; t < NB; t++) sumB[t] += rec[t];
      runB_ne = true;
    }
    if (++npA == RCAP) process_A();
  };
  auto flush_range = [&](int end) {
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
  };

  // ---- block sequence over dynamically grabbed items
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
  auto item_rows = [&](int it) {
    const int64_t r = (int64_t)it * ITEM;
    return (int)(N - r < ITEM ? N - r : ITEM);
  };
  struct Cur {
    int slot, b, seq, item;
  };
  auto adv = [&](Cur& u, bool may_grab) {
    u.seq++;
    if ((u.b + 1) * 32 < item_rows(u.item)) {
      u.b++;
    } else {
      u.b = 0;
      u.slot++;
      if (may_grab && u.slot >= nring) grab();
      u.item = ring_at(u.slot);
    }
  };
  // register prefetch of a block's operands (DMMA lane layout) and keys (lane = row)
  double px[8], pg[NB][8];
  int pk[3] = {-1, -1, -1};  // keys of the block whose operands are prefetched next
  int qk[3] = {-1, -1, -1};  // keys of the block after it
  auto row0_of = [&](const Cur& u) { return (int64_t)u.item * ITEM + u.b * 32; };
  auto nrows_of = [&](const Cur& u) { return min(32, item_rows(u.item) - u.b * 32); };
  auto load_keys = [&](const Cur& u, int (&kk)[3]) {
    kk[0] = kk[1] = kk[2] = -1;
    if (u.item < nitems && lane < nrows_of(u)) {
      const int64_t r = row0_of(u) + lane;
      kk[0] = g.kL[r];
      if (NS >= 1) kk[1] = g.kA[r];
      if (NS == 2) kk[2] = g.kB[r];
    }
  };
  auto load_ops = [&](const Cur& u) {  // operands of block u; pk holds its keys
    const int n = u.item < nitems ? nrows_of(u) : 0;
    const int64_t r0 = u.item < nitems ? row0_of(u) : 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int rj = 4 * j + k;
      const int key = __shfl_sync(FULL, pk[0], rj);
      const bool v = rj < n;
      px[j] = (isx0 && v) ? xcolm[r0 + rj] : 0.0;
      const double* row = g.VL + (unsigned)(v ? key : 0) * WL;
#pragma unroll
      for (int t = 0; t < NB; t++) {
        double val = v ? onev[t] : 0.0;
        if (v && isg[t]) val = row[gcol[t]];
        pg[t][j] = val;
      }
    }
  };
  auto park_ops = [&]() {
#pragma unroll
    for (int j = 0; j < 8; j++)
#pragma unroll
      for (int t = 0; t < NB; t++) ob[(j * NB + t) * 32 + lane] = (t == 0 && isx0) ? px[j] : pg[t][j];
  };

  grab();
  Cur c0{0, 0, 0, ring_at(0)};
  Cur c1 = c0, c2 = c0;  // c1: operands in flight (one ahead), c2: keys in flight (two ahead)
  int ck[3];             // keys (lane = row) of block c0
  load_keys(c0, pk);
  ck[0] = pk[0];
  ck[1] = pk[1];
  ck[2] = pk[2];
  load_ops(c0);
  adv(c1, true);
  adv(c2, true);
  adv(c2, true);
  load_keys(c1, pk);
  int range_end = -1;
  while (c0.item < nitems) {
    park_ops();  // operands of block c0 -> this lane's slots
    __syncwarp();
    load_keys(c2, qk);  // prefetch: keys two blocks ahead, operands of the next block
    load_ops(c1);
    const int irows = item_rows(c0.item);
    const int ro = c0.b * 32;
    const int nval = min(32, irows - ro);
    if (c0.b == 0) {  // new contiguous item: close the previous range
      if (range_end >= 0) flush_range(range_end);
#pragma unroll
      for (int t = 0; t < NB; t++) P[t] = Ps[t] = sumB[t] = 0.0;
      runA_ne = runB_ne = false;
      prevL = prevA = prevB = -1;
      runL_start = 0;
    }
    range_end = irows;
    const bool vr = lane < nval;
    const int kl = vr ? ck[0] : -1;
    const int ka = (NS >= 1 && vr) ? ck[1] : -1;
    const int kb = (NS == 2 && vr) ? ck[2] : -1;
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
    {
      const unsigned before = mL & ((1u << lane) - 1u);
      const int st = before ? ro + (31 - __clz(before)) : runL_start;
      const int len = ro + lane - st;
      hl_flush_lanes(dL && len > 0 && pl >= 0, pl, (unsigned)len);
      if (mL) runL_start = ro + (31 - __clz(mL));
    }
    const int ngr = (nval + 3) >> 2;
#pragma unroll 1
    for (int j = 0; j < ngr; j++) {
      double b[NB];
#pragma unroll
      for (int t = 0; t < NB; t++) b[t] = ob[(j * NB + t) * 32 + lane];
      const double xa = isx0 ? b[0] : 0.0;
#pragma unroll
      for (int t = 0; t < NB; t++) dmma(acc[t], xa, b[t]);
      if constexpr (NS >= 1) {
        const unsigned nib = (mA >> (4 * j)) & 0xFu;
        unsigned bits = nib;
        while (bits) {
          const int p = __ffs(bits) - 1;
          bits &= bits - 1;
          double rec[NB];
#pragma unroll
          for (int t = 0; t < NB; t++) {
            const double pb2 = P[t] + (k < p ? b[t] : 0.0);
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
#pragma unroll
        for (int t = 0; t < NB; t++) P[t] += b[t];
      }
    }
    __syncwarp();
    adv(c0, false);
    adv(c1, false);
    adv(c2, true);
    ck[0] = pk[0];
    ck[1] = pk[1];
    ck[2] = pk[2];
    pk[0] = qk[0];
    pk[1] = qk[1];
    pk[2] = qk[2];
  }
  if (range_end >= 0) flush_range(range_end);
  if constexpr (NS >= 1) {
    if (npA > 0) process_A();
  }
  __syncwarp();
  for (int i = lane; i < HCACHE; i += 32) {
    const unsigned long long e = hcache[i];
    if ((unsigned)(e >> 32) != 0xFFFFFFFFu) atomicAdd(&g.HL[(unsigned)(e >> 32)], (unsigned)e);
  }
  // deterministic CTA reduction (warps in order); the B block is summed from the warps' smem blocks
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem_raw + (size_t)nw * 24 * 16 * 8);  // reuse staging (all consumed)
  for (int i = threadIdx.x; i < TOT * 64; i += blockDim.x) red[i] = 0.0;
  __syncthreads();
  for (int w = 0; w < nw; w++) {
    if (wib == w) {
#pragma unroll
      for (int t = 0; t < TREG; t++) {
        red[t * 64 + m * 8 + 2 * k] += acc[t][0];
        red[t * 64 + m * 8 + 2 * k + 1] += acc[t][1];
      }
    }
    __syncthreads();
  }
  if constexpr (NS == 2) {
    const double* b0 = reinterpret_cast<const double*>(smem_raw);
    for (int i = threadIdx.x; i < 24 * 16; i += blockDim.x) {
      const int c = i / 16, f = i % 16;
      double v = 0.0;
      for (int w = 0; w < nw; w++) v += b0[(size_t)w * 24 * 16 + i];
      if (c < 8 * NB && f < 8 * NTS) red[(TREG + (c / 8) * NTS + f / 8) * 64 + (c % 8) * 8 + (f % 8)] = v;
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
  int cn = 0, WG = 2, nLe = 2, gslot = 16;
  CUtensorMap tmL;
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
  size_t smem = (size_t)(threads / 32) * (24 * 16 * 8 + g.smem_per_warp);
  CUDA_TRY(ensure_smem_attr((const void*)k_gram<NB, NS, NTS>, smem));
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
  g.nLe = nLe;
  g.gslot = gslot;
  g.tmL = tmL;
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
  fg->nLe = nLe;
  fg->gslot = (4 * nLe + 15) / 16 * 16;
  fg->NB = (cn + 1 + 7) / 8;
  if (fg->NB > 3) return nullptr;
  int maxs = std::max(fg->NS >= 1 ? (int)fg->A.attrs.size() : 0, fg->NS == 2 ? (int)fg->B.attrs.size() : 0);
  fg->NTS = maxs <= 8 ? 1 : 2;
  if (maxs > 16) return nullptr;
  fg->TOT = tiles_for(fg->NB, fg->NS, fg->NTS);
  {
    int pw = 8 * fg->NB * 32 * 8 + RCAP * 24 * 8 + 24 * 8 + HCACHE * 8 + 16;
    pw = (pw + 127) / 128 * 128;
    fg->smem_per_warp = pw;
    fg->threads = GW * 32;
    if (GW * (24 * 16 * 8 + pw) > 220 * 1024) return nullptr;
    if ((size_t)fg->TOT * 64 * 8 > (size_t)GW * (pw + 24 * 16 * 8)) return nullptr;
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
    if (!cp.empty() && cudaMemcpyAsync(l.colptrs.p, cp.data(), cp.size() * sizeof(void*), cudaMemcpyHostToDevice, st))
      return nullptr;
    l.nmom = 1 + n + n * n;
    l.moff = off;
    off += l.nmom;
    if (l.mom_partials.alloc((size_t)fg->mom_blocks * l.nmom * 8)) return nullptr;
  }
  fg->nsrc = off;
  fg->count_idx = fg->L.moff;
  {  // gather4 tensor map over V_L [nk x W] (fp64): box = nLe columns x 1 row
    typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess || !fn)
        return nullptr;
      encode = (EncodeFn)fn;
    }
    std::memset(&fg->tmL, 0, sizeof(fg->tmL));
    if (!fg->L.attrs.empty()) {
      cuuint64_t dims[2] = {(cuuint64_t)fg->L.W, (cuuint64_t)std::max<int64_t>(fg->L.nk, 1)};
      cuuint64_t strides[1] = {(cuuint64_t)fg->L.W * 8};
      cuuint32_t box[2] = {(cuuint32_t)fg->nLe, 1};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = encode(&fg->tmL, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, fg->L.V.p, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) return nullptr;
    }
  }
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
