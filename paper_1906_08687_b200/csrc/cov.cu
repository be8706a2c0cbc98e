// cov.cu — the covariance batch's fused root scan, B200 version 2 (k_cov).
//
// Same mathematics as gram.cu (§3 "covariance matrix" P:397-402: every
// aggregate is an entry of G = Σ_f u(f) u(f)^T with u = [1, x, s_L, s_A, s_B]),
// evaluated over the root sorted by its foreign keys in increasing domain size
// with the multi-output trie registration of P:1020-1214:
//   per row          x⊗x, x⊗s_L                (FP64 DMMA m8n8k4 on 4-row groups + 2 DFMA)
//   per level-A run  R_A⊗s_A, R_A = Σ_run [x, s_L, 1]  (4 runs per DMMA, "intermediate aggregates")
//   per level-B run  R_B⊗s_B, R_B = Σ_{A-runs} [R_A, n·s_A]  (record list, finished off-scan)
//   dimension side   Σ_k H_r[k] s_r(k) s_r(k)^T  ("each aggregate to its own root")
// What changed against gram.cu, and why (all measured on B200):
//  * the kernel is specialised at compile time for ≤ 8 fact features and ≤ 10
//    features per dimension level (C1, C2, C5's covariance), so the hot loop has
//    no runtime shape logic (the v12 kernel spent 45 warp-instructions per row);
//  * every warp runs its own TMA pipeline: `cp.async.bulk` of the fact columns and
//    keys of a 32-row block into a CS-deep shared-memory ring, and one
//    `cp.async.bulk.tensor.2d ... tile::gather4` per 4 rows for the view rows
//    s_L[k_L] (96-byte rows, L2-resident), issued one block ahead — no operand
//    prefetch lives in registers;
//  * level-A run records are stored unreduced (per lane) in shared memory and
//    reduced four at a time straight into the DMMA A-operand layout;
//  * level-B records go to a device list and are finished by a small kernel;
//  * H_L (root rows per L key, for s_L⊗s_L) is counted in a per-CTA open-
//    addressing table in shared memory (Zipf-hot keys would serialise global
//    atomics), spilling to global atomics when a probe misses twice.
// Runs split at block / item boundaries are exact (every update is linear in the
// run sums), so any row order is correct; the sort only makes runs long.
#include <cuda.h>

#include <set>

#include "ctx.h"

namespace lmfao {
namespace {

constexpr int CW = 8;        // warps per CTA (one CTA per SM)
constexpr int CS = 4;        // pipeline stages per warp
constexpr int CITEM = 512;   // rows per dynamically scheduled item
constexpr int XSTR = 36;     // doubles per staged x column (32 rows + pad: conflict-free DMMA-layout reads)
constexpr int GP = 12;       // doubles per view row (gather4 box width; cols >= n are 0)
constexpr int HT = 2048;     // per-CTA H_L hash slots
constexpr int PR = 97;       // doubles per pending record (3 x 32 lanes + 1: conflict-free transposed reads)
constexpr int STG_X = 8 * XSTR * 8;            // 2304 B
constexpr int STG_K = 3 * 32 * 4;              // 384 B
constexpr int STG_G = 32 * GP * 8;             // 3072 B
constexpr int STG = STG_X + STG_K + STG_G;     // 5760 B (45 x 128)
constexpr int PEND_B = (4 * PR * 8 + 127) / 128 * 128;
constexpr int WB = CS * STG + PEND_B + 128;    // per-warp shared bytes
constexpr int SMEM = HT * 8 + CW * WB;
constexpr int NPART = 384;   // per-CTA partial: XX[8][8] | XL[8][10] | RA[24][10]
constexpr int BRW = 36;      // doubles per B record
constexpr int NFIN = 707;    // RB[34][10] | TOT[34] | MB[111] | ML[111] | MA[111]
constexpr int FIN_BLOCKS = 148;
constexpr unsigned FULL = 0xffffffffu;

static_assert(SMEM <= 232448, "shared memory budget");

struct CovArgs {
  CUtensorMap tmL;  // gather4 map over V_L [nkL x GP] fp64 (first: 64-B aligned)
  int64_t nrows;
  const double* x[8];
  const int32_t* key[3];  // L, A, B dense key columns (A/B null if the level is absent)
  const double* VA;       // [nkA x GP] (a zero row if absent)
  unsigned* HL;
  unsigned* HA;
  double* brec;
  int* bcount;
  int bcap;
  int nx;
  double* partials;  // [grid][NPART]
  int* work;
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
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int r0, int r1, int r2, int r3, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(sa(dst)),
      "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(b))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
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

// NS = number of featured levels above L (0: L only, 1: A and L, 2: B, A and L).
template <int NS>
__global__ void __launch_bounds__(CW * 32, 1) k_cov(const __grid_constant__ CovArgs g) {
  const int lane = threadIdx.x & 31, k = lane & 3, m = lane >> 2, wib = threadIdx.x >> 5;
  extern __shared__ __align__(1024) unsigned char sm[];
  int* hkey = reinterpret_cast<int*>(sm);
  unsigned* hcnt = reinterpret_cast<unsigned*>(sm + HT * 4);
  unsigned char* wbase = sm + HT * 8 + wib * WB;
  double* pend = reinterpret_cast<double*>(wbase + CS * STG);
  uint64_t* bar_f = reinterpret_cast<uint64_t*>(wbase + CS * STG + PEND_B);
  uint64_t* bar_g = bar_f + CS;
  int* ring = reinterpret_cast<int*>(bar_g + CS);  // 8 grabbed item ids

  for (int i = threadIdx.x; i < HT; i += blockDim.x) {
    hkey[i] = -1;
    hcnt[i] = 0;
  }
  // x columns beyond nx stay zero for the whole kernel
  for (int s = 0; s < CS; s++) {
    double* xs = reinterpret_cast<double*>(wbase + s * STG);
    for (int i = g.nx * XSTR + lane; i < 8 * XSTR; i += 32) xs[i] = 0.0;
  }
  if (lane == 0) {
    for (int s = 0; s < CS; s++) {
      mbar_init(&bar_f[s], 1);
      mbar_init(&bar_g[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t N = g.nrows;
  const int nitems = (int)((N + CITEM - 1) / CITEM);
  auto item_rows = [&](int it) { const int64_t r = N - (int64_t)it * CITEM; return (int)(r < CITEM ? r : CITEM); };

  // per-lane TMA source of the fact block: lanes 0..7 x columns, 8..10 key columns
  const char* my_src = nullptr;
  int my_es = 0, my_off = 0;
  if (lane < 8) {
    if (lane < g.nx) {
      my_src = reinterpret_cast<const char*>(g.x[lane]);
      my_es = 8;
      my_off = lane * XSTR * 8;
    }
  } else if (lane < 8 + 1 + NS) {
    my_src = reinterpret_cast<const char*>(g.key[lane - 8]);
    my_es = 4;
    my_off = STG_X + (lane - 8) * 128;
  }

  // cursors over this warp's block sequence (items grabbed dynamically, in order)
  int nring = 0;
  auto grab = [&]() {
    int it = 0;
    if (lane == 0) it = atomicAdd(g.work, 1);
    it = __shfl_sync(FULL, it, 0);
    if (lane == 0) ring[nring & 7] = it;
    __syncwarp();
    nring++;
  };
  struct Cur {
    int slot, b, item;
  };
  auto item_at = [&](int slot) { return ring[slot & 7]; };
  auto advance = [&](Cur& c, bool may_grab) {
    if (c.item >= nitems) return;
    if ((c.b + 1) * 32 < item_rows(c.item)) {
      c.b++;
    } else {
      c.b = 0;
      c.slot++;
      if (may_grab && c.slot >= nring) grab();
      c.item = item_at(c.slot);
    }
  };
  auto block_rows = [&](const Cur& c) { return min(32, item_rows(c.item) - c.b * 32); };

  auto issue_fact = [&](const Cur& c, int stage) {
    if (c.item >= nitems) return;
    const int nv = block_rows(c);
    const int64_t row0 = (int64_t)c.item * CITEM + c.b * 32;
    const uint32_t bx = (uint32_t)((nv * 8 + 15) & ~15), bk = (uint32_t)((nv * 4 + 15) & ~15);
    unsigned char* st = wbase + stage * STG;
    __syncwarp();
    fence_proxy_async();
    if (lane == 0) mbar_expect(&bar_f[stage], bx * g.nx + bk * (1 + NS));
    __syncwarp();
    if (my_src) bulk_load(st + my_off, my_src + row0 * my_es, my_es == 8 ? bx : bk, &bar_f[stage]);
  };
  auto issue_gather = [&](const Cur& c, int stage) {
    if (c.item >= nitems) return;
    const int nv = block_rows(c);
    const int ngr = (nv + 3) >> 2;
    unsigned char* st = wbase + stage * STG;
    const int* kl = reinterpret_cast<const int*>(st + STG_X);
    __syncwarp();
    fence_proxy_async();
    if (lane == 0) mbar_expect(&bar_g[stage], (uint32_t)ngr * 4 * GP * 8);
    __syncwarp();
    if (lane < ngr) {
      const int4 q = reinterpret_cast<const int4*>(kl)[lane];
      const int r = 4 * lane;
      gather4(st + STG_X + STG_K + lane * 4 * GP * 8, &g.tmL, q.x, r + 1 < nv ? q.y : 0, r + 2 < nv ? q.z : 0,
              r + 3 < nv ? q.w : 0, &bar_g[stage]);
    }
  };

  // ---- accumulators
  double aXX[2] = {0, 0}, aXL[2] = {0, 0}, a8 = 0, a9 = 0;
  double aRA[3][2] = {{0, 0}, {0, 0}, {0, 0}}, r8[3] = {0, 0, 0}, r9[3] = {0, 0, 0};
  double SB0 = 0, SB1 = 0, SB2 = 0, SBn = 0, SBn8 = 0, SBn9 = 0;
  double Cx = 0, Cs = 0, Ct = 0;  // this lane's part of the open A run
  double pbA = 0;
  double2 pbA89 = make_double2(0, 0);
  int pkey = 0, pn = 0, npend = 0;
  bool openA = false, openB = false;
  int curA = 0, curB = 0, startA = 0;
  int prevL = -1, prevA = -1, prevB = -1;
  const int tcol = 8 + min(m, 2);

  auto hl_add = [&](int key, unsigned len) {
    unsigned h = ((unsigned)key * 2654435761u) >> (32 - 11);
#pragma unroll 1
    for (int probe = 0; probe < 2; probe++) {
      int t = hkey[h];
      if (t == -1) {
        const int old = atomicCAS(&hkey[h], -1, key);
        t = old == -1 ? key : old;
      }
      if (t == key) {
        atomicAdd(&hcnt[h], len);
        return;
      }
      h = (h + 1) & (HT - 1);
    }
    atomicAdd(&g.HL[key], len);
  };
  auto process_A = [&]() {
    __syncwarp();
    const bool rv = k < npend;
    const double* pk = pend + k * PR + 4 * m;
    double a0 = (pk[0] + pk[1]) + (pk[2] + pk[3]);
    double a1 = (pk[32] + pk[33]) + (pk[34] + pk[35]);
    double a2 = (pk[64] + pk[65]) + (pk[66] + pk[67]);
    const double nk = rv ? (double)pn : 0.0;
    if (m == 2) a2 = nk;
    if (!rv) a0 = a1 = a2 = 0.0;
    const double b0 = rv ? pbA : 0.0, b8 = rv ? pbA89.x : 0.0, b9 = rv ? pbA89.y : 0.0;
    dmma(aRA[0], a0, b0);
    dmma(aRA[1], a1, b0);
    dmma(aRA[2], a2, b0);
    r8[0] = fma(a0, b8, r8[0]);
    r8[1] = fma(a1, b8, r8[1]);
    r8[2] = fma(a2, b8, r8[2]);
    r9[0] = fma(a0, b9, r9[0]);
    r9[1] = fma(a1, b9, r9[1]);
    r9[2] = fma(a2, b9, r9[2]);
    SB0 += a0;
    SB1 += a1;
    SB2 += a2;
    SBn = fma(nk, b0, SBn);
    SBn8 = fma(nk, b8, SBn8);
    SBn9 = fma(nk, b9, SBn9);
    if (NS >= 1 && rv && m == 0) atomicAdd(&g.HA[pkey], (unsigned)pn);
    npend = 0;
    __syncwarp();
  };
  auto emit = [&](double rx, double rs, double rt, int n, int keyA) {
    double* pr = pend + npend * PR + lane;
    pr[0] = rx;
    pr[32] = rs;
    pr[64] = rt;
    if (k == npend) {
      pkey = keyA;
      pn = n;
      const double* row = g.VA + (size_t)(unsigned)keyA * GP;
      pbA = row[m];
      pbA89 = *reinterpret_cast<const double2*>(row + 8);
    }
    if (++npend == 4) process_A();
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
  auto flush_item = [&](int irows) {
    if (openA) emit(Cx, Cs, Ct, irows - startA, curA);
    if (npend) process_A();
    if (openB) push_B(curB);
    openA = openB = false;
    Cx = Cs = Ct = 0.0;
    prevL = prevA = prevB = -1;
  };

  // ---- pipeline prologue
  grab();
  Cur cc{0, 0, item_at(0)};
  Cur cf = cc;
  for (int s = 0; s < CS; s++) {
    issue_fact(cf, s);
    advance(cf, true);
  }
  if (cc.item < nitems) {
    mbar_wait(&bar_f[0], 0);
    issue_gather(cc, 0);
  }
  int blk = 0;
  int cur_item_rows = 0;
  bool have_item = false;
  while (cc.item < nitems) {
    const int s = blk % CS;
    const uint32_t par = (uint32_t)(blk / CS) & 1u;
    {  // gathers of the next block (its keys have landed)
      Cur cn = cc;
      advance(cn, false);
      if (cn.item < nitems) {
        const int s1 = (blk + 1) % CS;
        mbar_wait(&bar_f[s1], (uint32_t)((blk + 1) / CS) & 1u);
        issue_gather(cn, s1);
      }
    }
    if (cc.b == 0) {
      if (have_item) flush_item(cur_item_rows);
      have_item = true;
      cur_item_rows = item_rows(cc.item);
    }
    mbar_wait(&bar_g[s], par);
    unsigned char* st = wbase + s * STG;
    double* xs = reinterpret_cast<double*>(st);
    const int* ks = reinterpret_cast<const int*>(st + STG_X);
    double* gs = reinterpret_cast<double*>(st + STG_X + STG_K);
    const int nv = block_rows(cc);
    const int rowbase = cc.b * 32;
    if (nv < 32) {  // ragged tail: zero the stale rows of the stage
      if (lane >= nv) {
#pragma unroll
        for (int c = 0; c < 8; c++) xs[c * XSTR + lane] = 0.0;
#pragma unroll
        for (int c = 0; c < GP; c++) gs[lane * GP + c] = 0.0;
      }
      __syncwarp();
    }
    const bool vr = lane < nv;
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
    if (lead) {
      const unsigned above = mLd & ~((2u << lane) - 1u);
      const int end = above ? __ffs(above) - 1 : nv;
      hl_add(kl, (unsigned)(end - lane));
    }
    const double* xg = xs + m * XSTR + k;
    const double* gg = gs + k * GP;
    const int ngr = (nv + 3) >> 2;
#pragma unroll 2
    for (int j = 0; j < ngr; j++) {
      const double xa = xg[4 * j];
      const double* gr = gg + j * 4 * GP;
      const double sv = gr[m];
      const double2 s89 = *reinterpret_cast<const double2*>(gr + 8);
      const double tv = gr[tcol];
      dmma(aXX, xa, xa);
      dmma(aXL, xa, sv);
      a8 = fma(xa, s89.x, a8);
      a9 = fma(xa, s89.y, a9);
      unsigned nib = (mA >> (4 * j)) & 15u;
      if (nib == 0) {
        Cx += xa;
        Cs += sv;
        Ct += tv;
        continue;
      }
      int lo = 0;
      do {
        const int q = __ffs(nib) - 1;
        nib &= nib - 1;
        const int p = 4 * j + q;
        if (openA) {
          const bool in = k >= lo && k < q;
          emit(Cx + (in ? xa : 0.0), Cs + (in ? sv : 0.0), Ct + (in ? tv : 0.0), rowbase + p - startA, curA);
        }
        Cx = Cs = Ct = 0.0;
        if ((mB >> p) & 1u) {
          if (openB) {
            if (npend) process_A();
            push_B(curB);
          }
          openB = true;
          curB = __shfl_sync(FULL, kb, p);
        }
        openA = true;
        curA = __shfl_sync(FULL, ka, p);
        startA = rowbase + p;
        lo = q;
      } while (nib);
      const bool in = k >= lo;
      Cx = in ? xa : 0.0;
      Cs = in ? sv : 0.0;
      Ct = in ? tv : 0.0;
    }
    __syncwarp();
    issue_fact(cf, s);  // the slot just consumed takes the block CS ahead
    advance(cf, true);
    advance(cc, false);
    blk++;
  }
  if (have_item) flush_item(cur_item_rows);

  // ---- H_L table -> global
  __syncthreads();
  for (int i = threadIdx.x; i < HT; i += blockDim.x) {
    const int key = hkey[i];
    if (key != -1 && hcnt[i]) atomicAdd(&g.HL[key], hcnt[i]);
  }
  // ---- CTA reduction (warps in order) -> partials
  a8 = red4(a8);
  a9 = red4(a9);
#pragma unroll
  for (int t = 0; t < 3; t++) {
    r8[t] = red4(r8[t]);
    r9[t] = red4(r9[t]);
  }
  double* red = reinterpret_cast<double*>(sm + HT * 8);  // stage memory is free now
  __syncthreads();
  for (int i = threadIdx.x; i < NPART; i += blockDim.x) red[i] = 0.0;
  __syncthreads();
  for (int w = 0; w < CW; w++) {
    if (wib == w) {
      red[m * 8 + 2 * k] += aXX[0];
      red[m * 8 + 2 * k + 1] += aXX[1];
      red[64 + m * 10 + 2 * k] += aXL[0];
      red[64 + m * 10 + 2 * k + 1] += aXL[1];
      if (k == 0) {
        red[64 + m * 10 + 8] += a8;
        red[64 + m * 10 + 9] += a9;
      }
#pragma unroll
      for (int t = 0; t < 3; t++) {
        red[144 + (8 * t + m) * 10 + 2 * k] += aRA[t][0];
        red[144 + (8 * t + m) * 10 + 2 * k + 1] += aRA[t][1];
        if (k == 0) {
          red[144 + (8 * t + m) * 10 + 8] += r8[t];
          red[144 + (8 * t + m) * 10 + 9] += r9[t];
        }
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < NPART; i += blockDim.x) g.partials[(size_t)blockIdx.x * NPART + i] = red[i];
}

// V[k][f] = col_f[k] for f < n, 0 for n <= f < GP (primary-key leaf: row k has dense key k).
struct DimTables {
  const double* const* cols[3];
  int n[3];
  int64_t nk[3];
  double* V[3];
};
__global__ void k_cov_dims(DimTables d) {
  const int64_t tot0 = d.nk[0] * GP, tot1 = d.nk[1] * GP, tot2 = d.nk[2] * GP;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot0 + tot1 + tot2;
       i += (int64_t)gridDim.x * blockDim.x) {
    int l = 0;
    int64_t e = i;
    if (e >= tot0) {
      e -= tot0;
      l = 1;
      if (e >= tot1) {
        e -= tot1;
        l = 2;
      }
    }
    const int64_t kk = e / GP;
    const int f = (int)(e % GP);
    d.V[l][e] = f < d.n[l] ? d.cols[l][f][kk] : 0.0;
  }
}

// Off-scan finishing, per block b of FIN_BLOCKS: B records in its range (R_B⊗s_B,
// Σ R_B, B moments weighted by the record counts) and the L / A moments over its
// key ranges weighted by H_L / H_A.  Output: partials [FIN_BLOCKS][NFIN].
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
  double* partials;
};
__device__ __forceinline__ void moment_ij(int o, int& f, int& g2) {
  f = g2 = -1;
  if (o >= 1 && o <= 10) f = o - 1;
  if (o > 10) {
    f = (o - 11) / 10;
    g2 = (o - 11) % 10;
  }
}
__global__ void k_cov_fin(FinArgs a) {
  const int b = blockIdx.x, P = gridDim.x;
  const int nrec = min(*a.bcount, a.bcap);
  const int r0 = (int)((int64_t)nrec * b / P), r1 = (int)((int64_t)nrec * (b + 1) / P);
  const int64_t l0 = a.nkL * b / P, l1 = a.nkL * (b + 1) / P;
  const int64_t q0 = a.nkA * b / P, q1 = a.nkA * (b + 1) / P;
  for (int o = threadIdx.x; o < NFIN; o += blockDim.x) {
    double s = 0.0;
    if (o < 340) {
      const int r = o / 10, c = o % 10;
      for (int i = r0; i < r1; i++) {
        const double* rec = a.brec + (size_t)i * BRW;
        s = fma(rec[r], a.VB[(size_t)(unsigned)(int)rec[34] * GP + c], s);
      }
    } else if (o < 374) {
      const int r = o - 340;
      for (int i = r0; i < r1; i++) s += a.brec[(size_t)i * BRW + r];
    } else if (o < 485) {
      int f, g2;
      moment_ij(o - 374, f, g2);
      for (int i = r0; i < r1; i++) {
        const double* rec = a.brec + (size_t)i * BRW;
        const double* v = a.VB + (size_t)(unsigned)(int)rec[34] * GP;
        double t = rec[18];
        if (f >= 0) t *= v[f];
        if (g2 >= 0) t *= v[g2];
        s += t;
      }
    } else {
      const bool isL = o < 596;
      int f, g2;
      moment_ij(o - (isL ? 485 : 596), f, g2);
      const unsigned* H = isL ? a.HL : a.HA;
      const double* V = isL ? a.VL : a.VA;
      const int64_t k0 = isL ? l0 : q0, k1 = isL ? l1 : q1;
      for (int64_t kk = k0; kk < k1; kk++) {
        const unsigned h = H[kk];
        if (!h) continue;
        double t = (double)h;
        if (f >= 0) t *= V[kk * GP + f];
        if (g2 >= 0) t *= V[kk * GP + g2];
        s += t;
      }
    }
    a.partials[(size_t)b * NFIN + o] = s;
  }
}

// src[0:NPART] = Σ_cta scan partials; src[NPART:NPART+NFIN] = Σ_b fin partials (fixed order)
__global__ void k_cov_sum(const double* __restrict__ p1, int n1, const double* __restrict__ p2, int n2,
                          double* __restrict__ src) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < NPART) {
    double s = 0.0;
    for (int b = 0; b < n1; b++) s += p1[(size_t)b * NPART + e];
    src[e] = s;
  } else if (e < NPART + NFIN) {
    double s = 0.0;
    for (int b = 0; b < n2; b++) s += p2[(size_t)b * NFIN + e - NPART];
    src[e] = s;
  }
}

__global__ void k_cov_assemble(const double* __restrict__ src, const int32_t* __restrict__ toff,
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
struct CovLevel {
  int child = -1, rel = -1;
  std::vector<int> attrs;
  int64_t nk = 0;
  DevBuf V, colptrs;
};

struct FastCov : FastPaths {
  int NS = 0, nF = 0;
  std::vector<int> fattrs;
  CovLevel L, A, B;
  DevBuf zeros;  // one zero view row (absent levels)
  DevBuf zbuf;   // [work | bcount | pad] [HA] [HL], cleared every run
  size_t off_HA = 0, off_HL = 0, zbytes = 0;
  DevBuf brec, partials, finp, src, toff, tidx, tcoef;
  int bcap = 0, grid = 148, nout = 0;
  CUtensorMap tmL;
  bool only_scalar = true;

  std::string describe() const override {
    char b[256];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"cov\", \"NS\": %d, \"nF\": %d, \"nL\": %zu, \"nA\": %zu, \"nB\": %zu, \"grid\": %d, "
                  "\"threads\": %d, \"stages\": %d, \"item\": %d}",
                  NS, nF, L.attrs.size(), A.attrs.size(), B.attrs.size(), grid, CW * 32, CS, CITEM);
    return b;
  }
  bool skip_generic_views() const override { return only_scalar; }
  int run(lmfao_ctx* c, const NodeArgs& ra, cudaStream_t st, bool& scalar_done) override;
};

cudaError_t launch_cov(int NS, const CovArgs& g, int grid, cudaStream_t st) {
  static bool attr[3] = {false, false, false};
  auto go = [&](auto kern) -> cudaError_t {
    if (!attr[NS]) {
      CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
      attr[NS] = true;
    }
    kern<<<grid, CW * 32, SMEM, st>>>(g);
    return cudaGetLastError();
  };
  if (NS == 0) return go(k_cov<0>);
  if (NS == 1) return go(k_cov<1>);
  return go(k_cov<2>);
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
      d.n[i] = (int)lv[i]->attrs.size();
      d.nk[i] = lv[i]->rel >= 0 ? lv[i]->nk : 0;
      d.V[i] = lv[i]->V.as<double>();
      tot += d.nk[i] * GP;
    }
    if (tot > 0) {
      k_cov_dims<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16), 256, 0, st>>>(d);
      launches_add(1);
    }
  }
  CovArgs g{};
  g.tmL = tmL;
  g.nrows = R.nrows;
  g.nx = nF;
  for (int i = 0; i < 8; i++) g.x[i] = i < nF ? (const double*)R.cols[R.find_attr(fattrs[i])].buf.p : nullptr;
  g.key[0] = R.fk_dense[L.child].as<int32_t>();
  g.key[1] = NS >= 1 ? R.fk_dense[A.child].as<int32_t>() : nullptr;
  g.key[2] = NS == 2 ? R.fk_dense[B.child].as<int32_t>() : nullptr;
  g.VA = NS >= 1 ? A.V.as<double>() : zeros.as<double>();
  char* z = zbuf.as<char>();
  g.work = reinterpret_cast<int*>(z);
  g.bcount = reinterpret_cast<int*>(z + 4);
  g.HA = reinterpret_cast<unsigned*>(z + off_HA);
  g.HL = reinterpret_cast<unsigned*>(z + off_HL);
  g.brec = brec.as<double>();
  g.bcap = bcap;
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
  k_cov_fin<<<FIN_BLOCKS, 256, 0, st>>>(f);
  k_cov_sum<<<(NPART + NFIN + 127) / 128, 128, 0, st>>>(partials.as<double>(), grid, finp.as<double>(), FIN_BLOCKS,
                                                         src.as<double>());
  k_cov_assemble<<<(nout + 127) / 128 + 1, 128, 0, st>>>(src.as<double>(), toff.as<int32_t>(), tidx.as<int32_t>(),
                                                         tcoef.as<double>(), nout, c->scalar_out.as<double>(),
                                                         NPART + 340 + 18, c->scalar_count.as<unsigned long long>());
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
  for (int ch : R.children) {
    const Rel& D = c->rels[ch];
    if (!D.children.empty() || !D.unique_key) return nullptr;
  }
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
      if (R.children[j] == o) {
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
  if (fc->NS >= 1) setup(fc->A, featured[featured.size() - 2]);
  if (fc->NS == 2) setup(fc->B, featured[0]);
  // buffers
  if (fc->zeros.alloc(GP * 8)) return nullptr;
  if (cudaMemset(fc->zeros.p, 0, fc->zeros.bytes)) return nullptr;
  CovLevel* lv[3] = {&fc->L, &fc->A, &fc->B};
  for (int i = 0; i < 3; i++) {
    CovLevel& l = *lv[i];
    if (l.rel < 0) continue;
    if (l.V.alloc((size_t)std::max<int64_t>(l.nk, 1) * GP * 8)) return nullptr;
    std::vector<const double*> cp;
    const Rel& D = c->rels[l.rel];
    for (int a : l.attrs) cp.push_back((const double*)D.cols[D.find_attr(a)].buf.p);
    if (l.colptrs.alloc(std::max<size_t>(cp.size(), 1) * sizeof(void*))) return nullptr;
    if (!cp.empty() && cudaMemcpy(l.colptrs.p, cp.data(), cp.size() * sizeof(void*), cudaMemcpyHostToDevice))
      return nullptr;
  }
  const int64_t nkA = fc->NS >= 1 ? fc->A.nk : 0;
  fc->off_HA = 16;
  fc->off_HL = (fc->off_HA + (size_t)nkA * 4 + 15) / 16 * 16;
  fc->zbytes = fc->off_HL + (size_t)std::max<int64_t>(fc->L.nk, 1) * 4;
  if (fc->zbuf.alloc(fc->zbytes)) return nullptr;
  const int64_t nitems = (R.nrows + CITEM - 1) / CITEM;
  fc->bcap = (int)std::min<int64_t>((fc->NS == 2 ? fc->B.nk : 0) + 2 * nitems + 64, INT32_MAX / BRW);
  if (fc->brec.alloc((size_t)fc->bcap * BRW * 8)) return nullptr;
  if (fc->partials.alloc((size_t)fc->grid * NPART * 8)) return nullptr;
  if (fc->finp.alloc((size_t)FIN_BLOCKS * NFIN * 8)) return nullptr;
  if (fc->src.alloc((size_t)(NPART + NFIN) * 8)) return nullptr;
  {  // gather4 tensor map over V_L [nk x GP] fp64, box GP x 1
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
    std::memset(&fc->tmL, 0, sizeof(fc->tmL));
    cuuint64_t dims[2] = {(cuuint64_t)GP, (cuuint64_t)std::max<int64_t>(fc->L.nk, 1)};
    cuuint64_t strides[1] = {(cuuint64_t)GP * 8};
    cuuint32_t box[2] = {(cuuint32_t)GP, 1};
    cuuint32_t estr[2] = {1, 1};
    if (encode(&fc->tmL, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, fc->L.V.p, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return nullptr;
  }
  // source index of G[a][b] (a, b: attr id or -1 = "1"); see the layout above k_cov_sum
  auto fidx = [](const std::vector<int>& v, int a) {
    for (size_t i = 0; i < v.size(); i++)
      if (v[i] == a) return (int)i;
    return -1;
  };
  const int F0 = NPART, RB = F0, TOT = F0 + 340, MB = F0 + 374, ML = F0 + 485, MA = F0 + 596;
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
      case 0: return TOT + 18;                 // 1·1 = count
      case 1: return TOT + j;                  // 1·x
      case 2: return TOT + 8 + j;              // 1·s_L
      case 3: return TOT + 24 + j;             // 1·s_A
      case 4: return MB + 1 + j;               // 1·s_B
      case 6: return i * 8 + j;                // x·x
      case 7: return 64 + i * 10 + j;          // x·s_L
      case 8: return 144 + i * 10 + j;         // x·s_A
      case 9: return RB + i * 10 + j;          // x·s_B
      case 12: return ML + 11 + i * 10 + j;    // s_L·s_L
      case 13: return 144 + (8 + i) * 10 + j;  // s_L·s_A
      case 14: return RB + (8 + i) * 10 + j;   // s_L·s_B
      case 18: return MA + 11 + i * 10 + j;    // s_A·s_A
      case 19: return RB + (24 + i) * 10 + j;  // s_A·s_B
      case 24: return MB + 11 + i * 10 + j;    // s_B·s_B
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
  return fc.release();
}

}  // namespace lmfao
