// counts.cu — the histogram path (§8 row (e)) for count batches: COUNT GROUP BY over at
// most two attributes per query (§3 "Mutual information" / Chow-Liu trees
// Q_S for S ⊆ {i, j}; BASELINE.json configs[3]).  Every UDAF of the batch is a
// constant (SUM(c) = c · COUNT), so only the per-cell row counts of the join are needed
// (the compaction multiplies by c).  With primary-key leaves and no dangling rows every
// root row joins exactly one row per child, so
//  * a query over attributes of one dimension D only is finished at the dimension:
//    count[cell(D row k)] += H_D[k] with H_D[k] = root rows with key k ("each aggregate to
//    its own root");
//  * every other query (a root attribute, or attributes of two relations) is counted per
//    root row: its cell from the codes of the row (root attributes) and of the rows it
//    joins (dimension attributes through the foreign keys), lanes holding the same cell
//    merged with __match_any_sync so a Zipf-hot cell takes one atomic per warp.
// The attribute codes of a row are loaded once (not once per query).
//  * views with a join key and a group-by attribute (V_{S->C}(F_i; 1) with F_i the
//    join key plus the query's group-by attributes below S; P:929's L(X_k, X_i; c), "the counts
//    for X_i in the context of each value for X_k"): the pair queries (a, b) with a in child D
//    whose b is the same attribute share one table V_D[k][b] = root rows with key k and code b,
//    counted per root row once instead of once per query; each query is then finished at D:
//    count[x, b] = Σ_{k: a(k) = x} V_D[k][b] (k_cnt_vfin).
#include <cstdlib>
#include <map>
#include <set>

#include "ctx.h"

namespace lmfao {
namespace {

constexpr int CN_ATTR = 24;   // attributes with codes
constexpr int CN_LEV = 8;     // root children
constexpr unsigned CFULL = 0xffffffffu;
#ifndef CNT_UNROLL_SMALL
#define CNT_UNROLL_SMALL 4
#endif
#ifndef CNT_UNROLL_BIG
#define CNT_UNROLL_BIG 1
#endif
constexpr int kUnrollSmall = CNT_UNROLL_SMALL, kUnrollBig = CNT_UNROLL_BIG;

struct CntQuery {
  int8_t a, b;      // attribute slots (b = -1: one attribute); slot nattr + 1 + l is the dense
                    // key of child l (a view's key)
  int8_t run;       // >= 0: both attributes belong to dimensions, the deeper at sort position
                    // `run`: the cell is constant over a run at that level, counted once per run
                    // (segment) with the run's length; -1: per row
  int32_t sa;       // cell = code_a * sa + code_b
  unsigned long long* counts;
  int32_t soff;     // >= 0: counted in the CTA's shared table at this offset (small tables)
  int32_t ncell;
};
constexpr int CN_SMEM_CELLS = 32768;  // shared counters per CTA (128 KB) for the smallest tables
constexpr int CN_THREADS = 1024;      // k_cnt_rows block (one CTA per SM with the counters above)
struct CntArgs {
  int64_t nrows;
  int nattr, nlev, nq;
  const int32_t* code[CN_ATTR];  // root: per row; child: per dense key
  int8_t lev[CN_ATTR];           // -1 root, else child index (into fk)
  // a child's attribute codes packed into one u32 per dense key (plan time, from the dimension
  // alone): one gather per child and row instead of one per attribute
  const uint32_t* pk[CN_LEV];    // null: the child's attributes are gathered one by one
  int8_t pshift[CN_ATTR];        // >= 0: code = (packed >> pshift) & pmask
  uint32_t pmask[CN_ATTR];
  const int32_t* fk[CN_LEV];
  unsigned* H[CN_LEV];           // rows per key of the children with dimension-only queries (null: none)
  const CntQuery* q;             // [nq] per-row queries
  int nsmall;                    // shared counters of the small tables
  int nsq;                       // queries [0, nsq) count in shared memory
  int nsq_row, ngq_row;          // ... of which [0, nsq_row) per row; global ones [nsq, ngq_row) per row
  int8_t pos[CN_LEV];            // sort position (P:1052 order) of each child
  int8_t at[CN_LEV];             // child at each sort position
  unsigned long long* total;     // COUNT
  unsigned* work;                // chunk counter (zeroed per run)
};
constexpr int CN_CHUNK = 8;

// Per root row: the codes of every attribute, then each per-row query's cell.  Queries come
// sorted: the nsmall_q shared-counter tables first, then the global ones, so both loops are
// branch-free; a one-attribute query reads the all-zero code row (slot nattr) as its second code.
__global__ void __launch_bounds__(1024) k_cnt_rows(const __grid_constant__ CntArgs a) {
  extern __shared__ __align__(16) unsigned char cnsm[];
  int4* sq = reinterpret_cast<int4*>(cnsm);  // {a, b, sa, soff}; the run level in soff's top byte
  unsigned long long** sp = reinterpret_cast<unsigned long long**>(cnsm + (size_t)a.nq * 16);
  // per warp: codes [nattr + 1][32] (row nattr = 0), dense keys [nlev][32], packed codes [nlev][32]
  const int wrows = a.nattr + 1 + 2 * a.nlev;
  int* wsm = reinterpret_cast<int*>(cnsm + (size_t)a.nq * 24 + ((a.nq & 1) ? 8 : 0));
  unsigned* stab = reinterpret_cast<unsigned*>(wsm + (blockDim.x >> 5) * 32 * wrows);
  for (int i = threadIdx.x; i < a.nq; i += blockDim.x) {
    const CntQuery q = a.q[i];
    sq[i] = make_int4(q.a | ((int)(q.run + 1) << 8), q.b >= 0 ? q.b : a.nattr, q.sa, q.soff);
    sp[i] = q.counts;
  }
  for (int i = threadIdx.x; i < a.nsmall; i += blockDim.x) stab[i] = 0u;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int* scode = wsm + wib * 32 * wrows + lane;  // scode[32 i] = code of attribute i
  int* skey = scode + 32 * (a.nattr + 1);      // skey[32 l] = dense key at level l
  unsigned* spk = reinterpret_cast<unsigned*>(skey + 32 * a.nlev);  // spk[32 l] = packed codes
  scode[32 * a.nattr] = 0;
  __syncthreads();
  unsigned long long tot = 0;
  // warps take chunks of CN_CHUNK 32-row batches dynamically (a static interleave left SM active
  // cycles 27 % apart on C4: the atomics' cost differs between SMs)
  const int64_t nbatch = (a.nrows + 31) >> 5;
  int64_t cb0 = 0, cb1 = 0;
  for (int64_t bi = 0;; bi++) {
    if (cb0 + bi >= cb1) {
      long long ch = 0;
      if (lane == 0) ch = (long long)atomicAdd(a.work, 1u);
      ch = __shfl_sync(CFULL, ch, 0);
      cb0 = ch * CN_CHUNK;
      if (cb0 >= nbatch) break;
      cb1 = cb0 + CN_CHUNK < nbatch ? cb0 + CN_CHUNK : nbatch;
      bi = 0;
    }
    const int64_t base = (cb0 + bi) * 32 - (threadIdx.x & ~31);  // (row = base + warp offset + lane)
    const int64_t row = base + (threadIdx.x & ~31) + lane;
    const bool v = row < a.nrows;
    tot += v ? 1 : 0;
    int key[CN_LEV];
#pragma unroll
    for (int l = 0; l < CN_LEV; l++)
      if (l < a.nlev) {
        key[l] = v ? a.fk[l][row] : 0;
        skey[32 * l] = key[l];
        if (a.pk[l]) spk[32 * l] = v ? a.pk[l][key[l]] : 0u;
      }
    // run starts per sort position p: a key at a position <= p differs from the previous row's
    // (the block's first row always starts; runs split at block edges are counted in parts)
    unsigned smask[CN_LEV];
    {
      bool chg = lane == 0;
      const int64_t rem = a.nrows - base - (threadIdx.x & ~31);
      const int nvb = rem < 32 ? (int)rem : 32;
#pragma unroll
      for (int p = 0; p < CN_LEV; p++) {
        if (p >= a.nlev) break;
        const int l = a.at[p];
        int kl = 0;
#pragma unroll
        for (int t = 0; t < CN_LEV; t++)
          if (t == l) kl = key[t];
        const int kp = __shfl_up_sync(CFULL, kl, 1);
        chg = chg || kp != kl;
        smask[p] = __ballot_sync(CFULL, v && chg) | (nvb < 32 ? (~0u << (nvb > 0 ? nvb : 0)) : 0u);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < CN_ATTR; i++) {
      if (i >= a.nattr) break;
      const int l = a.lev[i];
      int cv;
      if (a.pshift[i] >= 0) {
        cv = (int)((spk[32 * l] >> a.pshift[i]) & a.pmask[i]);
      } else {
        const int64_t idx = l < 0 ? row : (int64_t)skey[32 * l];
        cv = v ? a.code[i][idx] : 0;
      }
      scode[32 * i] = cv;
    }
    __syncwarp();
    // a lane starting a run segment at position p: the segment's rows in this block
    auto seg_len = [&](int p, bool& start) -> unsigned {
      unsigned m = 0;
#pragma unroll
      for (int t = 0; t < CN_LEV; t++)
        if (t == p) m = smask[t];
      start = v && ((m >> lane) & 1u);
      const unsigned above = m & ~((2u << lane) - 1u);
      return (unsigned)((above ? __ffs(above) - 1 : 32) - lane);
    };
    // rows per key of the children that have dimension-only queries: one atomic per run segment
    // of the child's sort position (the key is constant over it)
#pragma unroll
    for (int l = 0; l < CN_LEV; l++) {
      if (l >= a.nlev) break;
      if (!a.H[l]) continue;
      bool start;
      const unsigned len = seg_len(a.pos[l], start);
      if (start) gred_add(&a.H[l][key[l]], len);
    }
    // small tables: the CTA's shared counters (native shared atomics)
#pragma unroll kUnrollSmall
    for (int qi = 0; qi < a.nsq_row; qi++) {
      const int4 d = sq[qi];
      const int ca = scode[32 * (d.x & 255)], cb = scode[32 * d.y];
      if (v) atomicAdd(&stab[d.w + ca * d.z + cb], 1u);
    }
    for (int qi = a.nsq_row; qi < a.nsq; qi++) {  // per run segment
      const int4 d = sq[qi];
      bool start;
      const unsigned len = seg_len((d.x >> 8) - 1, start);
      if (start) atomicAdd(&stab[d.w + scode[32 * (d.x & 255)] * d.z + scode[32 * d.y]], len);
    }
    // the others: lanes holding the same cell merged, one global atomic per distinct cell
#pragma unroll kUnrollBig
    for (int qi = a.nsq; qi < a.ngq_row; qi++) {
      const int4 d = sq[qi];
      const int ca = scode[32 * (d.x & 255)], cb = scode[32 * d.y];
      const int cell = v ? ca * d.z + cb : -1 - lane;
      const unsigned peers = __match_any_sync(CFULL, cell);
      if (v && (__ffs(peers) - 1) == lane) gred_add(&sp[qi][cell], (unsigned long long)__popc(peers));
    }
    for (int qi = a.ngq_row; qi < a.nq; qi++) {  // per run segment
      const int4 d = sq[qi];
      bool start;
      const unsigned len = seg_len((d.x >> 8) - 1, start);
      if (start) gred_add(&sp[qi][scode[32 * (d.x & 255)] * d.z + scode[32 * d.y]], (unsigned long long)len);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(CFULL, tot, o);
  if (lane == 0 && a.total) atomicAdd(a.total, tot);
  if (a.nsmall == 0) return;
  __syncthreads();
  for (int qi = 0; qi < a.nsq; qi++) {  // the shared counters -> the global tables
    const int4 d = sq[qi];
    const int ncell = a.q[qi].ncell;
    for (int c = threadIdx.x; c < ncell; c += blockDim.x) {
      const unsigned n = stab[d.w + c];
      if (n) gred_add(&sp[qi][c], (unsigned long long)n);
    }
  }
}

// Scalar queries of the batch: every UDAF is a constant c, value = c * COUNT.
__global__ void k_cnt_scalar(const double* __restrict__ coef, int nout, const unsigned long long* __restrict__ total,
                             double* __restrict__ out) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x)
    out[o] = coef[o] * (double)*total;
}

// Dimension-only queries: count[cell(k)] += H[k] over the child's dense keys.
struct CntDimQuery {
  const int32_t* ca;
  const int32_t* cb;  // null: one attribute
  int32_t sa;
  int lev;
  unsigned long long* counts;
};
struct CntDimArgs {
  int nq;
  const CntDimQuery* q;
  const unsigned* H[CN_LEV];
  int64_t nk[CN_LEV];
};
__global__ void k_cnt_dims(const __grid_constant__ CntDimArgs a) {
  const CntDimQuery q = a.q[blockIdx.y];
  const unsigned* H = a.H[q.lev];
  const int64_t nk = a.nk[q.lev];
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nk; k += (int64_t)gridDim.x * blockDim.x) {
    const unsigned h = H[k];
    if (!h) continue;
    const int cell = q.ca[k] * q.sa + (q.cb ? q.cb[k] : 0);
    gred_add(&q.counts[cell], (unsigned long long)h);
  }
}

// Queries finished from a view V_D[k][b] (cells [nk x domb]): count[x, b] = Σ_{k: a(k) = x}
// V_D[k][b], the keys of D grouped by their code x of the query's attribute a (plan time, from
// the dimension alone) and cut into pieces of at most CN_VPIECE keys (a Zipf-hot code owns
// thousands of keys: one serial sum would be a chain of dependent loads).  One warp per (piece,
// 32 consecutive b): coalesced reads of the view rows, one RED per cell and piece.
constexpr int CN_VPIECE = 16;
struct CntVQuery {
  const unsigned long long* view;
  int32_t domb;
  int32_t npiece;
  const int4* piece;     // [npiece] {x, first key index, end key index, 0} into kord
  const int32_t* kord;   // keys of D ordered by code
  int32_t first;         // 1: a is the query's first attribute (cell = x * sa + b), 0: cell = b * sa + x
  int32_t sa;
  unsigned long long* counts;
};
struct CntVArgs {
  int nv;  // views (for the plan summary)
  int nq;  // served queries
  const CntVQuery* q;
};
__global__ void __launch_bounds__(256) k_cnt_vfin(const __grid_constant__ CntVArgs a) {
  const CntVQuery q = a.q[blockIdx.y];
  const int lane = threadIdx.x & 31;
  const int nbc = (q.domb + 31) >> 5;
  const int ntask = q.npiece * nbc;
  for (int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < ntask; t += (gridDim.x * blockDim.x) >> 5) {
    const int pc = t / nbc;
    const int b = (t - pc * nbc) * 32 + lane;
    if (b >= q.domb) continue;
    const int4 p = q.piece[pc];
    unsigned long long sum = 0;
#pragma unroll 4
    for (int i = p.y; i < p.z; i++) sum += q.view[(int64_t)q.kord[i] * q.domb + b];
    if (sum) gred_add(&q.counts[q.first ? (int64_t)p.x * q.sa + b : (int64_t)b * q.sa + p.x], sum);
  }
}

struct FastCounts : FastPaths {
  CntArgs ra{};
  CntDimArgs da{};
  CntVArgs va{};
  DevBuf dq, ddq, Hbuf, scoef, vbuf, vqbuf;
  std::vector<DevBuf> kgroups;  // per served query: pieces | kord
  std::vector<DevBuf> pkbuf;    // packed codes per child
  DevBuf workbuf;
  int64_t vbytes = 0;
  int nscalar = 0;
  int64_t hwords = 0;
  int nrowq = 0, ndimq = 0, nvq = 0, grid = 148 * 8, threads = 256, cell_cap = 0;
  size_t smem = 0;
  bool scalar = false;
  std::string describe() const override {
    char b[160];
    std::snprintf(b, sizeof b,
                  "{\"kind\": \"counts\", \"attrs\": %d, \"row_queries\": %d, \"run_queries\": %d, \"dim_queries\": %d, "
                  "\"views\": %d, \"view_queries\": %d}",
                  ra.nattr, nrowq, (ra.nsq - ra.nsq_row) + (ra.nq - ra.ngq_row), ndimq, va.nv, nvq);
    return b;
  }
  bool handles_group(int) const override { return true; }
  bool handles_all_groups() const override { return true; }
  bool skip_generic_views() const override { return true; }
  int run(lmfao_ctx* c, const NodeArgs& root, cudaStream_t st, bool& scalar_done) override;
};

int FastCounts::run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool& scalar_done) {
  for (auto& gp : c->groups) CUDA_TRY(cudaMemsetAsync(gp.counts.p, 0, gp.ncells * 8, st));
  if (hwords) CUDA_TRY(cudaMemsetAsync(Hbuf.p, 0, hwords * 4, st));
  if (vbytes) CUDA_TRY(cudaMemsetAsync(vbuf.p, 0, vbytes, st));
  CUDA_TRY(cudaMemsetAsync(workbuf.p, 0, 4, st));
  CntArgs a = ra;
  a.nrows = c->rels[c->root].nrows;
  a.work = workbuf.as<unsigned>();
  a.total = nullptr;
  if (scalar) {
    CUDA_TRY(cudaMemsetAsync(c->scalar_count.p, 0, 8, st));
    a.total = c->scalar_count.as<unsigned long long>();
  }
  scan_timer_begin(c, st);
  if (a.nrows > 0) {
    k_cnt_rows<<<grid, threads, std::max<size_t>(smem, 16), st>>>(a);
    launches_add(1);
  }
  scan_timer_end(c, st);
  if (va.nv > 0) {
    k_cnt_vfin<<<dim3(64, (unsigned)va.nq), 256, 0, st>>>(va);
    launches_add(1);
  }
  if (ndimq > 0) {
    k_cnt_dims<<<dim3(64, (unsigned)ndimq), 256, 0, st>>>(da);
    launches_add(1);
  }
  if (scalar) {  // every scalar UDAF is a constant c: value = c * COUNT
    k_cnt_scalar<<<(nscalar + 127) / 128 + 1, 128, 0, st>>>(scoef.as<double>(), nscalar,
                                                           c->scalar_count.as<unsigned long long>(),
                                                           c->scalar_out.as<double>());
    launches_add(1);
    scalar_done = true;
  }
  return cudaGetLastError();
}

}  // namespace

// Planner hook: every UDAF of every query is a constant (SUM(c)), every group-by query has
// one or two attributes, scalar queries only count, and the root's children are
// primary-key leaves.  Otherwise nullptr.
FastPaths* plan_counts(lmfao_ctx* c) {
  if (c->groups.empty()) return nullptr;
  const Rel& R = c->rels[c->root];
  if (R.children.size() > (size_t)CN_LEV) return nullptr;
  for (int ch : R.children)
    if (!c->rels[ch].children.empty() || !c->rels[ch].unique_key) return nullptr;
  auto constant_udaf = [](const std::vector<QProduct>& u) {
    for (auto& p : u)
      for (auto& f : p.f)
        if (f.kind != LMFAO_F_CONST) return false;
    return true;
  };
  for (auto& Q : c->queries)
    for (auto& u : Q.udafs)
      if (!constant_udaf(u)) return nullptr;
  auto level_of = [&](int attr) -> int {
    const int o = c->owner[attr];
    if (o == c->root) return -1;
    for (size_t j = 0; j < R.children.size(); j++)
      if (R.children[j] == o) return (int)j;
    return -2;
  };
  std::unique_ptr<FastCounts> fc(new FastCounts());
  CntArgs& a = fc->ra;
  a.nlev = (int)R.children.size();
  // Tables whose cell is a function of the keys at sort positions <= p (both attributes in
  // dimensions, or a view's key and a dimension attribute) are counted once per run segment at
  // position p with the segment's length (registration at the lowest attribute of
  // the order that fixes the view's group-by attributes) when p <= LMFAO_CNT_RUN_POS (default 1:
  // long runs, no __match_any_sync); deeper ones per row, where warp-merged atomics measured
  // faster (C4: 4.42-4.76 vs 4.24 ms with every cross-dimension table per run).
  // LMFAO_CNT_RUNS=1: every such table per run, 0: none.
  const char* ro = std::getenv("LMFAO_CNT_RUNS");
  const int run_mode = ro ? (ro[0] == '1' ? 1 : 0) : 2;
  const bool run_off = run_mode == 0;
  const char* rpe = std::getenv("LMFAO_CNT_RUN_POS");
  const int run_pos = rpe ? std::atoi(rpe) : 1;
  for (size_t p = 0; p < c->levels.size(); p++) {
    a.at[p] = (int8_t)c->levels[p];
    a.pos[c->levels[p]] = (int8_t)p;
  }
  for (int j = 0; j < a.nlev; j++) a.fk[j] = R.fk_dense[j].as<int32_t>();
  std::map<int, int> slot;  // attr -> code slot
  int64_t slot_dom[CN_ATTR] = {};
  std::vector<CntQuery> rq;
  std::vector<CntDimQuery> dq;
  std::vector<int> needH(a.nlev, 0);
  // Views V_D[k][b]: a two-attribute query whose attributes lie in two
  // different relations, at least one a root child D, may take a candidate view (D the child
  // holding one attribute, b the other; nkeys(D) x |dom b| cells, at most LMFAO_CNT_VIEW_CELLS,
  // default 2^24); views are chosen greedily, the one serving the most queries first, while it
  // serves at least two (one table counted per row instead of two or more).  What a per-row
  // table costs is its atomics, and a view keyed by a deep level has about as many distinct cells
  // per warp as rows, so views are keyed only by children at sort position <= LMFAO_CNT_VIEW_POS
  // (default 0: the first level, long runs of equal keys) and take only queries of more than
  // LMFAO_CNT_VIEW_MIN cells (default 0).  C4: 4.18 -> 4.00 ms with the defaults;
  // position <= 1 4.28, position <= 1 and only global-sized queries 4.26.  LMFAO_CNT_VIEWS=0: off.
  struct VPick {
    int view = -1, side = 0;  // the view, and which of the query's attributes is D's
  };
  std::vector<VPick> vpick(c->groups.size());
  std::vector<std::pair<int, int>> views;  // (child level, attribute b)
  std::vector<int64_t> vcells;
  {
    const char* vo = std::getenv("LMFAO_CNT_VIEWS");
    const char* vc = std::getenv("LMFAO_CNT_VIEW_CELLS");
    const int64_t vcap = vc ? std::atoll(vc) : ((int64_t)1 << 24);
    const char* vmn = std::getenv("LMFAO_CNT_VIEW_MIN");
    const int64_t vmin = vmn ? std::atoll(vmn) : 0;
    const char* vps = std::getenv("LMFAO_CNT_VIEW_POS");
    const int vpos = vps ? std::atoi(vps) : 0;
    std::map<std::pair<int, int>, std::vector<std::pair<size_t, int>>> vm;
    if (!(vo && vo[0] == '0'))
      for (size_t gi = 0; gi < c->groups.size(); gi++) {
        const GroupPlan& gp = c->groups[gi];
        const Query& Q = c->queries[gp.q];
        if (Q.gb.size() != 2 || gp.ncells > INT32_MAX || gp.ncells <= vmin) continue;
        const int l0 = level_of(Q.gb[0]), l1 = level_of(Q.gb[1]);
        if (l0 == -2 || l1 == -2 || l0 == l1) continue;
        const int lv2[2] = {l0, l1};
        const int64_t dom[2] = {gp.ncells / std::max<int64_t>(gp.g.stride[0], 1), gp.g.stride[0]};
        for (int i = 0; i < 2; i++) {
          if (lv2[i] < 0 || a.pos[lv2[i]] > vpos) continue;
          const int64_t cells = std::max<int64_t>(c->rels[R.children[lv2[i]]].nkeys, 1) * dom[1 - i];
          if (cells > vcap || cells > INT32_MAX) continue;
          vm[{lv2[i], Q.gb[1 - i]}].push_back({gi, i});
        }
      }
    // greedy cover: the candidate serving the most unassigned queries (ties: fewer cells) while
    // it serves at least two
    auto cells_of = [&](const std::pair<int, int>& key, const std::pair<size_t, int>& e) {
      const GroupPlan& gp0 = c->groups[e.first];
      const int64_t domb = e.second == 0 ? gp0.g.stride[0] : gp0.ncells / gp0.g.stride[0];
      return std::max<int64_t>(c->rels[R.children[key.first]].nkeys, 1) * domb;
    };
    for (;;) {
      const std::pair<int, int>* bk = nullptr;
      size_t bn = 0;
      int64_t bcells = 0;
      for (auto& kv : vm) {
        size_t n = 0;
        for (auto& e : kv.second) n += vpick[e.first].view < 0 ? 1 : 0;
        if (n < 2) continue;
        const int64_t cl = cells_of(kv.first, kv.second[0]);
        if (!bk || n > bn || (n == bn && cl < bcells)) bk = &kv.first, bn = n, bcells = cl;
      }
      if (!bk) break;
      const int v = (int)views.size();
      views.push_back(*bk);
      vcells.push_back(bcells);
      for (auto& e : vm[*bk])
        if (vpick[e.first].view < 0) vpick[e.first] = VPick{v, e.second};
    }
  }
  std::vector<CntVQuery> vqs;
  std::vector<int> vq_view;
  std::vector<int> vslot_b(views.size(), -1);
  for (size_t gi = 0; gi < c->groups.size(); gi++) {
    GroupPlan& gp = c->groups[gi];
    const Query& Q = c->queries[gp.q];
    if (Q.gb.empty() || Q.gb.size() > 2) return nullptr;
    int lv[2] = {0, 0};
    for (size_t i = 0; i < Q.gb.size(); i++) {
      lv[i] = level_of(Q.gb[i]);
      if (lv[i] == -2) return nullptr;
    }
    if (gp.ncells > INT32_MAX) return nullptr;
    const bool dim_only = lv[0] >= 0 && (Q.gb.size() == 1 || lv[1] == lv[0]);
    if (dim_only) {
      CntDimQuery d{};
      d.ca = gp.g.code[0];
      d.cb = Q.gb.size() == 2 ? gp.g.code[1] : nullptr;
      d.sa = (int32_t)gp.g.stride[0];
      d.lev = lv[0];
      d.counts = gp.counts.as<unsigned long long>();
      dq.push_back(d);
      needH[lv[0]] = 1;
      continue;
    }
    if (vpick[gi].view >= 0) {  // finished from its view (k_cnt_vfin)
      const int v = vpick[gi].view, sd = vpick[gi].side;
      CntVQuery vq{};
      const int32_t* ca = gp.g.code[sd];
      vq.first = sd == 0 ? 1 : 0;
      vq.sa = (int32_t)gp.g.stride[0];
      vq.counts = gp.counts.as<unsigned long long>();
      {
        const int64_t nk = std::max<int64_t>(c->rels[R.children[views[v].first]].nkeys, 1);
        vq.domb = (int32_t)(vcells[v] / nk);
        // the keys of D grouped by their code of a (counting sort on the host, plan time), in
        // pieces of at most CN_VPIECE keys
        const int32_t doma = (int32_t)(sd == 0 ? gp.ncells / gp.g.stride[0] : gp.g.stride[0]);
        const int64_t nkr = c->rels[R.children[views[v].first]].nkeys;
        std::vector<int32_t> code(nkr), off(doma + 1, 0), ord(std::max<int64_t>(nkr, 1));
        if (nkr && (cudaMemcpyAsync(code.data(), ca, nkr * 4, cudaMemcpyDeviceToHost, c->stream) ||
                    cudaStreamSynchronize(c->stream)))
          return nullptr;
        for (int32_t x : code) off[x + 1]++;
        for (int x = 0; x < doma; x++) off[x + 1] += off[x];
        std::vector<int32_t> pos(off.begin(), off.end() - 1);
        for (int64_t k = 0; k < nkr; k++) ord[pos[code[k]]++] = (int32_t)k;
        std::vector<int4> pieces;
        for (int x = 0; x < doma; x++)
          for (int i = off[x]; i < off[x + 1]; i += CN_VPIECE)
            pieces.push_back(make_int4(x, i, std::min(i + CN_VPIECE, off[x + 1]), 0));
        vq.npiece = (int32_t)pieces.size();
        DevBuf kb;
        const size_t pb = std::max<size_t>(pieces.size(), 1) * sizeof(int4);
        if (kb.alloc(pb + ord.size() * 4) ||
            (!pieces.empty() && cudaMemcpyAsync(kb.p, pieces.data(), pieces.size() * sizeof(int4),
                                                cudaMemcpyHostToDevice, c->stream)) ||
            cudaMemcpyAsync((char*)kb.p + pb, ord.data(), ord.size() * 4, cudaMemcpyHostToDevice, c->stream) ||
            cudaStreamSynchronize(c->stream))
          return nullptr;
        vq.piece = kb.as<int4>();
        vq.kord = reinterpret_cast<const int32_t*>((const char*)kb.p + pb);
        fc->kgroups.push_back(std::move(kb));
      }
      vqs.push_back(vq);
      vq_view.push_back(v);
      if (vslot_b[v] < 0) {  // the view's attribute b needs a code slot
        auto it = slot.find(Q.gb[1 - sd]);
        if (it == slot.end()) {
          if ((int)slot.size() == CN_ATTR) return nullptr;
          const int s = (int)slot.size();
          slot[Q.gb[1 - sd]] = s;
          a.code[s] = gp.g.code[1 - sd];
          a.lev[s] = (int8_t)lv[1 - sd];
          slot_dom[s] = gp.d.radix[1 - sd];
          it = slot.find(Q.gb[1 - sd]);
        }
        vslot_b[v] = it->second;
      }
      continue;
    }
    CntQuery q{};
    for (size_t i = 0; i < Q.gb.size(); i++) {
      auto it = slot.find(Q.gb[i]);
      if (it == slot.end()) {
        if ((int)slot.size() == CN_ATTR) return nullptr;
        const int s = (int)slot.size();
        slot[Q.gb[i]] = s;
        a.code[s] = gp.g.code[i];
        a.lev[s] = (int8_t)lv[i];
        slot_dom[s] = gp.d.radix[i];
        it = slot.find(Q.gb[i]);
      }
      if (i == 0) q.a = (int8_t)it->second;
      else q.b = (int8_t)it->second;
    }
    if (Q.gb.size() == 1) q.b = -1;
    q.run = -1;
    if (Q.gb.size() == 2 && lv[0] >= 0 && lv[1] >= 0 && !run_off) {  // two dimensions: per run at the deeper one
      int p0 = 0, p1 = 0;
      for (size_t p = 0; p < c->levels.size(); p++) {
        if (c->levels[p] == lv[0]) p0 = (int)p;
        if (c->levels[p] == lv[1]) p1 = (int)p;
      }
      q.run = (int8_t)std::max(p0, p1);
    }
    q.sa = (int32_t)gp.g.stride[0];
    q.counts = gp.counts.as<unsigned long long>();
    q.soff = -1;
    q.ncell = (int32_t)gp.ncells;
    rq.push_back(q);
  }
  a.nattr = (int)slot.size();
  if (fc->workbuf.alloc(64)) return nullptr;
  // packed codes per child: its attributes' codes in one u32 per dense key while the bits fit
  // (LMFAO_CNT_PACK=0: off)
  for (int i = 0; i < CN_ATTR; i++) a.pshift[i] = -1;
  {
    const char* pe = std::getenv("LMFAO_CNT_PACK");
    const bool pack_on = !(pe && pe[0] == '0');
    for (int l = 0; l < a.nlev && pack_on; l++) {
      std::vector<int> at;
      int bits = 0;
      for (int i = 0; i < a.nattr; i++) {
        if (a.lev[i] != l) continue;
        int b = 1;
        while (((int64_t)1 << b) < slot_dom[i]) b++;
        if (bits + b > 32) continue;
        a.pshift[i] = (int8_t)bits;
        a.pmask[i] = b == 32 ? 0xffffffffu : ((1u << b) - 1u);
        bits += b;
        at.push_back(i);
      }
      if (at.size() < 2) {
        for (int i : at) a.pshift[i] = -1;
        continue;
      }
      const int64_t nk = c->rels[R.children[l]].nkeys;
      std::vector<uint32_t> pk(std::max<int64_t>(nk, 1), 0u);
      std::vector<int32_t> cd(std::max<int64_t>(nk, 1));
      for (int i : at) {
        if (nk && (cudaMemcpyAsync(cd.data(), a.code[i], nk * 4, cudaMemcpyDeviceToHost, c->stream) ||
                   cudaStreamSynchronize(c->stream)))
          return nullptr;
        for (int64_t k = 0; k < nk; k++) pk[k] |= (uint32_t)cd[k] << a.pshift[i];
      }
      DevBuf pb;
      if (pb.alloc(pk.size() * 4) ||
          cudaMemcpyAsync(pb.p, pk.data(), pk.size() * 4, cudaMemcpyHostToDevice, c->stream) ||
          cudaStreamSynchronize(c->stream))
        return nullptr;
      a.pk[l] = pb.as<uint32_t>();
      fc->pkbuf.push_back(std::move(pb));
    }
  }
  // one per-row table per view: cell = (dense key of D) * |dom b| + code b; the key of child l is
  // the kernel's code slot nattr + 1 + l
  if (fc->vbuf.alloc(std::max<int64_t>(1, [&] {
        int64_t t = 0;
        for (int64_t x : vcells) t += x;
        return t;
      }()) * 8))
    return nullptr;
  {
    int64_t off = 0;
    std::vector<const unsigned long long*> vptr(views.size());
    for (size_t v = 0; v < views.size(); v++) {
      CntQuery q{};
      q.a = (int8_t)(a.nattr + 1 + views[v].first);
      q.b = (int8_t)vslot_b[v];
      q.run = -1;
      const int lb = a.lev[vslot_b[v]];
      if (lb >= 0 && !run_off) q.run = (int8_t)std::max<int>(a.pos[views[v].first], a.pos[lb]);
      q.sa = (int32_t)(vcells[v] / std::max<int64_t>(c->rels[R.children[views[v].first]].nkeys, 1));
      q.counts = fc->vbuf.as<unsigned long long>() + off;
      vptr[v] = q.counts;
      q.soff = -1;
      q.ncell = (int32_t)vcells[v];
      rq.push_back(q);
      off += vcells[v];
    }
    fc->vbytes = off * 8;
    for (size_t i = 0; i < vqs.size(); i++) vqs[i].view = vptr[vq_view[i]];
    fc->va.nv = (int)views.size();
    fc->va.nq = fc->nvq = (int)vqs.size();
    if (fc->vqbuf.alloc(std::max<size_t>(vqs.size(), 1) * sizeof(CntVQuery))) return nullptr;
    if (!vqs.empty() && cudaMemcpyAsync(fc->vqbuf.p, vqs.data(), vqs.size() * sizeof(CntVQuery),
                                        cudaMemcpyHostToDevice, c->stream))
      return nullptr;
    fc->va.q = fc->vqbuf.as<CntVQuery>();
  }
  a.nq = (int)rq.size();
  {
    // one CTA of CN_THREADS per SM: the per-warp code rows plus as many small tables as fit the
    // shared budget (C4: 38 of its 60 per-row tables; 256 threads with 12288 cells: 30 tables,
    // 6.39 ms -> 4.33 ms).  LMFAO_CNT_THREADS / LMFAO_CNT_SMEM_CELLS: A/B knobs.
    const char* th = std::getenv("LMFAO_CNT_THREADS");
    fc->threads = th ? std::max(32, std::min(1024, std::atoi(th) / 32 * 32)) : CN_THREADS;
    int optin = 232448;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    const int64_t avail = (int64_t)optin - 2048 - (int64_t)rq.size() * 24;
    const int64_t rows = a.nattr + 1 + 2 * a.nlev;
    while (fc->threads > 64 && fc->threads * 4 * rows > avail / 2) fc->threads /= 2;
    fc->cell_cap = (int)std::max<int64_t>(0, (avail - fc->threads * 4 * rows) / 4);
  }
  {  // the smallest per-row tables get shared counters (no warp matching, no global atomics per row)
    const char* sc = std::getenv("LMFAO_CNT_SMEM_CELLS");
    const int budget = std::min(sc ? std::atoi(sc) : CN_SMEM_CELLS, fc->cell_cap);
    std::vector<int> order(rq.size());
    for (size_t i = 0; i < rq.size(); i++) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return rq[x].ncell < rq[y].ncell; });
    int used = 0;
    for (int i : order)
      if (used + rq[i].ncell <= budget) {
        rq[i].soff = used;
        used += rq[i].ncell;
      }
    a.nsmall = used;
    // shared-counter queries first (k_cnt_rows loops over the kinds separately), per-row before
    // per-run in each
    std::stable_partition(rq.begin(), rq.end(), [](const CntQuery& q) { return q.soff >= 0; });
    a.nsq = 0;
    for (auto& q : rq) a.nsq += q.soff >= 0 ? 1 : 0;
    if (run_mode == 2)
      for (auto& q : rq)
        if (q.run > run_pos) q.run = -1;
    std::stable_partition(rq.begin(), rq.begin() + a.nsq, [](const CntQuery& q) { return q.run < 0; });
    std::stable_partition(rq.begin() + a.nsq, rq.end(), [](const CntQuery& q) { return q.run < 0; });
    a.nsq_row = a.ngq_row = 0;
    for (int i = 0; i < a.nsq; i++) a.nsq_row += rq[i].run < 0 ? 1 : 0;
    a.ngq_row = a.nsq;
    for (size_t i = a.nsq; i < rq.size(); i++) a.ngq_row += rq[i].run < 0 ? 1 : 0;
  }
  fc->nrowq = (int)rq.size();
  fc->ndimq = (int)dq.size();
  // H buffers
  int64_t off = 0;
  std::vector<int64_t> hoff(a.nlev, -1);
  for (int j = 0; j < a.nlev; j++)
    if (needH[j]) {
      hoff[j] = off;
      off += std::max<int64_t>(c->rels[R.children[j]].nkeys, 1);
    }
  fc->hwords = off;
  if (fc->Hbuf.alloc(std::max<int64_t>(off, 1) * 4)) return nullptr;
  for (int j = 0; j < a.nlev; j++) {
    a.H[j] = hoff[j] >= 0 ? fc->Hbuf.as<unsigned>() + hoff[j] : nullptr;
    fc->da.H[j] = a.H[j];
    fc->da.nk[j] = c->rels[R.children[j]].nkeys;
  }
  // scalar outputs (constants times COUNT), in the order of the scalar program
  std::vector<double> sc;
  for (int qi : c->scalar_queries)
    for (auto& u : c->queries[qi].udafs) {
      double cf = 0.0;
      for (auto& p : u) {
        double v = p.coeff;
        for (auto& f : p.f) v *= f.param;
        cf += v;
      }
      sc.push_back(cf);
    }
  fc->scalar = !c->scalar_queries.empty();
  fc->nscalar = (int)sc.size();
  cudaStream_t st = c->stream;
  if (fc->scoef.alloc(std::max<size_t>(sc.size(), 1) * 8)) return nullptr;
  if (!sc.empty() && cudaMemcpyAsync(fc->scoef.p, sc.data(), sc.size() * 8, cudaMemcpyHostToDevice, st)) return nullptr;
  if (fc->dq.alloc(std::max<size_t>(rq.size(), 1) * sizeof(CntQuery)) ||
      fc->ddq.alloc(std::max<size_t>(dq.size(), 1) * sizeof(CntDimQuery)))
    return nullptr;
  if (!rq.empty() && cudaMemcpyAsync(fc->dq.p, rq.data(), rq.size() * sizeof(CntQuery), cudaMemcpyHostToDevice, st))
    return nullptr;
  if (!dq.empty() &&
      cudaMemcpyAsync(fc->ddq.p, dq.data(), dq.size() * sizeof(CntDimQuery), cudaMemcpyHostToDevice, st))
    return nullptr;
  a.q = fc->dq.as<CntQuery>();
  fc->da.nq = (int)dq.size();
  fc->da.q = fc->ddq.as<CntDimQuery>();
  if (cudaStreamSynchronize(st)) return nullptr;
  fc->smem = rq.size() * 24 + ((rq.size() & 1) ? 8 : 0) + (size_t)fc->threads * 4 * (a.nattr + 1 + 2 * a.nlev) +
             (size_t)a.nsmall * 4;
  // (static scode + dynamic above 48 KB needs the opt-in; the attribute is per device and
  // process-wide there: keep each device's max)
  if (ensure_smem_attr((const void*)k_cnt_rows, fc->smem)) return nullptr;
  {
    int per_sm = 0, nsm = 148;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cnt_rows, fc->threads, fc->smem) || per_sm < 1)
      per_sm = 1;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device);
    fc->grid = nsm * std::min(per_sm, 2048 / fc->threads);
  }
  return fc.release();
}

}  // namespace lmfao
