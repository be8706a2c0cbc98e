// poly.cu — scalar batches of polynomial aggregates on the FP64 tensor pipe (§8(f) NEXT-2:
// degree-2 polynomial regression, §3: the covariance of the degree-2
// monomials, i.e. sums of products of up to four features).
//
// Every product of the batch is split into two "halves", monomials of at most two features,
// from a small set H = {1, h_1 .. h_n} (n <= 24) chosen at plan time; the batch is then entries of
// the Gram matrix G = Σ_rows u u^T with u = [h_1(row) .. h_n(row)] — a dense contraction with K =
// the rows, as FP64 DMMA m8n8k4 tiles: per 4-row group one DMMA per (t, s) tile pair, t <= s.
// The features are root columns or columns of primary-key children of the root (one joined row
// per root row, dangling rows dropped at prepare), read once per 32-row block into shared
// memory (the children's through the dense foreign keys, L2-resident), the halves formed there.
// Work: contiguous per-warp ranges of blocks (static, equal rows), per-warp partial tiles
// summed in fixed order: deterministic.  (The interpreted path spent 10.9 ms on C2's 120-product
// degree-2 batch over four features.)
#include <cstdlib>
#include <map>

#include "ctx.h"

namespace lmfao {
namespace {

constexpr int PL_ATTR = 8;     // distinct features
constexpr int PL_MAXT = 3;     // tiles of 8 halves (n <= 24)
constexpr int PL_WARPS = 8;
constexpr unsigned PFULL = 0xffffffffu;

struct PolyArgs {
  int64_t nrows;
  int nattr, nt;
  const void* col[PL_ATTR];     // root column, or the child's column indexed by its dense key
  const int32_t* fk[PL_ATTR];   // null: root column
  int isint[PL_ATTR];
  int8_t ha[PL_MAXT * 8], hb[PL_MAXT * 8];  // half h = feature ha (or 1 if -1) × feature hb (or 1)
  double* partials;             // [warps][tile pairs × 64 | NT × 8 linear sums]
};
// The constant half 1 is not a tile column: its Gram row is the linear sums Σ h (lane sums, one
// DADD per half and group) and its corner the row count.  So C2-like covariance batches over 8
// features (halves 1, x_1..x_8) need one tile, one DMMA per 4-row group.

__device__ __forceinline__ void pdmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(PL_WARPS * 32) k_poly(const __grid_constant__ PolyArgs a) {
  __shared__ double fv[PL_WARPS][PL_ATTR][33];  // per warp: the block's feature values [attr][row]
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, k = lane & 3, m = lane >> 2;
  const int64_t nblk = (a.nrows + 31) / 32;
  const int64_t gw = (int64_t)blockIdx.x * PL_WARPS + wib, NW = (int64_t)gridDim.x * PL_WARPS;
  const int64_t b0 = nblk * gw / NW, b1 = nblk * (gw + 1) / NW;
  double acc[NT * (NT + 1) / 2][2], lin[NT];
#pragma unroll
  for (int t = 0; t < NT * (NT + 1) / 2; t++) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
  for (int t = 0; t < NT; t++) lin[t] = 0.0;
  double (*f)[33] = fv[wib];
  // the block's feature values, loaded one block ahead
  auto load = [&](int64_t b, double (&x)[PL_ATTR]) {
    const int64_t row = 32 * b + lane;
    const bool v = row < a.nrows;
#pragma unroll
    for (int i = 0; i < PL_ATTR; i++) {
      x[i] = 0.0;
      if (i < a.nattr && v) {
        const int64_t r = a.fk[i] ? (int64_t)a.fk[i][row] : row;
        x[i] = a.isint[i] ? (double)reinterpret_cast<const int32_t*>(a.col[i])[r] : reinterpret_cast<const double*>(a.col[i])[r];
      }
    }
  };
  double nx[PL_ATTR];
  if (b0 < b1) load(b0, nx);
  for (int64_t b = b0; b < b1; b++) {
#pragma unroll
    for (int i = 0; i < PL_ATTR; i++) f[i][lane] = nx[i];
    if (b + 1 < b1) load(b + 1, nx);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; j++) {
      const int r = 4 * j + k;
      const double one = (32 * b + r < a.nrows) ? 1.0 : 0.0;  // rows past the end weigh 0
      double h[NT];
#pragma unroll
      for (int t = 0; t < NT; t++) {
        const int ia = a.ha[8 * t + m], ib = a.hb[8 * t + m];
        double x = one;
        if (ia >= 0) x *= f[ia][r];
        if (ib >= 0) x *= f[ib][r];
        h[t] = x;
        lin[t] += x;
      }
      int p = 0;
#pragma unroll
      for (int t = 0; t < NT; t++)
#pragma unroll
        for (int s = t; s < NT; s++) pdmma(acc[p++], h[t], h[s]);
    }
    __syncwarp();
  }
  double* out = a.partials + (size_t)gw * (NT * (NT + 1) / 2 * 64 + NT * 8);
  int p = 0;
#pragma unroll
  for (int t = 0; t < NT; t++)
#pragma unroll
    for (int s = t; s < NT; s++, p++) {
      out[p * 64 + m * 8 + 2 * k] = acc[p][0];  // tile (t, s): D[m][n] = Σ h_{8t+m} h_{8s+n}
      out[p * 64 + m * 8 + 2 * k + 1] = acc[p][1];
    }
#pragma unroll
  for (int t = 0; t < NT; t++) {  // Σ h_{8t+m} over the warp's rows: the 4 lanes k of half m
    double l = lin[t];
    l += __shfl_xor_sync(PFULL, l, 1);
    l += __shfl_xor_sync(PFULL, l, 2);
    if (k == 0) out[NT * (NT + 1) / 2 * 64 + t * 8 + m] = l;
  }
}

// src[e] = Σ_w partials[w][e] in a fixed order: one CTA per element, its threads over strided
// warps, then a fixed tree; src[n] = the row count (the constant half's corner)
__global__ void k_poly_sum(const double* __restrict__ partials, int nw, int n, double* __restrict__ src, int64_t nrows) {
  __shared__ double red[256];
  for (int e = blockIdx.x; e < n; e += gridDim.x) {
    double s = 0.0;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) s += partials[(size_t)w * n + e];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) src[e] = red[0];
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) src[n] = (double)nrows;
}
__global__ void k_poly_assemble(const double* __restrict__ src, const int32_t* __restrict__ toff,
                                const int32_t* __restrict__ tidx, const double* __restrict__ tcoef, int nout,
                                double* __restrict__ out, int count_idx, unsigned long long* __restrict__ count) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < nout; o += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = toff[o]; t < toff[o + 1]; t++) s += tcoef[t] * src[tidx[t]];
    out[o] = s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = (unsigned long long)src[count_idx];
}

struct FastPoly : FastPaths {
  PolyArgs pa{};
  int grid = 148, nw = 0, npart = 0, nout = 0, count_idx = 0;
  DevBuf partials, src, toff, tidx, tcoef;
  std::string describe() const override {
    char b[128];
    std::snprintf(b, sizeof b, "{\"kind\": \"poly\", \"features\": %d, \"halves_tiles\": %d, \"outputs\": %d}", pa.nattr,
                  pa.nt, nout);
    return b;
  }
  bool skip_generic_views() const override { return true; }
  int run(lmfao_ctx* c, const NodeArgs&, cudaStream_t st, bool& scalar_done) override {
    PolyArgs a = pa;
    a.nrows = c->rels[c->root].nrows;
    a.partials = partials.as<double>();
    scan_timer_begin(c, st);
    if (pa.nt == 1) k_poly<1><<<grid, PL_WARPS * 32, 0, st>>>(a);
    else if (pa.nt == 2) k_poly<2><<<grid, PL_WARPS * 32, 0, st>>>(a);
    else k_poly<3><<<grid, PL_WARPS * 32, 0, st>>>(a);
    scan_timer_end(c, st);
    k_poly_sum<<<std::min(npart, 1024), 256, 0, st>>>(partials.as<double>(), nw, npart, src.as<double>(), a.nrows);
    k_poly_assemble<<<(nout + 127) / 128 + 1, 128, 0, st>>>(src.as<double>(), toff.as<int32_t>(), tidx.as<int32_t>(),
                                                            tcoef.as<double>(), nout, c->scalar_out.as<double>(),
                                                            count_idx, c->scalar_count.as<unsigned long long>());
    launches_add(3);
    scalar_done = true;
    return cudaGetLastError();
  }
};

}  // namespace

// Planner hook: a scalar batch (no group-by queries) whose products are constants times at most
// four identity factors over at most 8 features of the root and its primary-key children, with
// at most 24 distinct halves.  Otherwise nullptr.
FastPaths* plan_poly(lmfao_ctx* c) {
  if (c->scalar_queries.empty() || !c->groups.empty()) return nullptr;
  const Rel& R = c->rels[c->root];
  std::map<int, int> feat;  // attr -> feature slot
  std::unique_ptr<FastPoly> fp(new FastPoly());
  PolyArgs& a = fp->pa;
  auto slot_of = [&](int attr) -> int {
    auto it = feat.find(attr);
    if (it != feat.end()) return it->second;
    if ((int)feat.size() == PL_ATTR) return -2;
    const int o = c->owner[attr];
    const Rel* O = nullptr;
    const int32_t* fk = nullptr;
    if (o == c->root) {
      O = &R;
    } else {
      for (size_t j = 0; j < R.children.size(); j++)
        if (R.children[j] == o && c->rels[o].unique_key) {
          O = &c->rels[o];
          fk = R.fk_dense[j].as<int32_t>();
        }
      if (!O) return -2;  // deeper than a root child, or not a primary key
    }
    const int s = (int)feat.size();
    const Column& col = O->cols[O->find_attr(attr)];
    a.col[s] = col.buf.p;
    a.fk[s] = fk;
    a.isint[s] = col.dt == LMFAO_INT32;
    feat[attr] = s;
    return s;
  };
  // halves: monomials of <= 2 features, (slot a <= slot b; -1 = 1)
  std::map<std::pair<int, int>, int> half;
  std::vector<std::pair<int, int>> halves;
  auto half_of = [&](std::pair<int, int> h) -> int {
    auto it = half.find(h);
    if (it != half.end()) return it->second;
    if ((int)halves.size() == PL_MAXT * 8 + 1) return -1;  // the constant + 24 tile columns
    half[h] = (int)halves.size();
    halves.push_back(h);
    return (int)halves.size() - 1;
  };
  auto mono = [](int x, int y) { return x <= y ? std::make_pair(x, y) : std::make_pair(y, x); };
  half_of({-1, -1});  // h_0 = 1: not a tile column (linear sums and the count)
  struct T {
    double coef;
    int a, b;
  };
  std::vector<std::vector<T>> outs;
  bool higher = false;  // a product with more than two factors
  for (int q : c->scalar_queries)
    for (auto& u : c->queries[q].udafs) {
      std::vector<T> ts;
      for (auto& p : u) {
        double coef = p.coeff;
        std::vector<int> fs;
        for (auto& f : p.f) {
          if (f.kind == LMFAO_F_CONST) coef *= f.param;
          else if (f.kind == LMFAO_F_IDENT) {
            const int s = slot_of(f.attr);
            if (s < 0) return nullptr;
            fs.push_back(s);
          } else {
            return nullptr;
          }
        }
        if (fs.size() > 4) return nullptr;
        higher |= fs.size() > 2;
        while (fs.size() < 4) fs.push_back(-1);
        std::sort(fs.begin(), fs.end());
        // split into two halves of <= 2 features: prefer a split whose halves exist already
        const int splits[3][4] = {{0, 1, 2, 3}, {0, 2, 1, 3}, {0, 3, 1, 2}};
        int ha = -1, hb = -1;
        for (auto& sp : splits) {
          auto h1 = mono(fs[sp[0]], fs[sp[1]]), h2 = mono(fs[sp[2]], fs[sp[3]]);
          if (half.count(h1) && half.count(h2)) {
            ha = half[h1];
            hb = half[h2];
            break;
          }
        }
        if (ha < 0) {
          ha = half_of(mono(fs[0], fs[1]));
          hb = half_of(mono(fs[2], fs[3]));
          if (ha < 0 || hb < 0) return nullptr;
        }
        ts.push_back(T{coef, std::min(ha, hb), std::max(ha, hb)});
      }
      outs.push_back(ts);
    }
  // batches of products of at most two factors reach here only when cov.cu and gram.cu
  // declined them (e.g. a relation without children: the fact-only Gram)
  (void)higher;
  const int n = (int)halves.size() - 1;  // tile columns: halves 1..n (half 0 is the constant)
  if (n > PL_MAXT * 8) return nullptr;
  a.nattr = (int)feat.size();
  a.nt = std::max(1, (n + 7) / 8);
  for (int i = 0; i < PL_MAXT * 8; i++) {
    a.ha[i] = i < n ? (int8_t)halves[i + 1].first : (int8_t)-1;
    a.hb[i] = i < n ? (int8_t)halves[i + 1].second : (int8_t)-1;
  }
  // padded columns (i >= n) are the constant: harmless, their entries are never read
  // G entry (x, y), x <= y over the halves: (0, 0) the count; (0, y) the linear sum of column
  // y - 1; else tile pair (t, s) = ((x-1) / 8, (y-1) / 8), element [(x-1) % 8][(y-1) % 8]
  const int npairs = a.nt * (a.nt + 1) / 2;
  auto gidx = [&](int x, int y) {
    if (x == 0) return y == 0 ? npairs * 64 + a.nt * 8 : npairs * 64 + (y - 1);
    const int xx = x - 1, yy = y - 1, t = xx / 8, s = yy / 8;
    int p = 0;
    for (int tt = 0; tt < a.nt; tt++)
      for (int ss = tt; ss < a.nt; ss++, p++)
        if (tt == t && ss == s) return p * 64 + (xx % 8) * 8 + (yy % 8);
    return -1;
  };
  std::vector<int32_t> toff{0}, tidx;
  std::vector<double> tcoef;
  for (auto& ts : outs) {
    for (auto& t : ts) {
      tidx.push_back(gidx(t.a, t.b));
      tcoef.push_back(t.coef);
    }
    toff.push_back((int32_t)tidx.size());
  }
  fp->nout = (int)outs.size();
  fp->count_idx = gidx(0, 0);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int per = 0;  // one wave of resident CTAs (static per-warp ranges)
  const void* kfn = a.nt == 1 ? (const void*)k_poly<1> : a.nt == 2 ? (const void*)k_poly<2> : (const void*)k_poly<3>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, PL_WARPS * 32, 0) || per < 1) per = 1;
  fp->grid = sms * per;
  fp->nw = fp->grid * PL_WARPS;
  fp->npart = npairs * 64 + a.nt * 8;  // + the count at src[npart]
  cudaStream_t st = c->stream;
  if (fp->partials.alloc((size_t)fp->nw * fp->npart * 8) || fp->src.alloc((size_t)(fp->npart + 1) * 8) ||
      fp->toff.alloc(toff.size() * 4) || fp->tidx.alloc(std::max<size_t>(tidx.size(), 1) * 4) ||
      fp->tcoef.alloc(std::max<size_t>(tcoef.size(), 1) * 8))
    return nullptr;
  if (cudaMemcpyAsync(fp->toff.p, toff.data(), toff.size() * 4, cudaMemcpyHostToDevice, st) ||
      (!tidx.empty() && (cudaMemcpyAsync(fp->tidx.p, tidx.data(), tidx.size() * 4, cudaMemcpyHostToDevice, st) ||
                         cudaMemcpyAsync(fp->tcoef.p, tcoef.data(), tcoef.size() * 8, cudaMemcpyHostToDevice, st))) ||
      cudaStreamSynchronize(st))
    return nullptr;
  return fp.release();
}

}  // namespace lmfao
