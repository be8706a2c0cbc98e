// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU evaluation of an LMFAO aggregate batch
// (§3 "Problem Statement"):
//
//   Q(F_1..F_f; α_1..α_ℓ) += R_1(ω_1), …, R_m(ω_m)
//   SELECT F, SUM(α_1), …, SUM(α_ℓ) FROM R_1 NATURAL JOIN … NATURAL JOIN R_m GROUP BY F
//   α_i = Σ_j Π_k f_ijk, f ∈ {constant, identity, Kronecker 1_{X op t}}
//
// It MATERIALISES the natural join (streamed, tuple by tuple, never stored) by a
// depth-first enumeration over the join tree (the join tree of an
// acyclic join; matching on the attributes shared along each edge is the
// natural join because of the running-intersection property), with bag
// semantics (duplicates multiply; tuples with a dangling key vanish), and adds
// every UDAF's value into its group.  It does NOT use views, roots, merging,
// multi-output plans or any other LMFAO rewrite: it is the definition.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load this library.  It shares no code, header or
// table with the CUDA path (paper_1906_08687_b200/csrc) and never will.
//
// Precision (readings R3/R14): each product term is
// evaluated in IEEE double, left to right (coeff first, then factors in the
// listed order); the terms of one UDAF for one tuple are summed in long double,
// and that per-tuple value is accumulated per group in long double (x87, 64-bit
// mantissa).  Counts (the hidden join multiplicity of a group) are uint64.  The
// absolute mass A = Σ|term| is accumulated too (for the tolerance fallback).
//
// Accumulation modes ("long double (x87, 64-bit mantissa) or
// Neumaier-compensated double"): the default is long double as above; `ACC NEUMAIER`
// in the spec sums the terms of a tuple and the tuples of a group in double with
// Neumaier's compensation instead (used only to bound the oracle's own rounding error,
// tests/test_oracle_pins.py).
//
// Threads (SURVEY.md §8(d)(ii) "the same source built with OpenMP over fact-row chunks:
// private accumulators, merged in thread order"): `THREADS T` splits the root rows into
// T contiguous chunks, each enumerated by its own worker into private group tables;
// the tables are then added in chunk order (deterministic).  T = 1 is the plain loop.
//
// Input: a line-oriented text spec (see oracle/__init__.py, which writes it)
// plus one pointer per column (int32 or double arrays).
//
// Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC -o liboracle.so oracle.cpp
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

enum FactorKind { F_CONST = 0, F_IDENT, F_LT, F_LE, F_GT, F_GE, F_EQ, F_NE, F_IN };

struct Column {
  std::string name;
  bool is_int = false;
  const int32_t* ip = nullptr;
  const double* dp = nullptr;
};

struct Relation {
  std::string name;
  int64_t nrows = 0;
  std::vector<Column> cols;
  int find(const std::string& a) const {
    for (size_t i = 0; i < cols.size(); i++)
      if (cols[i].name == a) return (int)i;
    return -1;
  }
};

struct FactorSpec {
  int kind;
  std::string attr;  // empty for CONST
  double param;
};
struct ProductSpec {
  double coeff;
  std::vector<FactorSpec> factors;
};
struct QuerySpec {
  std::vector<std::string> groupby;
  std::vector<std::vector<ProductSpec>> udafs;
};

// A resolved attribute reference: which relation (by DFS position) and column.
struct AttrRef {
  int pos;  // position in DFS preorder
  int col;
  bool is_int;
};

struct Acc {
  uint64_t count = 0;
  std::vector<long double> sum;
  std::vector<long double> absmass;
  std::vector<double> nsum, ncomp;  // ACC NEUMAIER: running double sum and its compensation
};

// Neumaier's compensated addition: s + c carries the exact sum's rounding residue
inline void neumaier_add(double& s, double& c, double v) {
  const double t = s + v;
  if (std::fabs(s) >= std::fabs(v)) c += (s - t) + v;
  else c += (v - t) + s;
  s = t;
}

struct Result {
  int ngb = 0, nudaf = 0;
  std::map<std::vector<int64_t>, Acc> groups;
};

struct Oracle {
  std::vector<Relation> rels;
  std::vector<std::pair<std::string, std::string>> edges;  // parent, child
  std::string root;
  int64_t root_lo = 0, root_hi = -1;
  int threads = 1;
  bool neumaier = false;
  std::vector<QuerySpec> queries;
  std::vector<Result> results;

  // join-tree in DFS preorder
  std::vector<int> order;        // relation index at each position
  std::vector<int> parent_pos;   // position of the parent, -1 for the root
  std::vector<std::vector<std::pair<int, int>>> keycols;  // (child col, parent col) per position
  // per position (non-root): multimap key -> rows
  std::vector<std::map<std::vector<int64_t>, std::vector<int64_t>>> index;

  // one enumeration worker: its own tuple binding and private group tables
  struct Worker {
    std::vector<int64_t> binding;  // row bound at each position
    std::vector<Result> results;
  };

  // resolved queries
  struct RFactor { int kind; AttrRef ref; double param; };
  struct RProduct { double coeff; std::vector<RFactor> f; };
  struct RQuery { std::vector<AttrRef> gb; std::vector<std::vector<RProduct>> udafs; };
  std::vector<RQuery> rq;

  int rel_index(const std::string& n) const {
    for (size_t i = 0; i < rels.size(); i++)
      if (rels[i].name == n) return (int)i;
    throw std::runtime_error("unknown relation " + n);
  }

  double value(const Worker& w, const AttrRef& r) const {
    const Relation& R = rels[order[r.pos]];
    const Column& c = R.cols[r.col];
    int64_t row = w.binding[r.pos];
    return c.is_int ? (double)c.ip[row] : c.dp[row];
  }
  int64_t ivalue(const Worker& w, const AttrRef& r) const {
    const Relation& R = rels[order[r.pos]];
    const Column& c = R.cols[r.col];
    return (int64_t)c.ip[w.binding[r.pos]];
  }

  AttrRef resolve(const std::string& a) const {
    // any bound relation holding the attribute gives the same value in a joined
    // tuple (natural join); take the first in DFS order.
    for (size_t p = 0; p < order.size(); p++) {
      int c = rels[order[p]].find(a);
      if (c >= 0) return AttrRef{(int)p, c, rels[order[p]].cols[c].is_int};
    }
    throw std::runtime_error("unknown attribute " + a);
  }

  void build_tree() {
    int n = (int)rels.size();
    std::vector<std::vector<int>> children(n);
    std::vector<int> parent(n, -1);
    for (auto& e : edges) {
      int p = rel_index(e.first), c = rel_index(e.second);
      if (parent[c] != -1) throw std::runtime_error("node with two parents: " + e.second);
      parent[c] = p;
      children[p].push_back(c);
    }
    int r = rel_index(root);
    if (parent[r] != -1) throw std::runtime_error("root has a parent");
    // DFS preorder
    std::vector<int> stack{r};
    std::vector<int> pos_of(n, -1);
    while (!stack.empty()) {
      int u = stack.back();
      stack.pop_back();
      if (pos_of[u] != -1) throw std::runtime_error("cycle in join tree");
      pos_of[u] = (int)order.size();
      order.push_back(u);
      for (auto it = children[u].rbegin(); it != children[u].rend(); ++it) stack.push_back(*it);
    }
    if ((int)order.size() != n) throw std::runtime_error("join tree is disconnected");
    parent_pos.assign(n, -1);
    keycols.assign(n, {});
    index.assign(n, {});
    for (int p = 0; p < n; p++) {
      int u = order[p];
      if (parent[u] < 0) continue;
      parent_pos[p] = pos_of[parent[u]];
      const Relation& C = rels[u];
      const Relation& P = rels[parent[u]];
      for (size_t i = 0; i < C.cols.size(); i++) {
        int j = P.find(C.cols[i].name);
        if (j >= 0) {
          if (!C.cols[i].is_int || !P.cols[j].is_int)
            throw std::runtime_error("join attribute must be int: " + C.cols[i].name);
          keycols[p].push_back({(int)i, j});
        }
      }
      // multimap: key values -> rows of C
      for (int64_t row = 0; row < C.nrows; row++) {
        std::vector<int64_t> k;
        for (auto& kc : keycols[p]) k.push_back(C.cols[kc.first].ip[row]);
        index[p][k].push_back(row);
      }
    }
    // running intersection: attributes shared by two nodes appear on
    // the whole path between them.  Plain O(m^2 * path) check.
    for (int a = 0; a < n; a++)
      for (int b = a + 1; b < n; b++) {
        std::vector<int> pa, pb;  // ancestors incl. self
        for (int u = a; u != -1; u = parent[u]) pa.push_back(u);
        for (int u = b; u != -1; u = parent[u]) pb.push_back(u);
        std::set<int> sa(pa.begin(), pa.end());
        int lca = -1;
        for (int u : pb)
          if (sa.count(u)) { lca = u; break; }
        std::vector<int> path;
        for (int u = a; u != lca; u = parent[u]) path.push_back(u);
        for (int u = b; u != lca; u = parent[u]) path.push_back(u);
        path.push_back(lca);
        for (auto& col : rels[a].cols) {
          if (rels[b].find(col.name) < 0) continue;
          for (int u : path)
            if (rels[u].find(col.name) < 0)
              throw std::runtime_error("running intersection violated for attribute " + col.name);
        }
      }
  }

  void resolve_queries() {
    for (auto& q : queries) {
      RQuery r;
      for (auto& g : q.groupby) {
        AttrRef a = resolve(g);
        if (!a.is_int) throw std::runtime_error("group-by attribute must be int: " + g);
        r.gb.push_back(a);
      }
      for (auto& u : q.udafs) {
        std::vector<RProduct> ps;
        for (auto& p : u) {
          RProduct rp{p.coeff, {}};
          for (auto& f : p.factors) {
            RFactor rf{f.kind, AttrRef{-1, -1, false}, f.param};
            if (f.kind != F_CONST) rf.ref = resolve(f.attr);
            rp.f.push_back(rf);
          }
          ps.push_back(rp);
        }
        r.udafs.push_back(ps);
      }
      rq.push_back(r);
      Result res;
      res.ngb = (int)q.groupby.size();
      res.nudaf = (int)q.udafs.size();
      results.push_back(res);
    }
  }

  double eval_factor(const Worker& w, const RFactor& f) const {
    if (f.kind == F_CONST) return f.param;
    double x = value(w, f.ref);
    switch (f.kind) {
      case F_IDENT: return x;
      case F_LT: return x < f.param ? 1.0 : 0.0;
      case F_LE: return x <= f.param ? 1.0 : 0.0;
      case F_GT: return x > f.param ? 1.0 : 0.0;
      case F_GE: return x >= f.param ? 1.0 : 0.0;
      case F_EQ: return x == f.param ? 1.0 : 0.0;
      case F_NE: return x != f.param ? 1.0 : 0.0;
      case F_IN: {  // set inclusion, S as a bit mask over {0..52} (reading R20)
        if (!(x >= 0.0 && x <= 52.0) || x != std::floor(x)) return 0.0;
        const uint64_t mask = (uint64_t)f.param;
        return ((mask >> (int)x) & 1u) ? 1.0 : 0.0;
      }
    }
    throw std::runtime_error("bad factor kind");
  }

  // one joined tuple t is bound in w.binding
  void emit(Worker& w) const {
    for (size_t qi = 0; qi < rq.size(); qi++) {
      const RQuery& q = rq[qi];
      std::vector<int64_t> key;
      key.reserve(q.gb.size());
      for (auto& g : q.gb) key.push_back(ivalue(w, g));
      Acc& acc = w.results[qi].groups[key];
      if (acc.sum.empty()) {
        acc.sum.assign(q.udafs.size(), 0.0L);
        acc.absmass.assign(q.udafs.size(), 0.0L);
        if (neumaier) {
          acc.nsum.assign(q.udafs.size(), 0.0);
          acc.ncomp.assign(q.udafs.size(), 0.0);
        }
      }
      acc.count += 1;
      for (size_t j = 0; j < q.udafs.size(); j++) {
        long double s = 0.0L, a = 0.0L;
        double ns = 0.0, nc = 0.0;
        for (auto& p : q.udafs[j]) {
          double v = p.coeff;
          for (auto& f : p.f) v = v * eval_factor(w, f);
          if (neumaier) neumaier_add(ns, nc, v);
          else s += (long double)v;
          a += (long double)std::fabs(v);
        }
        if (neumaier) {
          neumaier_add(acc.nsum[j], acc.ncomp[j], ns);
          neumaier_add(acc.nsum[j], acc.ncomp[j], nc);
        } else {
          acc.sum[j] += s;
        }
        acc.absmass[j] += a;
      }
    }
  }

  void enumerate(Worker& w, size_t pos) const {
    if (pos == order.size()) {
      emit(w);
      return;
    }
    int pp = parent_pos[pos];
    const Relation& P = rels[order[pp]];
    std::vector<int64_t> k;
    for (auto& kc : keycols[pos]) k.push_back(P.cols[kc.second].ip[w.binding[pp]]);
    auto it = index[pos].find(k);
    if (it == index[pos].end()) return;  // dangling: the tuple vanishes
    for (int64_t row : it->second) {
      w.binding[pos] = row;
      enumerate(w, pos + 1);
    }
  }

  void run() {
    build_tree();
    resolve_queries();
    const Relation& R = rels[order[0]];
    int64_t hi = root_hi < 0 ? R.nrows : std::min(root_hi, R.nrows);
    const int64_t lo = std::min(root_lo, hi);
    const int T = threads < 1 ? 1 : threads;
    std::vector<Worker> ws(T);
    for (auto& w : ws) {
      w.binding.assign(order.size(), -1);
      w.results = results;  // empty tables of the right shape
    }
    // chunk t = root rows [lo + (hi-lo)·t/T, lo + (hi-lo)·(t+1)/T)
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; t++) {
      Worker& w = ws[t];
      const int64_t a = lo + (hi - lo) * t / T, b = lo + (hi - lo) * (t + 1) / T;
      for (int64_t row = a; row < b; row++) {
        w.binding[0] = row;
        enumerate(w, 1);
      }
    }
    // merge the private tables in chunk order
    for (int t = 0; t < T; t++)
      for (size_t qi = 0; qi < rq.size(); qi++)
        for (auto& kv : ws[t].results[qi].groups) {
          Acc& acc = results[qi].groups[kv.first];
          const Acc& part = kv.second;
          if (acc.sum.empty()) {
            acc = part;
            continue;
          }
          acc.count += part.count;
          for (size_t j = 0; j < acc.sum.size(); j++) {
            acc.sum[j] += part.sum[j];
            acc.absmass[j] += part.absmass[j];
            if (neumaier) {
              neumaier_add(acc.nsum[j], acc.ncomp[j], part.nsum[j]);
              neumaier_add(acc.nsum[j], acc.ncomp[j], part.ncomp[j]);
            }
          }
        }
    // P:134-139 SQL GROUP BY: with no group-by attribute the single output row
    // exists even over an empty join (value 0, count 0; reading R1).
    for (size_t qi = 0; qi < rq.size(); qi++) {
      if (rq[qi].gb.empty() && results[qi].groups.empty()) {
        Acc& acc = results[qi].groups[{}];
        acc.sum.assign(rq[qi].udafs.size(), 0.0L);
        acc.absmass.assign(rq[qi].udafs.size(), 0.0L);
        if (neumaier) {
          acc.nsum.assign(rq[qi].udafs.size(), 0.0);
          acc.ncomp.assign(rq[qi].udafs.size(), 0.0);
        }
      }
    }
  }
};

void parse(Oracle& o, const char* spec, const void* const* colptrs) {
  std::istringstream in(spec);
  std::string tok;
  size_t colk = 0;
  while (in >> tok) {
    if (tok == "REL") {
      Relation r;
      int ncols;
      in >> r.name >> r.nrows >> ncols;
      for (int c = 0; c < ncols; c++) {
        std::string ctok, name, ty;
        in >> ctok >> name >> ty;
        if (ctok != "COL") throw std::runtime_error("expected COL");
        Column col;
        col.name = name;
        col.is_int = (ty == "I");
        if (col.is_int) col.ip = (const int32_t*)colptrs[colk];
        else col.dp = (const double*)colptrs[colk];
        colk++;
        r.cols.push_back(col);
      }
      o.rels.push_back(r);
    } else if (tok == "ROOT") {
      in >> o.root;
    } else if (tok == "RANGE") {
      in >> o.root_lo >> o.root_hi;
    } else if (tok == "THREADS") {
      in >> o.threads;
    } else if (tok == "ACC") {
      std::string mode;
      in >> mode;
      if (mode == "NEUMAIER") o.neumaier = true;
      else if (mode != "LONGDOUBLE") throw std::runtime_error("bad ACC mode " + mode);
    } else if (tok == "EDGE") {
      std::string p, c;
      in >> p >> c;
      o.edges.push_back({p, c});
    } else if (tok == "QUERY") {
      QuerySpec q;
      int ngb, nudaf;
      in >> ngb;
      for (int i = 0; i < ngb; i++) {
        std::string g;
        in >> g;
        q.groupby.push_back(g);
      }
      in >> nudaf;
      for (int u = 0; u < nudaf; u++) {
        std::string ut;
        int nprod;
        in >> ut >> nprod;
        if (ut != "UDAF") throw std::runtime_error("expected UDAF");
        std::vector<ProductSpec> prods;
        for (int p = 0; p < nprod; p++) {
          std::string pt, coeff;
          int nf;
          in >> pt >> coeff >> nf;
          if (pt != "PROD") throw std::runtime_error("expected PROD");
          ProductSpec ps;
          ps.coeff = std::strtod(coeff.c_str(), nullptr);
          for (int f = 0; f < nf; f++) {
            FactorSpec fs;
            std::string attr, param;
            in >> fs.kind >> attr >> param;
            fs.attr = attr == "-" ? "" : attr;
            fs.param = std::strtod(param.c_str(), nullptr);
            ps.factors.push_back(fs);
          }
          prods.push_back(ps);
        }
        q.udafs.push_back(prods);
      }
      o.queries.push_back(q);
    } else {
      throw std::runtime_error("bad spec token " + tok);
    }
  }
}

}  // namespace

extern "C" {

void* oracle_eval(const char* spec, const void* const* cols, char* err, int errlen) {
  Oracle* o = new Oracle();
  try {
    parse(*o, spec, cols);
    o->run();
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "%s", e.what());
    delete o;
    return nullptr;
  }
  return o;
}

int oracle_nqueries(void* h) { return (int)((Oracle*)h)->results.size(); }

void oracle_shape(void* h, int q, int64_t* ngroups, int* ngb, int* nudaf) {
  Oracle* o = (Oracle*)h;
  *ngroups = (int64_t)o->results[q].groups.size();
  *ngb = o->results[q].ngb;
  *nudaf = o->results[q].nudaf;
}

void oracle_fetch(void* h, int q, int64_t* keys, double* vals, uint64_t* counts, double* absmass) {
  Oracle* o = (Oracle*)h;
  const Result& r = o->results[q];
  int64_t g = 0;
  for (auto& kv : r.groups) {  // std::map: ascending lexicographic key order
    for (int i = 0; i < r.ngb; i++) keys[g * r.ngb + i] = kv.first[i];
    for (int j = 0; j < r.nudaf; j++) {
      vals[g * r.nudaf + j] = o->neumaier ? kv.second.nsum[j] + kv.second.ncomp[j] : (double)kv.second.sum[j];
      absmass[g * r.nudaf + j] = (double)kv.second.absmass[j];
    }
    counts[g] = kv.second.count;
    g++;
  }
}

void oracle_free(void* h) { delete (Oracle*)h; }

}  // extern "C"
