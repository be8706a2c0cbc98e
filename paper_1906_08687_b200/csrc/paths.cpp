// paths.cpp — selection of the specialised kernels for a planned batch.
#include <cstdlib>
#include <memory>

#include "ctx.h"

namespace lmfao {
namespace {
// A scalar path (covariance / Gram scan, or none: the generic scalar scan) next to the
// cube path for the batch's group-by queries.
struct ComboPaths : FastPaths {
  std::unique_ptr<FastPaths> scalar, groups;
  ComboPaths(FastPaths* s, FastPaths* g) : scalar(s), groups(g) {}
  int run(lmfao_ctx* c, const NodeArgs& root, cudaStream_t st, bool& scalar_done) override {
    if (scalar)
      if (int e = scalar->run(c, root, st, scalar_done)) return e;
    bool unused = false;
    return groups->run(c, root, st, unused);
  }
  bool handles_group(int q) const override { return groups->handles_group(q); }
  bool graph_ok() const override { return groups->graph_ok() && (!scalar || scalar->graph_ok()); }
  bool handles_all_groups() const override { return groups->handles_all_groups(); }
  // the generic views feed only the generic scalar scan here
  bool skip_generic_views() const override { return scalar != nullptr || no_scalars; }
  bool no_scalars = false;
  std::string describe() const override {
    return "{\"kind\": \"combo\", \"scalar\": " + (scalar ? scalar->describe() : std::string("null")) +
           ", \"groups\": " + groups->describe() + "}";
  }
};
FastPaths* with_cube(lmfao_ctx* c, FastPaths* scalar) {
  if (c->groups.empty()) return scalar;
  FastPaths* g = plan_cube(c);
  if (!g) return scalar;
  auto* cp = new ComboPaths(scalar, g);
  cp->no_scalars = c->scalar_queries.empty();
  return cp;
}
}  // namespace

FastPaths* plan_fast_paths(lmfao_ctx* c) {
  // LMFAO_GENERIC_ONLY=1 forces the interpreted path (used by tests to cross-check the two)
  const char* env = std::getenv("LMFAO_GENERIC_ONLY");
  if (env && env[0] == '1') return nullptr;
  if (!c->revs.empty()) return nullptr;  // group-bys finished at a non-unique child: the generic scan
  const char* ng = std::getenv("LMFAO_NO_COV");  // tests: force the gram.cu kernel
  const char* nc = std::getenv("LMFAO_NO_CUBE");  // tests: keep group-bys on the generic scan
  const bool cube = !(nc && nc[0] == '1');
  if (!(ng && ng[0] == '1'))
    if (FastPaths* f = plan_cov(c)) return cube ? with_cube(c, f) : f;
  if (FastPaths* f = plan_counts(c)) return f;
  if (FastPaths* f = plan_rt(c)) return f;
  if (FastPaths* f = plan_gram(c)) return cube ? with_cube(c, f) : f;
  const char* np = std::getenv("LMFAO_NO_POLY");  // tests: the interpreted path instead
  if (!(np && np[0] == '1'))
    if (FastPaths* f = plan_poly(c)) return f;
  if (cube && c->groups.size() > 0)
    if (FastPaths* g = plan_cube(c)) {
      auto* cp = new ComboPaths(nullptr, g);
      cp->no_scalars = c->scalar_queries.empty();
      return cp;
    }
  return nullptr;
}
}  // namespace lmfao
