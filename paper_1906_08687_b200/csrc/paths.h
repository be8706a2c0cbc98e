// paths.h — specialised kernels selected by the planner for recognised batch
// shapes (the Gram path of the covariance batch, the histogram paths).
#pragma once
#include <string>

#include "internal.h"

struct lmfao_ctx;

namespace lmfao {
struct FastPaths {
  virtual ~FastPaths() {}
  // Launches the specialised root-scan work on `st`; sets scalar_done if it
  // produced all no-group-by outputs.  Returns a cudaError_t value (0 = ok).
  virtual int run(lmfao_ctx* c, const NodeArgs& root, cudaStream_t st, bool& scalar_done) = 0;
  virtual bool handles_group(int query) const { return false; }
  // true if run() fills every group-by table of the batch (the generic group scan is skipped)
  virtual bool handles_all_groups() const { return false; }
  // true if the specialised path builds its own dimension tables (skip generic views)
  virtual bool skip_generic_views() const { return false; }
  // false if run() synchronises with the host (data-dependent sizes): no CUDA Graph capture
  virtual bool graph_ok() const { return true; }
  virtual std::string describe() const = 0;
  // Dynamic functions: replace the planned batch's path condition (the
  // predicates every product carries) by factors[0..n), without re-planning.  0 = ok, else
  // unsupported (the path took no path condition, or an attribute it cannot evaluate).
  virtual int set_condition(lmfao_ctx* c, int n, const lmfao_factor* factors) { return -1; }
};
// Returns nullptr when no specialised path applies (the generic path runs).
FastPaths* plan_fast_paths(lmfao_ctx* c);
FastPaths* plan_gram(lmfao_ctx* c);
FastPaths* plan_cov(lmfao_ctx* c);
FastPaths* plan_rt(lmfao_ctx* c);
FastPaths* plan_counts(lmfao_ctx* c);
FastPaths* plan_cube(lmfao_ctx* c);  // group-by queries only (scalar queries: another path)
FastPaths* plan_poly(lmfao_ctx* c);  // scalar polynomial batches (products of up to 4 features)
}  // namespace lmfao
