// paths.cpp — selection of the specialised kernels for a planned batch.
#include <cstdlib>

#include "ctx.h"

namespace lmfao {
FastPaths* plan_fast_paths(lmfao_ctx* c) {
  // LMFAO_GENERIC_ONLY=1 forces the interpreted path (used by tests to cross-check the two)
  const char* env = std::getenv("LMFAO_GENERIC_ONLY");
  if (env && env[0] == '1') return nullptr;
  const char* ng = std::getenv("LMFAO_NO_COV");  // tests: force the gram.cu kernel
  if (!(ng && ng[0] == '1'))
    if (FastPaths* f = plan_cov(c)) return f;
  if (FastPaths* f = plan_counts(c)) return f;
  if (FastPaths* f = plan_rt(c)) return f;
  if (FastPaths* f = plan_gram(c)) return f;
  return nullptr;
}
}  // namespace lmfao
