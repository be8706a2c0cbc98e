#include "ctx.h"
namespace lmfao {
FastPaths* plan_fast_paths(lmfao_ctx*) { return nullptr; }
}
